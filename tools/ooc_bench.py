"""Throughput of the out-of-core transform (host-staged) vs the in-HBM e2e path."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1607_01039_b200 as bw
from paper_1607_01039_b200 import outofcore, signals

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
spec = signals.config(4, n)
t = signals.make(spec)
host = torch.empty(1 << n, dtype=torch.int64, pin_memory=True)
host.copy_(t)
del t
torch.cuda.empty_cache()
h = host.numpy()
for lw in (28, 30, 32):
    ws = torch.empty(1 << min(lw, n), dtype=torch.int64, device="cuda")
    outofcore.fwht_out_of_core(h, lw, ws)  # warm-up
    t0 = time.perf_counter()
    p = outofcore.fwht_out_of_core(h, lw, ws)
    dt = time.perf_counter() - t0
    print(f"n={n} workspace=2^{lw} ({(8 << lw) >> 30} GiB): {p} host passes, {dt:.3f} s, "
          f"{2**n/dt:.3e} pts/s, PCIe {(p * 16 * 2**n) / dt / 1e9:.1f} GB/s (both directions)", flush=True)
    del ws
    torch.cuda.empty_cache()
