"""Timing of the auxiliary device passes on a resident 2^n int64 signal:
the magnitude bound (k_minmax), exact Parseval (k_sumsq), the ordered
extraction (k_extract_*), and the fused transform + extraction, with CUDA
events; GB/s of the 8 B/point they read."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1607_01039_b200 as bw  # noqa: E402
from paper_1607_01039_b200 import signals  # noqa: E402


def timed(f, reps=5):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
x = signals.make(signals.config(4, n))
gb = 8 * (1 << n) / 1e9
for name, f in (("check_magnitude_bound", lambda: bw.check_magnitude_bound(x, n)),
                ("parseval_energy", lambda: bw.parseval_energy(bw.Signal(x))),
                ("extract_ge (few hits)", lambda: bw.extract_ge(x, 1 << 40))):
    ms = timed(f)
    print(f"{name:24s} n={n}: {ms:.3f} ms, {gb / (ms / 1e3):.0f} GB/s read", flush=True)
del x
torch.cuda.empty_cache()
ni = min(n, 30)  # the inverse's magnitude bound admits a +-1 signal's spectrum up to n = 30
x = signals.make(signals.config(4, ni))
sig = bw.Signal(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
tot = 0.0
for rep in range(4):
    bw.fwht_inplace(sig)  # time -> Walsh (untimed)
    torch.cuda.synchronize()
    e0.record()
    bw.inverse_wht_inplace(sig)  # bound, transform, divisibility check, exact shift
    e1.record()
    torch.cuda.synchronize()
    if rep:
        tot += e0.elapsed_time(e1)
print(f"inverse_wht_inplace n={ni}: {tot / 3:.3f} ms (bound + transform + check + shift)", flush=True)
for name, f in ():
    ms = timed(f)
    print(f"{name:24s} n={n}: {ms:.3f} ms, {gb / (ms / 1e3):.0f} GB/s read", flush=True)
