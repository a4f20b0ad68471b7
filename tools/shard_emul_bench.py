"""Single-GPU timing of the multi-GPU kernels: P shards as P buffers of one
device (same kernels and addressing as P GPUs, but every "peer" access is
local HBM, so this times the kernels' HBM efficiency, not NVLink).
Compares mode peer (full local transform + K6), mode fused (partial local
plan + K6') and mode narrow (int8 pack, int8 cross-shard exchange, local
transforms widening the packed shard)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1607_01039_b200 import sharded  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
for P in (2, 4, 8):
    p = P.bit_length() - 1
    nl = n - p
    shards = [torch.zeros(1 << nl, dtype=torch.int64, device="cuda") for _ in range(P)]
    for mode in ("peer", "fused", "narrow"):
        fused, narrow = mode == "fused", mode == "narrow"
        sharded.fwht_shards(shards, fused=fused, narrow=narrow)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record()
        for _ in range(reps):
            sharded.fwht_shards(shards, fused=fused, narrow=narrow)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        extra = ""
        if fused:
            w, r = sharded.fused_plan(nl, p)
            extra = f"local widths {w} + fused pass ({r} local + {p} shard stages)"
        print(f"n={n} P={P} {mode:6s} {ms:8.3f} ms  {2**n / (ms / 1e3):.3e} points/s  {extra}",
              flush=True)
    del shards
    torch.cuda.empty_cache()
