"""GPU fold timing (kernel k_fold, subspace.py:150-184): x'[L.j] += x[j] for a
resident 2^n int64 signal (8 B/point read) and for the on-the-fly generated
config input (no signal in memory), d_out = 12 / 14 (shared-memory bins) and
16 / 20 / 24 (the block fold; BW_FOLD_BLOCKS=0: L2 atomics).  CUDA events,
5 reps after one warm-up."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1607_01039_b200 import signals, subspace  # noqa: E402
from paper_1607_01039_b200.core import Domain, Signal  # noqa: E402


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
spec = signals.config(4, n)
x = signals.make(spec)
sig = Signal(x, Domain.TIME)
for d_out in (8, 10, 12, 14, 16, 20, 24):
    rows = subspace.random_full_rank(n, d_out, 7)
    ms = timed(lambda: subspace.fold(sig, rows))
    print(f"fold resident n={n} -> d_out={d_out}: {ms:.3f} ms, {(1 << n) / (ms / 1e3):.3e} points/s, "
          f"{8 * (1 << n) / ms / 1e6:.1f} GB/s read", flush=True)
    msg = timed(lambda: subspace.fold_generated(spec, rows))
    print(f"fold generated n={n} -> d_out={d_out}: {msg:.3f} ms, {(1 << n) / (msg / 1e3):.3e} points/s", flush=True)
rows = subspace.random_full_rank(n, 20, 7)
x.copy_(signals.make(signals.config(2, n)))  # wide values: the shared atomics' high words work too
ms = timed(lambda: subspace.fold(sig, rows))
print(f"fold resident n={n} (config 2 values) -> d_out=20: {ms:.3f} ms, {(1 << n) / (ms / 1e3):.3e} points/s",
      flush=True)
rows[:, 3] = rows[:, 1] ^ rows[:, 2]  # dependent low columns: the block fold with shared atomics
ms = timed(lambda: subspace.fold(sig, rows))
print(f"fold resident n={n} -> d_out=20, dependent low columns: {ms:.3f} ms, {(1 << n) / (ms / 1e3):.3e} points/s",
      flush=True)
del x, sig
torch.cuda.empty_cache()
if n < 34:
    spec = signals.config(5, 34)
    rows = np.asarray(subspace.random_full_rank(34, 20, 7))
    msg = timed(lambda: subspace.fold_generated(spec, rows), reps=2)
    print(f"fold generated n=34 (config 5) -> d_out=20: {msg:.3f} ms, {(1 << 34) / (msg / 1e3):.3e} points/s", flush=True)
