"""float64 transform timing (CUDA events, resident input): the ascending-
order pass kernels vs the int64 plan on the same n."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1607_01039_b200 as bw  # noqa: E402

for n in (24, 28, 30, 32):
    for dt in (torch.float64, torch.int64):
        x = torch.zeros(1 << n, dtype=dt, device="cuda")
        bw.fwht_array(x)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            bw.fwht_array(x)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"n={n} {str(dt):14s} {ms:8.3f} ms  {2**n / (ms / 1e3):.3e} points/s", flush=True)
        del x
        torch.cuda.empty_cache()
