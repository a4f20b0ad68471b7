"""Measure every pass shape the planner can emit: HBM TB/s of one pass of
(kind, r stages, cluster q) starting at stage bit k, on a resident 2^n
signal.  The table feeds the planner's cost model (bw_abi.cu shape_eff).

    python tools/sweep_shapes.py --n 32 --out gpurun_out/shapes_n32.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1607_01039_b200 import _lib  # noqa: E402


def fill(bits):
    """Split `bits` into filler passes of <= 10 stages."""
    out = []
    while bits > 0:
        w = min(10, bits)
        out.append(w)
        bits -= w
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    n = a.n
    L = _lib.lib()
    x = torch.zeros(1 << n, dtype=torch.int64, device="cuda")
    sh = torch.cuda.current_stream().cuda_stream
    gb = 16.0 * (1 << n) / 1e9
    res = []

    def measure(plan, idx):
        os.environ["BW_PLAN"] = ",".join(str(v) for v in plan)
        _lib.check(L.bw_fwht_i64_pass(x.data_ptr(), n, idx, sh))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            _lib.check(L.bw_fwht_i64_pass(x.data_ptr(), n, idx, sh))
        e1.record()
        torch.cuda.synchronize()
        return gb / (e0.elapsed_time(e1) / a.reps / 1e3) / 1e3  # TB/s

    for w0 in (13, 14, 15):
        tbs = measure([w0] + fill(n - w0), 0)
        res.append({"kind": "low", "r": w0, "q": w0 - 13, "k": 0, "tbs": round(tbs, 3)})
        print(res[-1], flush=True)
    for r in range(3, 11):
        for q in ((0,) if r <= 5 else (0, 1)):
            if r > 5 and not (3 <= 13 + q - r <= (7 if q == 0 else 8)) and not (q == 1 and 13 + q - r >= 4):
                continue
            if r > 5 and q == 0 and 13 - r < 3:
                continue
            for k in range(13, n - r + 1):
                entry = r | ((q + 1) << 4) if r > 5 else r
                plan = [13] + fill(k - 13) + [entry] + fill(n - k - r)
                idx = 1 + len(fill(k - 13))
                tbs = measure(plan, idx)
                res.append({"kind": "reg" if r <= 5 else "high", "r": r, "q": q, "k": k, "tbs": round(tbs, 3)})
                print(res[-1], flush=True)
    os.environ.pop("BW_PLAN", None)
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"n": n, "device": torch.cuda.get_device_name(), "passes": res}, f)


if __name__ == "__main__":
    main()
