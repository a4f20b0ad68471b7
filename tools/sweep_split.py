"""Time whole-transform plans that use split-row passes (bw_layouts.h) against
the default plan, on a resident 2^n signal: per-pass TB/s and the total.
Feeds the planner's split-plan choice (bw_abi.cu default_plan).

    python tools/sweep_split.py --n 34 --out gpurun_out/split_n34.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1607_01039_b200 import _lib  # noqa: E402


def split(r, q, a, k2):
    return r | ((q + 1) << 4) | (a << 8) | (k2 << 12)


def candidates(n):
    """(name, plan) pairs: the default plan, then 3-pass plans whose middle
    pass is one run and whose last pass takes the low rows {w0..w0+a-1} and
    the top rows."""
    out = [("default", None)]
    for w0 in (13, 14):
        h = n - w0
        for r_split in (9, 10):
            r_mid = h - r_split
            if not 6 <= r_mid <= 10:
                continue
            for a in range(1, r_split):
                k2 = n - (r_split - a)
                out.append((f"{w0} + [{w0 + a},{k2}) + split {{{w0}..{w0 + a - 1}}}u[{k2},{n})",
                            [w0, split(r_split, 1, a, k2), r_mid]))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=34)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    n = a.n
    L = _lib.lib()
    x = torch.zeros(1 << n, dtype=torch.int64, device="cuda")
    sh = torch.cuda.current_stream().cuda_stream
    gb = 16.0 * (1 << n) / 1e9
    res = []
    for name, plan in candidates(n):
        if plan is None:
            os.environ.pop("BW_PLAN", None)
        else:
            os.environ["BW_PLAN"] = ",".join(str(v) for v in plan)
        npasses = L.bw_plan_npasses(n)
        _lib.check(L.bw_fwht_i64(x.data_ptr(), n, sh, None))  # warm-up (and attributes)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(npasses + 1)]
        per = [0.0] * npasses
        for _ in range(a.reps):
            for i in range(npasses):
                ev[i].record()
                _lib.check(L.bw_fwht_i64_pass(x.data_ptr(), n, i, sh))
            ev[npasses].record()
            torch.cuda.synchronize()
            for i in range(npasses):
                per[i] += ev[i].elapsed_time(ev[i + 1]) / a.reps
        total = sum(per)
        res.append({"name": name, "plan": plan, "total_ms": round(total, 3),
                    "passes_ms": [round(t, 3) for t in per],
                    "passes_tbs": [round(gb / (t / 1e3) / 1e3, 3) for t in per]})
        print(json.dumps(res[-1]), flush=True)
    best = min(res, key=lambda r: r["total_ms"])
    print("best:", json.dumps(best))
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"n": n, "device": torch.cuda.get_device_name(), "plans": res}, f, indent=1)


if __name__ == "__main__":
    main()
