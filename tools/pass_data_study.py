"""Per-pass HBM rate of the default plan as a function of the DATA in the
signal: zeros (what tools/sweep_shapes.py and the walks measure), the
config-4 +-1 signal, the config-5 noisy signal, and uniform random 64-bit
values.  Every repetition regenerates the input and runs the passes in plan
order (each timed with CUDA events), as one real transform does.

    python tools/pass_data_study.py --n 34 [--plan 14,...] [--reps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1607_01039_b200 import _lib, sharded, signals  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=34)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--plan", default=None, help="BW_PLAN override")
    ap.add_argument("--kinds", default="zeros,pm1,noisy,random")
    a = ap.parse_args()
    if a.plan:
        os.environ["BW_PLAN"] = a.plan
    n = a.n
    L = _lib.lib()
    x = torch.empty(1 << n, dtype=torch.int64, device="cuda")
    sh = torch.cuda.current_stream().cuda_stream
    npasses = L.bw_plan_npasses(n)
    plan = sharded.plan(n, 0)
    gb = 16.0 * (1 << n) / 1e9
    out = {"n": n, "plan": plan["passes"], "kinds": {}}
    for kind in a.kinds.split(","):
        rows = []
        for _ in range(a.reps + 1):
            if kind == "zeros":
                x.zero_()
            elif kind == "pm1":
                signals.generate(signals.config(4, n), x)
            elif kind == "noisy":
                signals.generate(signals.config(5, n), x)
            else:  # uniform in [-2^62, 2^62]: full-entropy words
                signals.generate(signals.SignalSpec(n, _lib.GEN_UNIFORM, 7, (1 << 62,)), x)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(npasses + 1)]
            for i in range(npasses):
                ev[i].record()
                _lib.check(L.bw_fwht_i64_pass(x.data_ptr(), n, i, sh))
            ev[-1].record()
            torch.cuda.synchronize()
            rows.append([ev[i].elapsed_time(ev[i + 1]) for i in range(npasses)])
        rows = rows[1:]  # the first repetition warms up
        ms = [sum(r[i] for r in rows) / len(rows) for i in range(npasses)]
        out["kinds"][kind] = {"ms": [round(v, 3) for v in ms], "tbs": [round(gb / v, 3) for v in ms],
                              "total_ms": round(sum(ms), 3)}
        print(kind, out["kinds"][kind], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
