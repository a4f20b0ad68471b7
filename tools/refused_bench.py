"""What a signal the compact plan refuses pays for the attempt: fwht_array
(default: checked first pass, abort, exact restore, int64 plan) against
fwht_array(compact=False) on config 2's wide values at n = 26..32, and with a
single large value in the last tile of a +-1 signal (the worst case: every
tile but the last is written and restored).

    python tools/refused_bench.py [--n 32] [--reps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1607_01039_b200 as bw  # noqa: E402
from paper_1607_01039_b200 import signals  # noqa: E402


def timed(fn, prepare, reps):
    ts = []
    for r in range(reps + 1):
        prepare()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    return round(sorted(ts)[len(ts) // 2], 4)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    n = a.n
    x = torch.empty(1 << n, dtype=torch.int64, device="cuda")
    out = {"n": n}
    wide = signals.config(2, n)
    out["wide_default_ms"] = timed(lambda: bw.fwht_array(x), lambda: signals.generate(wide, x), a.reps)
    assert not bw.core.last_compact
    out["wide_int64_plan_ms"] = timed(lambda: bw.fwht_array(x, compact=False), lambda: signals.generate(wide, x), a.reps)
    pm1 = signals.config(4, n)

    def last_bad():
        signals.generate(pm1, x)
        x[-1] = 1 << 20

    out["last_tile_bad_default_ms"] = timed(lambda: bw.fwht_array(x), last_bad, a.reps)
    assert not bw.core.last_compact
    out["last_tile_bad_int64_plan_ms"] = timed(lambda: bw.fwht_array(x, compact=False), last_bad, a.reps)
    out["pm1_default_ms"] = timed(lambda: bw.fwht_array(x), lambda: signals.generate(pm1, x), a.reps)
    assert bw.core.last_compact
    print(json.dumps(out))


if __name__ == "__main__":
    main()
