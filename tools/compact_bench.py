"""Per-pass and whole-call device times of the compact in-place plan
(bw_fwht_i64_compact) against the int64 plan, on a config input:

    python tools/compact_bench.py --config 4 [--n 32] [--reps 5] [--rows 9,9] [--w 14]

Each repetition regenerates the input (outside the events), then times with
CUDA events: the int64 plan pass by pass, the compact plan pass by pass
(pass 0 unchecked and checked), and the public calls fwht_array (compact
and int64) and fwht_inplace.  Bytes per pass: 12 (int64 -> int32), 8
(int32 -> int32), 12 (int32 -> int64) per point.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1607_01039_b200 as bw  # noqa: E402
from paper_1607_01039_b200 import _lib, signals  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--rows", default=None)
    ap.add_argument("--w", default=None)
    ap.add_argument("--tpc", default=None)
    a = ap.parse_args()
    if a.rows:
        os.environ["BW_COMPACT_ROWS"] = a.rows
    if a.w:
        os.environ["BW_COMPACT_W"] = a.w
    if a.tpc:
        os.environ["BW_COMPACT_TPC"] = a.tpc
    spec = signals.config(a.config, a.n)
    n = spec.n
    L = _lib.lib()
    sh = torch.cuda.current_stream().cuda_stream
    x = torch.empty(1 << n, dtype=torch.int64, device="cuda")
    flags = torch.zeros(1 << (n - 13), dtype=torch.int32, device="cuda")
    abort = torch.zeros(1, dtype=torch.int32, device="cuda")
    npl = L.bw_plan_npasses(n)
    ncp = L.bw_compact_npasses(n)
    pts = float(1 << n)
    cp_bytes = [12.0] + [8.0] * (ncp - 2) + [12.0]

    def timed(fns):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(fns) + 1)]
        ev[0].record()
        for i, f in enumerate(fns):
            f()
            ev[i + 1].record()
        torch.cuda.synchronize()
        return [ev[i].elapsed_time(ev[i + 1]) for i in range(len(fns))]

    rows = {"int64_passes": [], "compact_passes": [], "compact_checked_pass0": [], "fwht_array_compact": [],
            "fwht_array_int64": [], "fwht_inplace": []}
    for rep in range(a.reps + 1):
        signals.generate(spec, x)
        torch.cuda.synchronize()
        r1 = timed([lambda i=i: _lib.check(L.bw_fwht_i64_pass(x.data_ptr(), n, i, sh)) for i in range(npl)])
        signals.generate(spec, x)
        r2 = timed([lambda i=i: _lib.check(L.bw_fwht_i64_compact_pass(x.data_ptr(), n, i, 0, None, None, sh))
                    for i in range(ncp)])
        signals.generate(spec, x)
        flags.zero_()
        abort.zero_()
        r3 = timed([lambda: _lib.check(L.bw_fwht_i64_compact_pass(x.data_ptr(), n, 0, 1, flags.data_ptr(),
                                                                  abort.data_ptr(), sh))])
        assert abort.item() == 0
        signals.generate(spec, x)
        r4 = timed([lambda: bw.fwht_array(x, compact=True)])
        assert bw.core.last_compact
        signals.generate(spec, x)
        r5 = timed([lambda: bw.fwht_array(x, compact=False)])
        signals.generate(spec, x)
        r6 = timed([lambda: bw.fwht_inplace(bw.Signal(x))])
        if rep == 0:
            continue
        rows["int64_passes"].append(r1)
        rows["compact_passes"].append(r2)
        rows["compact_checked_pass0"].append(r3)
        rows["fwht_array_compact"].append(r4)
        rows["fwht_array_int64"].append(r5)
        rows["fwht_inplace"].append(r6)

    def mean(v):
        return [round(sum(c) / len(c), 3) for c in zip(*v)]

    out = {"n": n, "config": a.config, "rows_env": a.rows, "w_env": a.w, "tpc_env": a.tpc,
           "compact_limit": L.bw_compact_limit(n)}
    for k, v in rows.items():
        ms = mean(v)
        out[k] = {"ms": ms, "total_ms": round(sum(ms), 3)}
    out["int64_passes"]["tbs"] = [round(16 * pts / m / 1e9, 3) for m in out["int64_passes"]["ms"]]
    out["compact_passes"]["tbs"] = [round(b * pts / m / 1e9, 3) for b, m in zip(cp_bytes, out["compact_passes"]["ms"])]
    out["compact_passes"]["bytes_per_point"] = cp_bytes
    out["compact_checked_pass0"]["tbs"] = [round(12 * pts / out["compact_checked_pass0"]["ms"][0] / 1e9, 3)]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
