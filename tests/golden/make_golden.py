"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Inputs are either literal vectors from the reference's own tests, seeded
numpy draws (stored), or this repository's counter-based generator
(regenerable anywhere, so only output digests are stored for big n).
Every output below is produced by the reference's functions:
bigwht.core.fwht_array / fwht_inplace / wht_bruteforce / inverse_wht_inplace,
bigwht.parallel.plan_parallel / run_parallel, bigwht.noisy.extract_above,
bigwht.subspace.random_full_rank / row_space / fold.
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, "/root/reference/pkg/src")

from bigwht.core import Domain, Signal, fwht_array, fwht_inplace, inverse_wht_inplace, wht_bruteforce  # noqa: E402
from bigwht.noisy import extract_above  # noqa: E402
from bigwht.parallel import plan_parallel, run_parallel  # noqa: E402
from bigwht.subspace import fold, random_full_rank, row_space  # noqa: E402

from oracle import oracle_np  # noqa: E402  (only for the counter-based inputs)


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()


def main():
    out = {}
    # 1. Known answers (test_core.py:44-55, 79-87).
    known = [[7], [3, 1], [1, 2, 3, 4], [1, 0, 0, 0], [1, 1, 1, 1]]
    out["known"] = [
        {"x": x, "y": fwht_inplace(Signal(np.array(x, dtype=np.int64))).data.tolist()} for x in known
    ]
    # 2. c01-style vectors: seed 2024, x in [-2^20, 2^20] inclusive
    #    (test_acceptance.py:33-50), 4 signals per n = 0..10, checked against
    #    both the fast path and the brute-force definition.
    rng = np.random.default_rng(2024)
    c01_x, c01_y = [], []
    for n in range(0, 11):
        for _ in range(4):
            x = rng.integers(-(1 << 20), (1 << 20) + 1, 1 << n).astype(np.int64)
            fast = fwht_inplace(Signal(x.copy())).data
            slow = wht_bruteforce(Signal(x.copy())).data
            assert np.array_equal(fast, slow)
            c01_x.append(x)
            c01_y.append(fast)
    np.savez_compressed(os.path.join(HERE, "c01_vectors.npz"),
                        **{f"x{i}": v for i, v in enumerate(c01_x)}, **{f"y{i}": v for i, v in enumerate(c01_y)})
    # 3. Larger arrays stored in full (n = 12, 14, 16).
    rng = np.random.default_rng(42)
    big = {}
    for n in (12, 14, 16):
        x = rng.integers(-(1 << 20), 1 << 20, 1 << n).astype(np.int64)
        y = x.copy()
        fwht_array(y)
        big[f"x{n}"], big[f"y{n}"] = x, y
    np.savez_compressed(os.path.join(HERE, "fwht_n12_16.npz"), **big)
    # 4. Counter-based inputs (regenerable) with reference output digests.
    gen_cases = []
    for n, kind, seed, params in [(18, 2, 18, [1 << 20]), (20, 1, 20, []), (21, 2, 21, [1 << 20]),
                                  (22, 2, 24, [1 << 20]), (24, 2, 24, [1 << 20])]:
        x = oracle_np.gen(kind, seed, params, 0, 1 << n)
        y = x.copy()
        bf = fwht_array(y)
        gen_cases.append({"n": n, "kind": kind, "seed": seed, "params": params,
                          "x_sha256": digest(x), "y_sha256": digest(y), "butterflies": bf,
                          "y_head": y[:8].tolist(), "y_tail": y[-8:].tolist()})
    out["gen_cases"] = gen_cases
    # 5. Wrap-around: the reference on unbounded int64 input (no bound check
    #    in fwht_array) -- arithmetic wraps mod 2^64.
    rng = np.random.default_rng(99)
    xw = rng.integers(np.iinfo(np.int64).min, np.iinfo(np.int64).max, 1 << 10, dtype=np.int64)
    yw = xw.copy()
    with np.errstate(over="ignore"):
        fwht_array(yw)
    np.savez_compressed(os.path.join(HERE, "wrap_n10.npz"), x=xw, y=yw)
    # 6. Parallel schedule (parallel.py:87-111) tuples and results.
    plans = []
    for n, p in [(6, 2), (12, 2), (20, 2), (9, 3), (5, 1)]:
        pl = plan_parallel(n, p)
        plans.append({"n": n, "p": p, "phases": [
            {"stage": ph.stage, "chunks": [list(c) for c in ph.chunks],
             "workloads": [[w.start, w.stride, w.count] for w in ph.workloads]} for ph in pl.phases]})
    out["plans"] = plans
    par = []
    for n, p in [(16, 1), (16, 2), (16, 3), (20, 3)]:
        x = oracle_np.gen(2, 1000 + n, [1 << 20], 0, 1 << n)
        y = run_parallel(Signal(x.copy()), plan_parallel(n, p)).data
        par.append({"n": n, "p": p, "seed": 1000 + n, "y_sha256": digest(y)})
    out["parallel"] = par
    # 7. Extraction (noisy.py:185-222).
    ext = []
    for data, tau in [([10, -2, -4, 0], 4), ([10, -2, -4, 0], 0), ([10, -2, -4, 0], 11), ([-5, 3, 5, -3], 3)]:
        hits = extract_above(Signal(np.array(data, dtype=np.int64), Domain.WALSH), tau)
        ext.append({"data": data, "tau": tau, "hits": [list(h) for h in hits]})
    rng = np.random.default_rng(12)
    data = rng.integers(-1000, 1000, 1 << 12).astype(np.int64)
    hits = extract_above(Signal(data, Domain.WALSH), 700)
    ext.append({"data": data.tolist(), "tau": 700, "hits": [list(h) for h in hits]})
    out["extract"] = ext
    # 7b. float64 Walsh-domain extraction (noisy.py:217-222: float values).
    rng = np.random.default_rng(13)
    data = rng.normal(scale=100.0, size=1 << 10)
    data[1], data[2], data[3] = -np.inf, -0.0, np.nan
    ext_f = []
    for tau in (0.0, 150.5, 250.0):
        hits = extract_above(Signal(data.copy(), Domain.WALSH), tau)
        ext_f.append({"tau": tau, "hits": [[int(i), float(v)] for i, v in hits]})
    out["extract_f64"] = {"data": [float(v) for v in data], "cases": ext_f}
    # 8. Noisy-secret construction of config 3 at n = 22 (threshold scaled
    #    by 2^-8 from 2^26): the reference recovers exactly the secret.
    from paper_1607_01039_b200.signals import config  # parameter derivation only (pure Python)
    spec = config(3, n=22)
    x = oracle_np.gen(spec.kind, spec.seed, list(spec.params), 0, 1 << 22)
    y = x.copy()
    fwht_array(y)
    tau = (1 << 26) >> 8
    hits = extract_above(Signal(y, Domain.WALSH), tau + 1)
    out["config3_n22"] = {"tau": tau, "hits": [list(h) for h in hits], "secret": spec.masks[0],
                          "y_sha256": digest(y)}
    spec5 = config(5, n=22)
    x5 = oracle_np.gen(spec5.kind, spec5.seed, list(spec5.params), 0, 1 << 22)
    y5 = x5.copy()
    fwht_array(y5)
    tau5 = (1 << 29) >> 12
    hits5 = extract_above(Signal(y5, Domain.WALSH), tau5 + 1)
    out["config5_n22"] = {"tau": tau5, "hits": [list(h) for h in hits5], "masks": spec5.masks,
                          "y_sha256": digest(y5)}
    # 9. Fold identity (subspace.py:150-161, test_acceptance.py:237-249).
    lmap = random_full_rank(16, 8, 7)
    xf = oracle_np.gen(1, 77, [], 0, 1 << 16)
    folded = fold(Signal(xf.copy()), lmap).data
    wf = folded.copy()
    fwht_array(wf)
    np.savez_compressed(os.path.join(HERE, "fold_16_8.npz"), rows=lmap.rows, row_space=row_space(lmap),
                        folded=folded, wfolded=wf)
    # 10. Inverse (core.py:147-173).
    inv = []
    for data in ([4, 0, 0, 0], [10, -2, -4, 0], [7]):
        inv.append({"w": data, "x": inverse_wht_inplace(Signal(np.array(data, dtype=np.int64), Domain.WALSH)).data.tolist()})
    out["inverse"] = inv
    # 11. float64 bitwise outputs.
    rng = np.random.default_rng(11)
    xf64 = {}
    for n in (4, 10, 15):
        x = rng.normal(size=1 << n)
        y = x.copy()
        fwht_array(y)
        xf64[f"x{n}"], xf64[f"y{n}"] = x, y
    np.savez_compressed(os.path.join(HERE, "float64.npz"), **xf64)
    # 12. Bound edges (test_core.py:129-136, 216-221).
    out["bound_edges"] = [
        {"value": 1 << 53, "n": 10, "ok": False},
        {"value": (1 << 53) - 1, "n": 10, "ok": True},
        {"value": 1 << 59, "n": 4, "ok": False},
        {"value": (1 << 59) - 1, "n": 4, "ok": True},
    ]
    # 13. A dataset written by the reference (dataset.py:427-446), kept as
    #     raw payload + sidecar for the format-compatibility pins.
    from bigwht import dataset as ref_dataset
    ds_path = os.path.join(HERE, "ref_dataset_n8.bin")
    for pth in (ds_path, ds_path + ".meta.json"):
        if os.path.exists(pth):
            os.remove(pth)
    ref_dataset.write_signal(ds_path, oracle_np.gen(2, 8, [1000], 0, 1 << 8), domain="time")
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote fixtures to", HERE)


if __name__ == "__main__":
    main()
