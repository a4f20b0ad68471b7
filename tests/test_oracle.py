"""Pin the CPU oracle (oracle/oracle_np.py, oracle/bw_oracle.c) against the
reference's own outputs (tests/golden, made by tests/golden/make_golden.py
from an import of /root/reference).  CPU only."""

import ctypes
import hashlib
import os

import numpy as np
import pytest

from oracle import oracle_np

REF_SRC = "/root/reference/pkg/src"


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()


def c_fwht(coracle, x):
    y = np.ascontiguousarray(x, dtype=np.int64).copy()
    bf = coracle.oracle_fwht_i64(y.ctypes.data, int(y.size).bit_length() - 1)
    return y, bf


def c_gen(coracle, kind, seed, params, base, count, threads=4):
    out = np.empty(count, dtype=np.int64)
    arr = (ctypes.c_uint64 * max(1, len(params)))(*[int(p) for p in params])
    assert coracle.oracle_gen_i64(out.ctypes.data, base, count, kind, seed, arr, len(params), threads) == 0
    return out


def test_known_answers(golden, coracle):
    for case in golden["known"]:
        x = np.array(case["x"], dtype=np.int64)
        y = x.copy()
        oracle_np.fwht_array(y)
        assert y.tolist() == case["y"]
        assert c_fwht(coracle, x)[0].tolist() == case["y"]


def test_c01_vectors_and_bruteforce(golden_npz, coracle):
    z = golden_npz("c01_vectors.npz")
    count = len([k for k in z.files if k.startswith("x")])
    assert count == 44
    for i in range(count):
        x, y = z[f"x{i}"], z[f"y{i}"]
        ynp = x.copy()
        oracle_np.fwht_array(ynp)
        assert np.array_equal(ynp, y)
        assert np.array_equal(c_fwht(coracle, x)[0], y)
        if x.size <= 256:
            assert np.array_equal(oracle_np.wht_bruteforce(x), y)


def test_fixture_arrays(golden_npz, coracle):
    z = golden_npz("fwht_n12_16.npz")
    for n in (12, 14, 16):
        y, bf = c_fwht(coracle, z[f"x{n}"])
        assert np.array_equal(y, z[f"y{n}"])
        assert bf == n << (n - 1)


def test_generated_inputs_match_reference_digests(golden, coracle):
    for case in golden["gen_cases"]:
        n = case["n"]
        x = oracle_np.gen(case["kind"], case["seed"], case["params"], 0, 1 << n)
        assert digest(x) == case["x_sha256"]
        xc = c_gen(coracle, case["kind"], case["seed"], case["params"], 0, 1 << n)
        assert np.array_equal(x, xc)
        y, bf = c_fwht(coracle, x)
        assert digest(y) == case["y_sha256"]
        assert bf == case["butterflies"]


def test_wraparound_matches_reference(golden_npz, coracle):
    z = golden_npz("wrap_n10.npz")
    assert np.array_equal(c_fwht(coracle, z["x"])[0], z["y"])


def test_parallel_plans_match_reference(golden):
    for case in golden["plans"]:
        phases = oracle_np.plan_parallel(case["n"], case["p"])
        ref = case["phases"]
        assert len(phases) == len(ref)
        assert ref[0]["stage"] is None and [tuple(c) for c in ref[0]["chunks"]] == phases[0][1]
        for (stage, loads), rp in zip(phases[1:], ref[1:]):
            assert stage == rp["stage"]
            assert [list(w) for w in loads] == rp["workloads"]


def test_parallel_results_match_reference(golden, coracle):
    for case in golden["parallel"]:
        n, p = case["n"], case["p"]
        x = oracle_np.gen(2, case["seed"], [1 << 20], 0, 1 << n)
        a = x.copy()
        oracle_np.run_parallel(a, n, p)
        assert digest(a) == case["y_sha256"]
        b = x.copy()
        assert coracle.oracle_run_parallel_i64(b.ctypes.data, n, p) == 0
        assert digest(b) == case["y_sha256"]


def test_extract_matches_reference(golden):
    for case in golden["extract"]:
        got = oracle_np.extract_above(np.array(case["data"], dtype=np.int64), case["tau"])
        assert [list(h) for h in got] == case["hits"]


def test_extract_float64_matches_reference(golden):
    g = golden["extract_f64"]
    data = np.array(g["data"], dtype=np.float64)
    for case in g["cases"]:
        got = oracle_np.extract_above(data, case["tau"])
        assert [[i, v] for i, v in got] == case["hits"]
        assert all(isinstance(v, float) for _, v in got)


def test_config_constructions(golden):
    from paper_1607_01039_b200.signals import config

    for key, idx, tau_shift in (("config3_n22", 3, 8), ("config5_n22", 5, 12)):
        spec = config(idx, n=22)
        x = oracle_np.gen(spec.kind, spec.seed, list(spec.params), 0, 1 << 22)
        oracle_np.fwht_array(x)
        assert digest(x) == golden[key]["y_sha256"]
        idxs, vals = oracle_np.extract_gt_by_index(x, golden[key]["tau"])
        ref = sorted(golden[key]["hits"])
        assert [[int(i), int(v)] for i, v in zip(idxs, vals)] == ref
        assert sorted(spec.masks) == sorted(i for i, _ in ref)


def test_fold_identity_matches_reference(golden_npz, coracle):
    z = golden_npz("fold_16_8.npz")
    rows = z["rows"]
    assert np.array_equal(oracle_np.row_space(rows), z["row_space"])
    x = oracle_np.gen(1, 77, [], 0, 1 << 16)
    assert np.array_equal(oracle_np.fold(x, rows), z["folded"])
    cols = oracle_np.column_masks(rows).astype(np.uint64)
    out = np.empty(1 << 8, dtype=np.int64)
    assert coracle.oracle_fold_i64(None, 16, cols.ctypes.data, 8, 1, 77, None, 0, 3, out.ctypes.data) == 0
    assert np.array_equal(out, z["folded"])
    # WHT(fold(x)) == WHT(x)[row_space] (subspace.py:1-11)
    w = x.copy()
    oracle_np.fwht_array(w)
    assert np.array_equal(w[z["row_space"]], z["wfolded"])


def test_random_full_rank_matches_reference(golden_npz):
    z = golden_npz("fold_16_8.npz")
    assert np.array_equal(oracle_np.random_full_rank(16, 8, 7), z["rows"])


def test_inverse_matches_reference(golden):
    for case in golden["inverse"]:
        assert oracle_np.inverse_wht(np.array(case["w"], dtype=np.int64)).tolist() == case["x"]


def test_float64_bitwise(golden_npz, coracle):
    z = golden_npz("float64.npz")
    for n in (4, 10, 15):
        y = z[f"x{n}"].copy()
        oracle_np.fwht_array(y)
        assert np.array_equal(y.view(np.int64), z[f"y{n}"].view(np.int64))
        yc = z[f"x{n}"].copy()
        coracle.oracle_fwht_f64(yc.ctypes.data, n)
        assert np.array_equal(yc.view(np.int64), z[f"y{n}"].view(np.int64))


def test_bound_edges(golden, coracle):
    for case in golden["bound_edges"]:
        data = np.array([case["value"], 0], dtype=np.int64)
        viol = coracle.oracle_bound_violated(data.ctypes.data, 2, case["n"], None)
        assert bool(viol) == (not case["ok"])
        if case["ok"]:
            oracle_np.check_magnitude_bound(data, case["n"])
        else:
            with pytest.raises(oracle_np.OracleOverflow):
                oracle_np.check_magnitude_bound(data, case["n"])


def test_c_extract_matches_numpy(coracle):
    rng = np.random.default_rng(5)
    x = rng.integers(-1000, 1000, 1 << 12).astype(np.int64)
    x[7] = np.iinfo(np.int64).min
    idx = np.empty(1 << 12, dtype=np.int64)
    val = np.empty(1 << 12, dtype=np.int64)
    h = coracle.oracle_extract_ge_i64(x.ctypes.data, x.size, 901, idx.ctypes.data, val.ctypes.data, 1 << 12)
    ref_i, ref_v = oracle_np.extract_gt_by_index(x, 900)
    assert h == ref_i.size and np.array_equal(idx[:h], ref_i) and np.array_equal(val[:h], ref_v)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not mounted (GPU box)")
def test_oracle_against_live_reference():
    """Extra pin when the reference is importable (build container only)."""
    import subprocess
    import sys

    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r);"
        "from bigwht.core import fwht_array; from oracle import oracle_np;"
        "x = oracle_np.gen(2, 5, [1<<20], 0, 1<<19); a = x.copy(); b = x.copy();"
        "fwht_array(a); oracle_np.fwht_array(b); assert np.array_equal(a, b); print('ok')"
    ) % (REF_SRC, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr


def test_subspace_host_helpers_match_reference(golden_npz):
    """The product's host-side map helpers restate subspace.py exactly."""
    from paper_1607_01039_b200 import subspace

    z = golden_npz("fold_16_8.npz")
    rows = subspace.random_full_rank(16, 8, 7)
    assert np.array_equal(rows, z["rows"])
    assert np.array_equal(subspace.row_space(rows), z["row_space"])
    assert subspace.column_masks(rows) == [int(c) for c in oracle_np.column_masks(rows)]
    assert subspace.gf2_rank(rows) == 8


def test_product_plan_parallel_matches_reference(golden):
    """The product's host-side plan objects (paper_1607_01039_b200.parallel)
    restate parallel.py:87-147 exactly."""
    from paper_1607_01039_b200 import errors, parallel

    for case in golden["plans"]:
        plan = parallel.plan_parallel(case["n"], case["p"])
        ref = case["phases"]
        assert len(plan.phases) == len(ref)
        assert ref[0]["stage"] is None and [list(c) for c in plan.phases[0].chunks] == [list(c) for c in ref[0]["chunks"]]
        for ph, rp in zip(plan.phases[1:], ref[1:]):
            assert ph.stage == rp["stage"]
            assert [[w.start, w.stride, w.count] for w in ph.workloads] == rp["workloads"]
        parallel.check_disjoint(plan)
        n = case["n"]
        assert parallel.total_butterflies(plan) == n << (n - 1)
    for n, p in ((4, 0), (4, 4), (1, 1)):
        with pytest.raises(errors.InvalidWorkerCount):
            parallel.plan_parallel(n, p)
    with pytest.raises(errors.InvalidWorkerCount):
        parallel.log2_workers_for(3)
    bad = parallel.plan_parallel(6, 2)
    broken = parallel.ParallelPlan(bad.log2_dim, bad.log2_workers,
                                   bad.phases[:1] + (parallel.Phase(stage=4, workloads=bad.phases[1].workloads[:1] * 2),))
    with pytest.raises(errors.ValidationError):
        parallel.check_disjoint(broken)
