"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden outputs and the CPU oracle.  int64 results must be bit-exact."""

import ctypes
import os
import hashlib

import numpy as np
import pytest
import torch

import paper_1607_01039_b200 as bw
from paper_1607_01039_b200 import _lib, errors, sharded, signals
from oracle import oracle_np

pytestmark = pytest.mark.gpu


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def gpu_fwht(x):
    t = dev(x)
    bf = bw.fwht_array(t)
    return t.cpu().numpy(), bf


def c_fwht(coracle, x):
    """The C oracle's transform of x: oracle_fwht_i64 (core.py:97-117) below
    n = 24; from there its restatement of the reference's run_parallel
    decomposition (parallel.py:162-198, one thread per worker) -- the same
    butterflies, so the same bits (tests/test_oracle.py pins both to the
    reference's digests), in a fraction of the single-threaded time."""
    y = np.ascontiguousarray(x, dtype=np.int64).copy()
    n = int(y.size).bit_length() - 1
    if n >= 24:
        p = max(1, min(4, (len(os.sched_getaffinity(0)) or 1).bit_length() - 1))
        assert coracle.oracle_run_parallel_i64(y.ctypes.data, n, p) == 0
    else:
        coracle.oracle_fwht_i64(y.ctypes.data, n)
    return y


def planned(x, bits):
    t = dev(x)
    n = int(t.numel()).bit_length() - 1
    if bits is None:
        _lib.check(_lib.lib().bw_fwht_i64_planned(t.data_ptr(), n, None, 0,
                                                  torch.cuda.current_stream().cuda_stream))
    else:
        arr = (ctypes.c_int * len(bits))(*bits)
        _lib.check(_lib.lib().bw_fwht_i64_planned(t.data_ptr(), n, arr, len(bits),
                                                  torch.cuda.current_stream().cuda_stream))
    return t.cpu().numpy()


# ------------------------------------------------------ reference pins ---

def test_device_is_b200():
    assert _lib.lib().bw_device_cc(0) == 100


def test_known_answers(golden):
    for case in golden["known"]:
        y, _ = gpu_fwht(np.array(case["x"], dtype=np.int64))
        assert y.tolist() == case["y"]
        sig = bw.fwht_inplace(bw.Signal(dev(np.array(case["x"], dtype=np.int64))))
        assert sig.data.cpu().tolist() == case["y"] and sig.domain == bw.Domain.WALSH


def test_c01_vectors(golden_npz):
    z = golden_npz("c01_vectors.npz")
    for i in range(44):
        y, bf = gpu_fwht(z[f"x{i}"])
        assert np.array_equal(y, z[f"y{i}"])
        n = z[f"x{i}"].size.bit_length() - 1
        assert bf == n << max(n - 1, 0)


def test_fixture_arrays(golden_npz):
    z = golden_npz("fwht_n12_16.npz")
    for n in (12, 14, 16):
        y, _ = gpu_fwht(z[f"x{n}"])
        assert np.array_equal(y, z[f"y{n}"])


def test_generated_cases_match_reference_digests(golden):
    for case in golden["gen_cases"]:
        n = case["n"]
        spec = signals.SignalSpec(n, case["kind"], case["seed"], tuple(case["params"]))
        t = signals.make(spec)
        assert digest(t.cpu().numpy()) == case["x_sha256"]
        assert bw.fwht_array(t) == case["butterflies"]
        assert digest(t.cpu().numpy()) == case["y_sha256"]


def test_wraparound_matches_reference(golden_npz):
    z = golden_npz("wrap_n10.npz")
    y, _ = gpu_fwht(z["x"])
    assert np.array_equal(y, z["y"])


def test_wraparound_large_n(coracle):
    """Unbounded int64 (the reference's fwht_array has no bound check and
    wraps mod 2^64): every pass kind must wrap identically."""
    rng = np.random.default_rng(3)
    for n in (14, 20, 24):
        x = rng.integers(np.iinfo(np.int64).min, np.iinfo(np.int64).max, 1 << n, dtype=np.int64)
        y, _ = gpu_fwht(x)
        assert np.array_equal(y, c_fwht(coracle, x))


def test_float64_bitwise(golden_npz):
    z = golden_npz("float64.npz")
    for n in (4, 10, 15):
        y, _ = gpu_fwht(z[f"x{n}"])
        assert np.array_equal(y.view(np.int64), z[f"y{n}"].view(np.int64))


@pytest.mark.parametrize("n", [13, 16, 20, 21, 24, 26])
def test_float64_bitwise_large(coracle, n):
    """float64 pass kernels (ascending stage order) vs numpy's order, bitwise."""
    rng = np.random.default_rng(8 + n)
    x = rng.normal(size=1 << n)
    y, _ = gpu_fwht(x)
    ref = x.copy()
    coracle.oracle_fwht_f64(ref.ctypes.data, n)
    assert np.array_equal(y.view(np.int64), ref.view(np.int64))


def test_numpy_buffers_are_staged_through_the_device(golden_npz):
    z = golden_npz("fwht_n12_16.npz")
    x = z["x14"].copy()
    assert bw.fwht_array(x) == 14 << 13
    assert np.array_equal(x, z["y14"])
    s = bw.fwht_inplace(bw.Signal(z["x12"].copy()))
    assert np.array_equal(s.data, z["y12"])


# -------------------------------------------------- oracle equivalence ---

@pytest.mark.parametrize("n", list(range(0, 27)))
def test_matches_oracle_every_n(coracle, n):
    x = oracle_np.gen(2, 500 + n, [1 << 20], 0, 1 << n)
    y, bf = gpu_fwht(x)
    assert np.array_equal(y, c_fwht(coracle, x))
    assert bf == n << max(n - 1, 0)


def test_every_pass_split_is_identical(coracle):
    """Block-size independence (test_external.py:120-129): every legal split
    of the high bits -- and every tile / cluster shape -- gives byte-identical
    output (entries r | (q + 1) << 4 force a cluster of 2^q CTAs)."""
    n = 22
    x = oracle_np.gen(2, 77, [1 << 20], 0, 1 << n)
    ref = c_fwht(coracle, x)
    assert np.array_equal(planned(x, None), ref)  # naive per-stage path
    plans = [[13, 9], [13, 1, 8], [13, 8, 1], [13, 3, 3, 3], [13, 5, 4], [13, 4, 5], [13, 6, 3], [13, 2, 7],
             [14, 8], [14, 4, 4], [14, 1, 7], [15, 7], [15, 2, 5], [13, 9 | (1 << 4)], [13, 9 | (2 << 4)],
             [14, 8 | (2 << 4)], [14, 8 | (3 << 4)], [15, 7 | (2 << 4)], [13, 6 | (2 << 4), 3],
             [13, 1, 1, 1, 1, 1, 1, 1, 1, 1]]
    for plan in plans:
        assert np.array_equal(planned(x, plan), ref), plan
    n = 24
    x = oracle_np.gen(1, 78, [], 0, 1 << n)
    ref = c_fwht(coracle, x)
    for plan in ([13, 10, 1], [13, 1, 10], [13, 6, 5], [14, 10], [15, 9], [14, 5, 5], [15, 4, 5],
                 [13, 10 | (1 << 4), 1], [14, 10 | (2 << 4)], [15, 9 | (3 << 4)]):
        assert np.array_equal(planned(x, plan), ref), plan


def split_entry(r, q, a, k2):
    return r | ((q + 1) << 4) | (a << 8) | (k2 << 12)


def test_split_row_plans_identical(coracle):
    """Split-row passes (rows [k, k+a) u [k2, k2+r-a), bw_layouts.h) on the
    device: 1- and 2-CTA tiles, the split pass first, in the middle or last,
    every split point a of a 10-row pass -- byte-identical to the oracle."""
    sp = split_entry
    cases = [
        (24, [[13, sp(6, 0, 3, 21), 5], [13, sp(9, 1, 4, 19), 2], [13, sp(10, 1, 1, 15), 1],
              [13, 2, sp(7, 0, 3, 20), 2], [14, sp(9, 1, 2, 17), 1], [13, sp(9, 1, 8, 21), 2]]),
        (27, [[14, sp(10, 1, a, 17 + a), 3] for a in range(1, 10)] +
             [[13, sp(9, 1, a, 18 + a), 5] for a in (1, 4, 8)] + [[13, sp(8, 0, 3, 22), 6]]),
    ]
    for n, plans in cases:
        x = oracle_np.gen(1, 90 + n, [], 0, 1 << n)
        ref = c_fwht(coracle, x)
        for plan in plans:
            assert np.array_equal(planned(x, plan), ref), plan


def test_split_row_pass_extraction(monkeypatch):
    """The fused extraction on a split-row pass (the hits' global indices come
    from the split address map).  Passes commute for int64, so the split pass
    runs last: pass 0, pass 2, then pass 1 with the |W| >= tau epilogue."""
    n = 24
    x = oracle_np.gen(2, 41, [1 << 10], 0, 1 << n)
    b = dev(x)
    bw.fwht_array(b)
    tau = 1 << 23  # ~4 sigma: about a thousand hits
    i2, v2 = bw.extract_ge(b, tau, cap=1 << 18)
    monkeypatch.setenv("BW_PLAN", ",".join(str(v) for v in [13, split_entry(6, 0, 3, 21), 5]))
    L = _lib.lib()
    a = dev(x)
    sh = torch.cuda.current_stream().cuda_stream
    cap = 1 << 18
    idx = torch.empty(cap, dtype=torch.int64, device="cuda")
    val = torch.empty(cap, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.check(L.bw_fwht_i64_pass(a.data_ptr(), n, 0, sh))
    _lib.check(L.bw_fwht_i64_pass(a.data_ptr(), n, 2, sh))
    _lib.check(L.bw_fwht_i64_pass_extract(a.data_ptr(), n, 1, tau, 0, idx.data_ptr(), val.data_ptr(), cap,
                                          cnt.data_ptr(), sh))
    assert torch.equal(a, b)
    k = int(cnt.item())
    assert k == i2.numel() and 10 < k < cap
    order = torch.argsort(idx[:k])
    assert torch.equal(idx[:k][order], i2) and torch.equal(val[:k][order], v2)


def narrow_run(x, plan=None, monkeypatch=None):
    """bw_fwht_i64_narrow on a copy of x: (result, used_narrow)."""
    t = dev(x)
    n = int(t.numel()).bit_length() - 1
    L = _lib.lib()
    need = int(L.bw_narrow_scratch_bytes(n))
    work = torch.empty(max(need, 16), dtype=torch.uint8, device="cuda")
    used = ctypes.c_int(-1)
    _lib.check(L.bw_fwht_i64_narrow(t.data_ptr(), n, work.data_ptr(), need, torch.cuda.current_stream().cuda_stream,
                                    ctypes.byref(used), None))
    return t.cpu().numpy(), used.value


def test_narrow_intermediates_match_oracle(coracle, monkeypatch):
    """int16 / int32 intermediates (k_pass_map, tile-major layouts): +-1 and
    small-magnitude signals at every default 2- and 3-pass plan up to n=28
    and on forced plans; wide inputs fall back to int64 -- all exact."""
    for n in (16, 18, 20, 22, 23, 24, 25, 26, 27, 28):
        has = _lib.lib().bw_narrow_npasses(n) > 0  # n = 25 plans a 4-CTA low pass: no narrow form
        for x, expect in ((oracle_np.gen(1, 300 + n, [], 0, 1 << n), has),
                          (np.random.default_rng(n).integers(-3, 4, 1 << n).astype(np.int64), has),
                          (oracle_np.gen(2, 310 + n, [1 << 20], 0, 1 << n), 0)):
            got, used = narrow_run(x)
            assert used == expect, (n, used)
            assert np.array_equal(got, c_fwht(coracle, x)), n
    for plan in ("13,5,6", "13,2,9", "14,4,6", "13,10,1", "13,1,10", "14,10", "13,6,5", "13,3,8", "14,9,1"):
        monkeypatch.setenv("BW_PLAN", plan)
        n = sum(int(v) for v in plan.split(","))
        x = oracle_np.gen(1, 77, [], 0, 1 << n)
        got, used = narrow_run(x)
        assert used == 1 and np.array_equal(got, c_fwht(coracle, x)), plan


def test_narrow_int16_edge(coracle):
    """The int16 check is exact: a low-pass output of +-32767 stays narrow,
    +-32768 falls back (the signal untouched by the failed first pass)."""
    n = 23  # plan 13 + 10: the low pass sums blocks of 2^13
    for sign in (1, -1):
        x = np.full(1 << n, sign, dtype=np.int64)
        x[: 1 << 13] = 4 * sign
        x[5] = 3 * sign  # block 0 sums to +-32767
        got, used = narrow_run(x)
        assert used == 1 and np.array_equal(got, c_fwht(coracle, x))
        x[5] = 4 * sign  # +-32768
        got, used = narrow_run(x)
        assert used == 0 and np.array_equal(got, c_fwht(coracle, x))


def test_fwht_array_narrow_option(coracle, monkeypatch):
    from paper_1607_01039_b200 import core

    x = oracle_np.gen(1, 5, [], 0, 1 << 24)
    for narrow, env, expect in ((True, "0", True), (None, "1", True), (None, "0", False), (False, "1", False)):
        monkeypatch.setenv("BW_NARROW", env)
        t = dev(x)
        bw.fwht_array(t, narrow=narrow)
        assert core.last_narrow == expect and np.array_equal(t.cpu().numpy(), c_fwht(coracle, x))


def test_involution_and_linearity():
    for n in (1, 5, 13, 14, 17, 23, 26):
        x = oracle_np.gen(2, 900 + n, [1000], 0, 1 << n)
        t = dev(x)
        bw.fwht_array(t)
        bw.fwht_array(t)
        assert np.array_equal(t.cpu().numpy(), x * (1 << n))
    n = 21
    a, b = 7, -3
    x = oracle_np.gen(2, 1, [500], 0, 1 << n)
    z = oracle_np.gen(2, 2, [500], 0, 1 << n)
    combo, _ = gpu_fwht(a * x + b * z)
    wx, _ = gpu_fwht(x)
    wz, _ = gpu_fwht(z)
    assert np.array_equal(combo, a * wx + b * wz)


# ------------------------------------------------------ error behaviour ---

def test_overflow_bound_raises_before_mutation(golden):
    for case in golden["bound_edges"]:
        n = case["n"]
        x = np.zeros(1 << n, dtype=np.int64)
        x[3] = case["value"]
        t = dev(x)
        if case["ok"]:
            bw.check_magnitude_bound(t, n)
            bw.fwht_inplace(bw.Signal(t))
        else:
            with pytest.raises(errors.OverflowBoundError):
                bw.fwht_inplace(bw.Signal(t))
            assert np.array_equal(t.cpu().numpy(), x)  # untouched
            h = x.copy()
            with pytest.raises(errors.OverflowBoundError):
                bw.fwht_inplace(bw.Signal(h))
            assert np.array_equal(h, x)
    # negative extreme: |INT64_MIN| = 2^63 never passes
    t = dev(np.array([np.iinfo(np.int64).min, 0], dtype=np.int64))
    with pytest.raises(errors.OverflowBoundError):
        bw.check_magnitude_bound(t, 1)


def test_argument_errors_before_launch():
    t = torch.arange(16, dtype=torch.int64, device="cuda")
    with pytest.raises(errors.BadArguments):
        bw.fwht_array(t[::2])
    with pytest.raises(errors.BadArguments):
        bw.fwht_array(t[:12])
    with pytest.raises(errors.BadArguments):
        bw.fwht_array(t.view(4, 4))
    with pytest.raises(errors.BadArguments):
        bw.fwht_array(t.to(torch.float32))  # int32 wraps like the reference; other dtypes are refused
    with pytest.raises(errors.BadArguments):
        bw.fwht_array(torch.arange(16, dtype=torch.int64))  # CPU tensor: no CPU path
    assert t.cpu().tolist() == list(range(16))


@pytest.mark.parametrize("n", [12, 13, 15, 19, 22, 26])
def test_misaligned_view_still_exact(coracle, n):
    """An odd-offset slice (8- but not 16-byte aligned) takes the 8-byte
    access layouts on the GPU and stays bit-exact (parallel.py:151 slices)."""
    base = torch.from_numpy(oracle_np.gen(2, 4 + n, [1 << 20], 0, (1 << n) + 1)).cuda()
    view = base[1:]
    ref = c_fwht(coracle, view.cpu().numpy())
    assert bw.fwht_array(view) == n << (n - 1)
    assert np.array_equal(view.cpu().numpy(), ref)
    assert base[0].item() == oracle_np.gen(2, 4 + n, [1 << 20], 0, 1)[0]  # the element before is untouched


def test_inverse(golden):
    for case in golden["inverse"]:
        s = bw.inverse_wht_inplace(bw.Signal(dev(np.array(case["w"], dtype=np.int64)), bw.Domain.WALSH))
        assert s.data.cpu().tolist() == case["x"] and s.domain == bw.Domain.TIME
    with pytest.raises(errors.BadArguments):
        bw.inverse_wht_inplace(bw.Signal(dev(np.array([1, 2, 3, 4], dtype=np.int64))))
    t = dev(np.array([1, 0, 0, 0], dtype=np.int64))
    with pytest.raises(errors.InexactDivision):
        bw.inverse_wht_inplace(bw.Signal(t, bw.Domain.WALSH))
    assert t.cpu().tolist() == [1, 0, 0, 0]
    for n in (1, 4, 9, 16, 22):
        x = oracle_np.gen(2, n, [9999], 0, 1 << n)
        s = bw.Signal(dev(x))
        bw.fwht_inplace(s)
        bw.inverse_wht_inplace(s)
        assert np.array_equal(s.data.cpu().numpy(), x)
    xf = np.random.default_rng(11).normal(size=1 << 10)
    s = bw.Signal(dev(xf))
    bw.fwht_inplace(s)
    bw.inverse_wht_inplace(s)
    np.testing.assert_allclose(s.data.cpu().numpy(), xf, rtol=1e-12, atol=1e-12)


# ----------------------------------------------------------- extraction ---

def test_extract_matches_reference(golden):
    for case in golden["extract"]:
        sig = bw.Signal(dev(np.array(case["data"], dtype=np.int64)), bw.Domain.WALSH)
        assert [list(h) for h in bw.extract_above(sig, case["tau"])] == case["hits"]


def test_extract_config_constructions(golden):
    for key, idx in (("config3_n22", 3), ("config5_n22", 5)):
        spec = signals.config(idx, n=22)
        t = signals.make(spec)
        bw.fwht_array(t)
        assert digest(t.cpu().numpy()) == golden[key]["y_sha256"]
        i, v = bw.extract_gt(t, golden[key]["tau"])
        assert [[a, b] for a, b in zip(i.tolist(), v.tolist())] == sorted(golden[key]["hits"])


def test_extract_dense_and_edges(coracle):
    rng = np.random.default_rng(21)
    for n in (0, 3, 16, 17, 20):
        x = rng.integers(-1000, 1000, 1 << n).astype(np.int64)
        if n >= 3:
            x[5] = np.iinfo(np.int64).min
        for tau in (0, 1, 500, 999, 1001):
            i, v = bw.extract_ge(dev(x), tau, cap=16)  # forces the capacity retry
            ri, rv = oracle_np.extract_gt_by_index(x, tau - 1) if tau > 0 else (np.arange(x.size), x)
            assert np.array_equal(i.cpu().numpy(), ri) and np.array_equal(v.cpu().numpy(), rv), (n, tau)


def test_extract_float64_matches_golden(golden):
    g = golden["extract_f64"]
    x = np.array(g["data"], dtype=np.float64)
    sig = bw.Signal(dev(x), bw.Domain.WALSH)
    for case in g["cases"]:
        assert [[i, v] for i, v in bw.extract_above(sig, case["tau"])] == case["hits"]


def test_extract_float64_matches_reference_semantics():
    """float64 Walsh-domain extraction (noisy.py:185-222 on a float array):
    |x| >= tau in double, NaN never hits, -0.0 / inf handled like numpy,
    float values, sorted by (-|x|, index)."""
    rng = np.random.default_rng(22)
    for n in (4, 16, 19):
        x = rng.normal(scale=100.0, size=1 << n)
        x[1] = np.nan
        x[2] = -np.inf
        x[3] = -0.0
        sig = bw.Signal(dev(x), bw.Domain.WALSH)
        for tau in (0.0, 50.0, 150.5, 1e300):
            got = bw.extract_above(sig, tau)
            assert got == oracle_np.extract_above(x, tau), (n, tau)
        i, v = bw.extract_ge(dev(x), 120.0, cap=4)  # capacity retry, index order, float values
        sel = np.nonzero(np.abs(x) >= 120.0)[0]
        assert np.array_equal(i.cpu().numpy(), sel) and v.dtype == torch.float64
        assert np.array_equal(v.cpu().numpy().view(np.int64), x[sel].view(np.int64))


# ----------------------------------------------------------- generators ---

def test_generators_match_oracle(coracle):
    for idx in (1, 2, 3, 5):
        spec = signals.config(idx, n=18)
        t = signals.make(spec)
        ref = oracle_np.gen(spec.kind, spec.seed, list(spec.params), 0, 1 << 18)
        assert np.array_equal(t.cpu().numpy(), ref)
        part = torch.empty(1000, dtype=torch.int64, device="cuda")
        signals.generate(spec, part, base=12345)
        assert np.array_equal(part.cpu().numpy(), oracle_np.gen(spec.kind, spec.seed, list(spec.params), 12345, 1000))


# ------------------------------------------------- multi-shard emulation ---

@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_sharded_emulation(coracle, P):
    """P shards as P buffers on one device, same kernels as the multi-GPU
    path (parallel.py: parallel == serial, test_acceptance.py:77-105)."""
    for n in (4, 12, 20):
        if n - (P.bit_length() - 1) < 1:
            continue
        x = oracle_np.gen(2, 60 + n, [1 << 20], 0, 1 << n)
        ref = c_fwht(coracle, x)
        shards = [dev(c) for c in np.split(x, P)]
        assert sharded.fwht_shards(shards) == n << (n - 1)
        assert np.array_equal(np.concatenate([s.cpu().numpy() for s in shards]), ref)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_sharded_fused_emulation(coracle, P):
    """The fused plan (K6' = last local pass + cross-shard stages in one
    kernel) on P buffers of one device equals the serial transform."""
    p = P.bit_length() - 1
    for nl in (14, 16, 19, 20, 22, 24):
        n = nl + p
        x = oracle_np.gen(2, 70 + n, [1 << 20], 0, 1 << n)
        ref = c_fwht(coracle, x)
        shards = [dev(c) for c in np.split(x, P)]
        assert sharded.fwht_shards(shards, fused=True) == n << (n - 1)
        assert np.array_equal(np.concatenate([s.cpu().numpy() for s in shards]), ref), (P, nl)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_sharded_fused_extraction_emulation(P):
    """Extraction fused into the cross-shard pass (K6' + |W| >= tau) on P
    buffers of one device equals a full transform + ordered extraction."""
    p = P.bit_length() - 1
    for nl in (14, 18, 21):
        n = nl + p
        tau = int(3.5 * 591 * 2 ** (n / 2))  # ~3.5 sigma of a transform of uniform +-1024: a few hits per 2^13
        x = oracle_np.gen(2, 60 + n, [1 << 10], 0, 1 << n)
        whole = dev(x)
        bw.fwht_array(whole)
        i2, v2 = bw.extract_ge(whole, tau, cap=1 << 18)
        shards = [dev(c) for c in np.split(x, P)]
        i1, v1 = sharded.fwht_shards_extract_ge(shards, tau, cap=1 << 18)
        assert torch.equal(torch.cat(shards), whole), (P, nl)
        assert i1.numel() > 0 and torch.equal(i1, i2) and torch.equal(v1, v2), (P, nl, i1.numel(), i2.numel())


@pytest.mark.parametrize("P", [2, 4, 8])
def test_sharded_narrow_emulation(coracle, P):
    """Narrow-wire exchange (int8 cross stages first, then widening local
    transforms) on P buffers of one device: +-1 signals, values at the wire
    limit +-(127 >> log2 P), and one value over it (falls back to fused)."""
    p = P.bit_length() - 1
    lim = 127 >> p
    rng = np.random.default_rng(P)
    for nl in (8, 13, 14, 18, 22):
        n = nl + p
        cases = [oracle_np.gen(1, 80 + n, [], 0, 1 << n),
                 rng.choice(np.array([-lim, lim, 0, 1], dtype=np.int64), 1 << n)]
        over = cases[1].copy()
        over[(1 << n) - 3] = lim + 1
        cases.append(over)
        for x in cases:
            ref = c_fwht(coracle, x)
            shards = [dev(c) for c in np.split(x, P)]
            assert sharded.fwht_shards(shards, narrow=True) == n << (n - 1)
            assert np.array_equal(np.concatenate([s.cpu().numpy() for s in shards]), ref), (P, nl)


def test_narrow_primitives():
    """bw_pack_narrow_i64 flags exactly the values over 127 >> log2 P;
    bw_fwht_widen on int8 / int16 / int32 sources equals the int64 transform."""
    L = _lib.lib()
    sh = torch.cuda.current_stream().cuda_stream
    for p in (1, 2, 3):
        lim = 127 >> p
        for bad_val, flagged in ((lim, 0), (-lim, 0), (lim + 1, 1), (-lim - 1, 1)):
            x = torch.zeros(1 << 12, dtype=torch.int64, device="cuda")
            x[777] = bad_val
            out = torch.empty(1 << 12, dtype=torch.int8, device="cuda")
            flag = torch.zeros(1, dtype=torch.int32, device="cuda")
            _lib.check(L.bw_pack_narrow_i64(x.data_ptr(), x.numel(), 1, p, out.data_ptr(), flag.data_ptr(), sh))
            assert int(flag.item()) == flagged, (p, bad_val)
            if not flagged:
                assert torch.equal(out.to(torch.int64), x)
    for dt, hi in ((torch.int8, 127), (torch.int16, 32767), (torch.int32, 1 << 30)):
        for n in (5, 13, 16, 21):
            src = torch.randint(-hi, hi + 1, (1 << n,), dtype=torch.int64, device="cuda")
            ref = src.clone()
            bw.fwht_array(ref)
            dst = torch.empty_like(ref)
            s8 = src.to(dt)
            _lib.check(L.bw_fwht_widen(s8.data_ptr(), s8.element_size(), dst.data_ptr(), n, sh, None))
            assert torch.equal(dst, ref), (dt, n)


@pytest.mark.parametrize("n,p", [(2, 1), (4, 3), (12, 2), (16, 1), (16, 3), (17, 4), (20, 2), (24, 3)])
def test_run_parallel_drop_in(coracle, n, p):
    """parallel.run_parallel (parallel.py:162-198) on the GPU equals the
    serial transform (test_parallel.py:104-129), calls on_phase_complete
    for every phase in order and flips the domain."""
    x = oracle_np.gen(2, 90 + n, [1 << 20], 0, 1 << n)
    ref = c_fwht(coracle, x)
    sig = bw.Signal(dev(x))
    seen = []
    out = bw.run_parallel(sig, bw.plan_parallel(n, p), on_phase_complete=seen.append)
    assert out is sig and sig.domain == bw.Domain.WALSH
    assert seen == list(range(p + 1))
    assert np.array_equal(sig.data.cpu().numpy(), ref)


def test_run_parallel_float64_and_host_buffers(coracle):
    rng = np.random.default_rng(31)
    x = rng.normal(size=1 << 18)
    ref = x.copy()
    coracle.oracle_fwht_f64(ref.ctypes.data, 18)
    sig = bw.Signal(x.copy())  # numpy buffer: staged through the device, written back
    bw.run_parallel(sig, bw.plan_parallel(18, 2))
    assert np.array_equal(sig.data.view(np.int64), ref.view(np.int64))
    with pytest.raises(errors.BadArguments):
        bw.run_parallel(bw.Signal(dev(np.zeros(16, dtype=np.int64))), bw.plan_parallel(5, 1))
    big = np.zeros(1 << 10, dtype=np.int64)
    big[0] = 1 << 60
    with pytest.raises(errors.OverflowBoundError):
        bw.run_parallel(bw.Signal(dev(big)), bw.plan_parallel(10, 1))


def test_xshard_strided_matches_per_pointer():
    x = oracle_np.gen(2, 9, [1 << 20], 0, 1 << 16)
    a = dev(x)
    b = dev(x)
    _lib.check(_lib.lib().bw_xshard_strided_i64(a.data_ptr(), 1 << 13, 3, 0, 1 << 13,
                                                torch.cuda.current_stream().cuda_stream))
    sharded.xshard(list(b.view(8, 1 << 13).unbind(0)))
    assert torch.equal(a, b)


# ------------------------------------------------- oracle + energy (GPU) ---

def test_bruteforce_matches_reference(golden_npz, golden):
    z = golden_npz("c01_vectors.npz")
    for i in range(44):
        x = z[f"x{i}"]
        sig = bw.Signal(dev(x))
        out = bw.wht_bruteforce(sig)
        assert np.array_equal(out.data.cpu().numpy(), z[f"y{i}"])
        assert out.domain == bw.Domain.WALSH and np.array_equal(sig.data.cpu().numpy(), x)
    # numpy input returns numpy (reference type), known answer (test_core.py:48-55)
    assert bw.wht_bruteforce(bw.Signal(np.array([1, 2, 3, 4], dtype=np.int64))).data.tolist() == [10, -2, -4, 0]
    with pytest.raises(errors.OracleTooLarge):
        bw.wht_bruteforce(bw.Signal(dev(np.zeros(16, dtype=np.int64))), limit=3)
    with pytest.raises(errors.OverflowBoundError):
        bw.wht_bruteforce(bw.Signal(dev(np.array([1 << 61, 0, 0, 0], dtype=np.int64))))
    x = oracle_np.gen(2, 5, [1 << 20], 0, 1 << 14)
    assert np.array_equal(bw.wht_bruteforce(bw.Signal(dev(x))).data.cpu().numpy(), oracle_np.wht_bruteforce(x))


def test_parseval_exact():
    E = bw.parseval_energy
    assert E(bw.Signal(dev(np.array([1, 1, 1, 1], dtype=np.int64)))) == 4
    assert E(bw.Signal(dev(np.array([10, -2, -4, 0], dtype=np.int64)))) == 120
    assert E(bw.Signal(dev(np.zeros(8, dtype=np.int64)))) == 0
    assert E(bw.Signal(dev(np.array([1 << 40] * 4, dtype=np.int64)))) == 4 * (1 << 80)  # beyond int64
    assert E(bw.Signal(dev(np.array([np.iinfo(np.int64).min, 3], dtype=np.int64)))) == (1 << 126) + 9
    for n in (0, 3, 8, 14, 20):
        x = oracle_np.gen(2, 70 + n, [1 << 20], 0, 1 << n)
        sig = bw.Signal(dev(x))
        before = E(sig)
        assert before == sum(int(v) * int(v) for v in x.tolist())
        bw.fwht_inplace(sig)
        assert E(sig) == before * (1 << n)  # Parseval, exactly (test_core.py:195-202)
    xf = np.random.default_rng(6).normal(size=1 << 10)
    sig = bw.Signal(dev(xf))
    before = E(sig)
    bw.fwht_inplace(sig)
    assert E(sig) == pytest.approx(before * (1 << 10), rel=1e-9)


def test_fused_extraction_matches_two_step():
    """Extraction fused into the last pass == transform then ordered
    extraction, for sparse hits, many hits (> 2048: fallback) and tau = 0."""
    for n, tau in ((14, 0), (16, 3000), (20, 1 << 14), (22, 1 << 17), (23, 1 << 30), (24, 25000)):
        x = oracle_np.gen(2, 40 + n, [1 << 10], 0, 1 << n)
        a, b = dev(x), dev(x)
        i1, v1 = bw.fwht_extract_ge(a, tau, cap=1 << 18)
        bw.fwht_array(b)
        i2, v2 = bw.extract_ge(b, tau, cap=1 << 18)
        assert torch.equal(a, b), n
        assert torch.equal(i1, i2) and torch.equal(v1, v2), (n, tau, i1.numel())
    # too many hits for the capacity: still complete and ordered
    x = oracle_np.gen(2, 3, [1 << 10], 0, 1 << 18)
    a, b = dev(x), dev(x)
    i1, v1 = bw.fwht_extract_ge(a, 0, cap=16)
    bw.fwht_array(b)
    assert torch.equal(i1, torch.arange(1 << 18, device="cuda")) and torch.equal(v1, b)


def test_fused_extraction_configs(golden):
    for key, idx in (("config3_n22", 3), ("config5_n22", 5)):
        spec = signals.config(idx, n=22)
        t = signals.make(spec)
        i, v = bw.fwht_extract_gt(t, golden[key]["tau"])
        assert digest(t.cpu().numpy()) == golden[key]["y_sha256"]
        assert [[a, b] for a, b in zip(i.tolist(), v.tolist())] == sorted(golden[key]["hits"])


def test_fold_matches_reference(golden_npz, coracle):
    from paper_1607_01039_b200 import subspace

    z = golden_npz("fold_16_8.npz")
    x = oracle_np.gen(1, 77, [], 0, 1 << 16)
    f = subspace.fold(bw.Signal(dev(x)), z["rows"])
    assert np.array_equal(f.data.cpu().numpy(), z["folded"])
    fn = subspace.fold(bw.Signal(x.copy()), z["rows"])  # numpy in, numpy out
    assert isinstance(fn.data, np.ndarray) and np.array_equal(fn.data, z["folded"])
    with pytest.raises(subspace.DimMismatch):
        subspace.fold(bw.Signal(dev(x[:1 << 15])), z["rows"])
    # large outputs (global atomics) and generated inputs
    for n, d_out, idx in ((22, 14, 2), (23, 13, 2), (24, 12, 2), (24, 20, 5), (20, 8, 3)):
        spec = signals.config(idx, n)
        rows = subspace.random_full_rank(n, d_out, n)
        want = np.empty(1 << d_out, dtype=np.int64)
        cols = oracle_np.column_masks(rows).astype(np.uint64)
        arr = (ctypes.c_uint64 * len(spec.params))(*spec.params) if spec.params else None
        assert coracle.oracle_fold_i64(None, n, cols.ctypes.data, d_out, spec.kind, spec.seed, arr,
                                       len(spec.params), 4, want.ctypes.data) == 0
        assert np.array_equal(subspace.fold_generated(spec, rows).cpu().numpy(), want)
        t = signals.make(spec)
        assert np.array_equal(subspace.fold(bw.Signal(t), rows).data.cpu().numpy(), want)


def test_fold_blocks_large_outputs(coracle, monkeypatch):
    """d_out > 14: the block fold (change of output basis, one 2^14-bin block
    per CTA in shared memory, chunks streamed without atomics) equals the
    oracle for resident and generated inputs, also when L's low columns are
    dependent (shared-memory atomics); BW_FOLD_BLOCKS=0 forces the shared-bin
    / L2-atomic fold."""
    from paper_1607_01039_b200 import subspace

    cases = [(20, 15, 1), (22, 16, 2), (24, 20, 5), (23, 22, 1), (26, 18, 3), (25, 16, 2)]
    for n, d_out, idx in cases:
        spec = signals.config(idx, n)
        rows = subspace.random_full_rank(n, d_out, 100 + n)
        if n == 26:  # dependent low columns: column 5 = column 3 ^ column 4 (still rank 18)
            rows[:, 5] = rows[:, 3] ^ rows[:, 4]
            assert subspace.gf2_rank(rows) == d_out
        if n == 25:  # a zero low column and a repeated one: chunk points share bins
            rows[:, 2] = 0
            rows[:, 9] = rows[:, 0]
            assert subspace.gf2_rank(rows) == d_out
        want = np.empty(1 << d_out, dtype=np.int64)
        cols = oracle_np.column_masks(rows).astype(np.uint64)
        arr = (ctypes.c_uint64 * len(spec.params))(*spec.params) if spec.params else None
        assert coracle.oracle_fold_i64(None, n, cols.ctypes.data, d_out, spec.kind, spec.seed, arr,
                                       len(spec.params), 4, want.ctypes.data) == 0
        t = signals.make(spec)
        for env in ("1", "0"):
            monkeypatch.setenv("BW_FOLD_BLOCKS", env)
            assert np.array_equal(subspace.fold_generated(spec, rows).cpu().numpy(), want), (n, d_out, env)
            assert np.array_equal(subspace.fold(bw.Signal(t), rows).data.cpu().numpy(), want), (n, d_out, env)


def test_int32_inputs_widened(coracle):
    """int32 inputs: the reference widened to int64 (overflow-free sums)."""
    rng = np.random.default_rng(32)
    for n in (0, 1, 5, 12, 13, 14, 15, 19, 22):
        x = rng.integers(np.iinfo(np.int32).min, np.iinfo(np.int32).max, 1 << n, dtype=np.int64).astype(np.int32)
        ref = c_fwht(coracle, x.astype(np.int64))
        out = bw.fwht_widen(torch.from_numpy(x).cuda())
        assert out.dtype == torch.int64 and np.array_equal(out.cpu().numpy(), ref), n
        assert np.array_equal(bw.fwht_widen(x).cpu().numpy(), ref)
    with pytest.raises(errors.BadArguments):
        bw.fwht_widen(torch.zeros(8, dtype=torch.int64, device="cuda"))


def test_concurrent_host_threads_do_not_share_scratch():
    """Calls that use the library's internal scratch (bound check, extraction)
    from several host threads on their own streams stay correct."""
    import threading

    results = {}

    def worker(tid):
        torch.cuda.set_device(0)
        stream = torch.cuda.Stream()
        rng = np.random.default_rng(100 + tid)
        x = rng.integers(-1000, 1000, 1 << 18).astype(np.int64)
        x[tid * 7 + 1] = 5000 + tid
        ok = True
        with torch.cuda.stream(stream):
            t = dev(x)
            for _ in range(20):
                bw.check_magnitude_bound(t, 18)
                i, v = bw.extract_ge(t, 4000)
                ok &= i.tolist() == [tid * 7 + 1] and v.tolist() == [5000 + tid]
        results[tid] = ok

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert results == {k: True for k in range(4)}


@pytest.mark.parametrize("n", [24, 26])
def test_host_buffer_transform_overlapped_copies(coracle, n):
    """fwht_array on a host numpy buffer (pageable and pinned): the copy /
    compute pipeline (chunked H2D + per-chunk passes, column-sliced last pass
    + 2-D D2H) equals the oracle."""
    x = oracle_np.gen(2, 500 + n, [1 << 20], 0, 1 << n)
    ref = c_fwht(coracle, x)
    a = x.copy()
    assert bw.fwht_array(a) == n << (n - 1)
    assert np.array_equal(a, ref)
    pinned = torch.from_numpy(x.copy()).pin_memory()
    b = pinned.numpy()
    assert bw.fwht_array(b) == n << (n - 1)
    assert np.array_equal(b, ref)


@pytest.mark.parametrize("count,n", [(1, 22), (2, 22), (3, 22), (5, 22), (3, 24), (5, 25)])
def test_host_batch_overlapped_signals(coracle, count, n):
    """fwht_arrays: consecutive host signals through two device buffers
    (H2D of one overlapping D2H of the previous), pinned and pageable, and a
    signal list that reuses buffers (each use sees the previous result).
    n >= 24: each signal's H2D in chunks with the inner passes as chunks
    land, its last pass in column slices with a 2-D D2H each."""
    xs = [oracle_np.gen(2, 700 + i, [1 << 20], 0, 1 << n) for i in range(count)]
    refs = [c_fwht(coracle, x) for x in xs]
    pageable = [x.copy() for x in xs]
    assert bw.fwht_arrays(pageable) == [n << (n - 1)] * count
    assert all(np.array_equal(a, r) for a, r in zip(pageable, refs))
    pinned = [torch.from_numpy(x.copy()).pin_memory() for x in xs]
    arrs = [t.numpy() for t in pinned]
    bw.fwht_arrays(arrs)
    assert all(np.array_equal(a, r) for a, r in zip(arrs, refs))
    # two buffers in turn, as bench.py's e2e leg uses them: H H x = 2^n x
    h = [torch.from_numpy(xs[0].copy()).pin_memory(), torch.from_numpy(xs[-1].copy()).pin_memory()]
    hn = [t.numpy() for t in h]
    bw.fwht_arrays([hn[i % 2] for i in range(4)])
    assert np.array_equal(hn[0], xs[0] << n) and np.array_equal(hn[1], xs[-1] << n)
    # the same buffer twice in a row runs in order: H H x = 2^n x
    one = torch.from_numpy(xs[0].copy()).pin_memory().numpy()
    bw.fwht_arrays([one, one])
    assert np.array_equal(one, xs[0] << n)


@pytest.mark.parametrize("nwork,n", [(2, 20), (3, 20), (4, 20), (2, 24), (3, 24)])
def test_host_batch_reused_buffers_any_work_count(nwork, n):
    """bw_fwht_host_batch_i64 with 2-4 device buffers and host lists that
    repeat a buffer 1..nwork-1 entries later ([h0, h1, h0, h1, ...],
    [h0, h1, h2, h0, ...]): each use must read the previous use's result
    (four uses: H^4 x = 2^(2n) x), also for partially overlapping views."""
    import ctypes

    from paper_1607_01039_b200 import _lib

    base = [oracle_np.gen(2, 900 + i, [1 << 10], 0, 1 << n) for i in range(3)]
    works = [torch.empty(1 << n, dtype=torch.int64, device="cuda") for _ in range(nwork)]
    warr = (ctypes.c_void_p * nwork)(*[w.data_ptr() for w in works])
    for period in (2, 3):
        hs = [torch.from_numpy(base[i].copy()).pin_memory() for i in range(period)]
        seq = [hs[i % period] for i in range(4 * period)]  # every buffer used 4 times: H^4 x = 2^(2n) x
        arr = (ctypes.c_void_p * len(seq))(*[t.data_ptr() for t in seq])
        _lib.check(_lib.lib().bw_fwht_host_batch_i64(arr, len(seq), n, warr, nwork,
                                                     torch.cuda.current_stream().cuda_stream, None))
        torch.cuda.synchronize()
        for i in range(period):
            assert np.array_equal(hs[i].numpy(), base[i] << (2 * n)), (nwork, period, i)
    # a partial overlap (a view starting inside another signal) also waits
    big = torch.from_numpy(np.concatenate([base[0], base[1]])).pin_memory()
    mid = big[(1 << n) // 2:(1 << n) // 2 + (1 << n)]
    seq = [big[: 1 << n], mid]
    arr = (ctypes.c_void_p * 2)(*[t.data_ptr() for t in seq])
    _lib.check(_lib.lib().bw_fwht_host_batch_i64(arr, 2, n, warr, nwork, torch.cuda.current_stream().cuda_stream,
                                                 None))
    torch.cuda.synchronize()
    first = base[0].copy()
    oracle_np.fwht_array(first)
    second = np.concatenate([first[(1 << n) // 2:], base[1][: (1 << n) // 2]])
    oracle_np.fwht_array(second)
    assert np.array_equal(big.numpy()[(1 << n) // 2:(1 << n) // 2 + (1 << n)], second)
    assert np.array_equal(big.numpy()[: (1 << n) // 2], first[: (1 << n) // 2])


def test_random_plans_on_device(coracle):
    """Random legal plans (tests/plan_fuzz.py) executed on the B200: every
    kernel shape, forced cluster sizes and split-row passes in any position,
    byte-identical to the oracle."""
    import random

    from plan_fuzz import random_plan

    rng = random.Random(34)
    for n in (18, 21, 24, 26, 27):
        x = oracle_np.gen(2, 40 + n, [1 << 20], 0, 1 << n)
        ref = c_fwht(coracle, x)
        for _ in range(10):
            plan = random_plan(rng, n)
            assert np.array_equal(planned(x, plan), ref), (n, plan)
