"""The compact in-place plan (bw_fwht_i64_compact: high-bit stages first on
int32 copies kept inside the signal's own buffer, then the low pass widening
back to int64) against the C oracle of fwht_array (core.py:97-117): bit-exact
for every plan shape, for inputs at the limit, and through the fallback
(inputs over the limit: the tiles already written are restored exactly and
the int64 plan runs)."""

import ctypes
import os

import numpy as np
import pytest
import torch

import paper_1607_01039_b200 as bw
from paper_1607_01039_b200 import _lib
from oracle import oracle_np

pytestmark = pytest.mark.gpu


def c_fwht(coracle, x):
    """The C oracle's transform of x.  From n = 24 up through its restatement
    of the reference's run_parallel decomposition (parallel.py:162-198, one
    thread per worker): the same butterflies, hence the same bits, as
    fwht_array (tests/test_oracle.py pins both to the reference's digests),
    in a fraction of the single-threaded time."""
    y = np.ascontiguousarray(x, dtype=np.int64).copy()
    n = int(y.size).bit_length() - 1
    if n >= 24:
        p = max(1, min(4, (len(os.sched_getaffinity(0)) or 1).bit_length() - 1))
        assert coracle.oracle_run_parallel_i64(y.ctypes.data, n, p) == 0
    else:
        coracle.oracle_fwht_i64(y.ctypes.data, n)
    return y


def compact(x, max_abs=-1):
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    n = int(t.numel()).bit_length() - 1
    used = ctypes.c_int(0)
    bf = ctypes.c_uint64(0)
    _lib.check(_lib.lib().bw_fwht_i64_compact(t.data_ptr(), n, max_abs, torch.cuda.current_stream().cuda_stream,
                                              ctypes.byref(used), ctypes.byref(bf)))
    assert bf.value == n << (n - 1)
    return t.cpu().numpy(), used.value


@pytest.mark.parametrize("n", [16, 18, 20, 21, 22, 23, 24, 25, 26])
def test_compact_pm1_every_n(coracle, n):
    x = oracle_np.gen(1, 100 + n, [], 0, 1 << n)
    for bound in (-1, 1):
        y, used = compact(x, bound)
        assert used == 1
        assert np.array_equal(y, c_fwht(coracle, x)), f"n={n} bound={bound}"


@pytest.mark.parametrize("rows,w", [("9,8", 13), ("6,5", 13), ("5,5,3", 13), ("4,4,3,2", 14),
                                    ("9,1", 14), ("4,3,3", 13), ("3,2", 14), ("8,9", 13)])
def test_compact_plan_shapes(coracle, monkeypatch, rows, w):
    """Every high-pass shape the plan can take (2-CTA tiles with 6..9 rows,
    register-only tiles with <= 5 rows, 1..4 high passes, low pass 13 / 14),
    checked statically and on the device at the limit value."""
    monkeypatch.setenv("BW_COMPACT_ROWS", rows)
    monkeypatch.setenv("BW_COMPACT_W", str(w))
    n = w + sum(int(r) for r in rows.split(","))
    if n <= 24:
        assert _lib.lib().bw_plan_check_compact(n) == 0, _lib.last_error()
    lim = _lib.lib().bw_compact_limit(n)
    rng = np.random.default_rng(n * 7 + w)
    x = rng.integers(-lim, lim + 1, size=1 << n, dtype=np.int64)
    x[rng.integers(0, 1 << n, size=64)] = lim
    x[rng.integers(0, 1 << n, size=64)] = -lim
    y, used = compact(x)
    assert used == 1
    assert np.array_equal(y, c_fwht(coracle, x))


@pytest.mark.parametrize("n,r2", [(16, "9"), (22, "9"), (23, "9"), (24, "9"), (24, "8"), (25, "9"), (26, "9"),
                                  (27, "8"), (28, "9"), (28, "6"), (29, "7"), (29, "8"), (30, "8")])
def test_compact_v2_limit_values(coracle, monkeypatch, n, r2):
    """The int32-engine plan (k32_high with 9 / 8 rows, k32_low with its last
    four stages in int64) on inputs at +-lim(n) = (2^31 - 1) >> (n - 4),
    with every first-pass shape (1..9 rows) over n = 24..30."""
    monkeypatch.setenv("BW_COMPACT_R2", r2)
    L = _lib.lib()
    lim = L.bw_compact_limit(n)
    assert lim == (2**31 - 1) >> (n - 4)
    rng = np.random.default_rng(n * 3 + int(r2))
    x = rng.integers(-lim, lim + 1, size=1 << n, dtype=np.int64)
    x[rng.integers(0, 1 << n, size=4096)] = lim
    x[rng.integers(0, 1 << n, size=4096)] = -lim
    y, used = compact(x)
    assert used == 1
    assert np.array_equal(y, c_fwht(coracle, x))
    y, used = compact(x, lim)  # known bound: unchecked, asynchronous
    assert used == 1
    assert np.array_equal(y, c_fwht(coracle, x))


@pytest.mark.parametrize("n", [16, 24])
def test_compact_v2_extreme_constant_signal(coracle, n):
    """x = lim everywhere: index 0 carries lim * 2^(n-4) <= 2^31 - 1 into the
    int64 stages -- the largest value the int32 engine ever holds."""
    lim = _lib.lib().bw_compact_limit(n)
    for v in (lim, -lim):
        x = np.full(1 << n, v, dtype=np.int64)
        y, used = compact(x)
        assert used == 1
        want = np.zeros(1 << n, dtype=np.int64)
        want[0] = v << n
        assert np.array_equal(y, want)


def test_compact_v1_still_selectable(coracle, monkeypatch):
    """BW_COMPACT_V2=0: the round-2 plan (int64-engine passes on int32 data)."""
    monkeypatch.setenv("BW_COMPACT_V2", "0")
    n = 24
    lim = _lib.lib().bw_compact_limit(n)
    assert lim == (2**31 - 1) >> (n - 13)
    x = np.random.default_rng(3).integers(-lim, lim + 1, size=1 << n, dtype=np.int64)
    y, used = compact(x)
    assert used == 1
    assert np.array_equal(y, c_fwht(coracle, x))


@pytest.mark.parametrize("n", [22, 23, 24])
@pytest.mark.parametrize("where", ["first", "last", "middle", "everywhere"])
def test_compact_fallback_restores_exactly(coracle, where, n):
    """One input over lim(n): the checked first pass leaves that tile (and
    every tile after the abort) untouched, the written tiles are restored by
    their own stages + an exact shift, and the int64 plan gives the
    reference's result.  n = 22 / 23: the first pass on the int32 engine
    (k32_first<6> / <5> and k32_restore); n = 24: the int64 engine's."""
    lim = _lib.lib().bw_compact_limit(n)
    rng = np.random.default_rng(5)
    x = rng.integers(-lim, lim + 1, size=1 << n, dtype=np.int64)
    if where == "first":
        x[3] = lim + 1
    elif where == "last":
        x[-1] = -(lim + 1)
    elif where == "middle":
        x[(1 << n) // 2 + 12345] = 1 << 40
    else:
        x = rng.integers(-(1 << 30), 1 << 30, size=1 << n, dtype=np.int64)
    y, used = compact(x)
    assert used == 0
    assert np.array_equal(y, c_fwht(coracle, x))


@pytest.mark.parametrize("n", [22, 23])
@pytest.mark.parametrize("bad", [2**31, -(2**31), 2**32, 2**32 + 1, -(2**32), -(2**32) + 1, 2**62, -(2**63), "lim+1", "-lim-1"])
def test_compact_first_pass_input_test_edges(coracle, n, bad):
    """k32_first's input test keeps the low word and must refuse every value
    whose high word is not its sign extension, and |low| > lim -- values
    whose low word alone looks small included."""
    lim = _lib.lib().bw_compact_limit(n)
    if bad == "lim+1":
        bad = lim + 1
    elif bad == "-lim-1":
        bad = -lim - 1
    x = oracle_np.gen(1, 40 + n, [], 0, 1 << n)
    x[(1 << n) - 77] = bad
    y, used = compact(x)
    assert used == 0
    assert np.array_equal(y, c_fwht(coracle, x))


@pytest.mark.parametrize("n", [22, 23])
def test_compact_first_pass_flags_say_which_tiles_were_written(n):
    """A violation in the LAST tile: the checked first pass aborts there; every
    tile is either written and flagged or untouched, and the restore gives the
    input back bit for bit."""
    L = _lib.lib()
    lim = L.bw_compact_limit(n)
    x = oracle_np.gen(1, 60 + n, [], 0, 1 << n)
    x[-1] = lim + 1
    t = torch.from_numpy(x.copy()).cuda()
    flags = torch.zeros(1 << (n - 13), dtype=torch.int32, device="cuda")
    abort = torch.zeros(1, dtype=torch.int32, device="cuda")
    sh = torch.cuda.current_stream().cuda_stream
    _lib.check(L.bw_fwht_i64_compact_pass(t.data_ptr(), n, 0, 1, flags.data_ptr(), abort.data_ptr(), sh))
    assert abort.item() == 1
    assert 0 <= int(flags.sum().item()) < 1 << (n - 14)
    _lib.check(L.bw_fwht_i64_compact_restore(t.data_ptr(), n, flags.data_ptr(), sh))
    assert np.array_equal(t.cpu().numpy(), x)


def test_compact_first_pass_engines_agree(coracle, monkeypatch):
    """BW_COMPACT_FIRST=0 runs the first pass on the int64 engine
    (k_pass_map) as before: same result."""
    n = 23
    x = oracle_np.gen(1, 5, [], 0, 1 << n)
    want = c_fwht(coracle, x)
    for first in ("1", "0"):
        monkeypatch.setenv("BW_COMPACT_FIRST", first)
        for bound in (-1, 1):
            y, used = compact(x, bound)
            assert used == 1
            assert np.array_equal(y, want)


def test_compact_restore_is_identity():
    """The restore step alone: a checked pass 0 that wrote every tile, then
    the restore, gives the input back bit for bit."""
    n = 22
    x = oracle_np.gen(2, 8, [1000], 0, 1 << n)
    t = torch.from_numpy(x.copy()).cuda()
    tiles = 1 << (n - 13)
    flags = torch.zeros(tiles, dtype=torch.int32, device="cuda")
    abort = torch.zeros(1, dtype=torch.int32, device="cuda")
    sh = torch.cuda.current_stream().cuda_stream
    L = _lib.lib()
    _lib.check(L.bw_fwht_i64_compact_pass(t.data_ptr(), n, 0, 1, flags.data_ptr(), abort.data_ptr(), sh))
    assert abort.item() == 0 and int(flags.sum().item()) == 1 << (n - 14)
    assert not np.array_equal(t.cpu().numpy(), x)
    _lib.check(L.bw_fwht_i64_compact_restore(t.data_ptr(), n, flags.data_ptr(), sh))
    assert np.array_equal(t.cpu().numpy(), x)


def test_fwht_array_and_inplace_pick_compact(coracle):
    n = 23
    x = oracle_np.gen(1, 23, [], 0, 1 << n)
    t = torch.from_numpy(x.copy()).cuda()
    bw.fwht_array(t, compact=True)
    assert bw.core.last_compact
    assert np.array_equal(t.cpu().numpy(), c_fwht(coracle, x))
    t = torch.from_numpy(x.copy()).cuda()
    bw.fwht_array(t, compact=1)  # a bound the caller guarantees
    assert bw.core.last_compact
    assert np.array_equal(t.cpu().numpy(), c_fwht(coracle, x))
    sig = bw.fwht_inplace(bw.Signal(torch.from_numpy(x.copy()).cuda()))
    assert np.array_equal(sig.data.cpu().numpy(), c_fwht(coracle, x))
    big = oracle_np.gen(2, 4, [1 << 30], 0, 1 << n)
    t = torch.from_numpy(big.copy()).cuda()
    bw.fwht_array(t, compact=True)
    assert not bw.core.last_compact
    assert np.array_equal(t.cpu().numpy(), c_fwht(coracle, big))
    t = torch.from_numpy(x.copy()).cuda()
    bw.fwht_array(t, compact=False)
    assert not bw.core.last_compact
    assert np.array_equal(t.cpu().numpy(), c_fwht(coracle, x))


def test_compact_unaligned_view_runs_int64_plan(coracle):
    n = 22
    x = oracle_np.gen(1, 9, [], 0, (1 << n) + 1)
    t = torch.from_numpy(x.copy()).cuda()
    v = t[1:]  # 8- but not 16-byte aligned
    bw.fwht_array(v, compact=True)
    assert not bw.core.last_compact
    assert np.array_equal(v.cpu().numpy(), c_fwht(coracle, x[1:]))


@pytest.mark.skipif(torch.cuda.is_available() and torch.cuda.get_device_properties(0).total_memory < (100 << 30),
                    reason="needs a B200")
@pytest.mark.parametrize("n", [28, 29, 30, 31, 32, 33, 34])
def test_compact_full_size_spot_check(n):
    """n = 32 (config 4: 9 + 9 rows), 31 (9 + 8), 30 (8 + 8), 29 (8 + 7), 28
    (8 + 6) and n = 33 / 34 (9 + 8 rows, then 2 / 3 in registers: 64 / 128 GiB
    in place) through the compact plan: the fold spot check of 2^20 outputs
    (subspace.py:1-11) against the CPU."""
    from paper_1607_01039_b200 import signals

    spec = signals.config(4, n)
    torch.cuda.empty_cache()
    if torch.cuda.mem_get_info()[0] < (8 << n) + (1 << 30):
        pytest.skip(f"needs {(8 << n) >> 30} GiB of free device memory")
    t = torch.empty(1 << n, dtype=torch.int64, device="cuda")
    signals.generate(spec, t)
    bw.fwht_array(t, compact=True)
    assert bw.core.last_compact
    d = 20
    rng = np.random.default_rng(77)
    while True:
        rows = rng.integers(0, 2, size=(d, n), dtype=np.uint8)
        if oracle_np.gf2_rank(rows) == d:
            break
    got = t[torch.from_numpy(oracle_np.row_space(rows)).cuda()].cpu().numpy()
    del t
    torch.cuda.empty_cache()  # up to 128 GiB: give it back before the next test asks for free memory
    from oracle import load_c

    lib = load_c()
    cols = oracle_np.column_masks(rows).astype(np.uint64)
    want = np.empty(1 << d, dtype=np.int64)
    params = (ctypes.c_uint64 * max(1, len(spec.params)))(*[int(v) for v in spec.params])
    rc = lib.oracle_fold_i64(None, n, cols.ctypes.data, d, spec.kind, spec.seed, params, len(spec.params),
                             len(os.sched_getaffinity(0)), want.ctypes.data)
    assert rc == 0
    lib.oracle_fwht_i64(want.ctypes.data, d)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n,cfg", [(26, 3), (27, 3), (26, 5), (28, 3)])
def test_compact_fused_extraction_matches_two_step(coracle, monkeypatch, n, cfg):
    """bw_fwht_extract_i64 on the noisy +-1 sums of configs 3 / 5: by default
    (n >= 26) the compact plan with |W| >= tau tested in k32_low's final
    registers; the same hits, in the same order, as the int64 plan
    (BW_COMPACT=0) and as transform-then-extract, and the planted masks."""
    from paper_1607_01039_b200 import signals

    spec = signals.config(cfg, n=n)
    assert spec.max_abs <= _lib.lib().bw_compact_limit(n)
    tau = 1 << 20  # between the noise floor (~2^(n/2) * 5 * sqrt(K)) and the planted bias (0.1 / 0.04 * 2^n)
    a = signals.make(spec)
    x = a.cpu().numpy().copy()
    i1, v1 = bw.fwht_extract_ge(a, tau)
    monkeypatch.setenv("BW_COMPACT", "0")
    b = torch.from_numpy(x.copy()).cuda()
    i2, v2 = bw.fwht_extract_ge(b, tau)
    monkeypatch.delenv("BW_COMPACT")
    want = c_fwht(coracle, x)
    assert np.array_equal(a.cpu().numpy(), want) and torch.equal(a, b)
    assert torch.equal(i1, i2) and torch.equal(v1, v2)
    hits = np.nonzero(np.abs(want) >= tau)[0]
    assert i1.tolist() == hits.tolist() and v1.tolist() == want[hits].tolist()
    assert sorted(spec.masks) == hits.tolist()


def test_compact_fused_extraction_many_hits_and_wide_values(coracle):
    """tau = 0 (every point hits: the ordered two-phase extraction takes
    over) and a wide-valued signal (the checked pass refuses it: int64 plan
    with its own fused extraction), both at a size the default tries the
    compact plan on."""
    n = 26
    x = oracle_np.gen(1, 5, [], 0, 1 << n)
    a = torch.from_numpy(x.copy()).cuda()
    i1, v1 = bw.fwht_extract_ge(a, 0, cap=16)
    want = c_fwht(coracle, x)
    assert np.array_equal(a.cpu().numpy(), want)
    assert torch.equal(i1, torch.arange(1 << n, device="cuda")) and np.array_equal(v1.cpu().numpy(), want)
    x = oracle_np.gen(2, 6, [1 << 20], 0, 1 << n)
    a = torch.from_numpy(x.copy()).cuda()
    want = c_fwht(coracle, x)
    tau = int(np.sort(np.abs(want))[-50])
    i1, v1 = bw.fwht_extract_ge(a, tau)
    hits = np.nonzero(np.abs(want) >= tau)[0]
    assert np.array_equal(a.cpu().numpy(), want)
    assert i1.tolist() == hits.tolist() and v1.tolist() == want[hits].tolist()


def test_default_picks_compact_from_n26(coracle):
    """bw_fwht_i64 / fwht_array / fwht_inplace with no arguments: the compact
    plan from n = 26 up (bw_compact_auto), the int64 plan below and for wide
    values; identical results."""
    L = _lib.lib()
    assert [L.bw_compact_auto(n) for n in (24, 25, 26, 30, 32, 33, 34)] == [0, 0, 1, 1, 1, 1, 1]
    for n in (25, 26):
        x = oracle_np.gen(1, n, [], 0, 1 << n)
        want = c_fwht(coracle, x)
        t = torch.from_numpy(x.copy()).cuda()
        bw.fwht_array(t)
        assert bw.core.last_compact == (n >= 26)
        assert np.array_equal(t.cpu().numpy(), want)
        t = torch.from_numpy(x.copy()).cuda()
        _lib.check(L.bw_fwht_i64(t.data_ptr(), n, torch.cuda.current_stream().cuda_stream, None))
        assert np.array_equal(t.cpu().numpy(), want)
        sig = bw.fwht_inplace(bw.Signal(torch.from_numpy(x.copy()).cuda()))
        assert np.array_equal(sig.data.cpu().numpy(), want)
        sig = bw.fwht_inplace(bw.Signal(torch.from_numpy(x.copy()).cuda()), max_abs=1)
        assert np.array_equal(sig.data.cpu().numpy(), want)
    n = 26
    x = oracle_np.gen(2, 9, [1 << 20], 0, 1 << n)  # wide values: the int64 plan after the exact restore
    want = c_fwht(coracle, x)
    t = torch.from_numpy(x.copy()).cuda()
    bw.fwht_array(t)
    assert not bw.core.last_compact and np.array_equal(t.cpu().numpy(), want)
    sig = bw.fwht_inplace(bw.Signal(torch.from_numpy(x.copy()).cuda()))
    assert np.array_equal(sig.data.cpu().numpy(), want)
    x[12345] = 1 << 40  # over the overflow bound: raised before mutation, as ever (core.py:122)
    t = torch.from_numpy(x.copy()).cuda()
    with pytest.raises(bw.errors.OverflowBoundError):
        bw.fwht_inplace(bw.Signal(t))
    assert np.array_equal(t.cpu().numpy(), x)


def test_default_under_stream_capture_runs_the_int64_plan(coracle):
    """The compact plan reads its first pass's verdict on the host, which a
    capturing stream cannot do: bw_fwht_i64 then launches the (asynchronous)
    int64 plan, so the call stays capturable; the replayed graph gives the
    reference's result."""
    n = 26
    x = oracle_np.gen(1, 77, [], 0, 1 << n)
    want = c_fwht(coracle, x)
    t = torch.from_numpy(x.copy()).cuda()
    L = _lib.lib()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        _lib.check(L.bw_fwht_i64_int64plan(t.data_ptr(), n, side.cuda_stream, None))  # warm-up: attributes, scratch
    side.synchronize()
    t.copy_(torch.from_numpy(x))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        _lib.check(L.bw_fwht_i64(t.data_ptr(), n, torch.cuda.current_stream().cuda_stream, None))
    assert np.array_equal(t.cpu().numpy(), x)  # captured, not run
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy(), want)


@pytest.mark.parametrize("rows", ["8,6,1", "8,6,2", "9,6,1", "8,4", "9,3"])
def test_compact_plans_with_register_passes(coracle, monkeypatch, rows):
    """k32_reg (1..4 rows, registers only) as the second or third high pass
    behind k32_first / k32_high -- the shapes of the n = 33 / 34 plans at sizes
    the oracle reaches -- on inputs at +-lim, unknown and known bound."""
    monkeypatch.setenv("BW_COMPACT_ROWS", rows)
    n = 14 + sum(int(r) for r in rows.split(","))
    L = _lib.lib()
    lim = L.bw_compact_limit(n)
    assert lim == (2**31 - 1) >> (n - 4) and L.bw_compact_npasses(n) == len(rows.split(",")) + 1
    rng = np.random.default_rng(n)
    x = rng.integers(-lim, lim + 1, size=1 << n, dtype=np.int64)
    x[rng.integers(0, 1 << n, size=4096)] = lim
    x[rng.integers(0, 1 << n, size=4096)] = -lim
    want = c_fwht(coracle, x)
    for bound in (-1, lim):
        y, used = compact(x, bound)
        assert used == 1
        assert np.array_equal(y, want)
