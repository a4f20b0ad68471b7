"""CPU-side tests of the boundary: the C-ABI library loads and exports every
declared symbol, the host plan checker (a static proof over the kernels' own
address tables, like parallel.py:114-147), error mapping and host-side
validation.  No kernel is launched here."""

import ctypes
import itertools
import os
import re

import numpy as np
import pytest

from paper_1607_01039_b200 import _lib, errors, sharded
from paper_1607_01039_b200.core import Signal

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "bigwht_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bw_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    decl = declared_symbols()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(_lib.exported_symbols()) == decl


def test_abi_version():
    assert _lib.lib().bw_abi_version() == 1


@pytest.mark.parametrize("n", list(range(0, 25)))
def test_default_plan_checker(n):
    assert sharded.plan_check(n) == n << max(n - 1, 0)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_fused_plan_checker(p):
    """The fused multi-device plan (local passes + K6' last pass with the
    shard bits): every element of every shard once per pass, every stage of
    the 2^(n_local+p) transform exactly once."""
    for nl in range(14, 31):
        widths, r = sharded.fused_plan(nl, p)
        assert widths[0] in (13, 14, 15) and sum(w & 15 for w in widths) + r == nl and 1 <= r <= 10 - p
        if nl > 24:  # the checker's bitmap limit; the plans above repeat the n=24 shapes
            continue
        n = nl + p
        assert sharded.plan_check_fused(nl, p) == n << (n - 1)


def splits(h):
    """Every composition of h into parts of 1..10."""
    if h == 0:
        yield ()
        return
    for first in range(1, min(10, h) + 1):
        for rest in splits(h - first):
            yield (first,) + rest


@pytest.mark.parametrize("low", [13, 14, 15])
@pytest.mark.parametrize("n", [16, 18, 20, 22])
def test_every_pass_split_checks(n, low):
    count = 0
    for parts in splits(n - low):
        if n == 22 and len(parts) > 3:
            continue
        assert sharded.plan_check(n, [low, *parts]) == n << (n - 1)
        count += 1
    assert count > 0


def test_bad_plans_rejected():
    with pytest.raises(errors.BadArguments):
        sharded.plan_check(20, [14, 11, -5])
    with pytest.raises(errors.BadArguments):
        sharded.plan_check(20, [12, 8])
    with pytest.raises(errors.BadArguments):
        sharded.plan_check(20, [16, 4])
    with pytest.raises(errors.BadArguments):
        sharded.plan_check(19, [14, 5 | (2 << 4)])  # 5 stages on a 2-CTA tile: 9 column bits, not built
    with pytest.raises(errors.BadArguments):
        sharded.plan_check(20, [14, 5])


def split(r, q, a, k2):
    """Plan entry of a split-row high pass: rows [k, k+a) u [k2, k2+r-a),
    k = the lowest bit no earlier pass covers (bw_layouts.h split rows)."""
    return r | ((q + 1) << 4) | (a << 8) | (k2 << 12)


SPLIT_PLANS = [
    (24, [13, split(6, 0, 3, 21), 5]),           # rows {13,14,15} u {21,22,23}, then 16..20 in registers
    (24, [13, split(9, 1, 4, 19), 2]),           # 2-CTA: {13..16} u {19..23}, then 17, 18
    (24, [13, split(10, 1, 1, 15), 1]),          # 2-CTA, 10 rows: {13} u {15..23}
    (24, [13, 2, split(7, 0, 3, 20), 2]),        # split pass in the middle
    (23, [13, split(8, 0, 2, 17), 2]),           # 1-CTA, 8 rows
    (24, [14, split(9, 1, 2, 17), 1]),         # n=34-like: 14 + split + contiguous rest
    (22, [13, split(9, 1, 8, 21)]),              # degenerate split (runs adjacent): one run in effect
]


@pytest.mark.parametrize("n,plan", SPLIT_PLANS)
def test_split_plan_checks(n, plan):
    """Split-row passes: every element once per pass, every stage once."""
    assert sharded.plan_check(n, plan) == n << (n - 1)


def test_split_plans_rejected():
    for n, plan in [
        (24, [13, split(6, 0, 3, 15), 5]),    # second run overlaps the first
        (24, [13, split(6, 0, 3, 22), 5]),    # reaches bit 24
        (24, [13, split(5, 0, 2, 20), 6]),    # no split register-only pass
        (24, [13, split(9, 0, 2, 20), 2]),    # 9 rows need a cluster of 2
        (24, [13, split(6, 0, 3, 21), 4]),    # leaves bit 20 uncovered
        (24, [13, split(6, 0, 3, 18), 5]),    # second run overlaps the contiguous pass
    ]:
        with pytest.raises(errors.BadArguments):
            sharded.plan_check(n, plan)


def test_narrow_wire_arguments_validated_before_launch():
    L = _lib.lib()
    buf = np.zeros(64, dtype=np.int64)
    flag = np.zeros(1, dtype=np.int32)
    ptr = (buf.ctypes.data + 15) & ~15
    for args in [(ptr, 64, 3, 1, ptr, flag.ctypes.data, None),   # wire of 3 bytes
                 (ptr, 60, 1, 1, ptr, flag.ctypes.data, None),   # count not a multiple of 8
                 (ptr + 8, 56, 1, 1, ptr, flag.ctypes.data, None),  # misaligned source
                 (ptr, 56, 1, 4, ptr, flag.ctypes.data, None)]:  # 16 shards
        with pytest.raises((errors.BadArguments, errors.InvalidWorkerCount)):
            _lib.check(L.bw_pack_narrow_i64(*args))
    arr = (ctypes.c_void_p * 2)(ptr, ptr)
    with pytest.raises(errors.BadArguments):
        _lib.check(L.bw_xshard_narrow(arr, 1, 1, 8, 16, None))  # begin not a multiple of 16
    with pytest.raises(errors.BadArguments):
        _lib.check(L.bw_fwht_widen(ptr, 3, ptr, 4, None, None))
    assert sharded.narrow_ok(1 << 10, 3) and not sharded.narrow_ok(64, 3) and not sharded.narrow_ok(1 << 10, 0)


def test_plan_describe():
    p = sharded.plan(32, 0)
    assert [x["kind"] for x in p["passes"]] == ["low", "high", "high"]
    assert all(x["cols_bits"] >= 4 for x in p["passes"][1:])  # >= 128-byte row segments
    assert sum(x["r"] for x in p["passes"]) == 32
    assert p["hbm_bytes_per_pass"] == 16 << 32
    q = sharded.plan(34, 3)
    assert q["local_log2n"] == 31 and q["cross_stages"] == [31, 32, 33]
    assert sharded.plan(18, 0)["passes"][1]["kind"] == "reg"
    assert sharded.plan(10, 0)["passes"][0]["kind"] == "small"


def test_status_mapping():
    assert errors.OverflowBoundError.exit_code == 3
    assert errors.DeviceError.exit_code == 2
    with pytest.raises(errors.BadArguments):
        _lib.check(1)
    with pytest.raises(errors.OverflowBoundError):
        _lib.check(2)
    with pytest.raises(errors.InexactDivision):
        _lib.check(3)
    with pytest.raises(errors.InvalidWorkerCount):
        _lib.check(4)
    with pytest.raises(errors.DeviceError):
        _lib.check(6)


def test_signal_validation_host_side():
    with pytest.raises(errors.BadArguments):
        Signal(np.zeros(3, dtype=np.int64))
    with pytest.raises(errors.BadArguments):
        Signal(np.zeros(4, dtype=np.int32))
    with pytest.raises(errors.BadArguments):
        Signal(np.zeros((2, 2), dtype=np.int64))
    assert Signal(np.zeros(8, dtype=np.int64)).log2_dim == 3
    assert Signal(np.array([5], dtype=np.int64)).log2_dim == 0


def test_shard_slices_partition():
    for world in (1, 2, 4, 8):
        for local in (2, 8, 1 << 10, 6):
            cover = np.zeros(local, dtype=np.int64)
            for r in range(world):
                b, c = sharded.slice_of(r, world, local)
                assert b % 2 == 0 and c % 2 == 0
                cover[b:b + c] += 1
            assert (cover == 1).all()


def test_shard_count_validation():
    for bad in (0, 3, 6, 16):
        with pytest.raises(errors.InvalidWorkerCount):
            sharded.log2_shards(bad)
    assert [sharded.log2_shards(p) for p in (1, 2, 4, 8)] == [0, 1, 2, 3]


def test_no_cpu_fallback_without_device(monkeypatch):
    import torch

    from paper_1607_01039_b200 import core

    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(errors.DeviceError):
        core.fwht_array(np.zeros(8, dtype=np.int64))


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1607_01039_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text, f


def emulate(x, bits=None):
    y = np.ascontiguousarray(x, dtype=np.int64).copy()
    n = int(y.size).bit_length() - 1
    if bits:
        arr = (ctypes.c_int * len(bits))(*bits)
        _lib.check(_lib.lib().bw_debug_emulate_i64(y.ctypes.data, n, arr, len(bits)))
    else:
        _lib.check(_lib.lib().bw_debug_emulate_i64(y.ctypes.data, n, None, 0))
    return y


@pytest.mark.parametrize("n", [0, 1, 5, 12, 13, 14, 15, 17, 19, 20, 23, 24])
def test_kernel_tables_emulated_on_host_match_oracle(coracle, n):
    """The pass kernels' address/stage/smem tables, executed on the host
    (bw_debug_emulate_i64), equal the oracle bit for bit."""
    from oracle import oracle_np

    x = oracle_np.gen(2, 300 + n, [1 << 20], 0, 1 << n)
    ref = x.copy()
    coracle.oracle_fwht_i64(ref.ctypes.data, n)
    assert np.array_equal(emulate(x), ref)


@pytest.mark.parametrize("n,plan", SPLIT_PLANS)
def test_split_plans_emulated_on_host_match_oracle(coracle, n, plan):
    from oracle import oracle_np

    x = oracle_np.gen(2, 700 + n, [1 << 20], 0, 1 << n)
    ref = x.copy()
    coracle.oracle_fwht_i64(ref.ctypes.data, n)
    assert np.array_equal(emulate(x, plan), ref)


@pytest.mark.parametrize("n", list(range(0, 25)))
def test_float64_plan_checker(n):
    """float64 plan: every stage once, every element's stages in ascending
    bit order (what bitwise numpy equality needs)."""
    bf = ctypes.c_uint64(0)
    _lib.check(_lib.lib().bw_plan_check_f64(n, ctypes.byref(bf)))
    assert bf.value == (n << (n - 1) if n else 0)


@pytest.mark.parametrize("n", [3, 12, 13, 14, 16, 19, 21, 22])
def test_float64_kernel_tables_emulated_on_host_bitwise(coracle, n):
    """The float64 pass kernels' tables with IEEE add/sub on the host equal
    numpy's float64 fwht_array bit for bit (oracle/bw_oracle.c restates it)."""
    rng = np.random.default_rng(40 + n)
    x = rng.normal(scale=1e3, size=1 << n)
    ref = x.copy()
    coracle.oracle_fwht_f64(ref.ctypes.data, n)
    y = x.copy()
    _lib.check(_lib.lib().bw_debug_emulate_f64(y.ctypes.data, n))
    assert np.array_equal(y.view(np.int64), ref.view(np.int64))


@pytest.mark.parametrize("low", [13, 14, 15])
def test_kernel_tables_every_split_emulated(coracle, low):
    from oracle import oracle_np

    n = 21
    x = oracle_np.gen(1, 5, [], 0, 1 << n)
    ref = x.copy()
    coracle.oracle_fwht_i64(ref.ctypes.data, n)
    for parts in splits(n - low):
        assert np.array_equal(emulate(x, [low, *parts]), ref), parts


@pytest.mark.parametrize("plan", [
    [14, 9 | (2 << 4)], [14, 8 | (2 << 4)], [14, 7 | (3 << 4)], [15, 8], [13, 10],
    [13, 9], [13, 10 | (3 << 4)], [13, 8 | (3 << 4)], [13, 6 | (2 << 4)], [13, 9 | (1 << 4)],
    [15, 7 | (2 << 4)], [13, 5 | (1 << 4)], [14, 6 | (3 << 4)], [13, 5 | (3 << 4), 4]])
def test_forced_cluster_shapes_emulated(coracle, plan):
    """Every cluster shape (forced with r | (q+1) << 4), on the host emulator."""
    from oracle import oracle_np

    n = sum(w & 15 for w in plan)
    x = oracle_np.gen(2, 11 + n, [1 << 20], 0, 1 << n)
    ref = x.copy()
    coracle.oracle_fwht_i64(ref.ctypes.data, n)
    assert sharded.plan_check(n, plan) == n << (n - 1)
    assert np.array_equal(emulate(x, plan), ref)


def _compile_c_consumer(tmp_path):
    import shutil
    import subprocess

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    out = str(tmp_path / "abi_smoke")
    cmd = [cc, "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "c", "abi_smoke.c"), "-L", os.path.dirname(_lib.LIB_PATH), "-lbigwht_b200",
           "-L", os.path.join(ROOT, "oracle"), "-loracle", "-L", "/usr/local/cuda/lib64", "-lcudart", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_c_consumer_compiles_against_the_header(tmp_path):
    """The header is plain C (no C++ or torch types) and the library links
    into a C program without Python."""
    _compile_c_consumer(tmp_path)


@pytest.mark.gpu
def test_c_consumer_runs(tmp_path):
    import subprocess

    exe = _compile_c_consumer(tmp_path)
    env = dict(os.environ)
    env["LD_LIBRARY_PATH"] = ":".join([os.path.dirname(_lib.LIB_PATH), os.path.join(ROOT, "oracle"),
                                       "/usr/local/cuda/lib64", env.get("LD_LIBRARY_PATH", "")])
    for n in ("13", "22", "24"):
        r = subprocess.run([exe, n], capture_output=True, text=True, env=env, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "c abi ok" in r.stdout


def test_random_plans_check_and_emulate(coracle):
    """Random legal plans (tests/plan_fuzz.py: every kernel shape, forced
    cluster sizes, split-row passes in any position): the static checker
    proves them at n <= 24 and the host emulator of the kernels' tables
    matches the oracle at n <= 20."""
    import random

    from oracle import oracle_np
    from plan_fuzz import random_plan

    rng = random.Random(1607)
    for i in range(60):
        n = rng.randint(14, 24)
        plan = random_plan(rng, n)
        assert sharded.plan_check(n, plan) == n << (n - 1), plan
        if n <= 20 and i % 3 == 0:
            x = oracle_np.gen(2, 900 + i, [1 << 20], 0, 1 << n)
            ref = x.copy()
            coracle.oracle_fwht_i64(ref.ctypes.data, n)
            assert np.array_equal(emulate(x, plan), ref), plan


def test_host_batch_validation_host_side():
    import paper_1607_01039_b200 as bw

    assert bw.fwht_arrays([]) == []
    with pytest.raises(errors.BadArguments):
        bw.fwht_arrays([np.zeros(8, dtype=np.float64)])
    with pytest.raises(errors.BadArguments):
        bw.fwht_arrays([np.zeros(8, dtype=np.int64), np.zeros(16, dtype=np.int64)])
    with pytest.raises(errors.BadArguments):
        bw.fwht_arrays([np.zeros(6, dtype=np.int64)])
    with pytest.raises(errors.BadArguments):
        bw.fwht_arrays([np.zeros((4, 4), dtype=np.int64)[:, 0]])  # not contiguous
    L = _lib.lib()
    with pytest.raises(errors.BadArguments):
        _lib.check(L.bw_fwht_host_batch_i64(None, 2, 10, None, 2, None, None))
    with pytest.raises(errors.BadArguments):
        _lib.check(L.bw_fwht_xfused_pass_extract_i64(None, 1, 20, 5, 0, 10, 0, None, None, 16, None, None))


@pytest.mark.parametrize("v2", ["0", "1", "first0"])
@pytest.mark.parametrize("n", [16, 19, 22, 23, 24])
def test_compact_plan_checks(monkeypatch, n, v2):
    """The compact in-place plan's exact address tables (bw_plan_check_compact):
    natural int64 in and out, every pass loads where the previous one
    stored, no tile stores over bytes another tile of the same pass loads,
    every bit staged once; for the int32-engine passes (v2) also every
    round's coverage, vector alignment and shared-memory bank conflicts.
    n = 22 / 23: the first pass (8 / 9 rows) is the int32 engine's k32_first
    ("first0": BW_COMPACT_FIRST=0 keeps it on the int64 engine)."""
    if v2 == "first0":
        monkeypatch.setenv("BW_COMPACT_FIRST", "0")
        v2 = "1"
    monkeypatch.setenv("BW_COMPACT_V2", v2)
    L = _lib.lib()
    assert L.bw_plan_check_compact(n) == 0, _lib.last_error()
    assert L.bw_compact_npasses(n) >= 2
    # v1: no int32 value of the high passes wraps (H = n - 13 high stages);
    # v2: every stage but the last four (int64) stays in int32
    assert L.bw_compact_limit(n) == (2**31 - 1) >> (n - 4 if v2 == "1" else n - 13)


@pytest.mark.parametrize("n,r2", [(16, "9"), (20, "9"), (22, "9"), (23, "9"), (24, "9"), (24, "8"), (24, "7"), (24, "6")])
def test_compact_v2_host_emulation_matches_oracle(monkeypatch, coracle, n, r2):
    """The int32-engine passes' exact tables (rounds, swizzled shared-memory
    slots, int32 / int64 arithmetic) run on the host (bw_debug_emulate_compact)
    on inputs at +-lim(n): bit-identical to the C oracle of fwht_array."""
    monkeypatch.setenv("BW_COMPACT_R2", r2)
    L = _lib.lib()
    lim = L.bw_compact_limit(n)
    rng = np.random.default_rng(n)
    x = rng.integers(-lim, lim + 1, size=1 << n, dtype=np.int64)
    x[rng.integers(0, 1 << n, size=256)] = lim
    x[rng.integers(0, 1 << n, size=256)] = -lim
    if n == 16:
        x[:] = lim  # the extreme: index 0 reaches lim * 2^(n-4) = 2^31 - 1 - ... before the int64 stages
    ref = x.copy()
    coracle.oracle_fwht_i64(ref.ctypes.data, n)
    y = x.copy()
    assert L.bw_debug_emulate_compact(y.ctypes.data, n) == 0, _lib.last_error()
    assert np.array_equal(y, ref)


@pytest.mark.parametrize("rows,w", [("4,4,3", 13), ("5,5", 14), ("9,1", 14), ("3,3,2,2", 14)])
def test_compact_plan_shapes_check(monkeypatch, rows, w):
    monkeypatch.setenv("BW_COMPACT_ROWS", rows)
    monkeypatch.setenv("BW_COMPACT_W", str(w))
    n = w + sum(int(r) for r in rows.split(","))
    assert _lib.lib().bw_plan_check_compact(n) == 0, _lib.last_error()


def test_compact_checker_catches_a_layout_that_is_not_in_place(monkeypatch):
    monkeypatch.setenv("BW_COMPACT_BREAK", "1")  # bit c trades places with the top bit
    monkeypatch.setenv("BW_COMPACT_V2", "0")
    assert _lib.lib().bw_plan_check_compact(20) != 0
    assert "not in place" in _lib.last_error()
    # v2: the int32-engine low pass reads its fixed layout, which the broken
    # first pass no longer writes
    monkeypatch.setenv("BW_COMPACT_V2", "1")
    assert _lib.lib().bw_plan_check_compact(20) != 0


@pytest.mark.parametrize("r2", ["6", "7", "8", "9"])
def test_compact_plan_checks_every_second_pass_shape(monkeypatch, r2):
    """k32_high with 6, 7, 8 and 9 rows as the second high pass (n = 24: 10 - r2
    rows first): the static checker on the kernels' exact address functions
    (coverage, bank conflicts, in place, every bit staged once)."""
    monkeypatch.setenv("BW_COMPACT_R2", r2)
    L = _lib.lib()
    assert L.bw_plan_check_compact(24) == 0, _lib.last_error()
    assert L.bw_compact_npasses(24) == 3
    k, r = ctypes.c_int(0), ctypes.c_int(0)
    assert L.bw_compact_pass_info(24, 1, ctypes.byref(k), ctypes.byref(r), None, None) == 0
    assert r.value == int(r2) and k.value == 14 + 10 - int(r2)


@pytest.mark.parametrize("rows", ["1,6,3", "2,7,1", "1,7,2", "2,6,2", "6,4", "7,3", "8,2", "9,1"])
def test_compact_plan_with_register_passes(monkeypatch, coracle, rows):
    """k32_reg (1..4 rows in registers, the third high pass of the n = 33 / 34
    plans) after k32_high or directly after the first pass, at n = 24: the
    static checker on the exact address functions and the host emulation
    against the oracle at +-lim."""
    monkeypatch.setenv("BW_COMPACT_ROWS", rows)
    n = 14 + sum(int(r) for r in rows.split(","))
    L = _lib.lib()
    assert L.bw_plan_check_compact(n) == 0, _lib.last_error()
    assert L.bw_compact_npasses(n) == len(rows.split(",")) + 1
    eng = ctypes.c_int(0)
    assert L.bw_compact_pass_info(n, 1, None, None, ctypes.byref(eng), None) == 0 and eng.value == 32
    lim = L.bw_compact_limit(n)
    assert lim == (2**31 - 1) >> (n - 4)
    rng = np.random.default_rng(n + len(rows))
    x = rng.integers(-lim, lim + 1, size=1 << n, dtype=np.int64)
    ref = x.copy()
    coracle.oracle_fwht_i64(ref.ctypes.data, n)
    y = x.copy()
    assert L.bw_debug_emulate_compact(y.ctypes.data, n) == 0, _lib.last_error()
    assert np.array_equal(y, ref)


def test_compact_plans_of_n33_n34():
    """n = 33 / 34: 9 rows (k32_first), 8 rows (k32_high), then 2 / 3 rows in
    registers (k32_reg), the 14-bit low pass; lim = 3 / 1; tried by default
    (bw_compact_auto) behind a sample of the first inputs."""
    L = _lib.lib()
    for n, third in ((33, 2), (34, 3)):
        assert L.bw_compact_npasses(n) == 4
        want = [(14, 9), (23, 8), (31, third), (0, 14)]
        for i, (k0, r0) in enumerate(want):
            k, r, e, b = (ctypes.c_int(0) for _ in range(4))
            assert L.bw_compact_pass_info(n, i, ctypes.byref(k), ctypes.byref(r), ctypes.byref(e), ctypes.byref(b)) == 0
            assert (k.value, r.value, e.value) == (k0, r0, 32)
            assert b.value == (12 if i in (0, 3) else 8)
        assert L.bw_compact_limit(n) == (2**31 - 1) >> (n - 4)
        assert L.bw_compact_auto(n) == 1
