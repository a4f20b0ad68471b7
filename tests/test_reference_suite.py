"""The drop-in through the reference's own callers and tests.

The shim (paper_1607_01039_b200/shim.py) rebinds
``bigwht.{core,parallel,external,noisy}.fwht_array`` and
``check_magnitude_bound`` to the B200 path and makes this package's
exceptions subclasses of ``bigwht.errors``.  The GPU tests run the
reference's unmodified test suite (/root/reference/pkg/tests, shipped to the
box as baseline/_ref/bigwht_tests by baseline/install_reference.sh) with
every butterfly on the device, and the reference CLI's error path
(cli.py:577-579: ``except BigWHTError`` -> exit code 3) on an overflow the
B200 bound check raises.

Every case runs in a subprocess: installing the shim patches ``bigwht`` for
the life of the interpreter.
"""

from __future__ import annotations

import os
import subprocess
import sys
import textwrap

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIPPED = os.path.join(REPO, "baseline", "_ref")


def _reference_path(gpu: bool) -> str | None:
    """Where ``bigwht`` can be imported from: the shipped install, or (CPU
    tests in the build container only) the read-only reference source."""
    if os.path.isdir(os.path.join(SHIPPED, "bigwht")):
        return SHIPPED
    src = "/root/reference/pkg/src"
    if not gpu and os.path.isdir(os.path.join(src, "bigwht")):
        return src
    return None


def _run(code: str, ref: str, timeout: int = 600, env_extra=None) -> subprocess.CompletedProcess:
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REPO, ref, env.get("PYTHONPATH", "")])
    env.update(env_extra or {})
    return subprocess.run([sys.executable, "-c", textwrap.dedent(code)], cwd=REPO, env=env,
                          capture_output=True, text=True, timeout=timeout)


def _need_ref(gpu: bool) -> str:
    ref = _reference_path(gpu)
    if ref is None:
        pytest.skip("reference package not installed (run baseline/install_reference.sh)")
    return ref


# ------------------------------------------------------------- CPU only ---

def test_errors_derive_from_reference_when_importable():
    ref = _need_ref(False)
    r = _run("""
        import bigwht.errors as R
        import paper_1607_01039_b200 as b
        from paper_1607_01039_b200 import errors as E
        assert E.bound_reference is R
        for ours, theirs in [(E.BigWHTError, R.BigWHTError), (E.ValidationError, R.ValidationError),
                             (E.StorageError, R.StorageError), (E.BadArguments, R.BadArguments),
                             (E.OverflowBoundError, R.OverflowBoundError), (E.InexactDivision, R.InexactDivision),
                             (E.OracleTooLarge, R.OracleTooLarge), (E.InvalidWorkerCount, R.InvalidWorkerCount),
                             (E.BadMetadata, R.BadMetadata), (E.SizeMismatch, R.SizeMismatch),
                             (E.PathExists, R.PathExists), (E.BadDims, R.BadDims), (E.DimMismatch, R.DimMismatch)]:
            assert issubclass(ours, theirs), ours
            assert ours.exit_code == theirs.exit_code, ours
        assert issubclass(E.DeviceError, R.BigWHTError) and E.DeviceError.exit_code == 2
        assert issubclass(E.NotPowerOfTwo, R.BadArguments) and issubclass(E.NotPowerOfTwo, ValueError)
        try:
            raise b.OverflowBoundError("x")
        except R.OverflowBoundError as exc:
            assert exc.exit_code == 3
        # Signal validation raises through the reference classes as well
        import numpy as np
        try:
            b.Signal(np.zeros(3, dtype=np.int64))
        except R.BadArguments:
            pass
        else:
            raise AssertionError("no BadArguments")
        print("ok")
    """, ref)
    assert r.returncode == 0, r.stdout + r.stderr


def test_errors_bind_when_reference_is_added_later():
    """Imported before bigwht is on sys.path: the shim's install() binds."""
    ref = _need_ref(False)
    r = _run(f"""
        import sys
        sys.path = [p for p in sys.path if p != {ref!r}]
        import paper_1607_01039_b200.errors as E
        assert E.bound_reference is None
        sys.path.append({ref!r})
        from paper_1607_01039_b200 import shim
        shim.install()
        import bigwht, bigwht.core, bigwht.parallel, bigwht.external, bigwht.noisy
        assert issubclass(E.OverflowBoundError, bigwht.errors.OverflowBoundError)
        for m in (bigwht, bigwht.core, bigwht.parallel, bigwht.external, bigwht.noisy):
            assert m.fwht_array.__wrapped__.__module__ == "paper_1607_01039_b200.core", m
        assert bigwht.core.check_magnitude_bound.__wrapped__.__module__ == "paper_1607_01039_b200.core"
        print("ok")
    """, ref, env_extra={"PYTHONPATH": REPO})
    assert r.returncode == 0, r.stdout + r.stderr


def test_errors_not_bound_when_disabled():
    ref = _need_ref(False)
    r = _run("""
        import paper_1607_01039_b200.errors as E
        assert E.bound_reference is None
        assert E.BigWHTError.__bases__ == (E._Root,)
        print("ok")
    """, ref, env_extra={"BW_REFERENCE_ERRORS": "0"})
    assert r.returncode == 0, r.stdout + r.stderr


def test_shim_without_device_raises_reference_class():
    """No GPU here: the shimmed fwht_array fails loudly (no CPU fallback),
    with an error a reference caller's ``except BigWHTError`` catches."""
    ref = _need_ref(False)
    r = _run("""
        import numpy as np, torch
        if torch.cuda.is_available():
            print("skip"); raise SystemExit(0)
        from paper_1607_01039_b200 import shim
        shim.install()
        import bigwht.core, bigwht.errors
        try:
            bigwht.core.fwht_array(np.zeros(8, dtype=np.int64))
        except bigwht.errors.BigWHTError as exc:
            assert type(exc).__name__ == "DeviceError" and exc.exit_code == 2
        else:
            raise AssertionError("transform ran without a device")
        print("ok")
    """, ref)
    assert r.returncode == 0, r.stdout + r.stderr


# ------------------------------------------------------------------ GPU ---

REFERENCE_TESTS = ["test_core.py", "test_parallel.py", "test_acceptance.py", "test_external.py",
                   "test_noisy.py", "test_subspace.py", "test_cli.py", "test_dataset.py",
                   "test_iobench.py", "test_perfmodel.py"]


@pytest.mark.gpu
def test_reference_suite_through_shim():
    """The reference's whole unmodified suite (244 tests in /root/reference
    /pkg/tests) with fwht_array and check_magnitude_bound on the B200."""
    ref = _need_ref(True)
    tests_dir = os.path.join(ref, "bigwht_tests")
    if not os.path.isdir(tests_dir):
        pytest.skip("reference tests not shipped (run baseline/install_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REPO, ref, env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "paper_1607_01039_b200.shim",
           "--rootdir", tests_dir, "-c", os.devnull, *[os.path.join(tests_dir, f) for f in REFERENCE_TESTS]]
    r = subprocess.run(cmd, cwd=tests_dir, env=env, capture_output=True, text=True, timeout=1800)
    out = r.stdout + r.stderr
    print(out[-3000:])
    assert r.returncode == 0, out[-6000:]
    line = [ln for ln in out.splitlines() if "bigwht_b200 shim:" in ln]
    assert line, out[-2000:]
    ncalls = int(line[-1].split("=")[1].split(",")[0])
    assert ncalls > 100, line  # the suite's transforms really ran through the B200 path


@pytest.mark.gpu
def test_reference_cli_exit_code_on_b200_overflow(tmp_path):
    """cli.run(['transform', 'mem', ...]) on data breaking the bound: the B200
    check raises, the reference CLI catches it as BigWHTError, exit 3
    (cli.py:577-579), and the dataset is untouched."""
    ref = _need_ref(True)
    path = str(tmp_path / "big.bin")
    r = _run(f"""
        import numpy as np
        from paper_1607_01039_b200 import shim, dataset
        shim.install()
        import bigwht.cli
        x = np.full(16, 1 << 59, dtype=np.int64)
        dataset.write_signal({path!r}, x, "time")
        code = bigwht.cli.run(["transform", "mem", "--in", {path!r}])
        assert code == 3, code
        assert shim.calls["check_magnitude_bound"] >= 1 and shim.calls["fwht_array"] == 0
        arr, kind, dom = dataset.read_signal({path!r})
        assert dom == "time" and np.array_equal(arr, x)
        # and a legal dataset transforms on the B200 through the same command
        ok = str({path!r}) + ".ok"
        y = np.arange(16, dtype=np.int64) - 8
        dataset.write_signal(ok, y, "time")
        assert bigwht.cli.run(["transform", "mem", "--in", ok]) == 0
        assert shim.calls["fwht_array"] == 1
        arr, kind, dom = dataset.read_signal(ok)
        h = np.array([[(-1) ** bin(i & j).count("1") for j in range(16)] for i in range(16)], dtype=np.int64)
        assert dom == "walsh" and np.array_equal(arr, h @ y)
        # run_parallel's chunk phase (parallel.py:151) from 4 threads
        z = np.arange(64, dtype=np.int64) * 3 - 50
        dataset.write_signal(ok + "2", z, "time")
        assert bigwht.cli.run(["transform", "mem", "--in", ok + "2", "--threads", "4"]) == 0
        arr, kind, dom = dataset.read_signal(ok + "2")
        h6 = np.array([[(-1) ** bin(i & j).count("1") for j in range(64)] for i in range(64)], dtype=np.int64)
        assert np.array_equal(arr, h6 @ z)
        print("ok")
    """, ref)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_fwht_array_reference_edge_semantics():
    """Edge behaviour of core.py:97-117 through the drop-in: empty buffer
    (returns 0), int32 (wrapping int32 arithmetic, in place), non-power-of-two
    (refused before mutation with an error that is a ValueError too)."""
    import numpy as np
    import torch

    import paper_1607_01039_b200 as b

    assert b.fwht_array(np.zeros(0, dtype=np.int64)) == 0
    rng = np.random.default_rng(5)
    for n in (0, 1, 5, 12, 17):
        x = rng.integers(-(1 << 31), 1 << 31, 1 << n, dtype=np.int64).astype(np.int32)
        want = x.copy()
        nref = 0
        for k in range(n):  # the reference loop, in int32 (wraps)
            p = want.reshape(-1, 2, 1 << k)
            lo, hi = p[:, 0, :], p[:, 1, :]
            d = lo - hi
            lo += hi
            hi[...] = d
            nref += d.size
        got = x.copy()
        assert b.fwht_array(got) == nref
        assert np.array_equal(got, want), n
        t = torch.from_numpy(x.copy()).cuda()
        b.fwht_array(t)
        assert np.array_equal(t.cpu().numpy(), want), n
    y = np.arange(6, dtype=np.int64)
    with pytest.raises(ValueError):
        b.fwht_array(y)
    assert np.array_equal(y, np.arange(6))


@pytest.mark.gpu
def test_fwht_inplace_known_bound():
    """fwht_inplace(sig, max_abs=M): host-side bound, no reduction pass;
    same result as the checked call; violations raise before mutation."""
    import torch

    import paper_1607_01039_b200 as b

    x = torch.randint(-1000, 1000, (1 << 20,), dtype=torch.int64, device="cuda")
    a = b.fwht_inplace(b.Signal(x.clone())).data
    c = b.fwht_inplace(b.Signal(x.clone()), max_abs=1000).data
    assert torch.equal(a, c)
    big = torch.full((16,), 1 << 59, dtype=torch.int64, device="cuda")
    with pytest.raises(b.OverflowBoundError):
        b.fwht_inplace(b.Signal(big), max_abs=1 << 59)
    assert bool((big == (1 << 59)).all())
    with pytest.raises(b.BadArguments):
        b.fwht_inplace(b.Signal(big), max_abs=-1)
    # numpy buffers take the host-staged call without the device check
    import numpy as np

    h = x.cpu().numpy().copy()
    b.fwht_inplace(b.Signal(h), max_abs=1000)
    assert np.array_equal(h, a.cpu().numpy())
