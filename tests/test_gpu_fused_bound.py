"""fwht_inplace with the magnitude bound fused into the low pass
(bw_fwht_inplace_i64 for n >= 22): the reference's semantics (core.py:80-94,
120-125) -- OverflowBoundError raised BEFORE any mutation when some
|x| * 2^n >= 2^63 -- with the tiles that were already transformed restored
exactly, and the transform bit-identical to the oracle otherwise."""

import numpy as np
import pytest
import torch

import paper_1607_01039_b200 as bw
from paper_1607_01039_b200 import errors
from oracle import oracle_np

pytestmark = pytest.mark.gpu


def c_fwht(coracle, x):
    y = np.ascontiguousarray(x, dtype=np.int64).copy()
    coracle.oracle_fwht_i64(y.ctypes.data, int(y.size).bit_length() - 1)
    return y


@pytest.mark.parametrize("n", [22, 23, 24])
def test_fused_bound_at_the_edge_transforms(coracle, n):
    edge = (1 << (63 - n)) - 1  # the largest |x| the bound allows
    rng = np.random.default_rng(n)
    x = rng.integers(-edge, edge + 1, size=1 << n, dtype=np.int64)
    x[rng.integers(0, 1 << n, size=32)] = edge
    x[rng.integers(0, 1 << n, size=32)] = -edge
    sig = bw.fwht_inplace(bw.Signal(torch.from_numpy(x.copy()).cuda()))
    assert sig.domain == bw.Domain.WALSH
    assert np.array_equal(sig.data.cpu().numpy(), c_fwht(coracle, x))


@pytest.mark.parametrize("where", ["first", "middle", "last", "everywhere", "min_int64"])
@pytest.mark.parametrize("n", [22, 24])
def test_fused_bound_violation_raises_before_mutation(n, where):
    edge = (1 << (63 - n)) - 1
    x = oracle_np.gen(2, 31 + n, [1 << 20], 0, 1 << n)
    if where == "first":
        x[5] = edge + 1
    elif where == "middle":
        x[(1 << n) // 2 + 77] = -(edge + 1)
    elif where == "last":
        x[-1] = edge + 1
    elif where == "everywhere":
        x = np.random.default_rng(1).integers(-(1 << 62), 1 << 62, size=1 << n, dtype=np.int64)
    else:
        x[(1 << n) - 3000] = np.iinfo(np.int64).min
    t = torch.from_numpy(x.copy()).cuda()
    sig = bw.Signal(t)
    with pytest.raises(errors.OverflowBoundError):
        bw.fwht_inplace(sig)
    assert sig.domain == bw.Domain.TIME
    assert np.array_equal(t.cpu().numpy(), x)  # untouched, bit for bit


def test_fused_bound_matches_the_separate_reduction(coracle, monkeypatch):
    n = 23
    x = oracle_np.gen(1, 5, [], 0, 1 << n)
    a = bw.fwht_inplace(bw.Signal(torch.from_numpy(x.copy()).cuda())).data.cpu().numpy()
    monkeypatch.setenv("BW_FUSED_BOUND", "0")  # read once per process: run the other path in a child
    import subprocess
    import sys
    code = ("import numpy as np, torch, sys; sys.path.insert(0, '.');"
            "import paper_1607_01039_b200 as bw; from oracle import oracle_np;"
            f"x = oracle_np.gen(1, 5, [], 0, 1 << {n});"
            "y = bw.fwht_inplace(bw.Signal(torch.from_numpy(x.copy()).cuda())).data.cpu().numpy();"
            "sys.stdout.write(str(int(np.bitwise_xor.reduce(y.view(np.uint64)))))")
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=root,
                       env=dict(os.environ, BW_FUSED_BOUND="0"), timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert int(r.stdout) == int(np.bitwise_xor.reduce(a.view(np.uint64)))
    assert np.array_equal(a, c_fwht(coracle, x))
