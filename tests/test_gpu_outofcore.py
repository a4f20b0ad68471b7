"""Out-of-core transform (external.py:65-283 semantics, host memory as the
disk): byte-identical to the in-memory transform for every workspace size,
on pinned, pageable and file-backed (np.memmap) host buffers."""

import numpy as np
import pytest
import torch

import paper_1607_01039_b200 as bw
from paper_1607_01039_b200 import outofcore
from oracle import oracle_np

pytestmark = pytest.mark.gpu


def c_fwht(coracle, x):
    y = x.copy()
    coracle.oracle_fwht_i64(y.ctypes.data, int(y.size).bit_length() - 1)
    return y


@pytest.mark.parametrize("n,log2_work", [(16, 16), (18, 16), (20, 16), (22, 17), (22, 20), (24, 18), (24, 24)])
def test_block_size_independence(coracle, n, log2_work):
    """External == in-memory for every block size (test_external.py:120-129,
    test_acceptance.py:135-189)."""
    x = oracle_np.gen(2, n * 7 + log2_work, [1 << 20], 0, 1 << n)
    buf = torch.from_numpy(x.copy()).pin_memory().numpy()
    passes = outofcore.fwht_out_of_core(buf, log2_work)
    assert passes == outofcore.plan_host_passes(n, min(log2_work, max(n, 15)))
    assert np.array_equal(buf, c_fwht(coracle, x))


def test_pageable_and_memmap(coracle, tmp_path):
    n = 21
    x = oracle_np.gen(1, 3, [], 0, 1 << n)
    ref = c_fwht(coracle, x)
    a = x.copy()  # pageable
    outofcore.fwht_out_of_core(a, 17)
    assert np.array_equal(a, ref)
    path = tmp_path / "signal.bin"  # raw little-endian int64, like dataset.py's payload
    x.astype("<i8").tofile(path)
    mm = np.memmap(path, dtype="<i8", mode="r+", shape=(1 << n,))
    outofcore.fwht_out_of_core(mm, 16)
    mm.flush()
    assert np.array_equal(np.fromfile(path, dtype="<i8"), ref)


def test_rejects_bad_buffers():
    with pytest.raises(bw.BadArguments):
        outofcore.fwht_out_of_core(np.zeros(1 << 10, dtype=np.int32), 16)
    with pytest.raises(bw.BadArguments):
        outofcore.fwht_out_of_core(np.zeros(3 << 10, dtype=np.int64), 16)
    with pytest.raises(bw.BadArguments):
        outofcore.fwht_out_of_core(np.zeros(1 << 20, dtype=np.int64)[::2], 16)


@pytest.mark.slow
def test_n30_through_a_1gib_workspace():
    """8 GiB host signal through a 1 GiB device workspace (2 host passes) ==
    the in-HBM transform of the same signal."""
    from paper_1607_01039_b200 import signals

    spec = signals.config(3, n=30)
    t = signals.make(spec)
    host = torch.empty(1 << 30, dtype=torch.int64, pin_memory=True)
    host.copy_(t)
    bw.fwht_array(t)
    passes = outofcore.fwht_out_of_core(host.numpy(), 27)
    assert passes == 2
    ht = host.to("cuda")
    assert torch.equal(ht, t)
