"""Threshold extraction of Walsh coefficients on the GPU (kernel K5).

Reference: /root/reference/pkg/src/bigwht/noisy.py:185-222 (``extract_above``
returns every (index, coefficient) with |coefficient| >= tau, sorted by
(-|coefficient|, index)).  The BASELINE configs 3 and 5 ask for |W| > tau
sorted by index, which for integers is ``>= tau + 1`` -- ``extract_gt``.

The device kernels produce hits already in index order (per-chunk counts,
an exclusive scan, then an ordered rewrite of the chunks that hold hits), so
no device sort is needed; ``extract_above`` re-sorts the (few) hits on the
host into the reference's magnitude order.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .core import Domain, Signal, _log2, _need_cuda, _stream_handle
from .errors import BadArguments


def _as_device(data) -> torch.Tensor:
    if isinstance(data, torch.Tensor):
        if not data.is_cuda:
            raise BadArguments("torch buffers must live on a CUDA device")
        return data
    return torch.from_numpy(np.ascontiguousarray(data)).cuda()


def extract_ge(data, tau, base: int = 0, cap: int = 1 << 16):
    """All hits with |x| >= tau as (index, value) CUDA tensors sorted by
    index (values int64, or float64 for float64 signals, noisy.py:217-222).
    ``base`` is added to every index (shards of a larger signal)."""
    if tau < 0:
        raise BadArguments(f"tau must be >= 0, got {tau}")
    _need_cuda()
    d = _as_device(data)
    if d.dtype not in (torch.int64, torch.float64):
        raise BadArguments("GPU extraction is implemented for int64 and float64 signals")
    if not d.is_contiguous():
        raise BadArguments("extraction needs a contiguous buffer")
    n = _log2(d)
    L = _lib.lib()
    while True:
        idx = torch.empty(max(cap, 1), dtype=torch.int64, device=d.device)
        val = torch.empty(max(cap, 1), dtype=d.dtype, device=d.device)
        count = ctypes.c_uint64(0)
        with torch.cuda.device(d.device):
            if d.dtype == torch.float64:
                st = L.bw_extract_ge_f64(d.data_ptr(), n, float(tau), int(base), idx.data_ptr(), val.data_ptr(),
                                         cap, None, _stream_handle(d), ctypes.byref(count))
            else:
                st = L.bw_extract_ge_i64(d.data_ptr(), n, int(tau), int(base), idx.data_ptr(), val.data_ptr(),
                                         cap, None, _stream_handle(d), ctypes.byref(count))
        if st == _lib.BW_CAPACITY:
            cap = int(count.value)
            continue
        _lib.check(st)
        k = int(count.value)
        return idx[:k], val[:k]


def fwht_extract_ge(data: torch.Tensor, tau: int, base: int = 0, cap: int = 1 << 16):
    """Transform ``data`` in place (fwht_array) and return every hit with
    |W| >= tau as (index, value) CUDA tensors sorted by index; the threshold
    test runs in the last pass's epilogue (configs 3/5 of BASELINE.json)."""
    if tau < 0:
        raise BadArguments(f"tau must be >= 0, got {tau}")
    _need_cuda()
    if not isinstance(data, torch.Tensor) or not data.is_cuda or data.dtype != torch.int64:
        raise BadArguments("fwht_extract needs a CUDA int64 tensor")
    if not data.is_contiguous():
        raise BadArguments("in-place transform needs a contiguous buffer")
    n = _log2(data)
    if data.numel() != 1 << n:
        raise BadArguments(f"signal length {data.numel()} is not a power of two")
    L = _lib.lib()
    idx = torch.empty(max(cap, 1), dtype=torch.int64, device=data.device)
    val = torch.empty(max(cap, 1), dtype=torch.int64, device=data.device)
    count = ctypes.c_uint64(0)
    with torch.cuda.device(data.device):
        st = L.bw_fwht_extract_i64(data.data_ptr(), n, int(tau), int(base), idx.data_ptr(), val.data_ptr(), cap,
                                   _stream_handle(data), ctypes.byref(count))
    if st == _lib.BW_CAPACITY:  # the transform is done; re-extract with room
        return extract_ge(data, tau, base, cap=int(count.value))
    _lib.check(st)
    k = int(count.value)
    return idx[:k], val[:k]


def fwht_extract_gt(data: torch.Tensor, tau: int, base: int = 0):
    """Config semantics: transform, then |W| > tau sorted by index."""
    return fwht_extract_ge(data, int(tau) + 1, base)


def extract_gt(data, tau: int, base: int = 0):
    """Config semantics: |W| > tau, (index, value) sorted by index."""
    return extract_ge(data, int(tau) + 1, base)


def extract_above(sig: Signal, tau) -> list[tuple[int, int | float]]:
    """noisy.py:185-198: (index, coefficient) with |coefficient| >= tau,
    largest magnitude first, ties by ascending index (int values for int64
    signals, float values for float64 ones, noisy.py:219-222)."""
    if sig.domain != Domain.WALSH:
        raise BadArguments("extraction expects a Walsh-domain signal")
    if tau < 0:
        raise BadArguments(f"tau must be >= 0, got {tau}")
    if sig.is_exact:
        t = int(-(-tau // 1)) if not isinstance(tau, int) else tau  # ceil for float tau
    else:
        t = float(tau)
    idx, val = extract_ge(sig.data, t)
    hits = list(zip(idx.tolist(), val.tolist()))
    hits.sort(key=lambda item: (-abs(item[1]), item[0]))
    return hits
