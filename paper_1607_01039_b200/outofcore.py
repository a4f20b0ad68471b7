"""Out-of-core transform of host arrays larger than the device workspace.

The paper's own contribution (Fig. 3; the reference implements it
for disk datasets in /root/reference/pkg/src/bigwht/external.py:65-283):
transform contiguous blocks in memory, then sweep the remaining high bits in
block passes.  Here host memory plays the disk and a bounded device
workspace plays RAM; every pass merges as many stages as the workspace
allows (external.py does one stage per disk pass after the first).  Works
on any host numpy buffer -- pinned memory for full PCIe speed, or an
np.memmap of a raw little-endian int64 dataset file.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .core import _check_contiguous, _check_shape, _need_cuda
from .errors import BadArguments


def plan_host_passes(n: int, log2_work: int) -> int:
    """Number of passes over host memory (cf. plan_external's q,
    external.py:65-97): 1 if the signal fits the workspace, else 1 + the
    high-bit passes of up to log2_work - 14 bits each."""
    if n <= log2_work:
        return 1
    cb = log2_work - 1
    g = cb - 13
    return 1 + -(-(n - cb) // g)


def fwht_out_of_core(buf: np.ndarray, log2_work: int = 30, workspace: torch.Tensor | None = None) -> int:
    """In-place FWHT of a host int64 array through a device workspace of
    2**log2_work elements.  Returns the number of host passes."""
    if not isinstance(buf, np.ndarray) or buf.dtype != np.int64:
        raise BadArguments("out-of-core transform needs a host int64 numpy buffer")
    _check_contiguous(buf)
    n = _check_shape(buf)
    _need_cuda()
    if log2_work < 15:
        raise BadArguments("the device workspace needs at least 2**15 elements")
    log2_work = min(log2_work, max(n, 15))
    if workspace is None:
        workspace = torch.empty(1 << log2_work, dtype=torch.int64, device="cuda")
    if workspace.numel() < (1 << log2_work) or workspace.dtype != torch.int64 or not workspace.is_cuda:
        raise BadArguments("workspace must be a CUDA int64 tensor of 2**log2_work elements")
    passes = ctypes.c_int(0)
    with torch.cuda.device(workspace.device):
        _lib.check(_lib.lib().bw_fwht_host_ooc_i64(buf.ctypes.data, n, workspace.data_ptr(), log2_work,
                                                   torch.cuda.current_stream().cuda_stream, ctypes.byref(passes)))
    return int(passes.value)
