"""Drop-in core API: ``Signal``, ``fwht_array``, ``fwht_inplace``, ...

Mirrors /root/reference/pkg/src/bigwht/core.py (same names, argument
meaning, return values and exceptions) with the arithmetic moved to the
B200 kernels behind the C ABI (include/bigwht_b200.h).

Accepted buffers:
  * torch CUDA tensors (int64 or float64, 1-D, contiguous) -- transformed in
    place in HBM, ordered on torch's current CUDA stream;
  * numpy arrays (the reference's own type) -- staged through the device
    (host -> HBM -> transform -> host, same call), so reference callers and
    tests work unchanged.  There is no CPU arithmetic path.
"""

from __future__ import annotations

import ctypes
import os
import threading
import enum
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import BadArguments, DeviceError, NotPowerOfTwo, OracleTooLarge, OverflowBoundError

# Brute force costs O(4**n); core.py:24-27 uses the same default limit.
ORACLE_LIMIT_DEFAULT = 14

_INT64_LIMIT = 1 << 63


class Domain(enum.Enum):
    """core.py:32-34."""

    TIME = "time"
    WALSH = "walsh"


def _is_power_of_two(value: int) -> bool:
    return value > 0 and (value & (value - 1)) == 0


def _length(buf) -> int:
    return int(buf.shape[0])


def _log2(buf) -> int:
    return _length(buf).bit_length() - 1


def _dtype_kind(buf) -> str:
    """'i64', 'f64' or a description of an unsupported dtype."""
    if isinstance(buf, torch.Tensor):
        if buf.dtype == torch.int64:
            return "i64"
        if buf.dtype == torch.float64:
            return "f64"
        return str(buf.dtype)
    if isinstance(buf, np.ndarray):
        if buf.dtype == np.dtype(np.int64):
            return "i64"
        if buf.dtype == np.dtype(np.float64):
            return "f64"
        return str(buf.dtype)
    raise BadArguments(f"unsupported buffer type {type(buf).__name__}")


def _stream_handle(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _require_cuda(t: torch.Tensor) -> None:
    if not t.is_cuda:
        raise BadArguments("torch buffers must live on a CUDA device (no CPU path)")


@dataclass
class Signal:
    """A 1-D array of 2**n samples tagged with its current domain
    (core.py:37-77).  ``data`` is a torch CUDA tensor or a numpy array of
    dtype int64 (exact) or float64."""

    data: object
    domain: Domain = Domain.TIME

    def __post_init__(self) -> None:
        if isinstance(self.data, torch.Tensor):
            arr = self.data
        else:
            arr = np.asarray(self.data)
        if arr.ndim != 1:
            raise BadArguments("signal data must be one-dimensional")
        if not _is_power_of_two(_length(arr)):
            raise BadArguments(f"signal length {_length(arr)} is not a power of two")
        kind = _dtype_kind(arr)
        if kind not in ("i64", "f64"):
            raise BadArguments(f"unsupported dtype {kind}; use int64 or float64")
        # The in-place kernels need contiguous storage (core.py:60-62).
        if isinstance(arr, torch.Tensor):
            self.data = arr.contiguous()
        else:
            self.data = np.ascontiguousarray(arr)

    @property
    def log2_dim(self) -> int:
        return _log2(self.data)

    @property
    def dim(self) -> int:
        return _length(self.data)

    @property
    def is_exact(self) -> bool:
        return _dtype_kind(self.data) == "i64"

    def copy(self) -> "Signal":
        return Signal(self.data.clone() if isinstance(self.data, torch.Tensor) else self.data.copy(), self.domain)


# ----------------------------------------------------------------- helpers ---

def _check_contiguous(buf) -> None:
    if isinstance(buf, torch.Tensor):
        ok = buf.is_contiguous()
    else:
        ok = buf.flags.c_contiguous
    if not ok:
        raise BadArguments("in-place transform needs a contiguous buffer")


def _check_shape(buf) -> int:
    if buf.ndim != 1:
        raise BadArguments("signal data must be one-dimensional")
    if not _is_power_of_two(_length(buf)):
        # The reference would raise numpy's ValueError after mutating part of
        # the buffer; we refuse before any launch, with
        # an error that is both a BadArguments and a ValueError.
        raise NotPowerOfTwo(f"signal length {_length(buf)} is not a power of two")
    return _log2(buf)


class _HostStage:
    """Device workspace for numpy buffers, reused between calls.  One per
    host thread (the calls using it are synchronous, so a thread never has
    two uses in flight and threads never share one)."""

    _local = threading.local()

    @classmethod
    def get(cls, n: int, dtype, slot: int = 0) -> torch.Tensor:
        work = getattr(cls._local, "work", None)
        if work is None:
            work = cls._local.work = {}
        dev = torch.cuda.current_device()
        key = (dev, dtype) if slot == 0 else (dev, dtype, slot)
        w = work.get(key)
        if w is None or w.numel() < (1 << n):
            w = torch.empty(1 << n, dtype=dtype, device=f"cuda:{dev}")
            work[key] = w
        return w[: 1 << n]


def _need_cuda() -> None:
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device is visible; the transform runs only on a B200")


# ------------------------------------------------------------------- API ---

def check_magnitude_bound(data, log2_dim: int) -> None:
    """Enforce M * 2**n < 2**63 for int64 data (core.py:80-94), on the GPU."""
    if _dtype_kind(data) != "i64" or _length(data) == 0:
        return
    if isinstance(data, np.ndarray):
        _need_cuda()
        data = np.ascontiguousarray(data).reshape(-1)
        if _is_power_of_two(_length(data)):
            work = _HostStage.get(_log2(data), torch.int64)
            work.copy_(torch.from_numpy(data))
        else:
            work = torch.from_numpy(data).cuda()
        data = work
    _require_cuda(data)
    with torch.cuda.device(data.device):
        if log2_dim > 63:
            raise OverflowBoundError(f"n = {log2_dim} cannot satisfy the int64 bound")
        m = ctypes.c_uint64(0)
        # bw_check_bound_i64 needs the signal length to be 2**log2n; for an
        # arbitrary length use the raw reduction and apply the bound here.
        if _length(data) == (1 << _log2(data)) and _log2(data) == log2_dim:
            _lib.check(_lib.lib().bw_check_bound_i64(data.data_ptr(), log2_dim, None,
                                                     _stream_handle(data), ctypes.byref(m)))
            return
        out = torch.empty(2, dtype=torch.int64, device=data.device)
        _lib.check(_lib.lib().bw_minmax_i64(data.data_ptr(), _length(data), out.data_ptr(),
                                            _stream_handle(data)))
        mx, mn = (int(v) for v in out.tolist())
        magnitude = max(mx, -mn)
        if magnitude << log2_dim >= _INT64_LIMIT:
            raise OverflowBoundError(
                f"max |x| = {magnitude} with n = {log2_dim} can overflow int64; need |x| * 2**n < 2**63"
            )


last_narrow = False  # whether the last fwht_array call ran the narrow plan (diagnostics)
NARROW_MIN_N = 22  # below this the transform is launch-bound and the flag readback costs more than it saves


def _narrow_wanted(n: int, narrow) -> int:
    """Work-buffer bytes of the narrow-intermediate plan if it should be
    tried for this call, else 0.  narrow=None follows BW_NARROW=1 (off by
    default: 5% faster at n = 32 on +-1 signals, but it needs a work buffer of
    3/4 of the signal (24 GiB at n = 32)),
    for n >= NARROW_MIN_N and when the work buffer fits in free device
    memory with 2 GiB left."""
    if narrow is False:
        return 0
    need = int(_lib.lib().bw_narrow_scratch_bytes(n))
    if need == 0:
        return 0
    if narrow is None:
        if os.environ.get("BW_NARROW", "0") != "1" or n < NARROW_MIN_N:
            return 0
        free, _ = torch.cuda.mem_get_info()
        if need + (2 << 30) > free:
            return 0
    return need


last_compact = False  # whether the last fwht_array call ran the compact in-place plan (diagnostics)


def _compact_wanted(n: int, compact) -> bool:
    """Whether fwht_array tries the compact in-place plan (int32
    intermediates inside the signal's own buffer, bw_fwht_i64_compact).
    compact=None follows the library's default (bw_compact_auto: n = 26..34,
    where the plan measured a fifth to a third faster; BW_COMPACT=1 / 0 widens
    it to n >= 22 / turns it off)."""
    if compact is False or _lib.lib().bw_compact_npasses(n) == 0:
        return False
    if compact is None:
        return bool(_lib.lib().bw_compact_auto(n))
    return True


def fwht_array(buf, narrow=None, compact=None) -> int:
    """Transform ``buf`` (length 2**n, contiguous) in place (core.py:97-117).

    Stage k pairs elements at stride 2**k and replaces (a, b) with
    (a + b, a - b).  Returns n * 2**(n-1).  No magnitude check, exactly like
    the reference: int64 arithmetic wraps mod 2**64 as numpy's does.

    narrow=True runs the narrow-intermediate plan on a CUDA int64 tensor
    (bw_fwht_i64_narrow: int16 / int32 intermediates for signals whose
    values stay within +-32767 after the low pass, e.g. +-1 Boolean
    signals; otherwise the int64 plan runs, results identical either way).
    It measured 5% faster at n = 32 (30.4 vs 32.1 ms, two tiles per CTA) but
    needs a work buffer of 3/4 of the signal, so the default (None) uses it
    only when BW_NARROW=1.

    compact (CUDA int64 tensors): the compact in-place plan
    (bw_fwht_i64_compact) -- the high-bit stages first with the signal kept
    as int32 inside its own buffer, then the low pass widening back to int64.
    Its first pass tests every input against lim(n) (7 at n = 32, 31 at
    n = 30); if one is larger, the tiles already written are restored exactly
    and the int64 plan runs.  Results are identical either way.  None: the
    library's default (tried at n = 26..34, where it measured faster: 21.7 vs
    31.4 ms at n = 32, 103.8 vs 140.1 at n = 34; BW_COMPACT=1 / 0: n >= 22 /
    never); True: the
    checked plan; False: the int64 plan; an int: a bound on |x| the caller
    guarantees (no test, no synchronisation).
    """
    global last_narrow, last_compact
    last_narrow = False
    last_compact = False
    _check_contiguous(buf)
    if buf.ndim == 1 and _length(buf) == 0:
        return 0  # core.py:106-107: n = -1, no stage runs
    n = _check_shape(buf)
    kind = _dtype_kind(buf)
    if kind in ("int32", "torch.int32"):
        return _fwht_int32(buf, n)
    if kind not in ("i64", "f64"):
        raise BadArguments(f"unsupported dtype {kind}; use int64 or float64 (or int32)")
    _need_cuda()
    bf = ctypes.c_uint64(0)
    L = _lib.lib()
    if isinstance(buf, np.ndarray):
        if kind == "i64":
            work = _HostStage.get(n, torch.int64)
            _lib.check(L.bw_fwht_host_i64(buf.ctypes.data, n, work.data_ptr(), 0,
                                          _stream_handle(work), ctypes.byref(bf)))
            return int(bf.value)
        work = _HostStage.get(n, torch.float64)
        work.copy_(torch.from_numpy(buf))
        with torch.cuda.device(work.device):
            _lib.check(L.bw_fwht_f64(work.data_ptr(), n, _stream_handle(work), ctypes.byref(bf)))
        buf[...] = work.cpu().numpy()
        return int(bf.value)
    _require_cuda(buf)
    with torch.cuda.device(buf.device):
        need = _narrow_wanted(n, narrow) if kind == "i64" else 0
        if kind == "i64" and not need and _compact_wanted(n, compact):
            used = ctypes.c_int(0)
            bound = -1 if compact is None or compact is True else int(compact)
            if bound < -1:
                raise BadArguments(f"compact bound must be >= 0, got {bound}")
            _lib.check(L.bw_fwht_i64_compact(buf.data_ptr(), n, bound, _stream_handle(buf), ctypes.byref(used),
                                             ctypes.byref(bf)))
            last_compact = bool(used.value)
        elif need:
            work = torch.empty(need, dtype=torch.uint8, device=buf.device)
            used = ctypes.c_int(0)
            _lib.check(L.bw_fwht_i64_narrow(buf.data_ptr(), n, work.data_ptr(), need, _stream_handle(buf),
                                            ctypes.byref(used), ctypes.byref(bf)))
            last_narrow = bool(used.value)
        elif kind == "i64":  # (the compact default was decided above: bw_fwht_i64 would ask again)
            _lib.check(L.bw_fwht_i64_int64plan(buf.data_ptr(), n, _stream_handle(buf), ctypes.byref(bf)))
        else:
            _lib.check(L.bw_fwht_f64(buf.data_ptr(), n, _stream_handle(buf), ctypes.byref(bf)))
    return int(bf.value)


def _fwht_int32(buf, n: int) -> int:
    """fwht_array on an int32 buffer: the reference transforms it in place
    in wrapping int32 arithmetic (core.py:108-115 on an int32 array;
    SURVEY.md 8b).  Reduction mod 2**32 commutes with every add/sub, so the
    exact int64 transform (bw_fwht_widen_i32: the first pass reads the
    int32 source) truncated to its low 32 bits is that result, bit for bit."""
    _need_cuda()
    src = torch.from_numpy(buf).cuda() if isinstance(buf, np.ndarray) else buf
    _require_cuda(src)
    bf = ctypes.c_uint64(0)
    out = torch.empty(1 << n, dtype=torch.int64, device=src.device)
    with torch.cuda.device(src.device):
        _lib.check(_lib.lib().bw_fwht_widen_i32(src.data_ptr(), out.data_ptr(), n, _stream_handle(src),
                                                ctypes.byref(bf)))
        low = out.to(torch.int32)  # two's-complement truncation, mod 2**32
        if isinstance(buf, np.ndarray):
            buf[...] = low.cpu().numpy()
        else:
            buf.copy_(low)
    return int(bf.value)


def fwht_arrays(buffers) -> list[int]:
    """fwht_array on each of several host int64 numpy buffers of the same
    length 2**n (each in place; core.py:97-117 per buffer).  The device
    alternates between two work buffers, so one buffer's host->device copy
    overlaps the previous one's device->host copy (bw_fwht_host_batch_i64);
    with pinned (page-locked) buffers PCIe then runs in both directions at
    once.  Returns the butterfly counts."""
    bufs = list(buffers)
    if not bufs:
        return []
    for b in bufs:
        if not isinstance(b, np.ndarray) or _dtype_kind(b) != "i64":
            raise BadArguments("fwht_arrays takes int64 numpy buffers")
        _check_contiguous(b)
    n = _check_shape(bufs[0])
    if any(b.shape != bufs[0].shape for b in bufs):
        raise BadArguments("fwht_arrays needs buffers of one length")
    _need_cuda()
    # two device buffers: the steady state then runs at the PCIe duplex rate
    # (~49 GB/s each way, tools/pcie_duplex.py); a third (BW_BATCH_BUFFERS=3)
    # measured no faster (profiles/r01_e2e_buffers.log)
    nwork = 1 if len(bufs) == 1 else 2
    if len(bufs) > 2 and os.environ.get("BW_BATCH_BUFFERS", "2") == "3":
        free, _ = torch.cuda.mem_get_info()
        have = sum(w.numel() * 8 for k, w in getattr(_HostStage._local, "work", {}).items()
                   if k[:2] == (torch.cuda.current_device(), torch.int64) and w.numel() >= (1 << n))
        if (8 << n) * 3 - have + (2 << 30) <= free:
            nwork = 3
    works = [_HostStage.get(n, torch.int64, slot=b) for b in range(nwork)]
    arr = (ctypes.c_void_p * len(bufs))(*[b.ctypes.data for b in bufs])
    warr = (ctypes.c_void_p * nwork)(*[w.data_ptr() for w in works])
    bf = ctypes.c_uint64(0)
    _lib.check(_lib.lib().bw_fwht_host_batch_i64(arr, len(bufs), n, warr, nwork, _stream_handle(works[0]),
                                                 ctypes.byref(bf)))
    return [int(bf.value)] * len(bufs)


def fwht_widen(x) -> torch.Tensor:
    """Out-of-place transform of an int32 signal into a new int64 CUDA
    tensor: the reference's fwht_array(x.astype(np.int64)) (core.py:97-117;
    a bare int32 buffer there would wrap in int32), computed with the first
    pass reading the int32 source directly.  Accepts a CUDA int32 tensor or a
    numpy int32 array."""
    if isinstance(x, np.ndarray):
        _need_cuda()
        x = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    if not isinstance(x, torch.Tensor) or x.dtype != torch.int32:
        raise BadArguments("fwht_widen expects int32 input")
    _require_cuda(x)
    _check_contiguous(x)
    n = _check_shape(x)
    out = torch.empty(1 << n, dtype=torch.int64, device=x.device)
    with torch.cuda.device(x.device):
        _lib.check(_lib.lib().bw_fwht_widen_i32(x.data_ptr(), out.data_ptr(), n, _stream_handle(x), None))
    return out


def _flip(domain: Domain) -> Domain:
    return Domain.WALSH if domain == Domain.TIME else Domain.TIME


def fwht_inplace(sig: Signal, max_abs: int | None = None) -> Signal:
    """Fast in-place WHT; flips the domain tag and returns its argument
    (core.py:120-125).  The magnitude bound is checked on the device before
    any mutation (OverflowBoundError leaves the data untouched).

    ``max_abs``: a bound M >= max|x| the caller already knows (a generator's
    range, an earlier check).  M * 2**n < 2**63 is then checked on the host
    and the 8 B/point reduction pass is skipped (bw_fwht_inplace_known_i64),
    so the call costs what fwht_array costs.  The caller vouches for M."""
    buf = sig.data
    n = sig.log2_dim
    _need_cuda()
    L = _lib.lib()
    bf = ctypes.c_uint64(0)
    if max_abs is not None:
        max_abs = int(max_abs)
        if max_abs < 0:
            raise BadArguments(f"max_abs must be >= 0, got {max_abs}")
        if sig.is_exact and max_abs << n >= _INT64_LIMIT:
            raise OverflowBoundError(
                f"max |x| = {max_abs} with n = {n} can overflow int64; need |x| * 2**n < 2**63")
    if sig.is_exact:
        if isinstance(buf, np.ndarray):
            work = _HostStage.get(n, torch.int64)
            _lib.check(L.bw_fwht_host_i64(buf.ctypes.data, n, work.data_ptr(), 1 if max_abs is None else 0,
                                          _stream_handle(work), ctypes.byref(bf)))
        else:
            _require_cuda(buf)
            with torch.cuda.device(buf.device):
                if max_abs is not None:
                    _lib.check(L.bw_fwht_inplace_known_i64(buf.data_ptr(), n, max_abs, _stream_handle(buf),
                                                           ctypes.byref(bf)))
                else:
                    _lib.check(L.bw_fwht_inplace_i64(buf.data_ptr(), n, None, _stream_handle(buf),
                                                     ctypes.byref(bf)))
    else:
        fwht_array(buf)
    sig.domain = _flip(sig.domain)
    return sig


def inverse_wht_inplace(sig: Signal) -> Signal:
    """Inverse transform in place (core.py:147-173): forward WHT then exact
    division by 2**n; on an inexact int64 division the buffer is restored
    and InexactDivision raised."""
    if sig.domain != Domain.WALSH:
        raise BadArguments("inverse transform expects a Walsh-domain signal")
    n = sig.log2_dim
    _need_cuda()
    L = _lib.lib()
    buf = sig.data
    host = None
    if isinstance(buf, np.ndarray):
        host = buf
        buf = _HostStage.get(n, torch.int64 if sig.is_exact else torch.float64)
        buf.copy_(torch.from_numpy(host))
    _require_cuda(buf)
    try:
        with torch.cuda.device(buf.device):
            if sig.is_exact:
                _lib.check(L.bw_inverse_i64(buf.data_ptr(), n, None, _stream_handle(buf)))
            else:
                _lib.check(L.bw_inverse_f64(buf.data_ptr(), n, _stream_handle(buf)))
    finally:
        if host is not None:
            host[...] = buf.cpu().numpy()
    sig.domain = Domain.TIME
    return sig


def _device_copy(buf) -> torch.Tensor:
    if isinstance(buf, torch.Tensor):
        _require_cuda(buf)
        return buf
    _need_cuda()
    return torch.from_numpy(np.ascontiguousarray(buf)).cuda()


def wht_bruteforce(sig: Signal, limit: int = ORACLE_LIMIT_DEFAULT) -> Signal:
    """Reference transform by the defining double sum (core.py:128-144);
    input unchanged, result returned as a new Signal of the same kind
    (torch CUDA or numpy) with the domain flipped.  O(4**n) on the GPU."""
    n = sig.log2_dim
    if n > limit:
        raise OracleTooLarge(f"n = {n} exceeds the oracle limit {limit}")
    if not sig.is_exact:
        raise BadArguments("the device brute force is implemented for int64 signals")
    check_magnitude_bound(sig.data, n)
    x = _device_copy(sig.data)
    y = torch.empty_like(x)
    with torch.cuda.device(x.device):
        _lib.check(_lib.lib().bw_wht_bruteforce_i64(x.data_ptr(), y.data_ptr(), n, _stream_handle(x)))
    out = y if isinstance(sig.data, torch.Tensor) else y.cpu().numpy()
    return Signal(out, _flip(sig.domain))


def parseval_energy(sig: Signal):
    """Sum of squared components (core.py:176-185).  int64: exact (Python
    int, beyond 2**63), from 192-bit partial sums computed on the GPU.
    float64: float."""
    x = _device_copy(sig.data)
    if not sig.is_exact:
        return float(torch.dot(x, x).item())
    nblocks = max(1, min(4096, x.numel() >> 16))  # contiguous ranges of >= 2^16 points per CTA
    part = torch.empty(3 * nblocks, dtype=torch.int64, device=x.device)
    with torch.cuda.device(x.device):
        _lib.check(_lib.lib().bw_sumsq_partials_i64(x.data_ptr(), x.numel(), part.data_ptr(), nblocks,
                                                    _stream_handle(x)))
    words = [w & ((1 << 64) - 1) for w in part.cpu().tolist()]
    return sum(words[3 * b] + (words[3 * b + 1] << 64) + (words[3 * b + 2] << 128) for b in range(nblocks))


def butterfly_count(n: int) -> int:
    """n * 2**(n-1), the value fwht_array returns (core.py:117)."""
    return n << max(n - 1, 0)
