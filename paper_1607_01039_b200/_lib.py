"""ctypes binding of the C ABI (include/bigwht_b200.h).

This is exactly the stub a maintainer of the reference would add to bind the
library.  There is no fallback: if the shared library is
missing or the device is not a B200, every call raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
# BW_LIB_PATH selects an alternative build of the same library (experiments).
LIB_PATH = os.environ.get("BW_LIB_PATH") or os.path.join(_HERE, "lib", "libbigwht_b200.so")

BW_OK = 0
_STATUS = {
    1: errors.BadArguments,
    2: errors.OverflowBoundError,
    3: errors.InexactDivision,
    4: errors.InvalidWorkerCount,
    5: errors.BadArguments,
    6: errors.DeviceError,
    7: errors.DeviceError,
}
BW_CAPACITY = 5

GEN_PM1 = 1
GEN_UNIFORM = 2
GEN_NOISY_MASKS = 3

_lib = None

P = ctypes.c_void_p
U64 = ctypes.c_uint64
I32 = ctypes.c_int
PU64 = ctypes.POINTER(ctypes.c_uint64)

_SIGNATURES = {
    "bw_abi_version": ([], I32),
    "bw_last_error": ([], ctypes.c_char_p),
    "bw_device_cc": ([I32], I32),
    "bw_fwht_i64": ([P, I32, P, PU64], I32),
    "bw_fwht_i64_planned": ([P, I32, ctypes.POINTER(I32), I32, P], I32),
    "bw_plan_npasses": ([I32], I32),
    "bw_fwht_i64_pass": ([P, I32, I32, P], I32),
    "bw_fwht_i64_pass_extract": ([P, I32, I32, U64, U64, P, P, U64, P, P], I32),
    "bw_sort_hits_i64": ([P, P, P, P], I32),
    "bw_fwht_widen_i32": ([P, P, I32, P, PU64], I32),
    "bw_fwht_widen": ([P, I32, P, I32, P, PU64], I32),
    "bw_fwht_i64_narrow": ([P, I32, P, U64, P, ctypes.POINTER(I32), PU64], I32),
    "bw_narrow_scratch_bytes": ([I32], U64),
    "bw_narrow_npasses": ([I32], I32),
    "bw_fwht_i64_narrow_pass": ([P, I32, P, U64, I32, P, P], I32),
    "bw_plan_check_narrow": ([I32], I32),
    "bw_fwht_i64_compact": ([P, I32, ctypes.c_longlong, P, ctypes.POINTER(I32), PU64], I32),
    "bw_compact_auto": ([I32], I32),
    "bw_fwht_i64_int64plan": ([P, I32, P, PU64], I32),
    "bw_compact_pass_info": ([I32, I32, ctypes.POINTER(I32), ctypes.POINTER(I32), ctypes.POINTER(I32), ctypes.POINTER(I32)], I32),
    "bw_fwht_i64_compact_pass_extract": ([P, I32, U64, U64, P, P, U64, P, P], I32),
    "bw_compact_limit": ([I32], ctypes.c_longlong),
    "bw_compact_npasses": ([I32], I32),
    "bw_fwht_i64_compact_pass": ([P, I32, I32, I32, P, P, P], I32),
    "bw_fwht_i64_compact_restore": ([P, I32, P, P], I32),
    "bw_plan_check_compact": ([I32], I32),
    "bw_debug_emulate_compact": ([P, I32], I32),
    "bw_pack_narrow_i64": ([P, U64, I32, I32, P, P, P], I32),
    "bw_xshard_narrow": ([ctypes.POINTER(P), I32, I32, U64, U64, P], I32),
    "bw_extract_ge_f64": ([P, I32, ctypes.c_double, ctypes.c_uint64, P, P, ctypes.c_uint64, P, P, PU64], I32),
    "bw_plan_check_f64": ([I32, PU64], I32),
    "bw_debug_emulate_f64": ([P, I32], I32),
    "bw_fwht_i64_partial": ([P, I32, ctypes.POINTER(I32), I32, P], I32),
    "bw_fwht_f64": ([P, I32, P, PU64], I32),
    "bw_minmax_i64": ([P, U64, P, P], I32),
    "bw_check_bound_i64": ([P, I32, P, P, PU64], I32),
    "bw_fwht_inplace_i64": ([P, I32, P, P, PU64], I32),
    "bw_fwht_inplace_known_i64": ([P, I32, ctypes.c_int64, P, PU64], I32),
    "bw_fwht_host_i64": ([P, I32, P, I32, P, PU64], I32),
    "bw_fwht_host_batch_i64": ([ctypes.POINTER(P), I32, I32, ctypes.POINTER(P), I32, P, PU64], I32),
    "bw_fwht_host_ooc_i64": ([P, I32, P, I32, P, ctypes.POINTER(I32)], I32),
    "bw_inverse_i64": ([P, I32, P, P], I32),
    "bw_inverse_f64": ([P, I32, P], I32),
    "bw_wht_bruteforce_i64": ([P, P, I32, P], I32),
    "bw_sumsq_partials_i64": ([P, U64, P, I32, P], I32),
    "bw_fold_i64": ([P, I32, PU64, I32, P, P], I32),
    "bw_fold_gen_i64": ([I32, I32, U64, PU64, I32, PU64, I32, P, P], I32),
    "bw_plan_fused": ([I32, I32, ctypes.POINTER(I32), ctypes.POINTER(I32), ctypes.POINTER(I32)], I32),
    "bw_fwht_xfused_pass_i64": ([ctypes.POINTER(P), I32, I32, I32, I32, P], I32),
    "bw_fwht_xfused_pass_extract_i64": ([ctypes.POINTER(P), I32, I32, I32, I32, U64, U64, P, P, U64, P, P], I32),
    "bw_xshard_i64": ([ctypes.POINTER(P), I32, U64, U64, P], I32),
    "bw_xshard_strided_i64": ([P, U64, I32, U64, U64, P], I32),
    "bw_ipc_get_handle": ([P, P, PU64], I32),
    "bw_ipc_open_handle": ([P, U64, ctypes.POINTER(P)], I32),
    "bw_ipc_close_handle": ([P, U64], I32),
    "bw_enable_peer_access": ([I32], I32),
    "bw_gen_i64": ([P, I32, I32, U64, PU64, I32, P], I32),
    "bw_gen_range_i64": ([P, U64, U64, I32, U64, PU64, I32, P], I32),
    "bw_extract_ge_i64": ([P, I32, U64, U64, P, P, U64, P, P, PU64], I32),
    "bw_fwht_extract_i64": ([P, I32, U64, U64, P, P, U64, P, PU64], I32),
    "bw_extract_scratch_bytes": ([I32], U64),
    "bw_plan_describe": ([I32, I32, ctypes.c_char_p, ctypes.c_size_t], I32),
    "bw_debug_emulate_i64": ([P, I32, ctypes.POINTER(I32), I32], I32),
    "bw_plan_check_fused": ([I32, I32, PU64], I32),
    "bw_plan_check": ([I32, ctypes.POINTER(I32), I32, PU64], I32),
}


def exported_symbols() -> list[str]:
    return sorted(_SIGNATURES)


def lib():
    """The loaded library; raises DeviceError if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise errors.DeviceError(
            f"native library {LIB_PATH} is missing; run __graft_entry__.build() "
            "(there is no CPU fallback)"
        )
    handle = ctypes.CDLL(LIB_PATH)
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(handle, name)
        fn.argtypes = args
        fn.restype = res
    _lib = handle
    return handle


def last_error() -> str:
    msg = lib().bw_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    """Raise the reference exception class that matches a bw_status."""
    if status == BW_OK:
        return
    cls = _STATUS.get(status, errors.DeviceError)
    raise cls(last_error() or f"bw status {status}")
