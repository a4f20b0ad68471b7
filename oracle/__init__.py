"""CPU oracle for the B200 FWHT -- TEST INFRASTRUCTURE ONLY.

``oracle_np`` (numpy) and ``bw_oracle.c`` (C, built to ``liboracle.so``)
restate the reference path (/root/reference/pkg/src/bigwht/core.py,
parallel.py, noisy.py, subspace.py).  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline legs may use them.  The product package never
imports this directory.
"""

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return LIB_PATH


def load_c():
    """ctypes handle of liboracle.so (built on first use if missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        build()
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    U64 = ctypes.c_uint64
    I = ctypes.c_int
    lib.oracle_fwht_i64.argtypes = [P, I]
    lib.oracle_fwht_i64.restype = U64
    lib.oracle_fwht_f64.argtypes = [P, I]
    lib.oracle_fwht_f64.restype = None
    lib.oracle_run_parallel_i64.argtypes = [P, I, I]
    lib.oracle_run_parallel_i64.restype = I
    lib.oracle_bound_violated.argtypes = [P, U64, I, ctypes.POINTER(U64)]
    lib.oracle_bound_violated.restype = I
    lib.oracle_hash64.argtypes = [U64, U64]
    lib.oracle_hash64.restype = U64
    lib.oracle_gen_i64.argtypes = [P, U64, U64, I, U64, P, I, I]
    lib.oracle_gen_i64.restype = I
    lib.oracle_fold_i64.argtypes = [P, I, P, I, I, U64, P, I, I, P]
    lib.oracle_fold_i64.restype = I
    lib.oracle_extract_ge_i64.argtypes = [P, U64, U64, P, P, U64]
    lib.oracle_extract_ge_i64.restype = U64
    _lib = lib
    return lib
