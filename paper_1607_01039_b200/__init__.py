"""B200-native fast Walsh-Hadamard transform -- drop-in for the hot path of
the reference package ``bigwht`` (arXiv:1607.01039).

Same names and semantics as /root/reference/pkg/src/bigwht/core.py
(``Signal``, ``Domain``, ``fwht_array``, ``fwht_inplace``,
``check_magnitude_bound``, ``inverse_wht_inplace``), noisy.py
(``extract_above``) and parallel.py (``plan_parallel`` / ``run_parallel``,
and multi-GPU sharding in ``sharded``),
computed by hand-written sm_100a kernels behind the C ABI in
include/bigwht_b200.h.  No CPU arithmetic path exists.
"""

from . import errors
from .core import (
    Domain,
    Signal,
    butterfly_count,
    check_magnitude_bound,
    fwht_array,
    fwht_arrays,
    fwht_inplace,
    fwht_widen,
    inverse_wht_inplace,
    parseval_energy,
    wht_bruteforce,
)
from .errors import (
    BadArguments,
    BigWHTError,
    DeviceError,
    InexactDivision,
    InvalidWorkerCount,
    OracleTooLarge,
    OverflowBoundError,
    ValidationError,
)
from .extract import extract_above, extract_ge, extract_gt, fwht_extract_ge, fwht_extract_gt
from .parallel import ParallelPlan, check_disjoint, plan_parallel, run_parallel, total_butterflies

__version__ = "0.1.0"

__all__ = [
    "Domain",
    "Signal",
    "butterfly_count",
    "check_magnitude_bound",
    "fwht_array",
    "fwht_arrays",
    "fwht_inplace",
    "fwht_widen",
    "inverse_wht_inplace",
    "parseval_energy",
    "wht_bruteforce",
    "extract_above",
    "extract_ge",
    "extract_gt",
    "fwht_extract_ge",
    "fwht_extract_gt",
    "ParallelPlan",
    "plan_parallel",
    "run_parallel",
    "check_disjoint",
    "total_butterflies",
    "errors",
    "BadArguments",
    "BigWHTError",
    "DeviceError",
    "InexactDivision",
    "InvalidWorkerCount",
    "OracleTooLarge",
    "OverflowBoundError",
    "ValidationError",
    "__version__",
]
