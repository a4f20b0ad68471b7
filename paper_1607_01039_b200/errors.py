"""Exception hierarchy of the drop-in, mirroring the reference names and
CLI exit codes (/root/reference/pkg/src/bigwht/errors.py:10-80) so callers'
``except`` clauses keep working.  ``DeviceError`` is new: CUDA failures have no
reference counterpart (the reference never touches a device).

When the reference package ``bigwht`` is importable, every class here also
derives from its ``bigwht.errors`` namesake (``bind_reference``), so a
reference caller's ``except OverflowBoundError`` / ``except BigWHTError``
(e.g. cli.py:577-579, exit code 3) catches what the B200 path raises.  The
binding happens at import when ``bigwht`` can be found, and again from
``paper_1607_01039_b200.shim.install`` (for a ``bigwht`` put on sys.path
later); BW_REFERENCE_ERRORS=0 turns the import-time binding off.
"""

from __future__ import annotations

import importlib.util
import os


class _Root(Exception):
    """Anchor below BigWHTError, so the reference base can be added to
    BigWHTError's bases later without an MRO conflict with Exception."""


class BigWHTError(_Root):
    """Base class of every error raised by this package (errors.py:10-13)."""

    exit_code = 3


class ValidationError(BigWHTError):
    exit_code = 3


class StorageError(BigWHTError):
    exit_code = 2


class BadArguments(ValidationError):
    """Arguments violate an operation's preconditions (errors.py:24)."""


class NotPowerOfTwo(BadArguments, ValueError):
    """A buffer length that is not a power of two.  The reference's
    fwht_array fails here with numpy's ValueError from the reshape
    (core.py:109, after mutating part of the buffer); this one is raised
    before any launch and is both a BadArguments and a ValueError."""


class OracleTooLarge(ValidationError):
    """Brute-force transform requested above the size limit (errors.py:28)."""


class OverflowBoundError(ValidationError):
    """Int64 magnitude bound M * 2**n < 2**63 does not hold (errors.py:32)."""


class InexactDivision(ValidationError):
    """Int64 inverse hit a coefficient not divisible by 2**n (errors.py:36)."""


class InvalidWorkerCount(ValidationError):
    """Worker / shard count not a power of two or out of range (errors.py:40)."""


class SizeMismatch(ValidationError):
    """Payload size disagrees with the sidecar (errors.py:48)."""


class BadMetadata(ValidationError):
    """Sidecar missing, unparsable, or semantically invalid (errors.py:52)."""


class BadDims(ValidationError):
    """Linear map dimensions are invalid (errors.py:64)."""


class DimMismatch(ValidationError):
    """Signal dimension does not match the linear map (errors.py:68)."""


class PathExists(StorageError):
    """Refusing to overwrite an existing dataset (errors.py:76)."""


class DeviceError(BigWHTError):
    """A CUDA call failed, the device is not a B200 (sm_100a), or the native
    library is missing.  After a failed in-place launch the buffer contents
    are unspecified, like a failed worker in parallel.py:167-169."""

    exit_code = 2


# class here -> name of its counterpart in bigwht.errors
_REFERENCE_NAMES = {
    BigWHTError: "BigWHTError",
    ValidationError: "ValidationError",
    StorageError: "StorageError",
    BadArguments: "BadArguments",
    OracleTooLarge: "OracleTooLarge",
    OverflowBoundError: "OverflowBoundError",
    InexactDivision: "InexactDivision",
    InvalidWorkerCount: "InvalidWorkerCount",
    SizeMismatch: "SizeMismatch",
    BadMetadata: "BadMetadata",
    BadDims: "BadDims",
    DimMismatch: "DimMismatch",
    PathExists: "PathExists",
}

bound_reference = None  # the bigwht.errors module the classes derive from, if any


def bind_reference(ref=None) -> bool:
    """Make every class above also a subclass of its ``bigwht.errors``
    namesake (``ref``, or the importable ``bigwht.errors``).  Idempotent;
    returns whether the binding is in place."""
    global bound_reference
    if ref is None:
        try:
            import bigwht.errors as ref  # noqa: PLC0415 -- the reference, only for its classes
        except Exception:  # not installed / its own imports fail: nothing to bind
            return False
    if bound_reference is ref:
        return True
    for cls, name in _REFERENCE_NAMES.items():
        target = getattr(ref, name, None)
        if target is None or issubclass(cls, target):
            continue
        cls.__bases__ = cls.__bases__ + (target,)
    bound_reference = ref
    return True


if os.environ.get("BW_REFERENCE_ERRORS", "1") != "0":
    try:
        _found = importlib.util.find_spec("bigwht") is not None
    except (ImportError, ValueError):
        _found = False
    if _found:
        bind_reference()
