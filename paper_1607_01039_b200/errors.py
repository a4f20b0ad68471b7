"""Exception hierarchy of the drop-in, mirroring the reference names and
CLI exit codes (/root/reference/pkg/src/bigwht/errors.py:10-41) so callers'
``except`` clauses keep working.  ``DeviceError`` is new: CUDA failures have no
reference counterpart (the reference never touches a device)."""


class BigWHTError(Exception):
    """Base class of every error raised by this package (errors.py:10-13)."""

    exit_code = 3


class ValidationError(BigWHTError):
    exit_code = 3


class StorageError(BigWHTError):
    exit_code = 2


class BadArguments(ValidationError):
    """Arguments violate an operation's preconditions (errors.py:24)."""


class OracleTooLarge(ValidationError):
    """Brute-force transform requested above the size limit (errors.py:28)."""


class OverflowBoundError(ValidationError):
    """Int64 magnitude bound M * 2**n < 2**63 does not hold (errors.py:32)."""


class InexactDivision(ValidationError):
    """Int64 inverse hit a coefficient not divisible by 2**n (errors.py:36)."""


class InvalidWorkerCount(ValidationError):
    """Worker / shard count not a power of two or out of range (errors.py:40)."""


class DeviceError(BigWHTError):
    """A CUDA call failed, the device is not a B200 (sm_100a), or the native
    library is missing.  After a failed in-place launch the buffer contents
    are unspecified, like a failed worker in parallel.py:167-169."""

    exit_code = 2
