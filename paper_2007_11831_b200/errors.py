"""Exception classes of the DBS package, mirroring the reference's hierarchy.

Reference: /root/reference/pkg/src/dbsim/errors.py:4-53.  Every class keeps the
reference's name and base class so ``except dbsim.errors.X`` call sites keep
working; ``from_status`` maps the C ABI's ``dbs_status`` codes
(include/dbs_b200.h) back onto them.
"""


class DbsError(Exception):
    """Root of every error raised by the DBS hot path."""


class InvalidMeasurementError(DbsError):
    """A measured epoch time or dataset share is non-positive or not finite."""


class InvalidPerformanceError(DbsError):
    """Performance estimates are empty, non-positive or not finite."""


class BudgetTooSmallError(DbsError):
    """The global batch budget is smaller than the number of workers."""


class InvalidBatchError(DbsError):
    """A (real or integer) batch size is negative or not finite."""


class EmptyPartitionError(DbsError):
    """No worker, or only zero batches, so no dataset partition exists."""


class DatasetTooSmallError(DbsError):
    """Fewer samples than workers."""


class ConfigurationError(DbsError):
    """Inconsistent training / strategy configuration."""


class ValidationError(ConfigurationError):
    """A configuration invariant failed; the message names the field."""


class EmptyBatchError(DbsError):
    """A gradient was requested for an empty batch."""


class InvalidStepSizeError(DbsError):
    """SGD step size outside (0, 1/mu)."""


class InvalidBaselineError(DbsError):
    """Savings requested against a non-positive baseline."""


class BaselineNotFoundError(DbsError):
    """The named baseline strategy is not among the reports."""


# dbs_status -> exception class (include/dbs_b200.h)
_STATUS = {
    1: InvalidMeasurementError,
    2: InvalidPerformanceError,
    3: BudgetTooSmallError,
    4: InvalidBatchError,
    5: EmptyPartitionError,
    6: DatasetTooSmallError,
    7: ConfigurationError,
    9: EmptyBatchError,
    10: InvalidStepSizeError,
    20: OverflowError,   # math.fsum intermediate overflow
    21: ValueError,      # math.fsum -inf + inf
    22: OverflowError,   # int64 range exceeded where Python has big ints
    30: IndexError,      # argument the reference would index out of range
}


class DeviceError(RuntimeError):
    """CUDA failure inside the DBS library (not a reference error)."""


def from_status(code: int, message: str) -> Exception:
    cls = _STATUS.get(int(code))
    if cls is None:
        return DeviceError(f"dbs_status {code}: {message}")
    return cls(message)
