"""Batch apportionment and dataset partitioning -- device-controller drop-in.

Same public surface as the reference module
/root/reference/pkg/src/dbsim/allocation.py (PerfEstimate :29-34,
BatchAllocation :37-44, PartitionPlan :47-75, evaluate_performance :78-88,
compute_batch_fractions :91-102, scale_to_real_batches :105-113,
round_twice :116-137, partition_ranges :140-155, spans_from_ranges :158-188,
_raise_zero_batches :191-204, plan_next_epoch :207-244).

Every numeric step runs in the single-CTA fp64 controller kernel of
csrc/controller.cu through the C ABI (dbs_* host-buffer entry points); this
module only marshals Python values, builds the frozen result objects and maps
status codes onto the reference's exception classes.  Results are bit-identical
to the reference (tests/test_controller_gpu.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from fractions import Fraction
from typing import Sequence

import numpy as np

from . import _lib
from .errors import InvalidPerformanceError

_I64_MIN, _I64_MAX = -(2**63), 2**63 - 1


@dataclass(frozen=True)
class PerfEstimate:
    """Throughput of one worker (dataset fraction per second)."""

    worker_id: int
    value: float


@dataclass(frozen=True)
class BatchAllocation:
    """Intermediate allocation state (exported for API parity)."""

    fractions: tuple[float, ...]
    real_batches: tuple[float, ...]
    int_batches: tuple[int, ...]
    total_budget: int


@dataclass(frozen=True)
class PartitionPlan:
    """One epoch's integer batches, exact fractional ranges and sample spans."""

    int_batches: tuple[int, ...]
    ranges: tuple[tuple[Fraction, Fraction], ...]
    epoch: int
    sample_spans: tuple[tuple[int, int], ...]

    @property
    def n_workers(self) -> int:
        return len(self.int_batches)

    @property
    def dataset_size(self) -> int:
        return self.sample_spans[-1][1]

    def span_sizes(self) -> tuple[int, ...]:
        return tuple(e - s for s, e in self.sample_spans)

    def shares(self) -> tuple[float, ...]:
        """Fraction of the dataset each worker actually holds (span / D)."""
        d = self.dataset_size
        return tuple((e - s) / d for s, e in self.sample_spans)


# ---------------------------------------------------------------------------
# marshalling helpers
# ---------------------------------------------------------------------------

def _f64(values) -> np.ndarray:
    return np.ascontiguousarray(np.asarray([float(v) for v in values], dtype=np.float64).reshape(-1))


def _i64(values) -> np.ndarray:
    vals = [int(v) for v in values]
    for v in vals:
        if not (_I64_MIN <= v <= _I64_MAX):
            raise OverflowError(f"integer {v} outside int64")
    return np.ascontiguousarray(np.asarray(vals, dtype=np.int64).reshape(-1))


def _pd(a: np.ndarray):
    return a.ctypes.data_as(_lib.P_dbl)


def _pi(a: np.ndarray):
    return a.ctypes.data_as(_lib.P_i64)


def _int_arg(v) -> int:
    v = int(v)
    if not (_I64_MIN <= v <= _I64_MAX):
        raise OverflowError(f"integer {v} outside int64")
    return v


# ---------------------------------------------------------------------------
# public API
# ---------------------------------------------------------------------------

def evaluate_performance(share: float, epoch_time: float) -> float:
    """Dataset fraction per second of the last epoch (allocation.py:78-88)."""
    s, t = _f64([share]), _f64([epoch_time])
    out = np.zeros(1)
    bad = ctypes.c_int64(-1)
    st = _lib.lib().dbs_evaluate_performance(_pd(s), _pd(t), 1, _pd(out), ctypes.byref(bad))
    if st:
        _lib.check(st, detail=(f"dataset share must be in (0, 1] and epoch time positive, "
                               f"got share={share}, time={epoch_time}"))
    return float(out[0])


def compute_batch_fractions(perfs: Sequence[PerfEstimate]) -> list[float]:
    """Normalise throughputs into fractions summing to 1 (allocation.py:91-102)."""
    if not perfs:
        raise InvalidPerformanceError("need at least one performance estimate")
    v = _f64([p.value for p in perfs])
    out = np.zeros(len(v))
    bad = ctypes.c_int64(-1)
    st = _lib.lib().dbs_compute_batch_fractions(_pd(v), len(v), _pd(out), ctypes.byref(bad))
    if st:
        detail = None
        if st == 2 and 0 <= bad.value < len(perfs):
            p = perfs[bad.value]
            detail = f"worker {p.worker_id} has invalid performance {p.value}"
        elif st == 20:
            detail = "intermediate overflow in fsum"
        _lib.check(st, "compute_batch_fractions", detail)
    return out.tolist()


def scale_to_real_batches(fractions: Sequence[float], total_budget: int) -> list[float]:
    """Real-valued batches for a fixed budget (allocation.py:105-113)."""
    f = _f64(fractions)
    out = np.zeros(max(len(f), 1))
    st = _lib.lib().dbs_scale_to_real_batches(_pd(f), len(f), _int_arg(total_budget), _pd(out))
    if st:
        detail = (f"budget {total_budget} is below worker count {len(f)}" if st == 3
                  else "fractions must sum to 1" if st == 2 else None)
        _lib.check(st, "scale_to_real_batches", detail)
    return out[: len(f)].tolist()


def round_twice(real_batches: Sequence[float], total_budget: int) -> list[int]:
    """Floor, then +1 to the largest decimals >= 0.5 within budget (allocation.py:116-137)."""
    r = _f64(real_batches)
    out = np.zeros(max(len(r), 1), dtype=np.int64)
    st = _lib.lib().dbs_round_twice(_pd(r), len(r), _int_arg(total_budget), _pi(out))
    if st:
        _lib.check(st, "round_twice", "batch sizes must be non-negative" if st == 4 else None)
    return [int(x) for x in out[: len(r)]]


def _raise_zero_batches(int_batches: list[int]) -> list[int]:
    """Lift zero batches to one sample, paid by the first largest (allocation.py:191-204)."""
    b = _i64(int_batches)
    out = np.zeros(max(len(b), 1), dtype=np.int64)
    if len(b):
        _lib.check(_lib.lib().dbs_raise_zero_batches(_pi(b), len(b), _pi(out)), "raise_zero_batches")
    return [int(x) for x in out[: len(b)]]


def _partition_cum(int_batches: Sequence[int]) -> list[int]:
    b = _i64(int_batches)
    cum = np.zeros(len(b) + 1, dtype=np.int64)
    st = _lib.lib().dbs_partition_ranges(_pi(b), len(b), _pi(cum))
    if st:
        detail = {5: "all integer batches are zero" if len(b) else "no workers to partition over",
                  4: "integer batches must be non-negative"}.get(st)
        _lib.check(st, "partition_ranges", detail)
    return [int(x) for x in cum]


def partition_ranges(int_batches: Sequence[int]) -> list[tuple[Fraction, Fraction]]:
    """Exact contiguous ranges proportional to integer batches (allocation.py:140-155)."""
    cum = _partition_cum(int_batches)
    total = cum[-1]
    return [(Fraction(cum[i], total), Fraction(cum[i + 1], total)) for i in range(len(cum) - 1)]


def _bound(x) -> _lib.Bound:
    if isinstance(x, Fraction):
        return _lib.Bound(0, 0, _int_arg(x.numerator), _int_arg(x.denominator), 0.0)
    if isinstance(x, (int, np.integer)) and not isinstance(x, bool):
        return _lib.Bound(0, 0, _int_arg(x), 1, 0.0)
    if isinstance(x, bool):
        return _lib.Bound(0, 0, int(x), 1, 0.0)
    return _lib.Bound(1, 0, 0, 1, float(x))


def spans_from_ranges(ranges: Sequence[tuple], dataset_size: int) -> list[tuple[int, int]]:
    """Half-open sample spans of fractional ranges (allocation.py:158-188)."""
    n = len(ranges)
    D = _int_arg(dataset_size)
    lo = (_lib.Bound * max(n, 1))(*[_bound(r[0]) for r in ranges])
    hi = (_lib.Bound * max(n, 1))(*[_bound(r[1]) for r in ranges])
    out = np.zeros(2 * max(n, 1), dtype=np.int64)
    st = _lib.lib().dbs_spans_from_ranges(lo, hi, n, D, _pi(out))
    if st:
        detail = (f"dataset of {dataset_size} samples cannot cover {n} workers" if st == 6
                  else "list index out of range" if st == 30 else None)
        _lib.check(st, "spans_from_ranges", detail)
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(n)]


def plan_next_epoch(
    prev_shares: Sequence[float],
    prev_times: Sequence[float],
    total_budget: int,
    dataset_size: int,
    epoch: int,
) -> PartitionPlan:
    """Whole per-epoch pipeline in one controller launch (allocation.py:207-244)."""
    n = len(prev_shares)
    if n == 0 or len(prev_times) != n:
        raise InvalidPerformanceError("share and time lists must be same non-empty length")
    B = _int_arg(total_budget)
    if B < n:
        from .errors import BudgetTooSmallError

        raise BudgetTooSmallError(f"budget {total_budget} is below worker count {n}")
    ep = int(epoch)
    ep_arg = 0 if ep == 0 else 1  # only `epoch == 0` matters to the pipeline
    s, t = _f64(prev_shares), _f64(prev_times)
    b = np.zeros(n, dtype=np.int64)
    cum = np.zeros(n + 1, dtype=np.int64)
    spans = np.zeros(2 * n, dtype=np.int64)
    bad = ctypes.c_int64(-1)
    st = _lib.lib().dbs_plan_next_epoch(_pd(s), _pd(t), n, B, _int_arg(dataset_size), ep_arg, _pi(b), _pi(cum),
                                        _pi(spans), ctypes.byref(bad))
    if st:
        detail = None
        if st == 1 and 0 <= bad.value < n:
            detail = (f"invalid measurement for worker {bad.value}: share={prev_shares[bad.value]}, "
                      f"time={prev_times[bad.value]}")
        elif st == 6:
            detail = f"dataset of {dataset_size} samples cannot cover {n} workers"
        _lib.check(st, "plan_next_epoch", detail)
    total = int(cum[-1])
    ranges = tuple((Fraction(int(cum[i]), total), Fraction(int(cum[i + 1]), total)) for i in range(n))
    return PartitionPlan(
        int_batches=tuple(int(x) for x in b),
        ranges=ranges,
        epoch=epoch,
        sample_spans=tuple((int(spans[2 * i]), int(spans[2 * i + 1])) for i in range(n)),
    )


def plan_from_arrays(int_batches, cum, spans, epoch: int) -> PartitionPlan:
    """PartitionPlan from the device controller's raw outputs (dbs_dev_replan)."""
    cum = [int(c) for c in cum]
    total = cum[-1]
    n = len(int_batches)
    return PartitionPlan(
        int_batches=tuple(int(x) for x in int_batches),
        ranges=tuple((Fraction(cum[i], total), Fraction(cum[i + 1], total)) for i in range(n)),
        epoch=epoch,
        sample_spans=tuple((int(spans[2 * i]), int(spans[2 * i + 1])) for i in range(n)),
    )
