"""Synchronous data-parallel SGD with per-worker variable batches -- on the B200.

Drop-in for /root/reference/pkg/src/dbsim/sgdlab.py: ConvexProblem (:33-95),
LogisticProblem (:98-159), SgdConfig (:165-189), SgdTrajectory (:191-197),
minibatch_gradient (:200-205), aggregate_gradients (:208-227), sgd_step
(:230-238), _epoch_layout (:320-340) and run_parallel_sgd (:343-396).

Problem construction (synthetic data, the logistic optimum via L-BFGS) is host
set-up exactly as in the reference; the data then lives in HBM and every
numeric step of the hot path runs in libdbs_b200 kernels:
  * sample assignment: PCG64 draws + Fisher-Yates on the device (permute.cu),
    bit-identical to numpy's Generator.permutation;
  * one fused single-CTA launch per epoch for the reference problems
    (problems.cu: worker gradients -> aggregate -> heavy-ball step -> ||x-x*||^2);
  * the drop-in functions call the same kernels one step at a time.
The theory estimators of the reference (theorem1_bound, estimate_gradient_noise
:252-272, verify_lemma1_variance :282-314) run on the device too (theory.cu):
numpy's Generator.integers / random draws reproduced bit-exactly from the same
PCG64 state, the Monte-Carlo arithmetic in fp64 kernels.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional, Sequence, Union

import numpy as np

from . import _lib
from . import allocation
from .allocation import PartitionPlan
from .errors import ConfigurationError, EmptyBatchError, InvalidStepSizeError

AGGREGATION_MODES = ("uniform_average", "batch_weighted")
_MODE = {"uniform_average": 0, "batch_weighted": 1}


def _torch():
    import torch

    return torch


def _dev():
    torch = _torch()
    _lib.require_device()
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev_f64(a):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device=_dev(), dtype=torch.float64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float64)), device=_dev())


def _like_input(t, ref):
    torch = _torch()
    if isinstance(ref, torch.Tensor):
        return t
    return t.cpu().numpy()


# ---------------------------------------------------------------------------
# reference problems (host construction, device-resident data)
# ---------------------------------------------------------------------------

@dataclass
class ConvexProblem:
    """f_i(x) = mu/2 ||x - x* - eps_i||^2 with centred Gaussian offsets (sgdlab.py:33-95)."""

    dimension: int
    mu: float
    optimum: np.ndarray
    sample_noise_scale: float
    sample_count: int
    offsets: np.ndarray = field(repr=False)
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    @classmethod
    def quadratic(cls, dimension: int, mu: float, sample_noise_scale: float, sample_count: int,
                  seed: int = 0, optimum: Optional[np.ndarray] = None) -> "ConvexProblem":
        if mu <= 0.0:
            raise ConfigurationError("mu must be positive")
        rng = np.random.default_rng(seed)
        opt = np.zeros(dimension) if optimum is None else np.asarray(optimum, dtype=float)
        if sample_noise_scale > 0.0:
            offsets = rng.normal(0.0, sample_noise_scale, (sample_count, dimension))
            offsets -= offsets.mean(axis=0)
        else:
            offsets = np.zeros((sample_count, dimension))
        return cls(dimension=dimension, mu=mu, optimum=opt, sample_noise_scale=sample_noise_scale,
                   sample_count=sample_count, offsets=offsets)

    kind = 0

    def device(self):
        """(data, labels, optimum) resident in HBM as fp64."""
        if "dev" not in self._cache:
            self._cache["dev"] = (_to_dev_f64(self.offsets), None, _to_dev_f64(self.optimum))
        return self._cache["dev"]

    def full_gradient(self, x):
        return self.mu * (np.asarray(x) - self.optimum)

    def sample_values(self, x, indices):
        torch = _torch()
        data, _, opt = self.device()
        idx = torch.as_tensor(np.asarray(indices, dtype=np.int64), device=data.device)
        d = _to_dev_f64(x) - opt - data[idx]
        return _like_input(0.5 * self.mu * (d * d).sum(dim=-1), x)

    def objective(self, x) -> float:
        torch = _torch()
        data, _, opt = self.device()
        d = _to_dev_f64(x) - opt - data
        return float((0.5 * self.mu * (d * d).sum(dim=-1)).mean().item())

    def objective_gap(self, x) -> float:
        return self.objective(x) - self.objective(self.optimum)


@dataclass
class LogisticProblem:
    """l2-regularised logistic regression, optimum by L-BFGS (sgdlab.py:98-159)."""

    dimension: int
    mu: float
    optimum: np.ndarray
    sample_count: int
    features: np.ndarray = field(repr=False)
    labels: np.ndarray = field(repr=False)
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    kind = 1

    @classmethod
    def synthetic(cls, dimension: int, mu: float, sample_count: int, seed: int = 0) -> "LogisticProblem":
        from scipy.optimize import minimize

        rng = np.random.default_rng(seed)
        labels = np.where(rng.random(sample_count) < 0.5, -1.0, 1.0)
        centers = labels[:, None] * np.full(dimension, 0.5)
        features = centers + rng.normal(0.0, 1.0, (sample_count, dimension))

        def loss(w):
            m = labels * (features @ w)
            return float(np.mean(np.logaddexp(0.0, -m)) + 0.5 * mu * np.dot(w, w))

        def grad(w):
            m = labels * (features @ w)
            c = -labels / (1.0 + np.exp(m))
            return features.T @ c / sample_count + mu * w

        res = minimize(loss, np.zeros(dimension), jac=grad, method="L-BFGS-B", tol=1e-12)
        return cls(dimension=dimension, mu=mu, optimum=res.x, sample_count=sample_count,
                   features=features, labels=labels)

    def device(self):
        if "dev" not in self._cache:
            self._cache["dev"] = (_to_dev_f64(self.features), _to_dev_f64(self.labels), _to_dev_f64(self.optimum))
        return self._cache["dev"]

    def sample_values(self, x, indices):
        torch = _torch()
        f, y, _ = self.device()
        idx = torch.as_tensor(np.asarray(indices, dtype=np.int64), device=f.device)
        xd = _to_dev_f64(x)
        m = -y[idx] * (f[idx] @ xd)
        v = torch.logaddexp(torch.zeros_like(m), m) + 0.5 * self.mu * torch.dot(xd, xd)
        return _like_input(v, x)

    def objective(self, x) -> float:
        torch = _torch()
        f, y, _ = self.device()
        xd = _to_dev_f64(x)
        m = -y * (f @ xd)
        return float((torch.logaddexp(torch.zeros_like(m), m) + 0.5 * self.mu * torch.dot(xd, xd)).mean().item())

    def objective_gap(self, x) -> float:
        return self.objective(x) - self.objective(self.optimum)


Problem = Union[ConvexProblem, LogisticProblem]


@dataclass
class SgdConfig:
    """Hyper-parameters of one SGD run; step size must lie in (0, 1/mu) (sgdlab.py:165-189)."""

    step_size: float
    n_iterations: int
    momentum: float = 0.0
    aggregation: str = "batch_weighted"
    seed: int = 0
    initial_point: Optional[np.ndarray] = None

    def __post_init__(self):
        if self.aggregation not in AGGREGATION_MODES:
            raise ConfigurationError(f"unknown aggregation {self.aggregation!r}")
        if not (0.0 <= self.momentum < 1.0):
            raise ConfigurationError("momentum must be in [0, 1)")
        if self.n_iterations < 1:
            raise ConfigurationError("n_iterations must be >= 1")

    def validate_step_size(self, mu: float) -> None:
        if not (0.0 < self.step_size * mu < 1.0):
            raise InvalidStepSizeError(f"step size {self.step_size} outside (0, {1.0 / mu})")


@dataclass
class SgdTrajectory:
    squared_distances: np.ndarray
    final_loss: float
    bound_values: Optional[np.ndarray] = None


# ---------------------------------------------------------------------------
# drop-in step functions
# ---------------------------------------------------------------------------

def minibatch_gradient(problem, x, indices):
    """Batch mean of per-sample gradients (sgdlab.py:200-205) on the device."""
    torch = _torch()
    idx_np = np.asarray(indices, dtype=np.int64).reshape(-1)
    if idx_np.size == 0:
        raise EmptyBatchError("mini-batch must contain at least one sample")
    if hasattr(problem, "minibatch_gradient_device"):
        return problem.minibatch_gradient_device(x, idx_np)
    data, labels, opt = problem.device()
    xd = _to_dev_f64(x)
    idx = torch.as_tensor(idx_np, device=xd.device)
    off = torch.tensor([0, idx_np.size], dtype=torch.int64, device=xd.device)
    out = torch.empty(problem.dimension, dtype=torch.float64, device=xd.device)
    s = _lib.stream_handle()
    if problem.kind == 0:
        st = _lib.lib().dbs_dev_quadratic_grads(xd.data_ptr(), opt.data_ptr(), data.data_ptr(), problem.dimension,
                                                idx.data_ptr(), off.data_ptr(), 1, float(problem.mu),
                                                out.data_ptr(), s)
    else:
        st = _lib.lib().dbs_dev_logistic_grads(xd.data_ptr(), data.data_ptr(), labels.data_ptr(), problem.dimension,
                                               idx.data_ptr(), off.data_ptr(), 1, float(problem.mu),
                                               out.data_ptr(), s)
    _lib.check(st, "minibatch_gradient")
    return _like_input(out, x)


def aggregate_gradients(grads: Sequence, batch_sizes: Sequence[int], mode: str):
    """Uniform or batch-weighted combination of worker gradients (sgdlab.py:208-227)."""
    if len(grads) != len(batch_sizes):
        raise ConfigurationError("gradients and batch sizes must align")
    if any(b <= 0 for b in batch_sizes):
        raise ConfigurationError("batch sizes must be positive")
    if mode not in _MODE:
        raise ConfigurationError(f"unknown aggregation {mode!r}")
    torch = _torch()
    gd = [_to_dev_f64(g).reshape(-1) for g in grads]
    P = gd[0].numel()
    if any(g.numel() != P for g in gd):
        raise ValueError("all input arrays must have the same shape")
    out = torch.empty(P, dtype=torch.float64, device=gd[0].device)
    ptrs = (ctypes.c_void_p * len(gd))(*[g.data_ptr() for g in gd])
    b = np.asarray([int(x) for x in batch_sizes], dtype=np.int64)
    st = _lib.lib().dbs_dev_aggregate_f64(ptrs, b.ctypes.data_as(_lib.P_i64), len(gd), _MODE[mode], P,
                                          out.data_ptr(), _lib.stream_handle())
    _lib.check(st, "aggregate_gradients")
    shape = np.shape(grads[0]) if not isinstance(grads[0], torch.Tensor) else tuple(grads[0].shape)
    return _like_input(out.reshape(shape), grads[0])


def sgd_step(x, gradient, config: SgdConfig, velocity):
    """Heavy-ball update v' = m v + g, x' = x - lr v', out of place (sgdlab.py:230-238)."""
    torch = _torch()
    xd, gd, vd = _to_dev_f64(x).reshape(-1), _to_dev_f64(gradient).reshape(-1), _to_dev_f64(velocity).reshape(-1)
    xo, vo = torch.empty_like(xd), torch.empty_like(vd)
    st = _lib.lib().dbs_dev_sgd_step_f64(xd.data_ptr(), gd.data_ptr(), vd.data_ptr(), xd.numel(),
                                         float(config.step_size), float(config.momentum), xo.data_ptr(),
                                         vo.data_ptr(), _lib.stream_handle())
    _lib.check(st, "sgd_step")
    shape = np.shape(x) if not isinstance(x, torch.Tensor) else tuple(x.shape)
    return _like_input(xo.reshape(shape), x), _like_input(vo.reshape(shape), x)


# ---------------------------------------------------------------------------
# the parallel loop
# ---------------------------------------------------------------------------

PlanSource = Union[Sequence[int], Sequence[PartitionPlan]]


def theorem1_bound(j: int, gamma: float, mu: float, initial_sq_dist: float, sigma_sq: float) -> float:
    """Geometric contraction bound (1 - gamma mu)^j d0 + gamma sigma^2 / mu (sgdlab.py:241-249)."""
    if not (0.0 < gamma * mu < 1.0):
        raise InvalidStepSizeError(f"gamma*mu must be in (0, 1), got {gamma * mu}")
    if sigma_sq < 0.0 or initial_sq_dist < 0.0:
        raise ConfigurationError("distances and noise must be non-negative")
    return (1.0 - gamma * mu) ** j * initial_sq_dist + gamma * sigma_sq / mu


def _epoch_layout(plan_source: PlanSource, epoch: int, n_workers: int,
                  sample_count: int) -> tuple[list[int], list[tuple[int, int]]]:
    """Per-epoch batches and spans (sgdlab.py:320-340); spans from the device controller."""
    if len(plan_source) == 0:
        raise ConfigurationError("plan source is empty")
    if isinstance(plan_source[0], PartitionPlan) or hasattr(plan_source[0], "int_batches"):
        plan = plan_source[min(epoch, len(plan_source) - 1)]
        if plan.n_workers != n_workers:
            raise ConfigurationError("plan worker count does not match run")
        batches = list(plan.int_batches)
        spans = allocation.spans_from_ranges(plan.ranges, sample_count)
    else:
        batches = [int(b) for b in plan_source]
        if len(batches) != n_workers:
            raise ConfigurationError("fixed batch list does not match worker count")
        spans = allocation.spans_from_ranges(allocation.partition_ranges([1] * n_workers), sample_count)
    if any(b < 1 for b in batches):
        raise ConfigurationError("every worker needs a positive batch size")
    return batches, spans


class DeviceRng:
    """numpy ``default_rng(seed)`` state resident in HBM (dbs_pcg64)."""

    def __init__(self, seed: int, device=None):
        torch = _torch()
        words = []
        s = int(seed)
        if s < 0:
            raise ValueError("expected non-negative integer")
        while True:
            words.append(s & 0xFFFFFFFF)
            s >>= 32
            if s == 0:
                break
        arr = (ctypes.c_uint32 * len(words))(*words)
        st = _lib.Pcg64()
        _lib.check(_lib.lib().dbs_pcg64_seed(arr, len(words), ctypes.byref(st)), "pcg64_seed")
        raw = np.frombuffer(bytes(st), dtype=np.uint8).copy()
        self.state = torch.as_tensor(raw, device=device or _dev())
        self._draws = None
        self._perm = None

    def host_state(self) -> _lib.Pcg64:
        st = _lib.Pcg64()
        ctypes.memmove(ctypes.byref(st), bytes(self.state.cpu().numpy()), ctypes.sizeof(st))
        return st

    def integers(self, high: int, size) -> "object":
        """Generator.integers(0, high, size) (int64) as a device tensor of shape `size`."""
        torch = _torch()
        shape = (size,) if isinstance(size, int) else tuple(size)
        n = int(np.prod(shape)) if shape else 1
        out = torch.empty(max(n, 1), dtype=torch.int64, device=self.state.device)
        _lib.check(_lib.lib().dbs_dev_pcg64_integers(self.state.data_ptr(), int(high), n, out.data_ptr(),
                                                     _lib.stream_handle()), "pcg64_integers")
        return out[:n].view(shape)

    def random(self, size) -> "object":
        """Generator.random(size) (float64) as a device tensor."""
        torch = _torch()
        shape = (size,) if isinstance(size, int) else tuple(size)
        n = int(np.prod(shape)) if shape else 1
        out = torch.empty(max(n, 1), dtype=torch.float64, device=self.state.device)
        _lib.check(_lib.lib().dbs_dev_pcg64_random(self.state.data_ptr(), n, out.data_ptr(), _lib.stream_handle()),
                   "pcg64_random")
        return out[:n].view(shape)

    def permute_spans(self, spans, only_span: int = -1, out=None, stream=None, total=None):
        """start + permutation(width) for every span, one generator (sgdlab.py:372-374).
        `spans` may be a device int64 tensor [2n] (e.g. the device controller's output,
        never copied to the host) when `total` (the sum of the widths) is given."""
        torch = _torch()
        dev = self.state.device
        if isinstance(spans, torch.Tensor) and spans.is_cuda:
            if total is None or only_span >= 0:
                raise ValueError("device spans need total= and the whole-plan permutation")
            flat = spans
            n_spans = int(spans.numel()) // 2
            widths = None
            total = int(total)
        else:
            flat = torch.as_tensor(np.asarray(spans, dtype=np.int64).reshape(-1), device=dev)
            n_spans = len(spans)
            widths = [e - s for s, e in spans]
            total = int(sum(widths))
        if self._draws is None or self._draws.numel() < max(total, 1):
            self._draws = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        n_out = total if only_span < 0 else widths[only_span]
        if out is None:
            out = torch.empty(max(n_out, 1), dtype=torch.int64, device=dev)
        st = _lib.lib().dbs_dev_permute_spans(self.state.data_ptr(), flat.data_ptr(), n_spans, total, only_span,
                                              out.data_ptr(), self._draws.data_ptr(), _lib.stream_handle(stream))
        _lib.check(st, "permute_spans")
        return out[:n_out], flat


def run_parallel_sgd(problem, config: SgdConfig, n_workers: int, plan_source: PlanSource) -> SgdTrajectory:
    """Synchronous data-parallel SGD with per-epoch layouts (sgdlab.py:343-396).

    One controller call (spans), one permutation and ONE fused epoch kernel per
    epoch; the squared distances stay on the device until the run ends.
    """
    torch = _torch()
    config.validate_step_size(problem.mu)
    if hasattr(problem, "run_parallel_sgd_device"):
        return problem.run_parallel_sgd_device(config, n_workers, plan_source)
    dev = _dev()
    rng = DeviceRng(config.seed, dev)
    x = (torch.ones(problem.dimension, dtype=torch.float64, device=dev) if config.initial_point is None
         else _to_dev_f64(np.asarray(config.initial_point, dtype=float).copy()))
    v = torch.zeros(problem.dimension, dtype=torch.float64, device=dev)
    sq = torch.empty(config.n_iterations, dtype=torch.float64, device=dev)
    data, labels, opt = problem.device()
    grads = torch.empty(n_workers * problem.dimension, dtype=torch.float64, device=dev)
    coeff = None
    done, epoch = 0, 0
    mode = _MODE[config.aggregation]
    s = _lib.stream_handle()
    while done < config.n_iterations:
        batches, spans = _epoch_layout(plan_source, epoch, n_workers, problem.sample_count)
        perm, _ = rng.permute_spans(spans)
        iters = min((e - st) // b for (st, e), b in zip(spans, batches))
        if iters == 0:
            raise ConfigurationError("worker span too small for its batch size")
        run = min(iters, config.n_iterations - done)
        span_off = np.cumsum([0] + [e - st for st, e in spans[:-1]]).astype(np.int64)
        b = np.asarray(batches, dtype=np.int64)
        if problem.kind == 1 and (coeff is None or coeff.numel() < int(b.sum())):
            coeff = torch.empty(int(b.sum()), dtype=torch.float64, device=dev)
        st = _lib.lib().dbs_dev_sgd_epoch(
            problem.kind, data.data_ptr(), labels.data_ptr() if labels is not None else None, opt.data_ptr(),
            problem.dimension, float(problem.mu), perm.data_ptr(), span_off.ctypes.data_as(_lib.P_i64),
            b.ctypes.data_as(_lib.P_i64), n_workers, mode, run, float(config.step_size), float(config.momentum),
            x.data_ptr(), v.data_ptr(), grads.data_ptr(), coeff.data_ptr() if coeff is not None else None,
            sq[done:].data_ptr(), s)
        _lib.check(st, "sgd_epoch")
        done += run
        epoch += 1
    return SgdTrajectory(squared_distances=sq.cpu().numpy(), final_loss=problem.objective_gap(x))


# ---------------------------------------------------------------------------
# theory estimators (sgdlab.py:252-314) on the device
# ---------------------------------------------------------------------------

def _problem_kind(problem):
    if isinstance(problem, ConvexProblem):
        return 0
    if isinstance(problem, LogisticProblem):
        return 1
    raise ConfigurationError(f"unsupported problem type {type(problem).__name__}")


def _row_moments(v):
    """(mean, sum (v - mean)^2, sum (v - mean)^4) of each row of a [rows][n] device tensor."""
    torch = _torch()
    v = v.contiguous()
    rows, n = v.shape
    out = torch.empty((rows, 3), dtype=torch.float64, device=v.device)
    _lib.check(_lib.lib().dbs_dev_row_moments(v.data_ptr(), rows, n, n, out.data_ptr(), _lib.stream_handle()),
               "row_moments")
    return out.cpu().numpy()


def estimate_gradient_noise(problem, x_set, batch_size: int, n_draws: int, seed: int = 0) -> float:
    """Max over probe points of the mean squared norm of the mini-batch gradient,
    i.i.d. draws (sgdlab.py:252-272)."""
    if n_draws < 100:
        raise ConfigurationError("need at least 100 draws for a usable estimate")
    torch = _torch()
    kind = _problem_kind(problem)
    data, labels, opt = problem.device()
    rng = DeviceRng(seed, data.device)
    worst = 0.0
    buf = torch.empty(n_draws, dtype=torch.float64, device=data.device)
    for x in x_set:
        idx = rng.integers(problem.sample_count, (n_draws, batch_size))
        xd = _to_dev_f64(x)
        _lib.check(_lib.lib().dbs_dev_minibatch_sqnorms(kind, data.data_ptr(), labels.data_ptr() if labels is not None
                                                        else None, opt.data_ptr(), problem.dimension,
                                                        float(problem.mu), xd.data_ptr(), idx.data_ptr(), n_draws,
                                                        int(batch_size), buf.data_ptr(), _lib.stream_handle()),
                   "minibatch_sqnorms")
        worst = max(worst, float(_row_moments(buf.view(1, -1))[0, 0]))
    return worst


@dataclass(frozen=True)
class VarianceEstimate:
    batch_size: int
    variance: float
    std_error: float


def verify_lemma1_variance(problem, x, m_values: Sequence[int], n_draws: int, seed: int = 0,
                           with_replacement: bool = True) -> list:
    """Empirical variance of the mini-batch mean objective value per size m, with the
    fourth-moment standard error (sgdlab.py:282-314)."""
    torch = _torch()
    kind = _problem_kind(problem)
    data, labels, opt = problem.device()
    rng = DeviceRng(seed, data.device)
    xd = _to_dev_f64(x)
    n = problem.sample_count
    values = torch.empty(n, dtype=torch.float64, device=data.device)
    _lib.check(_lib.lib().dbs_dev_sample_values(kind, data.data_ptr(), labels.data_ptr() if labels is not None else None,
                                                opt.data_ptr(), problem.dimension, float(problem.mu), xd.data_ptr(), n,
                                                values.data_ptr(), _lib.stream_handle()), "sample_values")
    means = torch.empty(n_draws, dtype=torch.float64, device=data.device)
    out = []
    for m in m_values:
        if with_replacement:
            idx = rng.integers(n, (n_draws, int(m)))
        else:
            # np.argsort(rng.random((n_draws, n)), axis=1)[:, :m]: the same uniforms, a
            # stable per-row sort (the draws are distinct with probability 1)
            idx = torch.argsort(rng.random((n_draws, n)), dim=1, stable=True)[:, :int(m)].contiguous()
        _lib.check(_lib.lib().dbs_dev_gather_means(values.data_ptr(), idx.data_ptr(), n_draws, int(m),
                                                   means.data_ptr(), _lib.stream_handle()), "gather_means")
        mean, m2, m4s = _row_moments(means.view(1, -1))[0]
        var = float(m2 / (n_draws - 1))
        m4 = float(m4s / n_draws)
        se = float(np.sqrt(max(m4 - var ** 2 * (n_draws - 3) / (n_draws - 1), 0.0) / n_draws))
        out.append(VarianceEstimate(batch_size=int(m), variance=var, std_error=se))
    return out
