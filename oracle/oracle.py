"""CPU parity oracle for the DBS hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  The product package
(paper_2007_11831_b200) never imports it; it is the checker, not the thing
measured or shipped.

Contents
* ``lib()``: ctypes handle on oracle/libdbs_oracle.so, the C restatement of
  allocation.py (controller), numpy's PCG64 permutation (sample assignment) and
  sgdlab.aggregate_gradients / sgd_step (dbs_oracle.c cites each line).
* ``MlpProblem``: a numpy 784-H-10 MLP implementing the reference's duck-typed
  ``Problem`` protocol (sgdlab.py:162; touched attributes listed at
  SURVEY.md 8b).  Its ``per_sample_gradients`` returns the batch-mean gradient as
  a single row, so ``minibatch_gradient``'s ``.mean(axis=0)``
  (sgdlab.py:205) yields exactly the mean of per-sample gradients.
* ``run_parallel_sgd``: a line-by-line numpy restatement of
  sgdlab.run_parallel_sgd (sgdlab.py:343-396) and _epoch_layout (320-340).

Parity status: the controller, the permutation and the SGD loop on the
reference's own problems are pinned against golden vectors produced by running
the reference (tests/golden/gen_golden.py).  The MLP model itself has no
counterpart in the reference ("parity unpinned" for the model);
only the loop around it is the reference's.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from fractions import Fraction
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libdbs_oracle.so"

ERROR_NAMES = {
    1: "InvalidMeasurementError",
    2: "InvalidPerformanceError",
    3: "BudgetTooSmallError",
    4: "InvalidBatchError",
    5: "EmptyPartitionError",
    6: "DatasetTooSmallError",
    7: "ConfigurationError",
    9: "EmptyBatchError",
    10: "InvalidStepSizeError",
    20: "OverflowError",
    21: "ValueError",
    22: "OverflowError",
    30: "IndexError",
}


class Bound(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("reserved", ctypes.c_int32), ("num", ctypes.c_int64),
                ("den", ctypes.c_int64), ("value", ctypes.c_double)]


class Pcg64(ctypes.Structure):
    _fields_ = [("state_hi", ctypes.c_uint64), ("state_lo", ctypes.c_uint64),
                ("inc_hi", ctypes.c_uint64), ("inc_lo", ctypes.c_uint64),
                ("has_uint32", ctypes.c_uint32), ("uinteger", ctypes.c_uint32)]

    @property
    def state(self) -> int:
        return (self.state_hi << 64) | self.state_lo

    @property
    def inc(self) -> int:
        return (self.inc_hi << 64) | self.inc_lo


_LIB = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        D = ctypes.POINTER(ctypes.c_double)
        I = ctypes.POINTER(ctypes.c_int64)
        i64 = ctypes.c_int64
        L.oracle_fsum.argtypes = [D, i64, D]
        L.oracle_compute_batch_fractions.argtypes = [D, i64, D]
        L.oracle_scale_to_real_batches.argtypes = [D, i64, i64, D]
        L.oracle_round_twice.argtypes = [D, i64, i64, I]
        L.oracle_raise_zero_batches.argtypes = [I, i64, I]
        L.oracle_partition_ranges.argtypes = [I, i64, I]
        L.oracle_spans_from_ranges.argtypes = [ctypes.POINTER(Bound), ctypes.POINTER(Bound), i64, i64, I]
        L.oracle_plan_next_epoch.argtypes = [D, D, i64, i64, i64, i64, I, I, I]
        L.oracle_replan.argtypes = [I, D, i64, i64, i64, i64, ctypes.c_int, ctypes.c_double, D,
                                    ctypes.POINTER(ctypes.c_int), I, I, I]
        L.oracle_iterations_for_plan.argtypes = [I, I, i64]
        L.oracle_iterations_for_plan.restype = i64
        L.oracle_pcg64_seed.argtypes = [ctypes.POINTER(ctypes.c_uint32), ctypes.c_int32, ctypes.POINTER(Pcg64)]
        L.oracle_permute_spans.argtypes = [ctypes.POINTER(Pcg64), I, i64, I]
        L.oracle_aggregate.argtypes = [ctypes.POINTER(D), I, i64, ctypes.c_int, i64, D]
        L.oracle_sgd_step.argtypes = [D, D, D, i64, ctypes.c_double, ctypes.c_double, D, D]
        _LIB = L
    return _LIB


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _i(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


class OracleError(Exception):
    def __init__(self, code):
        super().__init__(ERROR_NAMES.get(code, f"status {code}"))
        self.code = code
        self.name = ERROR_NAMES.get(code, f"status {code}")


def _check(st):
    if st:
        raise OracleError(st)


def fsum(values):
    v, pv = _d(values)
    out = ctypes.c_double()
    _check(lib().oracle_fsum(pv, len(v), ctypes.byref(out)))
    return out.value


def compute_batch_fractions(perfs):
    v, pv = _d(perfs)
    o, po = _d(np.zeros(len(v)))
    _check(lib().oracle_compute_batch_fractions(pv, len(v), po))
    return o.tolist()


def scale_to_real_batches(fr, budget):
    v, pv = _d(fr)
    o, po = _d(np.zeros(len(v)))
    _check(lib().oracle_scale_to_real_batches(pv, len(v), budget, po))
    return o.tolist()


def round_twice(reals, budget):
    v, pv = _d(reals)
    o, po = _i(np.zeros(len(v)))
    _check(lib().oracle_round_twice(pv, len(v), budget, po))
    return o.tolist()


def raise_zero_batches(b):
    v, pv = _i(b)
    o, po = _i(np.zeros(len(v)))
    _check(lib().oracle_raise_zero_batches(pv, len(v), po))
    return o.tolist()


def partition_ranges(b):
    v, pv = _i(b)
    o, po = _i(np.zeros(len(v) + 1))
    _check(lib().oracle_partition_ranges(pv, len(v), po))
    return o.tolist()


def make_bound(x) -> Bound:
    if isinstance(x, Fraction):
        return Bound(0, 0, x.numerator, x.denominator, 0.0)
    if isinstance(x, (int, np.integer)):
        return Bound(0, 0, int(x), 1, 0.0)
    return Bound(1, 0, 0, 1, float(x))


def spans_from_ranges(ranges, D):
    n = len(ranges)
    lo = (Bound * max(n, 1))(*[make_bound(r[0]) for r in ranges])
    hi = (Bound * max(n, 1))(*[make_bound(r[1]) for r in ranges])
    o, po = _i(np.zeros(2 * max(n, 1)))
    _check(lib().oracle_spans_from_ranges(lo, hi, n, D, po))
    return [(int(o[2 * i]), int(o[2 * i + 1])) for i in range(n)]


def plan_next_epoch(shares, times, B, D, epoch):
    n = len(shares)
    if n == 0 or len(times) != n:
        raise OracleError(2)
    s, ps = _d(shares)
    t, pt = _d(times)
    b, pb = _i(np.zeros(n))
    c, pc = _i(np.zeros(n + 1))
    sp, psp = _i(np.zeros(2 * n))
    _check(lib().oracle_plan_next_epoch(ps, pt, n, B, D, epoch, pb, pc, psp))
    return b.tolist(), c.tolist(), [(int(sp[2 * i]), int(sp[2 * i + 1])) for i in range(n)]


class ReplanState:
    """EMA carry of cluster.run_training (cluster.py:248, 263-266)."""

    def __init__(self, n):
        self.smoothed = np.zeros(n)
        self.has = ctypes.c_int(0)


def replan(prev_spans, times, B, D, epoch, adaptive, smoothing, state: ReplanState):
    n = len(times)
    ps_, pps = _i(np.asarray(prev_spans, dtype=np.int64).reshape(-1))
    t, pt = _d(times)
    b, pb = _i(np.zeros(n))
    c, pc = _i(np.zeros(n + 1))
    sp, psp = _i(np.zeros(2 * n))
    sm = state.smoothed
    _check(lib().oracle_replan(pps, pt, n, B, D, epoch, int(adaptive), smoothing,
                               sm.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                               ctypes.byref(state.has), pb, pc, psp))
    return b.tolist(), c.tolist(), [(int(sp[2 * i]), int(sp[2 * i + 1])) for i in range(n)]


def seed_words(seed: int):
    words = []
    s = int(seed)
    if s < 0:
        raise ValueError("seed must be non-negative")
    while True:
        words.append(s & 0xFFFFFFFF)
        s >>= 32
        if s == 0:
            break
    return words


def pcg64_seed(seed: int) -> Pcg64:
    w = seed_words(seed)
    arr = (ctypes.c_uint32 * len(w))(*w)
    out = Pcg64()
    _check(lib().oracle_pcg64_seed(arr, len(w), ctypes.byref(out)))
    return out


def permute_spans(g: Pcg64, spans):
    flat = np.asarray(spans, dtype=np.int64).reshape(-1)
    total = int(sum(e - s for s, e in spans))
    o, po = _i(np.zeros(max(total, 1)))
    f, pf = _i(flat)
    _check(lib().oracle_permute_spans(ctypes.byref(g), pf, len(spans), po))
    return o[:total]


def aggregate(grads, batches, mode):
    n = len(grads)
    gs = [np.ascontiguousarray(g, dtype=np.float64) for g in grads]
    arr = (ctypes.POINTER(ctypes.c_double) * n)(*[g.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) for g in gs])
    b, pb = _i(batches)
    P = gs[0].size
    o, po = _d(np.zeros(P))
    _check(lib().oracle_aggregate(arr, pb, n, int(mode), P, po))
    return o


def sgd_step(x, g, v, step, mom):
    x, px = _d(x)
    g, pg = _d(g)
    v, pv = _d(v)
    xo, pxo = _d(np.zeros_like(x))
    vo, pvo = _d(np.zeros_like(x))
    _check(lib().oracle_sgd_step(px, pg, pv, x.size, step, mom, pxo, pvo))
    return xo, vo


# ---------------------------------------------------------------------------
# numpy MLP Problem adapter + run_parallel_sgd restatement
# ---------------------------------------------------------------------------

def synthetic_mnist(n_samples=60000, in_dim=784, classes=10, seed=0):
    """C1 inputs: X ~ N(0,1) fp32, labels integers(0, classes)."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n_samples, in_dim), dtype=np.float32)
    y = rng.integers(0, classes, size=n_samples).astype(np.int32)
    return X, y


def mlp_init(in_dim=784, hidden=256, classes=10, seed=0):
    """Flat fp32 parameters [W1 (H x IN) | b1 | W2 (C x H) | b2], He-uniform-ish."""
    rng = np.random.default_rng(seed + 1)
    b1 = 1.0 / math.sqrt(in_dim)
    b2 = 1.0 / math.sqrt(hidden)
    W1 = rng.uniform(-b1, b1, (hidden, in_dim)).astype(np.float32)
    c1 = rng.uniform(-b1, b1, hidden).astype(np.float32)
    W2 = rng.uniform(-b2, b2, (classes, hidden)).astype(np.float32)
    c2 = rng.uniform(-b2, b2, classes).astype(np.float32)
    return np.concatenate([W1.ravel(), c1, W2.ravel(), c2]).astype(np.float32)


class MlpProblem:
    """Duck-typed reference ``Problem`` (sgdlab.py:162) for the 784-H-C MLP.

    Mean softmax cross-entropy over a batch; gradients in float64 (the
    reference computes in float64), inputs as given (fp32 data).
    ``emulate_bf16`` rounds the GEMM operands to bf16 first, matching the
    tensor-core operand precision of the GPU path.
    """

    def __init__(self, X, y, hidden=256, classes=10, emulate_bf16=False):
        self.X = X
        self.y = y
        self.in_dim = X.shape[1]
        self.hidden = hidden
        self.classes = classes
        self.sample_count = X.shape[0]
        self.dimension = hidden * self.in_dim + hidden + classes * hidden + classes
        self.mu = 1.0  # only used by SgdConfig.validate_step_size (sgdlab.py:184-188)
        self.optimum = np.zeros(self.dimension)
        self.emulate_bf16 = emulate_bf16

    def unpack(self, x):
        H, I, C = self.hidden, self.in_dim, self.classes
        o = 0
        W1 = x[o:o + H * I].reshape(H, I); o += H * I
        b1 = x[o:o + H]; o += H
        W2 = x[o:o + C * H].reshape(C, H); o += C * H
        b2 = x[o:o + C]
        return W1, b1, W2, b2

    @staticmethod
    def _bf16(a):
        a32 = np.asarray(a, dtype=np.float32)
        u = a32.view(np.uint32).astype(np.uint64)
        u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
        return u.astype(np.uint32).view(np.float32).astype(np.float64)

    def loss_and_grad(self, x, indices):
        W1, b1, W2, b2 = self.unpack(np.asarray(x, dtype=np.float64))
        Xb = self.X[indices].astype(np.float64)
        yb = self.y[indices]
        q = self._bf16 if self.emulate_bf16 else (lambda a: np.asarray(a, dtype=np.float64))
        h = q(Xb) @ q(W1).T + b1
        a = np.maximum(h, 0.0)
        z = q(a) @ q(W2).T + b2
        z = z - z.max(axis=1, keepdims=True)
        e = np.exp(z)
        p = e / e.sum(axis=1, keepdims=True)
        m = Xb.shape[0]
        loss = float(-np.mean(np.log(p[np.arange(m), yb])))
        dz = p
        dz[np.arange(m), yb] -= 1.0
        dz /= m
        gW2 = dz.T @ q(a)
        gb2 = dz.sum(axis=0)
        da = dz @ q(W2)
        dh = da * (h > 0)
        gW1 = dh.T @ q(Xb)
        gb1 = dh.sum(axis=0)
        g = np.concatenate([gW1.ravel(), gb1, gW2.ravel(), gb2])
        return loss, g

    def per_sample_gradients(self, x, indices):
        # batch mean as one row: minibatch_gradient's .mean(axis=0) (sgdlab.py:205)
        return self.loss_and_grad(x, np.asarray(indices))[1][None, :]

    def objective(self, x):
        losses = []
        for s in range(0, self.sample_count, 8192):
            idx = np.arange(s, min(s + 8192, self.sample_count))
            losses.append(self.loss_and_grad(x, idx)[0] * len(idx))
        return float(sum(losses) / self.sample_count)

    def objective_gap(self, x):
        return self.objective(x)


def epoch_layout(plan_source, epoch, n_workers, sample_count, plan_of=None):
    """sgdlab._epoch_layout (sgdlab.py:320-340) on (int_batches, cum) plans."""
    if len(plan_source) == 0:
        raise OracleError(7)
    first = plan_source[0]
    if isinstance(first, dict):
        plan = plan_source[min(epoch, len(plan_source) - 1)]
        batches = list(plan["int_batches"])
        cum = plan["cum"]
        rngs = [(Fraction(cum[i], cum[-1]), Fraction(cum[i + 1], cum[-1])) for i in range(len(batches))]
        spans = spans_from_ranges(rngs, sample_count)
    else:
        batches = [int(b) for b in plan_source]
        cum = partition_ranges([1] * n_workers)
        rngs = [(Fraction(cum[i], cum[-1]), Fraction(cum[i + 1], cum[-1])) for i in range(n_workers)]
        spans = spans_from_ranges(rngs, sample_count)
    if any(b < 1 for b in batches):
        raise OracleError(7)
    return batches, spans


def run_parallel_sgd(problem, step_size, n_iterations, momentum, aggregation, seed, n_workers,
                     plan_source, initial_point=None, record_loss=False, averaging_interval=None):
    """Restatement of sgdlab.run_parallel_sgd (sgdlab.py:343-396).

    averaging_interval=k switches the synchronous step to periodic model
    averaging (the reference counts its rounds, cluster.py:185-186, but has no
    numerics -- these are the declared semantics the GPU path implements):
    every worker keeps its own x_i, v_i and takes a local sgd_step with its own
    mean gradient; after iteration t of an epoch with (t + 1) % k == 0 the
    replicas are replaced by their aggregation-weighted average.  The reported
    x is the weighted average of the replicas."""
    if averaging_interval is not None:
        return _run_model_averaging(problem, step_size, n_iterations, momentum, aggregation, seed, n_workers,
                                    plan_source, initial_point, record_loss, int(averaging_interval))
    if not (0.0 < step_size * problem.mu < 1.0):
        raise OracleError(10)
    rng = np.random.default_rng(seed)
    x = np.ones(problem.dimension) if initial_point is None else np.asarray(initial_point, dtype=float).copy()
    velocity = np.zeros(problem.dimension)
    sq = np.empty(n_iterations)
    losses = []
    done = 0
    epoch = 0
    mode = 1 if aggregation == "batch_weighted" else 0
    while done < n_iterations:
        batches, spans = epoch_layout(plan_source, epoch, n_workers, problem.sample_count)
        perms = [start + rng.permutation(end - start) for start, end in spans]
        iters = min((end - start) // b for (start, end), b in zip(spans, batches))
        if iters == 0:
            raise OracleError(7)
        for t in range(iters):
            grads = []
            lsum = 0.0
            for perm, b in zip(perms, batches):
                idx = perm[t * b:(t + 1) * b]
                if record_loss and hasattr(problem, "loss_and_grad"):
                    l, g = problem.loss_and_grad(x, idx)
                    lsum += l * b
                else:
                    g = problem.per_sample_gradients(x, idx).mean(axis=0)
                grads.append(g)
            if record_loss:
                losses.append(lsum / sum(batches))
            stacked = np.stack(grads)
            if mode == 1:
                w = np.asarray(batches, dtype=float)
                w /= w.sum()
                grad = w @ stacked
            else:
                grad = stacked.mean(axis=0)
            velocity = momentum * velocity + grad
            x = x - step_size * velocity
            diff = x - problem.optimum
            sq[done] = float(diff @ diff)
            done += 1
            if done == n_iterations:
                break
        epoch += 1
    return {"squared_distances": sq, "x": x, "losses": np.asarray(losses),
            "final_loss": problem.objective_gap(x) if hasattr(problem, "objective_gap") else None}


def _run_model_averaging(problem, step_size, n_iterations, momentum, aggregation, seed, n_workers, plan_source,
                         initial_point, record_loss, interval):
    if not (0.0 < step_size * problem.mu < 1.0):
        raise OracleError(10)
    if interval < 1:
        raise OracleError(7)
    rng = np.random.default_rng(seed)
    x0 = np.ones(problem.dimension) if initial_point is None else np.asarray(initial_point, dtype=float).copy()
    xs = [x0.copy() for _ in range(n_workers)]
    vs = [np.zeros(problem.dimension) for _ in range(n_workers)]
    sq = np.empty(n_iterations)
    losses = []
    done = 0
    epoch = 0
    mode = 1 if aggregation == "batch_weighted" else 0

    def weights(batches):
        if mode == 1:
            w = np.asarray(batches, dtype=float)
            return w / w.sum()
        return np.full(len(batches), 1.0 / len(batches))

    batches = None
    while done < n_iterations:
        batches, spans = epoch_layout(plan_source, epoch, n_workers, problem.sample_count)
        perms = [start + rng.permutation(end - start) for start, end in spans]
        iters = min((end - start) // b for (start, end), b in zip(spans, batches))
        if iters == 0:
            raise OracleError(7)
        w = weights(batches)
        for t in range(iters):
            lsum = 0.0
            for i, (perm, b) in enumerate(zip(perms, batches)):
                idx = perm[t * b:(t + 1) * b]
                if record_loss and hasattr(problem, "loss_and_grad"):
                    l, g = problem.loss_and_grad(xs[i], idx)
                    lsum += l * b
                else:
                    g = problem.per_sample_gradients(xs[i], idx).mean(axis=0)
                vs[i] = momentum * vs[i] + g
                xs[i] = xs[i] - step_size * vs[i]
            if record_loss:
                losses.append(lsum / sum(batches))
            if (t + 1) % interval == 0:
                xbar = w @ np.stack(xs)
                xs = [xbar.copy() for _ in range(n_workers)]
            diff = (w @ np.stack(xs)) - problem.optimum
            sq[done] = float(diff @ diff)
            done += 1
            if done == n_iterations:
                break
        epoch += 1
    x = weights(batches) @ np.stack(xs)
    return {"squared_distances": sq, "x": x, "replicas": xs, "losses": np.asarray(losses),
            "final_loss": problem.objective_gap(x) if hasattr(problem, "objective_gap") else None}


# ---------------------------------------------------------------------------
# CPU baseline for the ResNet-18 configs: the run_parallel_sgd loop with a
# PyTorch-CPU ResNet-18 Problem (the reference itself has no ResNet; this is
# the same loop, a CPU model, on the host cores -- a reported baseline only)
# ---------------------------------------------------------------------------

def torch_cpu_resnet18(tensors):
    """Functional ResNet-18 (CIFAR stem) on the CPU with the given torchvision-order tensors."""
    import torch
    import torch.nn.functional as F

    params = [torch.as_tensor(np.asarray(t), dtype=torch.float32).requires_grad_(True) for t in tensors]

    def forward(x):
        it = iter(params)

        def conv_bn(h, stride, pad, relu=True):
            w, g, b = next(it), next(it), next(it)
            y = F.batch_norm(F.conv2d(h, w, stride=stride, padding=pad), None, None, g, b, training=True, eps=1e-5)
            return F.relu(y) if relu else y

        h = conv_bn(x, 1, 1)
        cin = 64
        for L, wdt in enumerate((64, 128, 256, 512)):
            for blk in range(2):
                stride = 2 if (L > 0 and blk == 0) else 1
                a = conv_bn(h, stride, 1)
                a = conv_bn(a, 1, 1, relu=False)
                sc = conv_bn(h, stride, 0, relu=False) if (stride != 1 or cin != wdt) else h
                h = F.relu(a + sc)
                cin = wdt
        wf, bf = next(it), next(it)
        return h.mean(dim=(2, 3)) @ wf.t() + bf

    return forward, params


def torch_cpu_resnet50(tensors):
    """Functional ResNet-50 (torchvision v1.5 topology) on the CPU; uint8 input
    rows are mapped to (u - 128) / 64 as on the device."""
    import torch
    import torch.nn.functional as F

    params = [torch.as_tensor(np.asarray(t), dtype=torch.float32).requires_grad_(True) for t in tensors]

    def forward(x):
        it = iter(params)
        if x.dtype == torch.uint8:
            x = (x.float() - 128.0) / 64.0

        def conv_bn(h, stride, pad, relu=True):
            w, g, b = next(it), next(it), next(it)
            y = F.batch_norm(F.conv2d(h, w, stride=stride, padding=pad), None, None, g, b, training=True, eps=1e-5)
            return F.relu(y) if relu else y

        h = F.max_pool2d(conv_bn(x, 2, 3), 3, 2, 1)
        cin = 64
        for L, (wdt, n) in enumerate(zip((64, 128, 256, 512), (3, 4, 6, 3))):
            for blk in range(n):
                stride = 2 if (L > 0 and blk == 0) else 1
                a = conv_bn(h, 1, 0)
                a = conv_bn(a, stride, 1)
                a = conv_bn(a, 1, 0, relu=False)
                sc = conv_bn(h, stride, 0, relu=False) if (stride != 1 or cin != 4 * wdt) else h
                h = F.relu(a + sc)
                cin = 4 * wdt
        wf, bf = next(it), next(it)
        return h.mean(dim=(2, 3)) @ wf.t() + bf

    return forward, params


def cpu_resnet_iteration_seconds(tensors, X, y, batches, lr=0.05, momentum=0.9, threads=None, depth=18):
    """One synchronous iteration (sgdlab.py:380-391) with CPU ResNet-18/50 workers:
    per-worker batch-mean gradient, batch-weighted aggregation, heavy-ball step."""
    import time

    import torch
    import torch.nn.functional as F

    if threads:
        torch.set_num_threads(threads)
    forward, params = (torch_cpu_resnet50 if depth == 50 else torch_cpu_resnet18)(tensors)
    vel = [torch.zeros_like(p) for p in params]
    t0 = time.perf_counter()
    grads = []
    off = 0
    for b in batches:
        xb = torch.as_tensor(X[off:off + b])
        yb = torch.as_tensor(y[off:off + b]).long()
        off += b
        for p in params:
            p.grad = None
        F.cross_entropy(forward(xb), yb).backward()
        grads.append([p.grad.detach().clone() for p in params])
    w = np.asarray(batches, dtype=np.float64)
    w /= w.sum()
    with torch.no_grad():
        for k, p in enumerate(params):
            g = sum(float(wi) * gr[k] for wi, gr in zip(w, grads))
            vel[k].mul_(momentum).add_(g)
            p.sub_(lr * vel[k])
    return time.perf_counter() - t0


# ---------------------------------------------------------------------------
# Workload inputs for bench.py's CPU legs (the reference arm must not touch the
# product package): the same numpy generators and torchvision-order
# initialisation as paper_2007_11831_b200.{mlp,resnet} (same draws, same order)
# ---------------------------------------------------------------------------

def synthetic_mnist(n_samples=60000, in_dim=784, classes=10, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n_samples, in_dim), dtype=np.float32)
    y = rng.integers(0, classes, size=n_samples).astype(np.int32)
    return X, y


def synthetic_cifar(n_samples=50000, classes=10, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n_samples, 3, 32, 32), dtype=np.float32)
    y = rng.integers(0, classes, size=n_samples).astype(np.int32)
    return X, y


def synthetic_imagenet(n_samples=20000, image=224, classes=1000, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.integers(0, 256, size=(n_samples, 3, image, image), dtype=np.uint8)
    y = rng.integers(0, classes, size=n_samples).astype(np.int32)
    return X, y


def resnet_shapes(classes=10, depth=18):
    """(kind, torch shape) of every parameter tensor in torchvision order
    (kind 0 conv weight, 1 BN gamma, 2 BN beta, 3 FC weight, 4 FC bias)."""
    if depth == 18:
        convs, cin = [(3, 64, 3)], 64
        for L, w in enumerate((64, 128, 256, 512)):
            for b in range(2):
                stride = 2 if (L > 0 and b == 0) else 1
                convs += [(cin, w, 3), (w, w, 3)] + ([(cin, w, 1)] if (stride != 1 or cin != w) else [])
                cin = w
    else:
        convs, cin = [(3, 64, 7)], 64
        for L, (w, n) in enumerate(zip((64, 128, 256, 512), (3, 4, 6, 3))):
            for b in range(n):
                stride = 2 if (L > 0 and b == 0) else 1
                convs += [(cin, w, 1), (w, w, 3), (w, 4 * w, 1)]
                convs += [(cin, 4 * w, 1)] if (stride != 1 or cin != 4 * w) else []
                cin = 4 * w
    out = []
    for ci, co, k in convs:
        out += [(0, (co, ci, k, k)), (1, (co,)), (2, (co,))]
    return out + [(3, (classes, cin)), (4, (classes,))]


def resnet_init(classes=10, seed=0, depth=18):
    """Kaiming-normal fan-out convolutions, BN (1, 0), uniform classifier."""
    rng = np.random.default_rng(seed)
    shapes = resnet_shapes(classes, depth)
    feat = shapes[-2][1][1]
    out = []
    for kind, shp in shapes:
        if kind == 0:
            out.append(rng.normal(0.0, math.sqrt(2.0 / (shp[0] * shp[2] * shp[3])), shp).astype(np.float32))
        elif kind == 1:
            out.append(np.ones(shp, dtype=np.float32))
        elif kind == 2:
            out.append(np.zeros(shp, dtype=np.float32))
        else:
            bound = 1.0 / math.sqrt(feat)
            out.append(rng.uniform(-bound, bound, shp).astype(np.float32))
    return out


# ---------------------------------------------------------------------------
# numpy Generator.integers / random restated (the draws of checks.py:42-142)
# ---------------------------------------------------------------------------

_PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
_M128 = (1 << 128) - 1


class Pcg64Ref:
    """PCG64 (XSL-RR 128/64) from a numpy bit-generator state dict."""

    def __init__(self, state: dict):
        self.state = int(state["state"]["state"])
        self.inc = int(state["state"]["inc"])

    def next64(self) -> int:
        self.state = (self.state * _PCG_MULT + self.inc) & _M128
        hi, lo = self.state >> 64, self.state & ((1 << 64) - 1)
        x, r = hi ^ lo, hi >> 58
        return ((x >> r) | (x << ((64 - r) & 63))) & ((1 << 64) - 1)

    def integers(self, n: int, count: int) -> list:
        """Generator.integers(0, n, size=count), int64, n <= 2^32: a 32-bit buffer local to
        the call (low half first), Lemire's multiply-and-reject (numpy distributions.c
        random_bounded_uint64_fill, use_masked = False)."""
        r = n - 1
        buf, bcnt = 0, 0
        out = []

        def b32():
            nonlocal buf, bcnt
            if not bcnt:
                buf, bcnt = self.next64(), 1
            else:
                buf, bcnt = buf >> 32, bcnt - 1
            return buf & 0xFFFFFFFF

        if r == 0:
            return [0] * count
        if r == 0xFFFFFFFF:
            return [b32() for _ in range(count)]
        rexcl = r + 1
        threshold = (0xFFFFFFFF - r) % rexcl
        for _ in range(count):
            m = b32() * rexcl
            left = m & 0xFFFFFFFF
            if left < rexcl:
                while left < threshold:
                    m = b32() * rexcl
                    left = m & 0xFFFFFFFF
            out.append(m >> 32)
        return out

    def random(self, count: int) -> list:
        return [(self.next64() >> 11) * (1.0 / 9007199254740992.0) for _ in range(count)]
