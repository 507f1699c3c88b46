"""Measured DBS vs fixed-batch synchronous training on B200s.

This is the GPU counterpart of cluster.run_training (cluster.py:234-275): the
same epoch loop and the same re-plan (cluster.next_plan -> the device
controller), but `per_worker_gpu` is MEASURED -- per-worker compute seconds
accumulated on the device from %globaltimer stamps around each worker's
forward/backward -- and the epoch wall time is a CUDA-event interval.  The
records are the reference's EpochStats (cluster.py:111-120), so
cumulative_times and the report schema apply unchanged.

Per epoch: controller plan -> device permutation of every span (sgdlab.py:
372-374) -> coalesced repack of each worker's rows into its HBM shard -> T
iterations of [every worker's forward/backward on its own stream || fused
batch-weighted aggregation + momentum SGD].  For ResNet-18 one iteration is
captured once per distinct plan as a CUDA graph (every kernel reads the
iteration index from device memory) and replayed T times.

Workers
  * one process, W simulated workers: each worker is a CUDA stream, confined
    to its own SM partition with a green context when ``partition=True``;
  * one process per GPU (torchrun): worker = rank (DistributedTrainer), the
    update is the fused NVLink kernel of comm.py.

Disturbance (DisturbanceEvent, cluster.py:25-56), realised on the device:
  * cost_multiplier m  -> a co-running spin kernel pins a fraction 1 - 1/m of
                          the worker's SMs for the whole epoch;
  * extra_epoch_seconds -> a timed spin on the worker's stream, spread over the
                          epoch's iterations (counted in its compute time, as
                          in epoch_gpu_time cluster.py:132-145).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib, cluster
from .cluster import EpochStats, StrategyConfig, WorkerProfile
from .errors import ConfigurationError
from .sgdlab import DeviceRng

_MODE = {"uniform_average": 0, "batch_weighted": 1}
MODEL_MLP, MODEL_RESNET18 = 0, 1


@dataclass
class Worker:
    index: int
    stream: object
    spin_stream: object
    sm_count: int
    green: object = None
    ctx: int = 0  # CUcontext of the worker's SM partition (0 = the current context)


def _green_supported() -> bool:
    try:
        import torch

        return bool(torch.cuda.green_contexts.SUPPORTED)
    except Exception:
        return False


_PARTITIONS = []  # keep green contexts alive for the process


def make_workers(n: int, partition: bool = True) -> list:
    """W simulated workers on the current device.  partition=True gives each
    worker a disjoint SM set (a green context created by the library, whose
    launches the iteration driver issues with that context current)."""
    import ctypes

    import torch

    dev = torch.cuda.current_device()
    total = torch.cuda.get_device_properties(dev).multi_processor_count
    workers = []
    if partition and n > 1:
        per = max(8, (total // n) // 8 * 8)
        h = ctypes.c_void_p()
        actual = ctypes.c_int32()
        _lib.check(_lib.lib().dbs_partition_create(n, per, ctypes.byref(h), ctypes.byref(actual)), "partition")
        _PARTITIONS.append(h)
        for i in range(n):
            ctx, st, side = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
            _lib.check(_lib.lib().dbs_partition_get(h, i, ctypes.byref(ctx), ctypes.byref(st), ctypes.byref(side)),
                       "partition_get")
            workers.append(Worker(i, torch.cuda.ExternalStream(st.value), torch.cuda.ExternalStream(side.value),
                                  actual.value, h, ctx.value))
        return workers
    for i in range(n):
        workers.append(Worker(i, torch.cuda.Stream(), torch.cuda.Stream(), total, None))
    return workers


@dataclass
class RunResult:
    stats: list
    losses: np.ndarray          # per-iteration batch-weighted mean loss
    samples: int                # samples processed (sum over epochs of T * sum b)
    wall_seconds: float         # sum of epoch wall times (device events, iterations only)
    plans: list = field(default_factory=list)
    timed_seconds: float = 0.0  # device time from the start of epoch `timed_from` to the end,
    timed_samples: int = 0      # whole epochs: re-plan, permutation, repack and iterations
    timed_launches: int = 0     # kernels of this library executed in that window
    timed_host_launches: int = 0  # launch calls the host issued in that window (kernels + graph launches)


class DevicePlanner:
    """cluster.run_training's re-plan (cluster.py:253-271) on the device: the
    measured per-worker seconds feed dbs_dev_replan where they were accumulated
    (shares of the previous spans -> perf -> optional EMA -> times = s / p ->
    plan_next_epoch, one single-CTA launch), and ONE pinned read-back per epoch
    carries the new plan, the seconds and the status for the host bookkeeping
    (EpochStats, launch sizes).  The epoch-0 / non-DBS even plan comes from the
    same kernel (cluster.py:254-255, 223-231)."""

    def __init__(self, torch, dev, n: int, config: StrategyConfig, D: int):
        self.torch, self.n, self.D = torch, n, D
        self.B = int(config.total_budget)
        self.adaptive = 1 if config.kind == "dbs" else 0
        self.smoothing = float(config.perf_smoothing) if self.adaptive else 0.0
        # device pack: [b n | cum n+1 | spans 2n | iters 1 | seconds n (f64) | flags 2 x i32]
        self.len = 5 * n + 3
        self.pack = torch.zeros(self.len, dtype=torch.int64, device=dev)
        self.host = torch.zeros(self.len, dtype=torch.int64, pin_memory=True)
        o = 0
        self.b = self.pack[o:o + n]; o += n
        self.cum = self.pack[o:o + n + 1]; o += n + 1
        self.spans_next = self.pack[o:o + 2 * n]; o += 2 * n
        self.iters = self.pack[o:o + 1]; o += 1
        self.secs = self.pack[o:o + n].view(torch.float64); o += n
        self.flags = self.pack[o:o + 1].view(torch.int32)
        self.spans = torch.zeros(2 * n, dtype=torch.int64, device=dev)  # the current epoch's spans (input)
        self.smoothed = torch.zeros(n, dtype=torch.float64, device=dev)

    def enqueue(self, epoch: int, seconds, stream: int, plan: bool = True) -> None:
        """Plan `epoch` from `seconds` (the previous epoch's measured compute times,
        device f64 [n]) and start the read-back; nothing waits here.  plan=False
        (after the last epoch): only the seconds are read back."""
        L = _lib.lib()
        if not plan:
            self.secs.copy_(seconds)
            self.host.copy_(self.pack, non_blocking=True)
            return
        if epoch > 0:
            self.spans.copy_(self.spans_next)
        _lib.check(L.dbs_dev_replan(self.spans.data_ptr(), seconds.data_ptr(), self.n, self.B, self.D, int(epoch),
                                    self.adaptive, self.smoothing, self.smoothed.data_ptr(), self.flags.data_ptr(),
                                    self.b.data_ptr(), self.cum.data_ptr(), self.spans_next.data_ptr(),
                                    self.iters.data_ptr(), stream), "dev_replan")
        self.secs.copy_(seconds)
        self.host.copy_(self.pack, non_blocking=True)

    def seconds(self) -> tuple:
        """The measured seconds carried by the last read-back (after a sync)."""
        n = self.n
        return tuple(float(x) for x in self.host.numpy()[4 * n + 2:5 * n + 2].view(np.float64))

    def result(self, epoch: int):
        """The plan of `epoch` from the read-back (after a sync); a controller error
        raises the reference's exception class (errors.py:4-53)."""
        from . import allocation
        from .errors import from_status

        h = self.host.numpy()
        n = self.n
        st = int(h[5 * n + 2:5 * n + 3].view(np.int32)[1])
        if st != 0:
            raise from_status(st, f"device re-plan of epoch {epoch} failed (dbs_status {st})")
        return allocation.plan_from_arrays(h[:n], h[n:2 * n + 1], h[2 * n + 1:4 * n + 1], epoch)

    def current_spans(self):
        """Device spans of the plan of the epoch just read back."""
        return self.spans_next


class SimulatedTrainer:
    """W simulated workers of synchronous S-SGD on one GPU.

    model = "mlp" (config 1: X fp32 [D][784]), "resnet18" (configs 3/4:
    X fp32 [D][3][32][32]) or "resnet50" (config 5: X uint8 [D][3][S][S],
    S = 224 for ImageNet-shaped data).
    """

    def __init__(self, X, y, n_workers: int, model: str = "mlp", hidden: int = 256, classes: int = 10,
                 seed: int = 0, partition: bool = False, params=None, max_batch: Optional[int] = None,
                 graphs: Optional[bool] = None, pin_sms: Optional[bool] = None, precision="f32"):
        import torch

        _lib.require_device()
        self.torch = torch
        self.dev = torch.device("cuda", torch.cuda.current_device())
        X = X if isinstance(X, torch.Tensor) else torch.as_tensor(X)
        y = y if isinstance(y, torch.Tensor) else torch.as_tensor(y)
        if model not in ("mlp", "resnet18", "resnet50"):
            raise ConfigurationError(f"unknown model {model!r}")
        x_dtype = torch.uint8 if model == "resnet50" else torch.float32
        self.X = X.to(self.dev, x_dtype).contiguous()
        self.y = y.to(self.dev, torch.int32).contiguous()
        self.D = int(self.X.shape[0])
        self.row_elems = int(np.prod(self.X.shape[1:]))
        self.row_bytes = self.row_elems * self.X.element_size()
        self.n = n_workers
        self.classes = classes
        self.kind = MODEL_MLP if model == "mlp" else MODEL_RESNET18
        # tensor-core operand precision: "f32" = 3xTF32 on S32 operands (the fp32 class), or "bf16"
        self.precision = _lib.precision_code(precision)
        self.depth, self.image = (50, int(self.X.shape[-1])) if model == "resnet50" else (18, 32)
        if self.kind == MODEL_MLP:
            from .mlp import MlpModel

            self.model = MlpModel(self.row_elems, hidden, classes, seed, self.dev, params=params,
                                  precision=self.precision)
        else:
            from .resnet import ResnetModel

            S = self.image
            if tuple(self.X.shape[1:]) != (3, S, S) or (model == "resnet18" and S != 32):
                raise ConfigurationError(f"{model} expects [D][3][{S}][{S}] rows, got {tuple(self.X.shape)}")
            self.model = ResnetModel(classes, seed, self.dev, params=params, depth=self.depth, image=S,
                                     precision=self.precision)
        self.workers = make_workers(n_workers, partition)
        partitioned = any(w.ctx for w in self.workers)
        # iteration graphs (one context: every kernel reads the iteration index from
        # device memory); partitioned workers launch eagerly from their own contexts
        # (a graph cannot span contexts)
        default_graphs = not partitioned
        self.graphs = default_graphs if graphs is None else bool(graphs and default_graphs)
        # partitioned workers: one graph per worker, captured in its own context
        self.worker_graphs = partitioned if graphs is None else bool(graphs and partitioned)
        if os.environ.get("DBS_WORKER_GRAPHS") == "0":  # A/B switch: eager launches from the host
            self.worker_graphs = False
        self._wg_cache = {}
        self._wg_retired = []
        # shared-context workers: the device-side epoch loop (a `while` conditional graph)
        self.epoch_graphs = os.environ.get("DBS_EPOCH_GRAPH", "1") != "0"
        self._eg_cache = {}
        self._eg_retired = []
        self.d_total = torch.zeros(1, dtype=torch.int64, device=self.dev)
        # SM-pinning disturbance only when each worker owns its SMs (one GPU per
        # worker, or green-context partitions); otherwise the proportional slow-down
        self.pin_sms = (n_workers == 1 or partition) if pin_sms is None else bool(pin_sms)
        # shared-GPU emulated devices (C1): when set, every worker's iteration also runs a
        # timed spin of m_w x b_w x device_per_sample_ns on its stream -- the reference's
        # cost law effective_cost x samples (cluster.py:123-145) on top of the real
        # (launch-latency-bound, nearly batch-independent) MLP compute, m_w the worker's
        # active cost multiplier.  None: a disturbed worker's spin is proportional to
        # its own measured forward/backward time.
        self.device_per_sample_ns: Optional[float] = None
        self.max_batch = max_batch
        self.scratch = {}
        P = self.model.P
        self.grads = [torch.zeros(P, dtype=torch.float32, device=self.dev) for _ in range(n_workers)]
        self.seconds = torch.zeros(n_workers, dtype=torch.float64, device=self.dev)
        self.stamps = [torch.zeros(2, dtype=torch.int64, device=self.dev) for _ in range(n_workers)]
        self.loss_scratch = torch.zeros(n_workers, dtype=torch.float32, device=self.dev)
        self.stop = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.d_iter = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.agg = torch.cuda.Stream()
        self.rng = None
        # fixed-address shards (graph replays need stable pointers); MLP rows are stored
        # in the GEMM operand form (S32 [in_ld] for "f32", bf16 for "bf16")
        if self.kind == MODEL_MLP and self.precision == _lib.PREC_F32:
            shard_shape, shard_dtype = (self.D, 2 * self.model.layout.in_ld), torch.float32
        else:
            shard_shape = (self.D, self.row_elems)
            shard_dtype = torch.bfloat16 if self.kind == MODEL_MLP else x_dtype
        self.shard_x = [torch.empty(shard_shape, dtype=shard_dtype, device=self.dev) for _ in range(n_workers)]
        self.shard_y = [torch.empty(self.D, dtype=torch.int32, device=self.dev) for _ in range(n_workers)]
        self.loss_buf = torch.zeros((n_workers, self.D + 1), dtype=torch.float32, device=self.dev)
        self._graph_cache = {}
        self.graph_iters = 8  # iterations per captured graph
        self._primed = False
        self._primed_batches = None

    # -- helpers --------------------------------------------------------------
    def _scratch(self, w: int, b: int):
        cur = self.scratch.get(w)
        if cur is None or cur.max_batch < b:
            cap = max(b, self.max_batch or 0)
            if self.kind == MODEL_MLP:
                from .mlp import MlpScratch

                cur = MlpScratch(self.model.layout, cap)
            else:
                from .resnet import ResnetScratch

                cur = ResnetScratch(cap, self.classes, self.depth, self.image, self.precision)
            self.scratch[w] = cur
            self._graph_cache.clear()  # scratch pointers changed
            if self._wg_cache:
                self.torch.cuda.synchronize()
                for h in self._wg_cache.values():
                    _lib.lib().dbs_worker_graphs_destroy(h)
                self._wg_cache.clear()
        return cur

    def _gather_mlp(self, idx, rows, xs, stream):
        """Repack MLP rows into the worker's shard in the GEMM operand form."""
        if self.precision == _lib.PREC_F32:
            return _lib.lib().dbs_dev_gather_rows_f32_s32(self.X.data_ptr(), idx.data_ptr(), rows, self.row_elems,
                                                          xs.data_ptr(), self.model.layout.in_ld, stream)
        return _lib.lib().dbs_dev_gather_rows_f32_bf16(self.X.data_ptr(), idx.data_ptr(), rows, self.row_elems,
                                                       xs.data_ptr(), stream)

    def _run_iters(self, slots, t0, t1, mode, lr, mom, params, vel, pb, skip, d_iter=None):
        st = _lib.lib().dbs_run_iterations(slots, self.n, t0, t1, mode, float(lr), float(mom), params.data_ptr(),
                                           vel.data_ptr(), pb.data_ptr(), int(skip), int(self.agg.cuda_stream),
                                           d_iter.data_ptr() if d_iter is not None else None)
        _lib.check(st, "run_iterations")

    def _replicas_begin(self, mode: int):
        """Per-worker model replicas for local SGD, copied from the shared model;
        the averaging kernel is loaded here (never lazily behind a spin kernel)."""
        torch = self.torch
        m = self.model
        self._rep_p = [m.params.clone() for _ in range(self.n)]
        self._rep_v = [m.velocity.clone() for _ in range(self.n)]
        self._rep_pb = [m.params_op.clone() for _ in range(self.n)]
        arr = lambda ts: (ctypes.c_void_p * self.n)(*[t.data_ptr() for t in ts])
        self._rep_ptrs = (arr(self._rep_p), arr(self._rep_v), arr(self._rep_pb))
        self._rep_mode = mode
        self._average_replicas(mode)
        torch.cuda.synchronize()

    def _average_replicas(self, mode: int, batches=None):
        b = np.asarray(batches if batches is not None else [1] * self.n, dtype=np.int64)
        st = _lib.lib().dbs_dev_average_replicas_f32_ex(self._rep_ptrs[0], b.ctypes.data_as(_lib.P_i64), self.n,
                                                        int(mode), self.model.P, self._rep_ptrs[2], self.precision,
                                                        int(self.agg.cuda_stream))
        _lib.check(st, "average_replicas")

    def _replicas_end(self, final_average: bool, batches):
        """Hand the (averaged) replica back to the shared model."""
        torch = self.torch
        if final_average:
            self._average_replicas(self._rep_mode, batches)
        torch.cuda.current_stream().wait_stream(self.agg)
        self.model.params.copy_(self._rep_p[0])
        self.model.velocity.copy_(self._rep_v[0])
        self.model.params_op.copy_(self._rep_pb[0])
        torch.cuda.synchronize()

    def _prime(self, slots, mode: int):
        """One throw-away iteration on scratch parameters before the first spin
        kernel or graph capture: every kernel of an iteration gets loaded (a lazily
        loaded module must never be needed while a spinning kernel owns SMs)."""
        if self._primed:
            return
        torch = self.torch
        p = self.model.params.clone()
        v = torch.zeros_like(p)
        pb = self.model.params_op.clone()
        # scratch first: the worker streams must see it initialised (they wait on `cur` below)
        st_scratch = torch.zeros(2 * self.n, dtype=torch.int64, device=self.dev)
        sec_scratch = torch.zeros(self.n, dtype=torch.float64, device=self.dev)
        it_scratch = torch.zeros(1, dtype=torch.int64, device=self.dev)
        cur = torch.cuda.current_stream()
        self.agg.wait_stream(cur)
        for wk in self.workers:
            wk.stream.wait_stream(cur)
        saved = [(slots[w].loss, slots[w].stamps, slots[w].seconds) for w in range(self.n)]
        for w in range(self.n):
            slots[w].loss = None
            slots[w].stamps = st_scratch[2 * w:].data_ptr()
            slots[w].seconds = sec_scratch.data_ptr()
        # device-indexed (d_iter) whenever graphs will run: the iteration-index kernels (iter_increment,
        # MLP row staging) must be loaded too
        self._run_iters(slots, 0, 1, mode, 0.0, 0.0, p, v, pb, 0,
                        it_scratch if (self.graphs or self.worker_graphs) else None)
        # (the update kernel advances the counter itself; the stand-alone increment other
        # paths launch -- multi-GPU, skip_update -- is loaded here too)
        _lib.check(_lib.lib().dbs_dev_iter_increment(it_scratch.data_ptr(), _lib.stream_handle()), "iter_increment")
        for w in range(self.n):
            slots[w].loss, slots[w].stamps, slots[w].seconds = saved[w]
        torch.cuda.synchronize()
        self._primed = True

    def _graph(self, key, k, slots, mode, lr, mom, skip):
        """(graph of k iterations, kernels per replay, kernels recorded by a fresh
        capture now).  Captured without a device-wide synchronisation (the queued
        permutation / repack keeps running while the host records), thread-local
        capture mode; every kernel reads the iteration index from d_iter, so one
        graph of k iterations serves any k consecutive iterations of the plan."""
        hit = self._graph_cache.get((key, k))
        if hit is not None:
            return hit[0], hit[1], 0
        torch = self.torch
        g = torch.cuda.CUDAGraph()
        c0 = _lib.lib().dbs_launch_count()
        with torch.cuda.stream(self.agg):
            g.capture_begin(capture_error_mode="thread_local")
            try:
                self._run_iters(slots, 0, k, mode, lr, mom, self.model.params, self.model.velocity,
                                self.model.params_op, skip, self.d_iter)
            finally:
                g.capture_end()
        per = _lib.lib().dbs_launch_count() - c0
        self._graph_cache[(key, k)] = (g, per)
        return g, per, per

    def _worker_graphs(self, key):
        """The per-worker graph set of a plan (captured by the library on first use);
        the last few plans' sets are kept, older ones released after the epoch's final
        synchronisation (never here: a disturbance spin kernel may be running, and a
        device-wide sync would wait for it forever)."""
        hit = self._wg_cache.pop(key, None)
        if hit is None:
            h = ctypes.c_void_p()
            _lib.check(_lib.lib().dbs_worker_graphs_create(self.n, ctypes.byref(h)), "worker_graphs_create")
            hit = h
        self._wg_cache[key] = hit  # most recent last
        while len(self._wg_cache) > 8:
            self._wg_retired.append(self._wg_cache.pop(next(iter(self._wg_cache))))
        return hit

    def _release_retired_graphs(self):
        """After a device-wide sync: the evicted graph sets are no longer in flight."""
        while self._wg_retired:
            _lib.lib().dbs_worker_graphs_destroy(self._wg_retired.pop())
        while self._eg_retired:
            _lib.lib().dbs_epoch_graph_destroy(self._eg_retired.pop())

    def _epoch_graph(self, key, slots, mode, lr, mom, skip):
        """The device-side epoch loop of a plan (dbs_epoch_graph_create: the iteration
        captured once into a `while` conditional node), or None when the driver cannot
        build one (the iteration graphs below are used instead)."""
        hit = self._eg_cache.pop(key, None)
        if hit is None:
            h = ctypes.c_void_p()
            st = _lib.lib().dbs_epoch_graph_create(slots, self.n, mode, float(lr), float(mom),
                                                   self.model.params.data_ptr(), self.model.velocity.data_ptr(),
                                                   self.model.params_op.data_ptr(), int(skip),
                                                   int(self.agg.cuda_stream), self.d_iter.data_ptr(),
                                                   self.d_total.data_ptr(), ctypes.byref(h))
            if st != 0:
                import warnings

                warnings.warn(f"device-side epoch loop unavailable ({_lib.last_error()}); using iteration graphs")
                self.epoch_graphs = False
                return None
            hit = h
        self._eg_cache[key] = hit
        while len(self._eg_cache) > 8:
            self._eg_retired.append(self._eg_cache.pop(next(iter(self._eg_cache))))
        return hit

    # -- the epoch loop -----------------------------------------------------------
    def run(self, config: StrategyConfig, n_epochs: int, lr: float = 0.05, momentum: float = 0.5,
            aggregation: str = "batch_weighted", profiles: Optional[Sequence[WorkerProfile]] = None,
            seed: int = 0, record_loss: bool = True, max_iters: Optional[int] = None,
            skip_update: bool = False, timed_from: Optional[int] = None,
            epoch_hook: Optional[Callable[[int], None]] = None,
            averaging_interval: Optional[int] = None, plan_source=None) -> RunResult:
        """Train n_epochs under `config`.  plan_source (a sequence of PartitionPlans),
        when given, replaces the re-plan: epoch e runs plan_source[min(e, len - 1)],
        the plan-list form of run_parallel_sgd's plan source (sgdlab.py:320-340).  epoch_hook(epoch), when given, runs at the
        start of every epoch inside the timed region (e.g. a host->device upload of
        that epoch's data, for end-to-end measurements).

        Synchronisation: S-SGD (aggregated gradient, one shared model) for
        "fixed_ssgd" / "dbs"; periodic model averaging (local SGD on per-worker
        replicas, averaged every `sync_interval` iterations) for "model_averaging",
        and a single average at the end of the run for "one_shot"
        (cluster.sync_rounds_for_epoch, cluster.py:173-189).  averaging_interval=k
        applies model averaging every k iterations on top of any plan kind -- with
        "dbs" that is the DBS model-averaging variant (BASELINE config 4)."""
        torch = self.torch
        local_interval = averaging_interval
        if local_interval is None and config.kind == "model_averaging":
            local_interval = config.sync_interval
        if local_interval is None and config.kind == "one_shot":
            local_interval = 1 << 30
        if local_interval is not None and local_interval < 1:
            raise ConfigurationError("averaging_interval must be >= 1")
        local = local_interval is not None and not skip_update
        if local:
            self._replicas_begin(mode=_MODE[aggregation])
        n, D = self.n, self.D
        self.rng = DeviceRng(seed, self.dev)
        # device-resident re-plan (no host controller round trip) unless a plan list is given
        planner = DevicePlanner(torch, self.dev, n, config, D) if plan_source is None else None
        next_secs = None
        if planner is not None:
            self.seconds.zero_()
            planner.enqueue(0, self.seconds, _lib.stream_handle())
            torch.cuda.synchronize()
        if record_loss and (getattr(self, "_loss_host", None) is None or self._loss_host.shape != self.loss_buf.shape):
            self._loss_host = torch.zeros(self.loss_buf.shape, dtype=torch.float32, pin_memory=True)
        stats: list = []
        smoothed = None
        losses, plans = [], []
        samples, wall, done = 0, 0.0, 0
        mode = _MODE[aggregation]
        t_start = t_end = None
        timed_samples = timed_launches = timed_host_launches = 0
        for epoch in range(n_epochs):
            if timed_from is not None and epoch == timed_from:
                torch.cuda.synchronize()
                t_start = torch.cuda.Event(enable_timing=True)
                t_start.record()
            timing = timed_from is not None and epoch >= timed_from
            if epoch_hook is not None:
                epoch_hook(epoch)
            launches0 = _lib.lib().dbs_launch_count()
            host0 = _lib.lib().dbs_host_launch_count()
            replays = 0
            captured = 0
            if plan_source is not None:
                plan = plan_source[min(epoch, len(plan_source) - 1)]
            else:
                plan = planner.result(epoch)
            plans.append(plan)
            batches = list(plan.int_batches)
            spans = list(plan.sample_spans)
            iters = cluster.iterations_for_plan(plan)
            if max_iters is not None:
                iters = min(iters, max_iters - done)
            # sample assignment (device) and the per-worker shard repack
            if planner is not None:
                perm, _ = self.rng.permute_spans(planner.current_spans(), total=D)
            else:
                perm, _ = self.rng.permute_spans(spans)
            offs = np.cumsum([0] + [e - s for s, e in spans[:-1]])
            s_main = _lib.stream_handle()
            slots = (_lib.WorkerSlot * n)()
            for w in range(n):
                rows = iters * batches[w]
                idx = perm[int(offs[w]):int(offs[w]) + rows]
                xs, ys = self.shard_x[w], self.shard_y[w]
                if rows:
                    if self.kind == MODEL_MLP:
                        st = self._gather_mlp(idx, rows, xs, s_main)
                    else:
                        st = _lib.lib().dbs_dev_gather_rows(self.X.data_ptr(), idx.data_ptr(), rows,
                                                            self.row_bytes, xs.data_ptr(), s_main)
                    _lib.check(st, "gather")
                    _lib.check(_lib.lib().dbs_dev_gather_i32(self.y.data_ptr(), idx.data_ptr(), rows, ys.data_ptr(),
                                                              s_main), "gather labels")
                sc = self._scratch(w, batches[w])
                sl = slots[w]
                sl.model = sc.handle.value
                sl.model_kind = self.kind
                sl.stream = int(self.workers[w].stream.cuda_stream)
                sl.x_shard = xs.data_ptr()
                sl.y_shard = ys.data_ptr()
                sl.batch = batches[w]
                sl.grad = self.grads[w].data_ptr()
                sl.loss = self.loss_buf[w].data_ptr() if record_loss else None
                sl.loss_scratch = self.loss_scratch[w:].data_ptr()
                sl.stamps = self.stamps[w].data_ptr()
                sl.seconds = self.seconds.data_ptr()
                sl.worker_index = w
                sl.spin_ns, sl.spin_ctas = 0, 0
                sl.ctx = self.workers[w].ctx or None
            self.seconds.zero_()
            self.d_iter.zero_()
            _lib.check(_lib.lib().dbs_dev_set_flag(self.stop.data_ptr(), 0, s_main), "set_flag")
            # disturbances of this epoch
            spinning, spin_key = [], []
            emulate = bool(self.device_per_sample_ns) and not self.pin_sms
            # a worker's device slowdown this epoch: its effective per-sample cost
            # (cluster.py:123-130: base cost x active multipliers) relative to the
            # cheapest worker's base cost -- a scenario's cost spread (e.g. the
            # robustness scenario's _geometric_costs) and its disturbances alike
            base_min = min(p.base_cost for p in profiles) if profiles is not None else 1.0
            for w in range(n):
                prof = profiles[w] if profiles is not None else None
                m = cluster.effective_cost(prof, epoch) / base_min if prof is not None else 1.0
                wk = self.workers[w]
                pinned = 0
                if emulate:
                    # emulated device: m x b x the per-sample time, whatever the batch
                    slots[w].spin_ns = int(m * batches[w] * self.device_per_sample_ns)
                    slots[w].spin_ctas = 2
                    spin_key.append((w, slots[w].spin_ns))
                elif m > 1.0:
                    if self.pin_sms:
                        # a co-running job pins 1 - 1/m of the worker's SMs
                        ctas = int(round(wk.sm_count * (1.0 - 1.0 / m)))
                        ctas = max(0, min(ctas, wk.sm_count - 1))
                        if ctas:
                            spinning.append((wk, ctas))
                            pinned = ctas
                    else:
                        # simulated workers share the GPU's SMs: the slow worker's
                        # device is emulated as m x its own forward/backward time
                        slots[w].slow_scale = float(m - 1.0)
                        slots[w].slow_ctas = 8
                        spin_key.append((w, "x", float(m)))
                ev = prof.active_disturbance(epoch) if prof is not None else None
                if ev is not None and ev.extra_epoch_seconds:
                    # flat extra seconds (cluster.py:141-143), spread over the epoch's iterations
                    slots[w].spin_ns += int(ev.extra_epoch_seconds * 1e9 / max(iters, 1))
                    # in its own partition the spin occupies the worker's free SMs (one wave:
                    # the SMs a co-running pinning spin holds are not available to it); on a
                    # shared GPU a 2-CTA timed spin delays only this worker's stream
                    slots[w].spin_ctas = max(1, wk.sm_count - pinned) if wk.ctx else 2
                    spin_key.append((w, "+", slots[w].spin_ns))
            if iters > 0 and spinning and not self.worker_graphs and tuple(batches) != self._primed_batches:
                # eager launches behind a running spin: a new plan may select kernel
                # instantiations not loaded yet (lazy loading would wait behind the spin)
                self._primed = False
            if iters > 0 and (spinning or self.graphs):
                self._prime(slots, mode)
                self._primed_batches = tuple(batches)
            wg = None
            if self.worker_graphs and iters > 0 and not local:
                # capture this plan's per-worker graphs now, before any spin starts
                wg = self._worker_graphs((tuple(batches), tuple(spin_key), bool(record_loss)))
                _lib.check(_lib.lib().dbs_worker_graphs_capture(
                    slots, self.n, mode, float(lr), float(momentum), self.model.params.data_ptr(),
                    self.model.velocity.data_ptr(), self.model.params_op.data_ptr(), int(skip_update),
                    int(self.agg.cuda_stream), self.d_iter.data_ptr(), wg), "worker_graphs_capture")
            elif self.worker_graphs and iters > 0 and local:
                # local SGD: per-worker graphs over the replicas (their addresses are part of the key)
                if getattr(self, "_local_iters", None) is None or self._local_iters.numel() != n:
                    self._local_iters = torch.zeros(n, dtype=torch.int64, device=self.dev)
                self._local_iters.zero_()
                wg = self._worker_graphs(("local", tuple(batches), tuple(spin_key), bool(record_loss), float(lr),
                                          float(momentum), self._rep_ptrs[0][0]))
                _lib.check(_lib.lib().dbs_run_iterations_local_graphed(
                    slots, self.n, 0, 0, mode, float(lr), float(momentum), int(local_interval), self._rep_ptrs[0],
                    self._rep_ptrs[1], self._rep_ptrs[2], int(self.agg.cuda_stream), self._local_iters.data_ptr(),
                    wg, 1), "worker_graphs_capture (local)")
            graph = graph_r = None
            egraph = None
            per_replay = per_r = 0
            k_it = 1
            key = (tuple(batches), tuple(spin_key), mode, float(lr), float(momentum), bool(skip_update),
                   bool(record_loss))
            if (self.graphs and iters > 0 and not local and self.epoch_graphs and
                    ((key, 1) in self._graph_cache or key in self._eg_cache)):
                # a plan seen before: the device-side epoch loop (building one -- capture plus
                # instantiation of the conditional graph -- is not worth it for a plan that
                # may live one epoch, as DBS re-plans by a sample or two)
                egraph = self._epoch_graph(key, slots, mode, lr, momentum, skip_update)
                if egraph is not None:
                    self.d_total.fill_(iters)  # the loop's trip count (d_iter is 0)
            if self.graphs and iters > 0 and not local and egraph is None:
                key = (tuple(batches), tuple(spin_key), mode, float(lr), float(momentum), bool(skip_update),
                       bool(record_loss))
                # a plan seen before gets k-iteration graphs; a new one (DBS re-plans move
                # batches by a sample or two from epoch to epoch) a one-iteration graph,
                # whose capture hides under the queued permutation and repack
                if (key, 1) in self._graph_cache:
                    k_it = min(iters, self.graph_iters)
                # graphs of k_it iterations (fewer dependent graph launches per epoch) + the remainder
                graph, per_replay, captured = self._graph(key, k_it, slots, mode, lr, momentum, skip_update)
                if iters % k_it:
                    graph_r, per_r, cap_r = self._graph(key, iters % k_it, slots, mode, lr, momentum, skip_update)
                    captured += cap_r
                self.d_iter.zero_()
            cur = torch.cuda.current_stream()
            for wk, ctas in spinning:
                wk.spin_stream.wait_stream(cur)
                _lib.check(_lib.lib().dbs_dev_spin_until_ctx(ctas, self.stop.data_ptr(), int(wk.spin_stream.cuda_stream),
                                                             wk.ctx or None), "spin")
            self.agg.wait_stream(cur)
            for wk in self.workers:
                wk.stream.wait_stream(cur)
            start = torch.cuda.Event(enable_timing=True)
            end = torch.cuda.Event(enable_timing=True)
            start.record(self.agg)
            if iters > 0:
                if egraph is not None:
                    _lib.check(_lib.lib().dbs_epoch_graph_launch(egraph, iters, int(self.agg.cuda_stream)),
                               "epoch_graph_launch")
                    replays = 0  # counted by the library
                elif graph is not None:
                    with torch.cuda.stream(self.agg):
                        for _ in range(iters // k_it):
                            graph.replay()
                        if graph_r is not None:
                            graph_r.replay()
                    replays = iters // k_it + (graph_r is not None)
                elif local and wg is not None:
                    st = _lib.lib().dbs_run_iterations_local_graphed(
                        slots, self.n, 0, iters, mode, float(lr), float(momentum), int(local_interval),
                        self._rep_ptrs[0], self._rep_ptrs[1], self._rep_ptrs[2], int(self.agg.cuda_stream),
                        self._local_iters.data_ptr(), wg, 0)
                    _lib.check(st, "run_iterations_local_graphed")
                elif local:
                    st = _lib.lib().dbs_run_iterations_local(slots, self.n, 0, iters, mode, float(lr), float(momentum),
                                                             int(local_interval), self._rep_ptrs[0], self._rep_ptrs[1],
                                                             self._rep_ptrs[2], int(self.agg.cuda_stream))
                    _lib.check(st, "run_iterations_local")
                elif wg is not None:
                    st = _lib.lib().dbs_run_iterations_graphed(
                        slots, self.n, 0, iters, mode, float(lr), float(momentum), self.model.params.data_ptr(),
                        self.model.velocity.data_ptr(), self.model.params_op.data_ptr(), int(skip_update),
                        int(self.agg.cuda_stream), self.d_iter.data_ptr(), wg)
                    _lib.check(st, "run_iterations_graphed")
                else:
                    self._run_iters(slots, 0, iters, mode, lr, momentum, self.model.params, self.model.velocity,
                                    self.model.params_op, skip_update)
            end.record(self.agg)
            # stop the disturbance once the epoch's work is done (copy engine, no kernel)
            _lib.check(_lib.lib().dbs_dev_set_flag(self.stop.data_ptr(), 1, int(self.agg.cuda_stream)), "set_flag")
            for wk, _ in spinning:
                self.agg.wait_stream(wk.spin_stream)
            cur.wait_stream(self.agg)
            last = epoch == n_epochs - 1 or (max_iters is not None and done + iters >= max_iters)
            if planner is not None:
                # the next epoch's plan from this epoch's measured seconds, on the device;
                # the read-back carries the seconds too (the only host round trip)
                planner.enqueue(epoch + 1, self.seconds, _lib.stream_handle(), plan=not last)
            if record_loss and iters > 0:
                self._loss_host[:, :iters].copy_(self.loss_buf[:, :iters], non_blocking=True)
            torch.cuda.synchronize()
            self._release_retired_graphs()
            ep_wall = start.elapsed_time(end) / 1e3
            if planner is not None:
                secs = planner.seconds()
            else:
                secs = tuple(float(x) for x in self.seconds.cpu().tolist())
            slowest = max(secs) if secs else 0.0
            stats.append(EpochStats(epoch=epoch, per_worker_gpu=secs, per_worker_wait=tuple(slowest - s for s in secs),
                                    sync_time=max(0.0, ep_wall - slowest), epoch_wall_time=ep_wall, plan=plan))
            if record_loss and iters > 0:
                lb = self._loss_host[:, :iters].double().numpy()
                bw = np.asarray(batches, dtype=np.float64)[:, None]
                losses.append((lb * bw).sum(axis=0) / bw.sum())
            samples += iters * sum(batches)
            wall += ep_wall
            done += iters
            if timing:
                timed_samples += iters * sum(batches)
                timed_launches += (_lib.lib().dbs_launch_count() - launches0 - captured
                                   + (per_replay * (iters // k_it) + per_r if graph is not None else 0))
                timed_host_launches += _lib.lib().dbs_host_launch_count() - host0 + replays
            if max_iters is not None and done >= max_iters:
                break
        timed = 0.0
        if t_start is not None:
            t_end = torch.cuda.Event(enable_timing=True)
            t_end.record()
            torch.cuda.synchronize()
            timed = t_start.elapsed_time(t_end) / 1e3
        if local:
            self._replicas_end(final_average=(config.kind == "one_shot"),
                               batches=list(plans[-1].int_batches) if plans else None)
        return RunResult(stats=stats, losses=np.concatenate(losses) if losses else np.zeros(0), samples=samples,
                         wall_seconds=wall, plans=plans, timed_seconds=timed, timed_samples=timed_samples,
                         timed_launches=timed_launches, timed_host_launches=timed_host_launches)


# ---------------------------------------------------------------------------
# one process per GPU: the same workers, plus the fused NVLink all-reduce
# ---------------------------------------------------------------------------

def gather_worker_times(local_secs, group=None) -> list:
    """All ranks learn every worker's measured compute time (Alg. 2 step 1,
    PAPER.md:115): rank-major order, so every rank runs the identical
    (deterministic, bit-exact) controller on the same inputs."""
    from .comm import gather_times

    out = []
    for r_times in _gather_lists(list(local_secs), group):
        out.extend(r_times)
    return out


def _gather_lists(values: list, group=None) -> list:
    import torch.distributed as dist

    got = [None] * dist.get_world_size(group)
    dist.all_gather_object(got, [float(v) for v in values], group=group)
    return got


def distributed_plan(config, epoch, n_global, D, prev_stats, smoothed, planner=None):
    """cluster.run_training's re-plan (cluster.py:253-271) on the gathered times."""
    planner = planner or cluster.next_plan
    return planner(config, epoch, n_global, D, prev_stats, smoothed)


class DistributedTrainer(SimulatedTrainer):
    """Synchronous DBS S-SGD across GPUs (one process per GPU, torchrun).

    Each rank hosts ``workers_per_rank`` workers (SM partitions of its GPU, or the
    whole GPU for one worker); the global plan covers world * workers_per_rank
    workers.  Per iteration: local forward/backward, local weighted reduce, then
    the fused NVLink weighted all-reduce + momentum SGD (comm.cu) -- the only
    data-path exchange.  The dataset is generated identically on every rank
    (device RNG) so a rank repacks its own spans locally.
    """

    def __init__(self, D_per_rank: int, workers_per_rank: int = 1, model: str = "resnet18", classes: int = 10,
                 seed: int = 0, partition: Optional[bool] = None, max_batch: Optional[int] = None, group=None,
                 image: int = 224, precision="f32"):
        import torch
        import torch.distributed as dist

        from .comm import Communicator

        self.group = group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        dev = torch.device("cuda", torch.cuda.current_device())
        D = D_per_rank * self.world
        g = torch.Generator(device=dev).manual_seed(seed + 1234)
        if model == "resnet18":
            X = torch.randn((D, 3, 32, 32), generator=g, device=dev)
        elif model == "resnet50":
            X = torch.randint(0, 256, (D, 3, image, image), generator=g, device=dev, dtype=torch.uint8)
        else:
            X = torch.randn((D, 784), generator=g, device=dev)
        y = torch.randint(0, classes, (D,), generator=g, device=dev, dtype=torch.int32)
        part = (workers_per_rank > 1) if partition is None else partition
        super().__init__(X, y, workers_per_rank, model=model, classes=classes, seed=seed, partition=part,
                         max_batch=max_batch, graphs=False, pin_sms=True, precision=precision)
        P = self.model.P
        self.comm = Communicator.create(P, group)
        # the communicator pads P to a multiple of 32 * world: the model's P elements are its prefix
        self.comm.params.zero_()
        self.comm.params[:P].copy_(self.model.params)
        if self.precision == _lib.PREC_F32:
            # S32 operand copy kept locally, refreshed after every update (comm.cu pushes fp32 only)
            self.comm_shadow = torch.zeros(2 * self.comm.P, dtype=torch.float32, device=self.dev)
            _lib.refresh_shadow(self.comm.params, self.comm_shadow, self.precision)
            self.comm.set_shadow(self.comm_shadow, self.precision)
            shadow = self.comm_shadow[:2 * P]
        else:
            self.comm.params_bf16.copy_(self.comm.params.to(torch.bfloat16))
            shadow = self.comm.params_bf16[:P]
        torch.cuda.synchronize()
        dist.barrier(group)
        # the model's tensors now alias the symmetric blocks (their unpadded prefix)
        self.model.params, self.model.params_op = self.comm.params[:P], shadow
        if workers_per_rank == 1:
            self.grads = [self.comm.grad[:P]]

    def run(self, config: StrategyConfig, n_epochs: int, lr: float = 0.05, momentum: float = 0.5,
            aggregation: str = "batch_weighted", profiles: Optional[Sequence[WorkerProfile]] = None,
            seed: int = 0, record_loss: bool = True, max_iters: Optional[int] = None,
            skip_update: bool = False, timed_from: Optional[int] = None,
            epoch_hook: Optional[Callable[[int], None]] = None,
            averaging_interval: Optional[int] = None) -> RunResult:
        """S-SGD across GPUs (fused NVLink all-reduce + SGD every iteration), or --
        for "model_averaging" / "one_shot" / averaging_interval=k -- local SGD on
        per-worker replicas with a global batch-weighted parameter average every k
        iterations (local average, then the NVLink average across ranks)."""
        import ctypes

        import torch

        from .comm import max_over_ranks

        local_interval = averaging_interval
        if local_interval is None and config.kind == "model_averaging":
            local_interval = config.sync_interval
        if local_interval is None and config.kind == "one_shot":
            local_interval = 1 << 30
        if local_interval is not None and local_interval < 1:
            raise ConfigurationError("averaging_interval must be >= 1")
        local = local_interval is not None and not skip_update
        if local:
            # replica 0 IS the symmetric parameter block the cross-rank average runs on
            Pm = self.model.P
            self._rep_p = [self.comm.params] + [self.comm.params.clone() for _ in range(self.n - 1)]
            self._rep_pb = [self.model.params_op] + [self.model.params_op.clone() for _ in range(self.n - 1)]
            self._rep_v = [torch.zeros(Pm, dtype=torch.float32, device=self.dev) for _ in range(self.n)]
            arr = lambda ts: (ctypes.c_void_p * self.n)(*[t.data_ptr() for t in ts])
            rep_ptrs = (arr(self._rep_p), arr(self._rep_v), arr(self._rep_pb))

        n_loc, W, R = self.n, self.n * self.world, self.rank
        D = self.D
        self.rng = DeviceRng(seed, self.dev)
        stats, losses, plans = [], [], []
        smoothed = None
        samples = done = 0
        wall = 0.0
        mode = _MODE[aggregation]
        t_start = None
        timed_samples = timed_launches = 0
        for epoch in range(n_epochs):
            if timed_from is not None and epoch == timed_from:
                torch.cuda.synchronize()
                torch.distributed.barrier(self.group)
                t_start = torch.cuda.Event(enable_timing=True)
                t_start.record()
            if epoch_hook is not None:
                epoch_hook(epoch)
            launches0 = _lib.lib().dbs_launch_count()
            plan, smoothed = distributed_plan(config, epoch, W, D, stats[-1] if stats else None, smoothed)
            plans.append(plan)
            batches = list(plan.int_batches)
            spans = list(plan.sample_spans)
            iters = cluster.iterations_for_plan(plan)
            if max_iters is not None:
                iters = min(iters, max_iters - done)
            perm, _ = self.rng.permute_spans(spans)
            offs = np.cumsum([0] + [e - s for s, e in spans[:-1]])
            s_main = _lib.stream_handle()
            slots = (_lib.WorkerSlot * n_loc)()
            for w in range(n_loc):
                gw = R * n_loc + w
                rows = iters * batches[gw]
                idx = perm[int(offs[gw]):int(offs[gw]) + rows]
                xs, ys = self.shard_x[w], self.shard_y[w]
                if rows:
                    if self.kind == MODEL_MLP:
                        st = self._gather_mlp(idx, rows, xs, s_main)
                    else:
                        st = _lib.lib().dbs_dev_gather_rows(self.X.data_ptr(), idx.data_ptr(), rows,
                                                            self.row_bytes, xs.data_ptr(), s_main)
                    _lib.check(st, "gather")
                    _lib.check(_lib.lib().dbs_dev_gather_i32(self.y.data_ptr(), idx.data_ptr(), rows, ys.data_ptr(),
                                                              s_main), "gather labels")
                sc = self._scratch(w, batches[gw])
                sl = slots[w]
                sl.model = sc.handle.value
                sl.model_kind = self.kind
                sl.stream = int(self.workers[w].stream.cuda_stream)
                sl.ctx = self.workers[w].ctx or None
                sl.x_shard, sl.y_shard = xs.data_ptr(), ys.data_ptr()
                sl.batch = batches[gw]
                sl.grad = self.grads[w].data_ptr()
                sl.loss = self.loss_buf[w].data_ptr() if record_loss else None
                sl.loss_scratch = self.loss_scratch[w:].data_ptr()
                sl.stamps = self.stamps[w].data_ptr()
                sl.seconds = self.seconds.data_ptr()
                sl.worker_index = w
            self.seconds.zero_()
            _lib.check(_lib.lib().dbs_dev_set_flag(self.stop.data_ptr(), 0, s_main), "set_flag")
            spinning = []
            if profiles is not None:
                for w in range(n_loc):
                    ev = profiles[R * n_loc + w].active_disturbance(epoch)
                    if ev is not None and ev.cost_multiplier is not None and ev.cost_multiplier > 1.0:
                        wk = self.workers[w]
                        ctas = max(0, min(int(round(wk.sm_count * (1.0 - 1.0 / ev.cost_multiplier))), wk.sm_count - 1))
                        if ctas:
                            spinning.append((wk, ctas))
                    elif ev is not None and ev.extra_epoch_seconds:
                        slots[w].spin_ns = int(ev.extra_epoch_seconds * 1e9 / max(iters, 1))
                        # own partition: the whole partition; shared GPU: a 2-CTA timed spin that
                        # delays only this worker's stream
                        slots[w].spin_ctas = self.workers[w].sm_count if self.workers[w].ctx else 2
            rank_batches = np.asarray([sum(batches[r * n_loc:(r + 1) * n_loc]) for r in range(self.world)],
                                      dtype=np.int64)
            if iters > 0:
                # a new plan: load its kernels before the spin starts -- decided on the GLOBAL
                # plan (identical on every rank), since the prime runs the collective kernel
                any_spin = profiles is not None and any(
                    (lambda ev: ev is not None and ev.cost_multiplier is not None and ev.cost_multiplier > 1.0)(
                        p.active_disturbance(epoch)) for p in profiles)
                if any_spin and tuple(batches) != self._primed_batches:
                    self._primed = False
                self._prime_comm(slots, mode, rank_batches)
                self._primed_batches = tuple(batches)
            wg = None
            if self.worker_graphs and iters > 0 and not local:
                # this plan's per-worker graphs, captured before any spin starts
                self.d_iter.zero_()
                wg = self._worker_graphs(("comm", tuple(batches), tuple((w, slots[w].spin_ns) for w in range(n_loc)),
                                          bool(record_loss)))
                _lib.check(_lib.lib().dbs_run_iterations_comm_graphed(
                    slots, n_loc, 0, 0, mode, float(lr), float(momentum), self.comm.h,
                    rank_batches.ctypes.data_as(_lib.P_i64), self.comm.velocity.data_ptr(), int(self.agg.cuda_stream),
                    self.d_iter.data_ptr(), wg, 1), "worker_graphs_capture (comm)")
            cur = torch.cuda.current_stream()
            for wk, ctas in spinning:
                wk.spin_stream.wait_stream(cur)
                _lib.check(_lib.lib().dbs_dev_spin_until_ctx(ctas, self.stop.data_ptr(), int(wk.spin_stream.cuda_stream),
                                                             wk.ctx or None), "spin")
            self.agg.wait_stream(cur)
            for wk in self.workers:
                wk.stream.wait_stream(cur)
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record(self.agg)
            if iters > 0 and local:
                st = _lib.lib().dbs_run_iterations_local_comm(
                    slots, n_loc, 0, iters, mode, float(lr), float(momentum), int(local_interval), rep_ptrs[0],
                    rep_ptrs[1], rep_ptrs[2], self.comm.h, rank_batches.ctypes.data_as(_lib.P_i64),
                    int(self.agg.cuda_stream))
                _lib.check(st, "run_iterations_local_comm")
            elif iters > 0 and wg is not None:
                st = _lib.lib().dbs_run_iterations_comm_graphed(
                    slots, n_loc, 0, iters, mode, float(lr), float(momentum), self.comm.h,
                    rank_batches.ctypes.data_as(_lib.P_i64), self.comm.velocity.data_ptr(), int(self.agg.cuda_stream),
                    self.d_iter.data_ptr(), wg, 0)
                _lib.check(st, "run_iterations_comm_graphed")
            elif iters > 0:
                st = _lib.lib().dbs_run_iterations_comm(slots, n_loc, 0, iters, mode, float(lr), float(momentum),
                                                        self.comm.h, rank_batches.ctypes.data_as(_lib.P_i64),
                                                        self.comm.velocity.data_ptr(), int(self.agg.cuda_stream), None)
                _lib.check(st, "run_iterations_comm")
            end.record(self.agg)
            _lib.check(_lib.lib().dbs_dev_set_flag(self.stop.data_ptr(), 1, int(self.agg.cuda_stream)), "set_flag")
            for wk, _ in spinning:
                self.agg.wait_stream(wk.spin_stream)
            cur.wait_stream(self.agg)
            torch.cuda.synchronize()
            self._release_retired_graphs()
            ep_wall = max_over_ranks(start.elapsed_time(end) / 1e3, self.group)
            secs = tuple(gather_worker_times(self.seconds.cpu().tolist(), self.group))
            slowest = max(secs)
            stats.append(EpochStats(epoch=epoch, per_worker_gpu=secs, per_worker_wait=tuple(slowest - s for s in secs),
                                    sync_time=max(0.0, ep_wall - slowest), epoch_wall_time=ep_wall, plan=plan))
            if record_loss and iters > 0:
                lb = self.loss_buf[:, :iters].double().cpu().numpy()
                bw = np.asarray(batches[R * n_loc:(R + 1) * n_loc], dtype=np.float64)[:, None]
                losses.append((lb * bw).sum(axis=0) / bw.sum())
            samples += iters * sum(batches)
            wall += ep_wall
            done += iters
            if timed_from is not None and epoch >= timed_from:
                timed_samples += iters * sum(batches)
                timed_launches += _lib.lib().dbs_launch_count() - launches0
            if max_iters is not None and done >= max_iters:
                break
        timed = 0.0
        if t_start is not None:
            t_end = torch.cuda.Event(enable_timing=True)
            t_end.record()
            torch.cuda.synchronize()
            timed = max_over_ranks(t_start.elapsed_time(t_end) / 1e3, self.group)
        if local and config.kind == "one_shot" and plans:
            # the single averaging round of one-shot averaging (cluster.py:187-188)
            last = list(plans[-1].int_batches)
            b_loc = np.asarray(last[R * n_loc:(R + 1) * n_loc], dtype=np.int64)
            _lib.check(_lib.lib().dbs_dev_average_replicas_f32_ex(rep_ptrs[0], b_loc.ctypes.data_as(_lib.P_i64),
                                                                  n_loc, mode, self.model.P, rep_ptrs[2],
                                                                  self.precision, int(self.agg.cuda_stream)),
                       "average_replicas")
            rb = np.asarray([sum(last[r * n_loc:(r + 1) * n_loc]) for r in range(self.world)], dtype=np.int64)
            self.comm.average_params(rb, mode=mode, stream=self.agg)
            if self.precision == _lib.PREC_F32:
                _lib.refresh_shadow(self.model.params, self.model.params_op, self.precision, stream=self.agg)
            torch.cuda.synchronize()
        return RunResult(stats=stats, losses=np.concatenate(losses) if losses else np.zeros(0), samples=samples,
                         wall_seconds=wall, plans=plans, timed_seconds=timed, timed_samples=timed_samples,
                         timed_launches=timed_launches)

    def _prime_comm(self, slots, mode, rank_batches):
        """Load every kernel of an iteration (local workers, local reduce, the fused
        NVLink kernel) before any spin kernel runs: a lazily loaded module must
        never be needed while a spinning kernel owns SMs.  The all-reduce runs
        with lr = 0, so the parameters are untouched; the velocity is reset."""
        if self._primed:
            return
        import ctypes

        import torch

        self._prime(slots, mode)
        self._primed = True
        if self.n > 1:
            ptrs = (ctypes.c_void_p * self.n)(*[g.data_ptr() for g in self.grads])
            b = np.asarray([slots[w].batch for w in range(self.n)], dtype=np.int64)
            _lib.check(_lib.lib().dbs_dev_aggregate_f32(ptrs, b.ctypes.data_as(_lib.P_i64), self.n, mode,
                                                        self.model.P, self.comm.grad.data_ptr(),
                                                        _lib.stream_handle()), "aggregate_f32")
        self.comm.allreduce_sgd(rank_batches, 0.0, 0.0, mode=mode)
        # the model-averaging round's kernels too (identical parameters on every rank: no change)
        self.comm.average_params(rank_batches, mode=mode)
        ptr1 = (ctypes.c_void_p * 1)(self.model.params.data_ptr())
        ptrb = (ctypes.c_void_p * 1)(self.model.params_op.data_ptr())
        one = np.ones(1, dtype=np.int64)
        _lib.check(_lib.lib().dbs_dev_average_replicas_f32_ex(ptr1, one.ctypes.data_as(_lib.P_i64), 1, mode,
                                                              self.model.P, ptrb, self.precision, _lib.stream_handle()),
                   "average_replicas")
        if self.precision == _lib.PREC_F32:
            _lib.refresh_shadow(self.model.params, self.model.params_op, self.precision)
        torch.cuda.synchronize()
        self.comm.velocity.zero_()
        torch.distributed.barrier(self.group)
