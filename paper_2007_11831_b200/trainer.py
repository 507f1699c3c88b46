"""Measured DBS vs fixed-batch synchronous training on B200s.

This is the GPU counterpart of cluster.run_training (cluster.py:234-275): the
same epoch loop and the same re-plan (cluster.next_plan -> the device
controller), but `per_worker_gpu` is MEASURED -- per-worker compute seconds
accumulated on the device from %globaltimer stamps around each worker's
forward/backward -- and the epoch wall time is a CUDA-event interval.  The
records are the reference's EpochStats (cluster.py:111-120), so
cumulative_times / the report schema apply unchanged.

Workers
  * one process, W simulated workers (config 1): each worker is a CUDA stream,
    optionally confined to its own SM partition with a green context;
  * one process per GPU (torchrun): worker = rank, gradients combined by the
    fused NVLink kernel of comm.py (see DistributedTrainer).

Disturbance (DisturbanceEvent, cluster.py:25-56), realised on the device:
  * cost_multiplier m  -> a co-running spin kernel pins a fraction 1 - 1/m of
                          the worker's SMs for the whole epoch;
  * extra_epoch_seconds -> a timed spin on the worker's stream, spread over the
                          epoch's iterations (counted in its compute time, as
                          in epoch_gpu_time cluster.py:132-145).
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib, cluster
from .allocation import PartitionPlan
from .cluster import EpochStats, StrategyConfig, WorkerProfile
from .mlp import MlpModel, MlpScratch
from .sgdlab import DeviceRng

_MODE = {"uniform_average": 0, "batch_weighted": 1}


@dataclass
class Worker:
    index: int
    stream: object
    spin_stream: object
    sm_count: int
    green: object = None


def make_workers(n: int, partition: bool = True) -> list[Worker]:
    """W simulated workers on the current device; SM partitions via green contexts."""
    import torch

    dev = torch.cuda.current_device()
    total = torch.cuda.get_device_properties(dev).multi_processor_count
    workers = []
    use_green = partition and n > 1 and _green_supported()
    per = max(8, (total // n) // 8 * 8) if use_green else total
    for i in range(n):
        if use_green:
            g = torch.cuda.green_contexts.GreenContext.create(per, dev)
            s = g.Stream()
            g.set_context()
            try:
                spin = torch.cuda.Stream()
            finally:
                g.pop_context()
            workers.append(Worker(i, s, spin, per, g))
        else:
            workers.append(Worker(i, torch.cuda.Stream(), torch.cuda.Stream(), total, None))
    return workers


def _green_supported() -> bool:
    try:
        import torch

        return bool(torch.cuda.green_contexts.SUPPORTED)
    except Exception:
        return False


@dataclass
class RunResult:
    stats: list
    losses: np.ndarray          # per-iteration batch-weighted mean loss
    samples: int                # samples processed (sum over epochs of T * sum b)
    wall_seconds: float         # sum of epoch wall times (device events)
    plans: list = field(default_factory=list)


class SimulatedTrainer:
    """W simulated workers of synchronous S-SGD on one GPU (config 1)."""

    def __init__(self, X, y, n_workers: int, hidden: int = 256, classes: int = 10, seed: int = 0,
                 partition: bool = True, params=None, max_batch: Optional[int] = None):
        import torch

        _lib.require_device()
        self.torch = torch
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.X = torch.as_tensor(X, device=self.dev) if not isinstance(X, torch.Tensor) else X.to(self.dev)
        self.y = torch.as_tensor(y, device=self.dev) if not isinstance(y, torch.Tensor) else y.to(self.dev)
        self.X = self.X.to(torch.float32).contiguous()
        self.y = self.y.to(torch.int32).contiguous()
        self.D, self.in_dim = self.X.shape
        self.n = n_workers
        self.model = MlpModel(self.in_dim, hidden, classes, seed, self.dev, params=params)
        self.workers = make_workers(n_workers, partition)
        self.max_batch = max_batch
        self.scratch = {}
        self.grads = [torch.zeros(self.model.P, dtype=torch.float32, device=self.dev) for _ in range(n_workers)]
        self.seconds = torch.zeros(n_workers, dtype=torch.float64, device=self.dev)
        self.stamps = [torch.zeros(2, dtype=torch.int64, device=self.dev) for _ in range(n_workers)]
        self.loss_scratch = torch.zeros(n_workers, dtype=torch.float32, device=self.dev)
        self.stop = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.agg = torch.cuda.Stream()
        self.rng = None

    def _scratch(self, w: int, b: int) -> MlpScratch:
        cur = self.scratch.get(w)
        if cur is None or cur.max_batch < b:
            cap = max(b, self.max_batch or 0)
            cur = MlpScratch(self.model.layout, cap)
            self.scratch[w] = cur
        return cur

    def _prime(self, slots, iters: int, mode: int):
        """Run one throw-away iteration (scratch parameters) before a spin kernel
        starts, so every kernel of the epoch is resident: a lazily loaded module
        must never be needed while a spinning kernel owns SMs."""
        if getattr(self, "_primed", False) or iters <= 0:
            return
        torch = self.torch
        p = self.model.params.clone()
        v = torch.zeros_like(p)
        pb = self.model.params_bf16.clone()
        cur = torch.cuda.current_stream()
        self.agg.wait_stream(cur)
        for wk in self.workers:
            wk.stream.wait_stream(cur)
        saved = [(slots[w].loss, slots[w].stamps, slots[w].seconds) for w in range(self.n)]
        st_scratch = torch.zeros(2 * self.n, dtype=torch.int64, device=self.dev)
        sec_scratch = torch.zeros(self.n, dtype=torch.float64, device=self.dev)
        for w in range(self.n):
            # same kernel set as a real iteration (incl. the timing stamps), scratch outputs
            slots[w].loss = None
            slots[w].stamps = st_scratch[2 * w:].data_ptr()
            slots[w].seconds = sec_scratch.data_ptr()
        _lib.check(_lib.lib().dbs_mlp_run_iterations(slots, self.n, 0, 1, mode, 0.0, 0.0, p.data_ptr(), v.data_ptr(),
                                                      pb.data_ptr(), 0, int(self.agg.cuda_stream)), "prime")
        for w in range(self.n):
            slots[w].loss, slots[w].stamps, slots[w].seconds = saved[w]
        torch.cuda.synchronize()
        self._primed = True

    def run(self, config: StrategyConfig, n_epochs: int, lr: float = 0.05, momentum: float = 0.5,
            aggregation: str = "batch_weighted", profiles: Optional[Sequence[WorkerProfile]] = None,
            seed: int = 0, record_loss: bool = True, max_iters: Optional[int] = None,
            skip_update: bool = False) -> RunResult:
        torch = self.torch
        n, D = self.n, self.D
        self.rng = DeviceRng(seed, self.dev)
        stats: list[EpochStats] = []
        smoothed = None
        losses = []
        samples = 0
        wall = 0.0
        plans = []
        mode = _MODE[aggregation]
        done = 0
        for epoch in range(n_epochs):
            plan, smoothed = cluster.next_plan(config, epoch, n, D, stats[-1] if stats else None, smoothed)
            plans.append(plan)
            batches = list(plan.int_batches)
            spans = list(plan.sample_spans)
            iters = cluster.iterations_for_plan(plan)
            if max_iters is not None:
                iters = min(iters, max_iters - done)
            # sample assignment: device permutation of every span (sgdlab.py:372-374)
            perm, _ = self.rng.permute_spans(spans)
            # repartition gather: each worker's used rows, in epoch order, fp32 -> bf16
            slots = (_lib.WorkerSlot * n)()
            shards = []
            offs = np.cumsum([0] + [e - s for s, e in spans[:-1]])
            loss_buf = torch.zeros((n, max(iters, 1)), dtype=torch.float32, device=self.dev)
            s_main = _lib.stream_handle()
            for w in range(n):
                rows = iters * batches[w]
                xs = torch.empty((max(rows, 1), self.in_dim), dtype=torch.bfloat16, device=self.dev)
                ys = torch.empty(max(rows, 1), dtype=torch.int32, device=self.dev)
                idx = perm[int(offs[w]):int(offs[w]) + rows]
                if rows:
                    _lib.check(_lib.lib().dbs_dev_gather_rows_f32_bf16(self.X.data_ptr(), idx.data_ptr(), rows,
                                                                        self.in_dim, xs.data_ptr(), s_main), "gather")
                    _lib.check(_lib.lib().dbs_dev_gather_i32(self.y.data_ptr(), idx.data_ptr(), rows, ys.data_ptr(),
                                                              s_main), "gather labels")
                shards.append((xs, ys))
                sc = self._scratch(w, batches[w])
                sl = slots[w]
                sl.model = sc.handle.value
                sl.stream = int(self.workers[w].stream.cuda_stream)
                sl.x_shard = xs.data_ptr()
                sl.y_shard = ys.data_ptr()
                sl.batch = batches[w]
                sl.grad = self.grads[w].data_ptr()
                sl.loss = loss_buf[w].data_ptr() if record_loss else None
                sl.loss_scratch = self.loss_scratch[w:].data_ptr()
                sl.stamps = self.stamps[w].data_ptr()
                sl.seconds = self.seconds.data_ptr()
                sl.worker_index = w
                sl.spin_ns, sl.spin_ctas = 0, 0
            self.seconds.zero_()
            _lib.check(_lib.lib().dbs_dev_set_flag(self.stop.data_ptr(), 0, s_main), "set_flag")
            # disturbances of this epoch
            spinning = []
            if profiles is not None and any(p.active_disturbance(epoch) for p in profiles):
                self._prime(slots, iters, mode)
                for w, prof in enumerate(profiles):
                    ev = prof.active_disturbance(epoch)
                    if ev is None:
                        continue
                    wk = self.workers[w]
                    if ev.cost_multiplier is not None and ev.cost_multiplier > 1.0:
                        ctas = int(round(wk.sm_count * (1.0 - 1.0 / ev.cost_multiplier)))
                        ctas = max(0, min(ctas, wk.sm_count - 1))
                        if ctas:
                            wk.spin_stream.wait_stream(torch.cuda.current_stream())
                            _lib.check(_lib.lib().dbs_dev_spin_until(ctas, self.stop.data_ptr(),
                                                                     int(wk.spin_stream.cuda_stream)), "spin")
                            spinning.append(wk)
                    elif ev.extra_epoch_seconds:
                        slots[w].spin_ns = int(ev.extra_epoch_seconds * 1e9 / max(iters, 1))
                        slots[w].spin_ctas = wk.sm_count
            cur = torch.cuda.current_stream()
            self.agg.wait_stream(cur)
            for wk in self.workers:
                wk.stream.wait_stream(cur)
            start = torch.cuda.Event(enable_timing=True)
            end = torch.cuda.Event(enable_timing=True)
            start.record(self.agg)
            if iters > 0:
                st = _lib.lib().dbs_mlp_run_iterations(
                    slots, n, 0, iters, mode, float(lr), float(momentum), self.model.params.data_ptr(),
                    self.model.velocity.data_ptr(), self.model.params_bf16.data_ptr(), int(skip_update),
                    int(self.agg.cuda_stream))
                _lib.check(st, "mlp_run_iterations")
            end.record(self.agg)
            # stop the disturbance once the epoch's work is done (memset: no kernel launch)
            _lib.check(_lib.lib().dbs_dev_set_flag(self.stop.data_ptr(), 1, int(self.agg.cuda_stream)), "set_flag")
            for wk in spinning:
                self.agg.wait_stream(wk.spin_stream)
            cur.wait_stream(self.agg)
            torch.cuda.synchronize()
            ep_wall = start.elapsed_time(end) / 1e3
            secs = tuple(float(x) for x in self.seconds.cpu().tolist())
            slowest = max(secs) if secs else 0.0
            stat = EpochStats(epoch=epoch, per_worker_gpu=secs, per_worker_wait=tuple(slowest - s for s in secs),
                              sync_time=max(0.0, ep_wall - slowest), epoch_wall_time=ep_wall, plan=plan)
            stats.append(stat)
            if record_loss and iters > 0:
                lb = loss_buf[:, :iters].double().cpu().numpy()
                bw = np.asarray(batches, dtype=np.float64)[:, None]
                losses.append((lb * bw).sum(axis=0) / bw.sum())
            samples += iters * sum(batches)
            wall += ep_wall
            done += iters
            if max_iters is not None and done >= max_iters:
                break
        return RunResult(stats=stats, losses=np.concatenate(losses) if losses else np.zeros(0), samples=samples,
                         wall_seconds=wall, plans=plans)
