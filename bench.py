#!/usr/bin/env python
"""DBS benchmark: samples/s and epoch time under skewed load, DBS vs fixed batch.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload resnet18|mlp]

Prints ONE JSON line on rank 0.  Definitions ("Measurement"):
  * a "step" is one synchronous S-SGD EPOCH of the hot path: device controller
    re-plan -> device permutation of every span -> coalesced shard repack ->
    T iterations of per-worker variable-batch forward/backward on tcgen05 +
    fused batch-weighted aggregation / momentum SGD (CUDA-graph replays);
  * value = samples processed by all workers in the K timed epochs / device
    time of those K whole epochs (CUDA events, inputs resident in HBM);
  * e2e = the same through the public trainer API with the dataset uploaded
    from pinned host memory every epoch and the losses read back;
  * roofline of the dominant kernel (the tcgen05 implicit-GEMM convolution),
    cpu_baseline (the reference loop with a CPU model on the host cores),
    clocks sampled in-process with NVML during the timed region.
Workload at N=1 (config 3, BASELINE.json): ResNet-18 on synthetic CIFAR-shaped
data, 3 simulated workers = 3 disjoint 48-SM partitions (green contexts; 144 of the
148 SMs -- partitions come in multiples of 8 SMs) of the B200, B=510 (170/worker
fixed); worker 0 shares its partition with a co-running spin kernel that pins
half of its SMs (cost_multiplier 2, the paper's SM disturbance).  Under torchrun
every rank hosts the same workers on its own GPU, the global plan spans all
ranks' workers, and the gradients meet every iteration in the fused NVLink
all-reduce + SGD kernel (comm.cu); the epoch time is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "DBS samples/sec & epoch time under skewed load vs fixed batch"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--report", default=None,
                    help="directory for the reference-format run reports (epoch CSV per strategy + run JSON)")
    ap.add_argument("--workload", default="resnet18", choices=["resnet18", "resnet18_4w", "resnet18_ma", "resnet50", "resnet50_3w", "mlp", "allreduce"])
    ap.add_argument("--precision", default="f32", choices=["f32", "bf16"],
                    help="tensor-core arithmetic of the models: f32 = 3xTF32 on S32 operands (fp32 class, the "
                         "headline), bf16 = bf16 operands")
    ap.add_argument("--no-bf16", action="store_true", help="skip the labelled bf16 variant of the headline workload")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def bench_device(local, world):
    """One process per GPU.  DBS_BENCH_SHARE_GPU=1 (testing the multi-rank path on a
    one-GPU box only) maps every rank onto the visible devices round-robin."""
    import torch

    if world <= 1:
        return 0
    if os.environ.get("DBS_BENCH_SHARE_GPU") == "1":
        return local % torch.cuda.device_count()
    return local


def init_group():
    """Host-side process group (IPC handles, worker times, max over ranks): NCCL
    over NVLink; gloo when ranks share a GPU (NCCL refuses duplicate devices)."""
    import torch
    import torch.distributed as dist

    if os.environ.get("DBS_BENCH_SHARE_GPU") == "1":
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "bf16_tflops": d.get("bf16_tflops", 1590.0),
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", 1400.0), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """SM clock + throttle reasons sampled in-process (NVML) DURING the timed region."""

    def __init__(self, index=0):
        self.index, self.samples, self.power = index, [], []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            names = [("hw_slowdown", pynvml.nvmlClocksEventReasonHwSlowdown),
                     ("hw_thermal_slowdown", pynvml.nvmlClocksEventReasonHwThermalSlowdown),
                     ("sw_thermal_slowdown", pynvml.nvmlClocksEventReasonSwThermalSlowdown),
                     ("sw_power_cap", pynvml.nvmlClocksEventReasonSwPowerCap)]
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((sm, [n for n, b in names if r & b]))
                        try:
                            self.power.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1e3)
                        except Exception:
                            pass
                    except Exception:
                        pass
                    self._stop.wait(0.25)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception as exc:  # no NVML: record why
            self.error = repr(exc)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=5)
        sm = [s for s, _ in self.samples]
        reasons = sorted({r for _, rs in self.samples for r in rs})
        out = {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": getattr(self, "max_mhz", None),
               "reasons": reasons, "samples": len(sm)}
        if self.power:
            out["power_w"] = round(float(np.median(self.power)), 1)
        return out


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
WL = {
    "resnet18": dict(D=50000, workers=3, per_worker=170, lr=0.05, mom=0.9, mult=2.0,
                     desc="C3: ResNet-18 (CIFAR stem), synthetic CIFAR-10-shaped 50000x3x32x32 fp32, 3 simulated "
                          "workers = 3 disjoint 48-SM partitions (green contexts, 144 of the 148 SMs) of the B200, "
                          "B=510 (170/worker fixed), step = 1 epoch (98 iterations)"),
    "resnet18_4w": dict(D=50000, workers=4, per_worker=128, lr=0.05, mom=0.9, mult=2.0,
                        desc="C3 variant: ResNet-18 CIFAR, 4 simulated workers = 4 disjoint 32-SM partitions (128 of "
                             "148 SMs; partitions come in multiples of 8 SMs), B=512"),
    "resnet18_ma": dict(D=50000, workers=3, per_worker=170, lr=0.05, mom=0.9, mult=2.0, avg=4,
                        desc="C4: C3 with periodic model averaging (local SGD on per-worker replicas, averaged every "
                             "step=4 iterations), DBS vs fixed plan, step = 1 epoch"),
    "resnet50_3w": dict(D=12800, workers=3, per_worker=85, lr=0.05, mom=0.9, mult=None, image=224, classes=1000,
                        max_batch=200, cpu_per_worker=16, smoothing=0.7,
                        desc="C5 variant: ResNet-50 224, 3 simulated workers = 3 disjoint 48-SM partitions, B=255"),
    "resnet50": dict(D=12800, workers=4, per_worker=64, lr=0.05, mom=0.9, mult=None, image=224, classes=1000,
                     max_batch=160, cpu_per_worker=16, smoothing=0.7,
                     desc="C5: ResNet-50 (torchvision v1.5) on synthetic ImageNet-shaped 12800x3x224x224 uint8, 1000 "
                          "classes, 4 simulated workers = 4 disjoint 32-SM partitions (green contexts) of the B200, "
                          "B=256 (64/worker fixed), step = 1 epoch (50 iterations)"),
    "mlp": dict(D=60000, workers=3, per_worker=128, lr=0.05, mom=0.5, mult=2.0,
                desc="C1: MLP 784-256-10, synthetic MNIST 60000x784, 3 simulated workers sharing the GPU, B=384 "
                     "(128/worker fixed), step = 1 epoch (156 iterations)"),
}


def varying_multipliers(n_epochs=64, seed=2007):
    """Per-epoch SM fractions f ~ U(0.25, 0.6) stolen from workers 0 and 1
    (cost multiplier 1 / (1 - f)): persistent disturbed workers whose intensity
    changes every epoch."""
    rng = np.random.default_rng(seed)
    f = rng.uniform(0.25, 0.6, size=(2, n_epochs))
    return 1.0 / (1.0 - f)


def profiles(n, mult):
    from paper_2007_11831_b200 import cluster

    if mult is None:
        m = varying_multipliers()
        prof = [cluster.WorkerProfile(w, 1.0, disturbances=tuple(
            cluster.DisturbanceEvent(e, e + 1, cost_multiplier=float(m[w, e])) for e in range(m.shape[1])))
            for w in range(2)]
        return prof + [cluster.WorkerProfile(i, 1.0) for i in range(2, n)]
    # a persistent slow worker (rotating disturbances defeat the
    # one-epoch-lag estimator; persistent ones are what DBS absorbs)
    prof = [cluster.WorkerProfile(0, 1.0, disturbances=(cluster.DisturbanceEvent(0, cost_multiplier=mult),))]
    return prof + [cluster.WorkerProfile(i, 1.0) for i in range(1, n)]


PRECISION_DESC = {
    "f32": "fp32 class: 3xTF32 tcgen05 GEMMs on S32 (hi/lo tf32 split) operands, fp32 accumulation, fp32 "
           "parameters / BN / gradients",
    "bf16": "bf16 tensor-core operands, fp32 accumulation, fp32 master parameters",
}


def workload_config(wl, precision):
    """The config dict both arms print (same workload, same disturbance)."""
    w = WL[wl]
    cfg = {"workload": w["desc"], "disturbance": disturbance_desc(wl), "lr": w["lr"], "momentum": w["mom"],
           "parallelism": f"{w['workers']} simulated DP workers/GPU", "arithmetic": PRECISION_DESC[precision]}
    return cfg


def make_trainer(wl, rank, world=1, precision="f32"):
    import torch

    from paper_2007_11831_b200.trainer import DistributedTrainer, SimulatedTrainer

    w = WL[wl]
    if world > 1:
        # one process per GPU: the same SM-partition workers per GPU, the global
        # plan spans workers x world workers, gradients meet in the fused NVLink kernel
        model = "resnet50" if wl.startswith("resnet50") else ("resnet18" if wl.startswith("resnet18") else "mlp")
        tr = DistributedTrainer(w["D"], workers_per_rank=w["workers"], model=model, seed=0, partition=True,
                                max_batch=w.get("max_batch", 3 * w["per_worker"]), classes=w.get("classes", 10),
                                image=w.get("image", 224), precision=precision)
        return tr, (None, None)
    if wl.startswith("resnet50"):
        from paper_2007_11831_b200.resnet import synthetic_imagenet

        X, y = synthetic_imagenet(w["D"], w["image"], w["classes"], seed=rank, device=torch.device("cuda"))
        tr = SimulatedTrainer(X, y, n_workers=w["workers"], model="resnet50", classes=w["classes"], seed=0,
                              partition=True, max_batch=w["max_batch"], precision=precision)
        return tr, (X.cpu().numpy(), y.cpu().numpy())
    if wl.startswith("resnet18"):
        from paper_2007_11831_b200.resnet import synthetic_cifar

        X, y = synthetic_cifar(w["D"], seed=rank)
        return SimulatedTrainer(X, y, n_workers=w["workers"], model="resnet18", seed=0, partition=True,
                                max_batch=w["workers"] * w["per_worker"], precision=precision), (X, y)
    from paper_2007_11831_b200.mlp import synthetic_mnist

    X, y = synthetic_mnist(w["D"], seed=rank)
    tr = SimulatedTrainer(X, y, n_workers=w["workers"], model="mlp", seed=0,
                          max_batch=w["workers"] * w["per_worker"], precision=precision)
    calibrate_slow_device(tr, w)
    return tr, (X, y)


def calibrate_slow_device(tr, w):
    """C1's three workers share one GPU and the MLP's iteration is launch-latency bound
    (its time hardly depends on the batch), so the workers are emulated devices with
    the reference's cost law t = effective_cost x samples (cluster.py:123-145): every
    worker's iteration adds a timed spin of m_w x b_w x the per-sample time measured
    here on one undisturbed fixed-plan epoch (the median worker's compute seconds /
    (T b)), m_w = 2 for the disturbed worker -- so a worker's time follows the batch
    DBS assigns it, as on real devices."""
    from paper_2007_11831_b200 import cluster

    cfg = cluster.StrategyConfig("fixed_ssgd", w["workers"] * w["per_worker"])
    res = tr.run(cfg, n_epochs=2, lr=0.0, momentum=0.0, record_loss=False)
    st = res.stats[-1]
    iters = cluster.iterations_for_plan(st.plan)
    per = sorted(t / (iters * b) for t, b in zip(st.per_worker_gpu, st.plan.int_batches))
    tr.device_per_sample_ns = per[len(per) // 2] * 1e9
    tr.model.velocity.zero_()
    tr._graph_cache.clear()


def run_strategy(tr, wl, kind, args, world=1):
    import torch

    from paper_2007_11831_b200 import cluster

    w = WL[wl]
    n_global = w["workers"] * world
    # the reference's perf-smoothing EMA (cluster.py:263-266) for a disturbance
    # redrawn every epoch: the plan follows the mean speed, not last epoch's draw
    cfg = cluster.StrategyConfig(kind, n_global * w["per_worker"], perf_smoothing=w.get("smoothing", 0.0))
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    extra = {"averaging_interval": w["avg"]} if w.get("avg") else {}
    res = tr.run(cfg, n_epochs=args.warmup + args.steps, lr=w["lr"], momentum=w["mom"],
                 profiles=profiles(n_global, w["mult"]), record_loss=True, timed_from=args.warmup, **extra)
    clocks = sampler.stop()
    timed = res.stats[args.warmup:]
    return {"samples_per_s": res.timed_samples / res.timed_seconds, "epoch_s": res.timed_seconds / len(timed),
            "stats": timed, "clocks": clocks, "launches": res.timed_launches, "host_launches": res.timed_host_launches, "loss_last": float(res.losses[-1]),
            "samples": res.timed_samples, "seconds": res.timed_seconds}


TF32_DENSE_TFLOPS = 1100.0  # B200 dense tf32 tensor rate, B200_PROFILING.md (nominal, for context)


def measure_tf32_peak(reps=10):
    """Measured dense tf32 tensor rate of this GPU, the same recipe as the driver's bf16
    burst figure in MEASURED_PEAKS.json: a cuBLAS 8192^3 fp32 matmul with TF32 math
    (torch.backends.cuda.matmul.allow_tf32), best of `reps`, CUDA events.  Library code
    used only as the roofline denominator, never on the measured path."""
    import torch

    n = 8192
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        a = torch.randn(n, n, device="cuda")
        b = torch.randn(n, n, device="cuda")
        c = torch.empty(n, n, device="cuda")
        for _ in range(3):
            torch.matmul(a, b, out=c)
        torch.cuda.synchronize()
        best = None
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b, out=c)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            best = t if best is None or t < best else best
        del a, b, c
        torch.cuda.empty_cache()
        return 2.0 * n ** 3 / best / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev

ROOFLINE_CONV = {
    # workload -> (H, Cin, Cout, k, stride, description): the dominant conv shape
    "resnet18": (32, 64, 64, 3, 1, "3x3 64->64 @32x32"),
    "resnet50": (14, 256, 256, 3, 1, "3x3 256->256 @14x14 (layer 3 carries the most FLOPs)"),
}


def kernel_roofline(peaks, wl, precision, tr=None):
    """Dominant kernel: the tcgen05 implicit-GEMM convolution of the workload's most
    expensive conv shape, timed where the bench runs it -- inside worker 0's SM
    partition (green context; its SM count sizes the persistent grid) at the
    workload's per-worker batch -- with 100 launches on the partition's stream
    between CUDA events.  Peak: the measured bf16 dense rate, divided by 6 for the
    fp32-class kernel (kind::tf32 runs at half the bf16 rate and 3xTF32 issues
    three MMAs per product), scaled by the partition's share of the SMs."""
    import ctypes

    import torch

    from paper_2007_11831_b200 import _lib

    w = WL[wl]
    key = "resnet50" if wl.startswith("resnet50") else "resnet18"
    H, C, Co, k, stride, desc = ROOFLINE_CONV[key]
    N = w["per_worker"]
    pad = k // 2
    OH = (H + 2 * pad - k) // stride + 1
    f32 = precision == "f32"
    L = _lib.lib()
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(N * H * H, C, device="cuda", generator=g)
    wt = torch.randn(Co, k * k * C, device="cuda", generator=g) / (k * k * C) ** 0.5
    if f32:
        def s32(t):
            o = torch.empty(t.shape[0], 2 * t.shape[1], device="cuda")
            assert L.dbs_dev_split_s32(t.data_ptr(), t.shape[0], t.shape[1], t.shape[1], o.data_ptr(), t.shape[1],
                                       _lib.stream_handle()) == 0, _lib.last_error()
            return o

        xs, ws = s32(x), s32(wt)
        y = torch.empty(N * OH * OH, Co, device="cuda")
        fn = L.dbs_dev_conv2d_fwd_s32
    else:
        xs, ws = x.to(torch.bfloat16), wt.to(torch.bfloat16)
        y = torch.empty(N * OH * OH, Co, dtype=torch.bfloat16, device="cuda")
        fn = L.dbs_dev_conv2d_fwd
    wk = tr.workers[0] if tr is not None and tr.workers and tr.workers[0].ctx else None
    ctx = wk.ctx if wk else None
    stream = wk.stream if wk else torch.cuda.Stream()
    sms = wk.sm_count if wk else torch.cuda.get_device_properties(0).multi_processor_count
    torch.cuda.synchronize()
    if ctx:
        _lib.check(L.dbs_partition_push(ctx), "partition_push")
    try:
        h = int(stream.cuda_stream)

        def launch():
            st = fn(xs.data_ptr(), N, H, H, C, ws.data_ptr(), Co, k, stride, pad, y.data_ptr(), h)
            assert st == 0, _lib.last_error()

        for _ in range(10):
            launch()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 100
        e0.record(stream)
        for _ in range(reps):
            launch()
        e1.record(stream)
        torch.cuda.synchronize()
    finally:
        if ctx:
            _lib.check(L.dbs_partition_pop(ctx), "partition_pop")
    dur = e0.elapsed_time(e1) / 1e3 / reps
    flops = 2.0 * N * OH * OH * Co * k * k * C
    achieved = flops / dur / 1e12
    share = sms / torch.cuda.get_device_properties(0).multi_processor_count
    # fp32 class: 3 kind::tf32 MMAs per product at the tf32 dense rate (no measured tf32 peak in
    # MEASURED_PEAKS.json: B200_PROFILING.md's 1.1 PFLOP/s dense tf32, which the 256-/512-channel
    # convs of this kernel reach ~0.8 of); bf16: the measured dense bf16 rate
    tf32 = measure_tf32_peak() if f32 else None
    peak_full = tf32 / 3.0 if f32 else peaks["bf16_tflops"]
    peak = peak_full * share
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic_r2.json"
    if tf.exists():
        rec = json.loads(tf.read_text()).get(f"{key}_{precision}")
        if rec:
            traffic = rec["dram_read_bytes"] + rec["dram_write_bytes"]
    if f32:
        # (64 -> 64 3x3: the S32 halo kernel unless DBS_HALO_TF=0; wider convs: the streamed BN = 128 kernel)
        halo = Co == 64 and C == 64 and k == 3 and stride == 1 and os.environ.get("DBS_HALO_TF", "1") != "0"
        kname = ("gemm_bf16_kernel<64, true, true> (3xTF32, S32 halo)" if halo else
                 f"gemm_bf16_kernel<{64 if Co <= 64 else 128}, false, true> (3xTF32)")
    else:
        kname = "gemm_bf16_kernel<64, true> (halo)" if Co == 64 else "gemm_bf16_kernel<128, false> (bf16)"
    return {"bound": "tensor", "kernel": f"{kname} implicit-GEMM conv {desc}, b={N} per worker, inside a "
                                         f"{sms}-SM partition",
            "achieved": round(achieved, 2), "peak": round(peak, 1), "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "traffic_unit": "bytes per launch (ncu --set full, profiles/ncu_traffic_r2.json)",
            "algorithmic_flops_per_launch": flops,
            "algorithmic_bytes_per_launch": (8.0 if f32 else 2.0) * (N * H * H * C + Co * k * k * C) +
                                            (4.0 if f32 else 2.0) * N * OH * OH * Co,
            "avg_launch_us": round(dur * 1e6, 2), "partition_sms": sms,
            "peak_note": (f"measured tf32 dense {tf32:.0f} TF/s (cuBLAS 8192^3, best of 10, this run) / 3 MMAs per "
                          f"fp32-class product x {sms}/148 SMs" if f32 else
                          f"measured bf16 {peaks['bf16_tflops']} TF/s x {sms}/148 SMs"),
            "peak_source": "measured (tf32, in bench.py)" if f32 else peaks["source"],
            **({"frac_of_nominal": round(achieved / (TF32_DENSE_TFLOPS / 3.0 * share), 4),
                "tf32_measured_tflops": round(tf32, 1)} if f32 else {})}


def _graph_time(launch, reps=20):
    """Mean device time of `launch(stream)` over `reps` launches captured in a CUDA
    graph (CUDA events on the capturing stream)."""
    import torch

    from paper_2007_11831_b200 import _lib

    for _ in range(3):
        launch(_lib.stream_handle())
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=cs):
        for _ in range(reps):
            launch(int(cs.cuda_stream))
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cs):
        e0.record(cs)
        g.replay()
        e1.record(cs)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def aux_rooflines(tr, peaks):
    """HBM rooflines of the two other hot-path kernels, on the workload's own
    buffers: the repartition gather (gather.cu; 2 * row_bytes + 8 B per row:
    every dataset row to a shard in a random order) and the fused batch-weighted
    aggregate + momentum SGD of the simulated workers (sgd.cu; (4n + 4 * 4 + s) B
    per parameter: n gradients, x and v read, x, v and the operand shadow written,
    s = 8 for the S32 shadow of the fp32 class, 2 for bf16)."""
    import ctypes

    import torch

    from paper_2007_11831_b200 import _lib

    L = _lib.lib()
    out = {}
    D, rb = tr.D, tr.row_bytes
    perm = torch.randperm(D, device=tr.dev)
    dst = torch.empty_like(tr.X)  # the dataset's own row format (MLP shards hold bf16 rows)

    def gather(st):
        assert L.dbs_dev_gather_rows(tr.X.data_ptr(), perm.data_ptr(), D, rb, dst.data_ptr(), st) == 0, _lib.last_error()

    t = _graph_time(gather, 10)
    byt = 2.0 * D * rb + 8.0 * D
    out["repartition_gather"] = {"bound": "hbm", "achieved": round(byt / t / 1e9, 1), "peak": peaks["hbm_gbs"],
                                 "unit": "GB/s", "frac": round(byt / t / 1e9 / peaks["hbm_gbs"], 4),
                                 "bytes_per_launch": byt, "avg_launch_us": round(t * 1e6, 2),
                                 "launch": f"{D} rows x {rb} B, random permutation"}
    n, P = tr.n, tr.model.P
    ptrs = (ctypes.c_void_p * n)(*[g.data_ptr() for g in tr.grads])
    b = np.asarray([37 + 36 * (i % 2) for i in range(n)], dtype=np.int64)
    x = tr.model.params.clone()
    v = torch.zeros_like(x)
    xb = tr.model.params_op.clone()
    sh_bytes = 8.0 if tr.precision == _lib.PREC_F32 else 2.0  # S32 / bf16 operand shadow written per parameter

    def agg(st):
        assert L.dbs_dev_aggregate_sgd_f32_ex(ptrs, b.ctypes.data_as(_lib.P_i64), n, 1, P, 0.0, 0.9, x.data_ptr(),
                                              v.data_ptr(), xb.data_ptr(), tr.precision, st) == 0, _lib.last_error()

    t = _graph_time(agg, 20)
    byt = (4.0 * n + 16.0 + sh_bytes) * P
    out["aggregate_sgd"] = {"bound": "hbm", "achieved": round(byt / t / 1e9, 1), "peak": peaks["hbm_gbs"],
                            "unit": "GB/s", "frac": round(byt / t / 1e9 / peaks["hbm_gbs"], 4),
                            "bytes_per_launch": byt, "avg_launch_us": round(t * 1e6, 2),
                            "launch": f"{n} worker gradients x {P} fp32 parameters"}
    if tr.kind != 0 and tr.depth == 18 and tr.precision == _lib.PREC_F32 and tr.workers and tr.workers[0].ctx:
        out.update(bn_rooflines(tr, peaks))
    return out


def bn_rooflines(tr, peaks, reps=20):
    """The fp32-class BatchNorm passes (resnet.cu; the network's own kernels through
    dbs_dev_bn_*_s32) at the bench's largest BN shape (b per worker x 32 x 32 x 64),
    timed where the bench runs them -- inside worker 0's SM partition, eager launches
    between CUDA events on the partition's stream -- against the copy bandwidth the
    same partition reaches (the repartition gather with an identity index over the
    same bytes in 16 KB rows).  Bytes per element: forward 4 (y) + 8 (S32 out); backward 12 (reduce:
    g, y, mask hi plane) + 24 (apply: g, y, mask, S32 dy, g_out)."""
    import torch

    from paper_2007_11831_b200 import _lib

    L = _lib.lib()
    wk = tr.workers[0]
    M, C = tr.max_batch // tr.n * 1024, 64
    dev = tr.dev
    g0 = torch.Generator(device=dev).manual_seed(0)
    y = torch.randn(M, C, device=dev, generator=g0)
    acc = torch.cat([y.double().sum(0), (y.double() ** 2).sum(0)]).contiguous()
    gamma, beta = torch.ones(C, device=dev), torch.zeros(C, device=dev)
    mean, invstd = torch.empty(C, device=dev), torch.empty(C, device=dev)
    out = torch.empty(M, 2 * C, device=dev)
    g = torch.randn(M, C, device=dev, generator=g0)
    dgam, dbet = torch.zeros(C, device=dev), torch.zeros(C, device=dev)
    dy, gout = torch.empty(M, 2 * C, device=dev), torch.empty(M, C, device=dev)
    # the copy reference: the same bytes as y moved by the repartition gather in 16 KB rows
    # (its efficient regime; 256-byte rows would understate the partition's bandwidth)
    cp_rows = M * C * 4 // 16384
    idx = torch.arange(cp_rows, device=dev)
    cp = torch.empty_like(y)
    h = int(wk.stream.cuda_stream)
    fns = {
        "copy": lambda: L.dbs_dev_gather_rows(y.data_ptr(), idx.data_ptr(), cp_rows, 16384, cp.data_ptr(), h),
        "bn_forward": lambda: L.dbs_dev_bn_apply_s32(y.data_ptr(), acc.data_ptr(), gamma.data_ptr(), beta.data_ptr(),
                                                    C, M, 1, mean.data_ptr(), invstd.data_ptr(), out.data_ptr(), h),
        "bn_backward": lambda: L.dbs_dev_bn_backward_s32(g.data_ptr(), out.data_ptr(), y.data_ptr(), mean.data_ptr(),
                                                        invstd.data_ptr(), gamma.data_ptr(), C, M, dgam.data_ptr(),
                                                        dbet.data_ptr(), dy.data_ptr(), gout.data_ptr(), h),
    }
    byts = {"copy": 2.0 * cp_rows * 16384 + 8.0 * cp_rows, "bn_forward": 12.0 * M * C, "bn_backward": 36.0 * M * C}
    res = {}
    torch.cuda.synchronize()
    _lib.check(L.dbs_partition_push(wk.ctx), "partition_push")
    try:
        for name, fn in fns.items():
            for _ in range(3):
                assert fn() == 0, _lib.last_error()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(wk.stream)
            for _ in range(reps):
                fn()
            e1.record(wk.stream)
            torch.cuda.synchronize()
            res[name] = e0.elapsed_time(e1) / 1e3 / reps
    finally:
        _lib.check(L.dbs_partition_pop(wk.ctx), "partition_pop")
    copy_gbs = byts["copy"] / res["copy"] / 1e9
    out_ = {}
    for name in ("bn_forward", "bn_backward"):
        a = byts[name] / res[name] / 1e9
        out_[name] = {"bound": "hbm", "achieved": round(a, 1), "peak": round(copy_gbs, 1), "unit": "GB/s",
                      "frac": round(a / copy_gbs, 4), "frac_of_full_gpu_hbm": round(a / peaks["hbm_gbs"], 4),
                      "bytes_per_launch": byts[name], "avg_launch_us": round(res[name] * 1e6, 2),
                      "launch": f"M = {M} rows x C = {C} (b = {M // 1024} x 32 x 32), inside a {wk.sm_count}-SM "
                                "partition; peak = the copy bandwidth measured in the same partition",
                      "partition_copy_GBps": round(copy_gbs, 1)}
    return out_


def disturbance_desc(wl):
    w = WL[wl]
    if w["mult"] is None:
        return ("workers 0 and 1: co-running spin kernels pin a fraction f ~ U(0.25, 0.6) of their SM partitions, "
                "redrawn every epoch (seeded; cost_multiplier 1/(1-f)); DBS plans with the reference's "
                f"perf-smoothing EMA a = {w.get('smoothing', 0.0)}")
    if wl.startswith("resnet"):
        return (f"worker 0: a co-running spin kernel pins {1 - 1 / w['mult']:.0%} of its SM partition for every "
                f"epoch (cost_multiplier {w['mult']})")
    return (f"worker 0 on a {w['mult']}x slower emulated device (per-sample cost m x the calibrated time; the "
            "other two at 1x)")


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_iteration_seconds(wl, X, y, threads, k=3):
    """Best of k timed samples of the reference loop (sgdlab.py:380-391) with a CPU
    model on `threads` host threads (torch intra-op threads for the PyTorch-CPU
    ResNet, BLAS threads via threadpoolctl for the numpy MLP).  Imports only the
    oracle (test infrastructure) -- never the product package."""
    from threadpoolctl import threadpool_limits

    from oracle import oracle as O

    w = WL[wl]
    batches = [w.get("cpu_per_worker", w["per_worker"])] * w["workers"]
    ts = []
    with threadpool_limits(limits=threads):
        if wl.startswith("resnet"):
            import torch

            torch.set_num_threads(threads)
            depth = 50 if wl.startswith("resnet50") else 18
            tens = O.resnet_init(w.get("classes", 10), 0, depth)
            for _ in range(k):
                ts.append(O.cpu_resnet_iteration_seconds(tens, X[:sum(batches)], y[:sum(batches)], batches,
                                                         threads=threads, depth=depth))
            sample = (f"best of {k}: 1 synchronous iteration x {w['workers']} workers x {batches[0]} samples, "
                      f"ResNet-{depth} fwd+bwd on PyTorch-CPU (fp32) inside the restated run_parallel_sgd loop")
        else:
            prob = O.MlpProblem(X, y)
            p0 = O.mlp_init().astype(np.float64)
            for _ in range(k):
                t0 = time.perf_counter()
                O.run_parallel_sgd(prob, w["lr"], 4, w["mom"], "batch_weighted", 0, w["workers"], batches,
                                   initial_point=p0)
                ts.append((time.perf_counter() - t0) / 4)
            sample = f"best of {k}: 4 iterations of the numpy float64 oracle loop (MLP Problem, 3 x 128 samples)"
    return sum(batches) / min(ts), sample


def cpu_inputs(wl):
    """The workload's inputs from the oracle's generators (identical to the package's)."""
    from oracle import oracle as O

    w = WL[wl]
    if wl.startswith("resnet18"):
        return O.synthetic_cifar(w["workers"] * w["per_worker"], seed=0)
    if wl.startswith("resnet50"):
        return O.synthetic_imagenet(w["workers"] * w["cpu_per_worker"], w["image"], w["classes"], seed=0)
    return O.synthetic_mnist(w["D"], seed=0)


def cpu_baseline(wl, threads=None):
    """The reported CPU baseline (BASELINE.md CPU plan): all host cores, plus the
    single-thread figure."""
    cores = host_cores()
    X, y = cpu_inputs(wl)
    val, sample = cpu_iteration_seconds(wl, X, y, threads or cores)
    one, _ = cpu_iteration_seconds(wl, X, y, 1, k=2)
    return {"value": round(val, 2), "unit": "samples/s", "cores": threads or cores, "kind": "port",
            "sample": sample, "single_thread": round(one, 2),
            "env": {"OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"),
                    "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"),
                    "thread_limits": "threadpoolctl / torch.set_num_threads per measurement"}}


def e2e_run(tr, wl, X, y, args, world=1):
    """Public API end to end: the same DBS run (same disturbance, plan carried across
    epochs) with the dataset uploaded from pinned host memory at the start of every
    epoch and the per-iteration losses / worker times read back every epoch.  Under
    torchrun every rank uploads its own dataset copy; the time is the max over ranks."""
    import torch

    from paper_2007_11831_b200 import cluster

    w = WL[wl]
    if X is None:  # the distributed trainer generated its data on the device
        X, y = tr.X.cpu().numpy(), tr.y.cpu().numpy()
    Xh = torch.from_numpy(np.ascontiguousarray(X)).pin_memory()
    yh = torch.from_numpy(np.ascontiguousarray(y)).pin_memory()
    h2d_per_epoch = Xh.numel() * Xh.element_size() + yh.numel() * yh.element_size()

    # double-buffered upload: epoch e trains on the buffer whose copy ran during
    # epoch e - 1 and starts the copy for epoch e + 1 on a side stream, so every
    # epoch still moves one full dataset host -> device inside the timed region,
    # overlapped with compute instead of serialised before it
    bufX, bufy = [tr.X, torch.empty_like(tr.X)], [tr.y, torch.empty_like(tr.y)]
    copy_stream = torch.cuda.Stream()
    ready = [None, None]

    def start_copy(slot):
        copy_stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(copy_stream):
            bufX[slot].copy_(Xh.view(tr.X.shape), non_blocking=True)
            bufy[slot].copy_(yh, non_blocking=True)
            ready[slot] = torch.cuda.Event()
            ready[slot].record(copy_stream)

    def upload(epoch):
        cur = epoch % 2
        if ready[cur] is None:
            start_copy(cur)
        torch.cuda.current_stream().wait_event(ready[cur])
        ready[cur] = None
        tr.X, tr.y = bufX[cur], bufy[cur]
        start_copy(1 - cur)

    cfg = cluster.StrategyConfig("dbs", w["workers"] * world * w["per_worker"], perf_smoothing=w.get("smoothing", 0.0))
    extra = {"averaging_interval": w["avg"]} if w.get("avg") else {}
    res = tr.run(cfg, n_epochs=args.warmup + args.steps, lr=w["lr"], momentum=w["mom"],
                 profiles=profiles(w["workers"] * world, w["mult"]), record_loss=True, timed_from=args.warmup,
                 epoch_hook=upload, **extra)
    timed = res.stats[args.warmup:]
    iters = [cluster.iterations_for_plan(s.plan) for s in timed]
    # read back per epoch: the [workers x iters] fp32 loss rows and the fp64 worker times
    d2h = [4 * tr.n * it + tr.seconds.numel() * tr.seconds.element_size() for it in iters]
    return {"value": round(res.timed_samples / res.timed_seconds, 1), "unit": "samples/s",
            "h2d_bytes_per_step": int(h2d_per_epoch), "d2h_bytes_per_step": int(sum(d2h) // max(len(d2h), 1)),
            "epochs": len(timed),
            "note": "DBS epochs; every epoch uploads one full dataset copy from pinned host memory inside the timed "
                    "region (double-buffered: the copy for epoch e + 1 overlaps epoch e) and reads the losses back"}


def reference_arm_allreduce(args, world):
    """Reference arm of C2: aggregate_gradients(batch_weighted) + sgd_step
    (sgdlab.py:208-238) restated in C (oracle/dbs_oracle.c, fp64 like the
    reference), W rank gradients of a bounded 16 MiB-equivalent size."""
    from oracle import oracle as O

    n = max(world, 1)
    P = 16 * (1 << 20) // 4
    rng = np.random.default_rng(0)
    grads = [rng.standard_normal(P) for _ in range(n)]
    x, v = rng.standard_normal(P), np.zeros(P)
    b = [C2_BATCHES[r % len(C2_BATCHES)] for r in range(n)]
    ts = []
    for _ in range(max(1, min(args.steps, 3))):
        t0 = time.perf_counter()
        g = O.aggregate(grads, b, 1)
        x, v = O.sgd_step(x, g, v, 0.05, 0.9)
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    val = round(22.0 * P / t / 1e9, 3)
    out = {"impl": "reference", "metric": "batch-weighted aggregate + momentum SGD, GB/s (22 B per parameter)",
           "value": val, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "higher_is_better": True, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"C2 reference: {n} rank gradients x 16 MiB-equivalent on the host"},
           "cpu_baseline": {"value": val, "unit": "GB/s", "cores": 1, "kind": "port",
                            "sample": f"aggregate_gradients + sgd_step over {n} x {P} fp64 (C restatement)"},
           "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def reference_arm(args):
    """The reference's CPU implementation of the path on the host cores (the oracle
    port of run_parallel_sgd with a CPU model), on the same workload / config as
    our arm.  Imports only the oracle: no product code, no product .so."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    wl = args.workload
    if wl == "allreduce":
        return reference_arm_allreduce(args, world)
    base = cpu_baseline(wl)
    out = {"impl": "reference", "metric": METRIC, "value": base["value"], "unit": "samples/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
           "dtype": "f32" if wl.startswith("resnet") else "f64", "data": "synthetic",
           "config": workload_config(wl, args.precision), "cpu_baseline": base,
           "e2e": {"value": base["value"], "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


C2_BATCHES = [37, 37, 73, 73, 73, 73, 73, 73]  # a DBS plan of 8 ranks, sum 512
C2_SIZES_MIB = [1, 4, 16, 64, 256, 1024]


def run_allreduce(args):
    """C2: the fused batch-weighted all-reduce + momentum SGD (comm.cu) swept over
    1 MiB .. 1 GiB of fp32 gradient per rank with unequal batch weights.  One
    launch per step; CUDA events on the launching stream, max over ranks.
    Bytes per rank and direction over NVLink: 4P(W-1)/W of gradient shards
    pulled + 6P(W-1)/W of updated parameters (fp32 + bf16 shadow) pushed, i.e.
    10P(W-1)/W; busbw is NCCL's all-reduce convention 2(W-1)/W * 4P / t.  At
    W = 1 there is no exchange: the kernel is the HBM-bound local update
    (22 B per parameter: read g, x, v; write x, v and the bf16 shadow)."""
    import torch

    from paper_2007_11831_b200.comm import Communicator, max_over_ranks

    rank, world, local = dist_env()
    torch.cuda.set_device(bench_device(local, world))
    group = None
    if world > 1:
        import torch.distributed as dist

        init_group()
    else:
        import torch.distributed as dist

        dist.init_process_group("gloo", init_method="tcp://127.0.0.1:29517", rank=0, world_size=1)
    peaks = load_peaks()
    b = [C2_BATCHES[r % len(C2_BATCHES)] for r in range(world)]
    rows = []
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    for mib in C2_SIZES_MIB:
        P = mib * (1 << 20) // 4
        comm = Communicator.create(P, group) if world > 1 else Communicator.local(1, P)[0]
        g = torch.Generator(device="cuda").manual_seed(1000 + rank)
        comm.grad.copy_(torch.randn(comm.P, generator=g, device="cuda"))
        comm.params.copy_(torch.randn(comm.P, generator=g, device="cuda"))
        s = torch.cuda.current_stream()
        for _ in range(args.warmup):
            comm.allreduce_sgd(b, 0.05, 0.9, stream=s)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(args.steps):
            comm.allreduce_sgd(b, 0.05, 0.9, stream=s)
        e1.record(s)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / args.steps
        if world > 1:
            t = max_over_ranks(t)
        Pp = comm.P
        row = {"MiB": mib, "us": round(t * 1e6, 2)}
        if world > 1:
            nv = 10.0 * Pp * (world - 1) / world
            row.update({"busbw_GBps": round(2.0 * (world - 1) / world * 4 * Pp / t / 1e9, 1),
                        "nvlink_GBps_per_dir": round(nv / t / 1e9, 1),
                        "nvlink_frac_of_770": round(nv / t / 1e9 / 770.0, 3)})
        else:
            row.update({"hbm_GBps": round(22.0 * Pp / t / 1e9, 1),
                        "hbm_frac": round(22.0 * Pp / t / 1e9 / peaks["hbm_gbs"], 3)})
        rows.append(row)
        comm.close()
        del comm
        torch.cuda.empty_cache()
    clocks = sampler.stop()
    top = rows[-1]
    out = {
        "metric": "batch-weighted all-reduce + momentum SGD (fused NVLink kernel), bus bandwidth at 1 GiB"
                  if world > 1 else "batch-weighted aggregate + momentum SGD (W=1: local update), HBM GB/s at 1 GiB",
        "value": top["busbw_GBps"] if world > 1 else top["hbm_GBps"], "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(top["us"] / 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "C2: fused batch-weighted all-reduce + SGD sweep 1 MiB-1 GiB fp32 per rank, "
                               f"batch weights {b}, lr 0.05, momentum 0.9",
                   "l2": "1 GiB gradient + parameters per rank exceed L2"},
        "sweep": rows,
        "roofline": ({"bound": "nvlink", "achieved": top["nvlink_GBps_per_dir"], "peak": 770.0, "unit": "GB/s",
                      "frac": top["nvlink_frac_of_770"], "traffic": None,
                      "peak_source": "B200_PROFILING.md measured peer copy per direction"} if world > 1 else
                     {"bound": "hbm", "achieved": top["hbm_GBps"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
                      "frac": top["hbm_frac"], "traffic": None, "peak_source": peaks["source"]}),
        "e2e": None, "cpu_baseline": None, "clocks": clocks,
        "gpu_launches": (args.warmup + args.steps) * len(C2_SIZES_MIB),
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    if args.workload == "allreduce" and args.impl != "reference":
        return run_allreduce(args)
    if args.impl == "reference":
        return reference_arm(args)
    rank, world, local = dist_env()
    import torch

    torch.cuda.set_device(bench_device(local, world))
    if world > 1:
        import torch.distributed as dist

        init_group()
    peaks = load_peaks()
    wl = args.workload
    w = WL[wl]
    tr, (X, y) = make_trainer(wl, rank, world, args.precision)
    if world > 1:
        dist.barrier()
    # (multi-GPU: the trainer's timed seconds are already the max over ranks and
    # its samples count every worker of every rank)
    res = {k: run_strategy(tr, wl, k, args, world) for k in ("fixed_ssgd", "dbs")}
    dbs, fixed = res["dbs"], res["fixed_ssgd"]
    if args.report and rank == 0:
        from pathlib import Path

        from paper_2007_11831_b200 import report as rpt

        out = Path(args.report)
        out.mkdir(parents=True, exist_ok=True)
        reps = [rpt.RunReport.from_stats(f"bench_{wl}_n{world}", k, 0, res[k]["stats"]) for k in ("fixed_ssgd", "dbs")]
        for r in reps:
            rpt.write_epoch_csv(r, out / f"{r.scenario_name}_{r.strategy}.csv")
        rpt.write_run_json(reps, [], out / f"bench_{wl}_n{world}.json")
    roof = kernel_roofline(peaks, wl, args.precision, tr) if wl in ("resnet18", "resnet18_4w", "resnet18_ma", "resnet50",
                                                                   "resnet50_3w") else None
    aux = aux_rooflines(tr, peaks) if world == 1 else None
    e2e = None if args.no_e2e else e2e_run(tr, wl, X, y, args, world)
    gaps = [np.mean(s.per_worker_wait) / max(s.per_worker_gpu) for s in fixed["stats"]]
    cfg = workload_config(wl, args.precision)
    cfg["l2"] = (f"inputs > L2: {tr.X.numel() * tr.X.element_size() / 1e6:.0f} MB dataset repacked into per-worker "
                 "shards every epoch")
    if getattr(tr, "device_per_sample_ns", None):
        cfg["emulated_devices"] = (f"every worker adds a timed spin of m_w x b_w x {tr.device_per_sample_ns:.0f} ns "
                                   "per iteration (the reference's cost law, per-sample time calibrated on an "
                                   "undisturbed epoch; m_w = 2 on the disturbed worker)")
    variant = None
    if world == 1 and not args.no_bf16 and args.precision == "f32":
        # the same workload with bf16 tensor-core operands: a labelled variant, not the headline
        del tr
        torch.cuda.empty_cache()
        trb, _ = make_trainer(wl, rank, world, "bf16")
        rb = {k: run_strategy(trb, wl, k, args, world) for k in ("fixed_ssgd", "dbs")}
        variant = {"dtype": "bf16", "arithmetic": PRECISION_DESC["bf16"],
                   "value": round(rb["dbs"]["samples_per_s"], 1),
                   "fixed_samples_per_s": round(rb["fixed_ssgd"]["samples_per_s"], 1),
                   "dbs_vs_fixed_speedup": round(rb["dbs"]["samples_per_s"] / rb["fixed_ssgd"]["samples_per_s"], 4),
                   "ms_per_step": round(rb["dbs"]["epoch_s"] * 1e3, 3)}
        del trb
        torch.cuda.empty_cache()
    cpu = None if (args.no_cpu or world > 1) else cpu_baseline(wl)
    out = {
        "metric": METRIC,
        "value": round(dbs["samples_per_s"], 1),
        "unit": "samples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(dbs["epoch_s"] * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": args.precision,
        "data": "synthetic",
        "config": cfg,
        "fixed": {"samples_per_s": round(fixed["samples_per_s"], 1), "ms_per_epoch": round(fixed["epoch_s"] * 1e3, 3)},
        "dbs_vs_fixed_speedup": round(dbs["samples_per_s"] / fixed["samples_per_s"], 4),
        "dbs_saving": round(1.0 - fixed["samples_per_s"] / dbs["samples_per_s"], 4),
        "utilisation_gap_fixed": round(float(np.mean(gaps)), 4),
        "final_plan": list(dbs["stats"][-1].plan.int_batches),
        "per_worker_gpu_s_last_epoch": {"fixed": [round(v, 4) for v in fixed["stats"][-1].per_worker_gpu],
                                        "dbs": [round(v, 4) for v in dbs["stats"][-1].per_worker_gpu]},
        "roofline": roof,
        "kernel_rooflines": aux,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "bf16_variant": variant,
        "clocks": dbs["clocks"],
        # (the fixed-plan epochs' own timed region: on one GPU the emulated workers share one
        # power budget, and balanced DBS epochs keep every partition busy)
        "clocks_fixed": fixed["clocks"],
        "gpu_launches": int(dbs["launches"]),
        "host_launches_per_epoch": round(dbs["host_launches"] / max(len(dbs["stats"]), 1), 1),
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
