"""Dev probe: the fp32-class (3xTF32) path inside one worker's 48-SM partition.

    python scripts/time_f32.py [convs] [step] [prof]

convs: fwd / dgrad / wgrad of every ResNet-18 conv shape at the bench's per-worker
batch (170), eager launches on the partition stream between CUDA events.
step:  one worker's full forward/backward (b=170) in the partition.
prof:  kernel-time breakdown of that step (torch.profiler / CUPTI).
"""
import collections
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2007_11831_b200 import _lib, resnet  # noqa: E402

L = _lib.lib()
B = int(dict(a.split("=") for a in sys.argv[1:] if "=" in a).get("b", 170))
prec = dict(a.split("=") for a in sys.argv[1:] if "=" in a).get("prec", "f32")
f32 = prec == "f32"
h = ctypes.c_void_p()
act = ctypes.c_int32()
_lib.check(L.dbs_partition_create(3, 48, ctypes.byref(h), ctypes.byref(act)), "partition")
ctx, st, side = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
_lib.check(L.dbs_partition_get(h, 0, ctypes.byref(ctx), ctypes.byref(st), ctypes.byref(side)), "get")
stream = torch.cuda.ExternalStream(st.value)
S = int(stream.cuda_stream)


def timed(fn, reps=20):
    _lib.check(L.dbs_partition_push(ctx), "push")
    try:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
    finally:
        L.dbs_partition_pop(ctx)
    return e0.elapsed_time(e1) / reps * 1e3


def s32(t):
    t = t.reshape(-1, t.shape[-1]).contiguous()
    o = torch.empty(t.shape[0], 2 * t.shape[1], device="cuda")
    assert L.dbs_dev_split_s32(t.data_ptr(), t.shape[0], t.shape[1], t.shape[1], o.data_ptr(), t.shape[1], 0) == 0
    return o


SHAPES = [(32, 64, 64, 3, 1), (32, 64, 128, 3, 2), (32, 64, 128, 1, 2), (16, 128, 128, 3, 1), (16, 128, 256, 3, 2),
          (8, 256, 256, 3, 1), (8, 256, 512, 3, 2), (4, 512, 512, 3, 1)]
peak = (1100.0 / 3.0 if f32 else 1648.0) * act.value / 148
print(f"partition {act.value} SMs, b={B}, {prec}, peak {peak:.1f} TF/s", flush=True)
if "convs" in sys.argv:
    for (H, C, K, k, s) in SHAPES:
        OH = (H + 2 * (k // 2) - k) // s + 1
        x = torch.randn(B, H, H, C, device="cuda")
        w = torch.randn(K, k, k, C, device="cuda") / (k * k * C) ** 0.5
        dy = torch.randn(B, OH, OH, K, device="cuda")
        fl = 2.0 * B * OH * OH * K * k * k * C
        if f32:
            xs, ws, dys = s32(x), s32(w), s32(dy)
            y = torch.empty(B, OH, OH, K, device="cuda")
            dx = torch.empty(B, H, H, C, device="cuda")
            fwd = lambda: L.dbs_dev_conv2d_fwd_s32(xs.data_ptr(), B, H, H, C, ws.data_ptr(), K, k, s, k // 2, y.data_ptr(), S)
            dgr = lambda: L.dbs_dev_conv2d_dgrad_s32(dys.data_ptr(), B, H, H, C, ws.data_ptr(), K, k, s, k // 2, dx.data_ptr(), S)
        else:
            xs, ws, dys = x.to(torch.bfloat16), w.to(torch.bfloat16), dy.to(torch.bfloat16)
            y = torch.empty(B, OH, OH, K, dtype=torch.bfloat16, device="cuda")
            dx = torch.empty(B, H, H, C, dtype=torch.bfloat16, device="cuda")
            fwd = lambda: L.dbs_dev_conv2d_fwd(xs.data_ptr(), B, H, H, C, ws.data_ptr(), K, k, s, k // 2, y.data_ptr(), S)
            dgr = lambda: L.dbs_dev_conv2d_dgrad(dys.data_ptr(), B, H, H, C, ws.data_ptr(), K, k, s, k // 2, dx.data_ptr(), None, S)
        dw = torch.zeros(K, k, k, C, device="cuda")
        wfn = L.dbs_dev_conv2d_wgrad_s32 if f32 else L.dbs_dev_conv2d_wgrad
        wgr = lambda: wfn(dys.data_ptr(), xs.data_ptr(), B, H, H, C, K, k, s, k // 2, dw.data_ptr(), S)
        tf, td, tw = timed(fwd), timed(dgr), timed(wgr)
        print(f"conv {C:4d}->{K:4d} k{k} s{s} @{H:2d}: fwd {tf:8.1f} us ({fl / tf / 1e6:6.1f} TF/s {fl / tf / 1e6 / peak:5.2f})"
              f"  dgrad {td:8.1f} us ({fl / td / 1e6 / peak:5.2f})  wgrad {tw:8.1f} us ({fl / tw / 1e6 / peak:5.2f})",
              flush=True)
if "step" in sys.argv or "prof" in sys.argv:
    m = resnet.ResnetModel(seed=0, precision=prec)
    _lib.check(L.dbs_partition_push(ctx), "push")
    sc = resnet.ResnetScratch(B, precision=prec)
    L.dbs_partition_pop(ctx)
    X, yy = resnet.synthetic_cifar(B, seed=0)
    x = torch.as_tensor(X, device="cuda")
    yl = torch.as_tensor(yy, device="cuda")
    gr = torch.zeros(m.P, device="cuda")
    loss = torch.zeros(1, device="cuda")

    def step():
        st_ = L.dbs_resnet_forward_backward(sc.handle, m.params_op.data_ptr(), m.params.data_ptr(), x.data_ptr(),
                                            yl.data_ptr(), B, None, gr.data_ptr(), loss.data_ptr(), S)
        assert st_ == 0, _lib.last_error()

    us = timed(step, 10)
    print(f"ResNet-18 worker step b={B}: {us / 1e3:.3f} ms ({3.33e9 * B / us / 1e6:.1f} TF/s, "
          f"{3.33e9 * B / us / 1e6 / peak:.2f} of the partition peak)", flush=True)
    if "prof" in sys.argv:
        from torch.profiler import ProfilerActivity, profile

        _lib.check(L.dbs_partition_push(ctx), "push")
        with profile(activities=[ProfilerActivity.CUDA]) as p:
            for _ in range(2):
                step()
            torch.cuda.synchronize()
        L.dbs_partition_pop(ctx)
        agg = collections.defaultdict(lambda: [0, 0.0])
        for e in p.events():
            if e.device_type == torch.autograd.DeviceType.CUDA:
                agg[e.name[:100]][0] += 1
                agg[e.name[:100]][1] += e.device_time_total
        tot = sum(v[1] for v in agg.values())
        print(f"== kernel time per 2 steps {tot / 1e3:.2f} ms")
        for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]:
            print(f"{t / 1e3:9.3f} ms {100 * t / tot:5.1f}% {c:5d}x  {k}")
