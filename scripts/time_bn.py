"""Dev probe: the fp32-class BatchNorm passes (dbs_dev_bn_*_s32, the network's own kernels)
at every ResNet-18 BN shape of the bench's per-worker batch, inside one worker's 48-SM
partition, against the copy bandwidth of the same partition.

    python scripts/time_bn.py [b=170]

Bytes per element: forward 4 (y) + 8 (S32 out); backward 12 (reduce: g, y, mask hi plane)
+ 24 (apply: g, y, mask hi plane, S32 dy, g_out).
"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2007_11831_b200 import _lib  # noqa: E402

L = _lib.lib()
B = int(dict(a.split("=") for a in sys.argv[1:] if "=" in a).get("b", 170))
h = ctypes.c_void_p()
act = ctypes.c_int32()
_lib.check(L.dbs_partition_create(3, 48, ctypes.byref(h), ctypes.byref(act)), "partition")
ctx, st, side = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
_lib.check(L.dbs_partition_get(h, 0, ctypes.byref(ctx), ctypes.byref(st), ctypes.byref(side)), "get")
stream = torch.cuda.ExternalStream(st.value)
S = int(stream.cuda_stream)


def timed(fn, reps=30):
    _lib.check(L.dbs_partition_push(ctx), "push")
    try:
        for _ in range(3):
            assert fn() == 0, _lib.last_error()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
    finally:
        L.dbs_partition_pop(ctx)
    return e0.elapsed_time(e1) / reps / 1e3


big = torch.empty(B * 1024 * 64, device="cuda")
cp_rows = big.numel() * 4 // 16384
idx = torch.arange(cp_rows, device="cuda")
cp = torch.empty_like(big)
t = timed(lambda: L.dbs_dev_gather_rows(big.data_ptr(), idx.data_ptr(), cp_rows, 16384, cp.data_ptr(), S))
copy = (2.0 * cp_rows * 16384 + 8.0 * cp_rows) / t / 1e9
print(f"partition {act.value} SMs, b={B}: copy {copy:.0f} GB/s", flush=True)
tot_f = tot_b = byt_f = byt_b = 0.0
for HW, C in ((1024, 64), (256, 128), (64, 256), (16, 512)):
    M = B * HW
    g0 = torch.Generator(device="cuda").manual_seed(C)
    y = torch.randn(M, C, device="cuda", generator=g0)
    acc = torch.cat([y.double().sum(0), (y.double() ** 2).sum(0)]).contiguous()
    gamma, beta = torch.ones(C, device="cuda"), torch.zeros(C, device="cuda")
    mean, invstd = torch.empty(C, device="cuda"), torch.empty(C, device="cuda")
    out = torch.empty(M, 2 * C, device="cuda")
    g = torch.randn(M, C, device="cuda", generator=g0)
    dgam, dbet = torch.zeros(C, device="cuda"), torch.zeros(C, device="cuda")
    dy, gout = torch.empty(M, 2 * C, device="cuda"), torch.empty(M, C, device="cuda")
    tf = timed(lambda: L.dbs_dev_bn_apply_s32(y.data_ptr(), acc.data_ptr(), gamma.data_ptr(), beta.data_ptr(), C, M, 1,
                                              mean.data_ptr(), invstd.data_ptr(), out.data_ptr(), S))
    tb = timed(lambda: L.dbs_dev_bn_backward_s32(g.data_ptr(), out.data_ptr(), y.data_ptr(), mean.data_ptr(),
                                                 invstd.data_ptr(), gamma.data_ptr(), C, M, dgam.data_ptr(),
                                                 dbet.data_ptr(), dy.data_ptr(), gout.data_ptr(), S))
    bf, bb = 12.0 * M * C, 36.0 * M * C
    tot_f += tf
    tot_b += tb
    byt_f += bf
    byt_b += bb
    print(f"M {M:7d} x C {C:3d}: forward {tf * 1e6:7.1f} us {bf / tf / 1e9:6.0f} GB/s ({bf / tf / 1e9 / copy:.2f})  "
          f"backward {tb * 1e6:7.1f} us {bb / tb / 1e9:6.0f} GB/s ({bb / tb / 1e9 / copy:.2f})", flush=True)
print(f"all four shapes: forward {byt_f / tot_f / 1e9 / copy:.2f}, backward {byt_b / tot_b / 1e9 / copy:.2f} of copy")
