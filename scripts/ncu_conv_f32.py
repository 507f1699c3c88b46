"""ncu target: warm-up + a few launches of one fp32-class (3xTF32, S32 operands) conv forward.

    python scripts/ncu_conv_f32.py N H Cin Cout k stride [reps]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2007_11831_b200 import _lib  # noqa: E402

N, H, Cin, Cout, k, stride = (int(v) for v in sys.argv[1:7])
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 4
pad = k // 2
OH = (H + 2 * pad - k) // stride + 1
L = _lib.lib()
s = _lib.stream_handle()


def s32(t):
    o = torch.empty(t.shape[0], 2 * t.shape[1], device="cuda")
    assert L.dbs_dev_split_s32(t.data_ptr(), t.shape[0], t.shape[1], t.shape[1], o.data_ptr(), t.shape[1], s) == 0
    return o


x = s32(torch.randn(N * H * H, Cin, device="cuda"))
w = s32(torch.randn(Cout, k * k * Cin, device="cuda") / (k * k * Cin) ** 0.5)
y = torch.empty(N * OH * OH, Cout, device="cuda")
for _ in range(reps):
    st = L.dbs_dev_conv2d_fwd_s32(x.data_ptr(), N, H, H, Cin, w.data_ptr(), Cout, k, stride, pad, y.data_ptr(), s)
    assert st == 0, _lib.last_error()
torch.cuda.synchronize()
print("ok f32 fwd", N, H, Cin, Cout, k, stride)
