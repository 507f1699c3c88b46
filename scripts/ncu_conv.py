"""ncu target: warm-up + a few launches of one implicit-GEMM conv (fwd | dgrad | wgrad).

    python scripts/ncu_conv.py N H Cin Cout k stride [fwd|dgrad|wgrad] [reps]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2007_11831_b200 import _lib  # noqa: E402

N, H, Cin, Cout, k, stride = (int(v) for v in sys.argv[1:7])
op = sys.argv[7] if len(sys.argv) > 7 else "fwd"
reps = int(sys.argv[8]) if len(sys.argv) > 8 else 4
pad = k // 2
OH = (H + 2 * pad - k) // stride + 1
L = _lib.lib()
x = torch.randn(N, H, H, Cin, device="cuda").to(torch.bfloat16)
w = (torch.randn(Cout, k, k, Cin, device="cuda") / (k * k * Cin) ** 0.5).to(torch.bfloat16)
y = torch.empty(N, OH, OH, Cout, dtype=torch.bfloat16, device="cuda")
dy = torch.randn(N, OH, OH, Cout, device="cuda").to(torch.bfloat16)
dx = torch.empty_like(x)
dw = torch.zeros(Cout, k, k, Cin, device="cuda")
s = _lib.stream_handle()
for _ in range(reps):
    if op == "fwd":
        st = L.dbs_dev_conv2d_fwd(x.data_ptr(), N, H, H, Cin, w.data_ptr(), Cout, k, stride, pad, y.data_ptr(), s)
    elif op == "dgrad":
        st = L.dbs_dev_conv2d_dgrad(dy.data_ptr(), N, H, H, Cin, w.data_ptr(), Cout, k, stride, pad, dx.data_ptr(),
                                    None, s)
    else:
        st = L.dbs_dev_conv2d_wgrad(dy.data_ptr(), x.data_ptr(), N, H, H, Cin, Cout, k, stride, pad, dw.data_ptr(), s)
    assert st == 0, _lib.last_error()
torch.cuda.synchronize()
print("ok", op, N, H, Cin, Cout, k, stride)
