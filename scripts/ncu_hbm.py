"""ncu target: the HBM-bound hot-path kernels on bench-sized buffers --
the repartition gather (50000 CIFAR rows of 12 KB, random permutation) and the
fused batch-weighted aggregate + momentum SGD (4 workers x ResNet-18 gradient)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2007_11831_b200 import _lib  # noqa: E402

L = _lib.lib()
s = _lib.stream_handle()
D, rb = 50000, 12288
X = torch.randn(D, rb // 4, device="cuda")
dst = torch.empty_like(X)
perm = torch.randperm(D, device="cuda")
P, n = 11174304, 4
grads = [torch.randn(P, device="cuda") for _ in range(n)]
ptrs = (ctypes.c_void_p * n)(*[g.data_ptr() for g in grads])
b = np.asarray([37, 73, 73, 73], dtype=np.int64)
x = torch.randn(P, device="cuda")
v = torch.zeros(P, device="cuda")
xb = torch.empty(P, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    assert L.dbs_dev_gather_rows(X.data_ptr(), perm.data_ptr(), D, rb, dst.data_ptr(), s) == 0
    assert L.dbs_dev_aggregate_sgd_f32(ptrs, b.ctypes.data_as(_lib.P_i64), n, 1, P, 0.05, 0.9, x.data_ptr(),
                                       v.data_ptr(), xb.data_ptr(), s) == 0
torch.cuda.synchronize()
print("ok")
