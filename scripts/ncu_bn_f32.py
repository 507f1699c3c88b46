"""ncu target: the fp32-class BatchNorm passes (dbs_dev_bn_apply_s32 / dbs_dev_bn_backward_s32)
at the bench's largest BN shape (b = 170 x 32 x 32 x 64), after warm-up."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2007_11831_b200 import _lib  # noqa: E402

L = _lib.lib()
s = _lib.stream_handle()
M, C = 170 * 1024, 64
y = torch.randn(M, C, device="cuda")
acc = torch.cat([y.double().sum(0), (y.double() ** 2).sum(0)]).contiguous()
gamma, beta = torch.ones(C, device="cuda"), torch.zeros(C, device="cuda")
mean, invstd = torch.empty(C, device="cuda"), torch.empty(C, device="cuda")
out = torch.empty(M, 2 * C, device="cuda")
g = torch.randn(M, C, device="cuda")
dg, db = torch.zeros(C, device="cuda"), torch.zeros(C, device="cuda")
dy, gout = torch.empty(M, 2 * C, device="cuda"), torch.empty(M, C, device="cuda")
for _ in range(3):
    assert L.dbs_dev_bn_apply_s32(y.data_ptr(), acc.data_ptr(), gamma.data_ptr(), beta.data_ptr(), C, M, 1,
                                  mean.data_ptr(), invstd.data_ptr(), out.data_ptr(), s) == 0
    assert L.dbs_dev_bn_backward_s32(g.data_ptr(), out.data_ptr(), y.data_ptr(), mean.data_ptr(), invstd.data_ptr(),
                                     gamma.data_ptr(), C, M, dg.data_ptr(), db.data_ptr(), dy.data_ptr(),
                                     gout.data_ptr(), s) == 0
torch.cuda.synchronize()
print("ok")
