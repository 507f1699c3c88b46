"""ncu target: one plain tcgen05 GEMM launch (after warm-up) of shape M N K (bf16 out)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2007_11831_b200 import _lib
M, N, K = (int(v) for v in sys.argv[1:4])
L = _lib.lib()
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
d = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(4):
    assert L.dbs_dev_gemm_bf16(a.data_ptr(), 0, K, b.data_ptr(), 0, K, d.data_ptr(), N, M, N, K, 4, None, None, _lib.stream_handle()) == 0
torch.cuda.synchronize()
