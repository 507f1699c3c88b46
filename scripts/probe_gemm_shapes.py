"""Dev probe: plain 2-D tcgen05 GEMM vs implicit-GEMM conv at the ResNet-18 stage-1 shape."""
import torch
from paper_2007_11831_b200 import _lib
L = _lib.lib()


def timed(fn, reps=50):
    for _ in range(3): fn(_lib.stream_handle())
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); cs = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=cs):
        for _ in range(reps): fn(int(cs.cuda_stream))
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(cs):
        e0.record(cs); g.replay(); e1.record(cs)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for M, N, K in [(131072, 64, 576), (131072, 128, 576), (131072, 256, 576), (131072, 64, 64), (16384, 512, 4608),
                (32768, 256, 2304)]:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    d = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    t = timed(lambda st: L.dbs_dev_gemm_bf16(a.data_ptr(), 0, K, b.data_ptr(), 0, K, d.data_ptr(), N, M, N, K, 4, None, None, st))
    fl = 2.0 * M * N * K
    byt = 2.0 * (M * K + N * K + M * N)
    print(f"gemm M={M} N={N} K={K}: {t:7.1f} us  {fl/t/1e6:7.1f} TF/s  {byt/t/1e3:7.1f} GB/s(min bytes)", flush=True)
