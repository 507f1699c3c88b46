"""Dev probe: plain tcgen05 GEMM timings (CUDA graph of 50 launches) for a few shapes."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2007_11831_b200 import _lib  # noqa: E402
L = _lib.lib()
shapes = [(200704, 256, 64), (200704, 64, 256), (16384, 256, 2304), (50176, 256, 1024), (12544, 1024, 256)]
if len(sys.argv) > 1 and sys.argv[1] == "transposed":
    # normal (M = pixels, N = Cout) vs transposed (M = Cout, N = pixels) orientation
    shapes = [(50176, 128, 1152), (128, 50176, 1152), (50176, 64, 576), (64, 50176, 576), (32768, 128, 1152),
              (128, 32768, 1152)]
for M, N, K in shapes:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    d = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    def run(st):
        assert L.dbs_dev_gemm_bf16(a.data_ptr(), 0, K, b.data_ptr(), 0, K, d.data_ptr(), N, M, N, K, 4, None, None, st) == 0
    for _ in range(3): run(_lib.stream_handle())
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); cs = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=cs):
        for _ in range(50): run(int(cs.cuda_stream))
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(cs):
        e0.record(cs); g.replay(); e1.record(cs)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    byt = 2 * (M * K + N * K + M * N)
    print(f"gemm M={M} N={N} K={K}: {us:8.1f} us  {2*M*N*K/us/1e6:7.1f} TF/s  {byt/us/1e3:7.1f} GB/s", flush=True)
