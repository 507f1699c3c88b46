"""Dev probe: tcgen05 conv kernels (fwd / dgrad / wgrad) timed in CUDA graphs + one ResNet step."""
import sys, torch
sys.path.insert(0, ".")
from paper_2007_11831_b200 import _lib, resnet
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
SETS = {
    "r18": [(128, 32, 64, 64, 3, 1), (128, 16, 128, 128, 3, 1), (128, 8, 256, 256, 3, 1), (128, 4, 512, 512, 3, 1),
            (128, 32, 64, 128, 3, 2)],
    "r50": [(64, 56, 64, 64, 3, 1), (64, 56, 64, 256, 1, 1), (64, 56, 256, 64, 1, 1), (64, 28, 128, 128, 3, 1),
            (64, 14, 256, 256, 3, 1), (64, 14, 1024, 256, 1, 1), (64, 7, 512, 512, 3, 1), (64, 7, 512, 2048, 1, 1),
            (64, 56, 128, 128, 3, 2)],
    "l2": [(128, 4, 512, 512, 3, 1), (256, 4, 512, 512, 3, 1), (512, 4, 512, 512, 3, 1),
           (32, 14, 256, 256, 3, 1), (64, 14, 256, 256, 3, 1), (96, 14, 256, 256, 3, 1)],
}
which = sys.argv[1:] or ["r18"]
for (N, H, C, K, k, s) in [sh for w in which if w in SETS for sh in SETS[w]]:
    OH = (H + 2*(k//2) - k)//s + 1
    x = torch.randn(N, H, H, C, device="cuda").to(torch.bfloat16)
    w = (torch.randn(K, k, k, C, device="cuda") / 24).to(torch.bfloat16)
    y = torch.empty(N, OH, OH, K, dtype=torch.bfloat16, device="cuda")
    dy = torch.randn(N, OH, OH, K, device="cuda").to(torch.bfloat16)
    dx = torch.empty(N, H, H, C, dtype=torch.bfloat16, device="cuda")
    dw = torch.zeros(K, k, k, C, device="cuda")
    scr = torch.empty(2*(K*k*k*C+64) + 8*N*H*H*K + 1024, dtype=torch.uint8, device="cuda")
    fl = 2.0 * N * OH * OH * K * k * k * C
    tf = timed(lambda st: L.dbs_dev_conv2d_fwd(x.data_ptr(), N, H, H, C, w.data_ptr(), K, k, s, k//2, y.data_ptr(), st))
    td = timed(lambda st: L.dbs_dev_conv2d_dgrad(dy.data_ptr(), N, H, H, C, w.data_ptr(), K, k, s, k//2, dx.data_ptr(), scr.data_ptr(), st))
    tw = timed(lambda st: L.dbs_dev_conv2d_wgrad(dy.data_ptr(), x.data_ptr(), N, H, H, C, K, k, s, k//2, dw.data_ptr(), st))
    print(f"conv {C}->{K} k{k} s{s} @{H}: fwd {tf:7.1f} us ({fl/tf/1e6:6.1f} TF/s)  dgrad {td:7.1f} us ({fl/td/1e6:6.1f})  wgrad {tw:7.1f} us ({fl/tw/1e6:6.1f})", flush=True)
if "step" not in which:
    sys.exit(0)
if "r50" in which:
    B = 64
    m = resnet.ResnetModel(1000, seed=0, depth=50, image=224); sc = resnet.ResnetScratch(B, 1000, depth=50, image=224)
    X, yy = resnet.synthetic_imagenet(B, 224, 1000, seed=0)
    x = torch.as_tensor(X, device="cuda"); yl = torch.as_tensor(yy, device="cuda")
    gr = torch.zeros(m.P, device="cuda"); loss = torch.zeros(1, device="cuda")
    for _ in range(3): resnet.forward_backward(m, sc, x, yl, gr, loss)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): resnet.forward_backward(m, sc, x, yl, gr, loss)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"ResNet-50 step B={B}: {ms:.3f} ms  ({24.3e9*B/ms/1e9:.1f} TFLOP/s, {B/ms*1e3:.0f} img/s)", flush=True)
    sys.exit(0)
B = 128
m = resnet.ResnetModel(seed=0); sc = resnet.ResnetScratch(B)
X, yy = resnet.synthetic_cifar(B, seed=0)
x = torch.as_tensor(X, device="cuda"); yl = torch.as_tensor(yy, device="cuda")
gr = torch.zeros(m.P, device="cuda"); loss = torch.zeros(1, device="cuda")
for _ in range(3): resnet.forward_backward(m, sc, x, yl, gr, loss)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(10): resnet.forward_backward(m, sc, x, yl, gr, loss)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"ResNet-18 step B=128: {ms:.3f} ms  ({3.33e9*B/ms/1e9:.1f} TFLOP/s)", flush=True)
