"""ncu target: warm-up + ONE ResNet-18 worker forward/backward (b=128), or the 64->64 conv alone."""
import sys, torch
sys.path.insert(0, ".")
from paper_2007_11831_b200 import resnet, _lib
what = sys.argv[1] if len(sys.argv) > 1 else "step"
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
if what == "conv":
    N, H, C = 128, 32, 64
    x = torch.randn(N, H, H, C, device="cuda").to(torch.bfloat16)
    w = (torch.randn(C, 3, 3, C, device="cuda") / 24).to(torch.bfloat16)
    y = torch.empty(N, H, H, C, dtype=torch.bfloat16, device="cuda")
    for _ in range(4):
        assert _lib.lib().dbs_dev_conv2d_fwd(x.data_ptr(), N, H, H, C, w.data_ptr(), C, 3, 1, 1, y.data_ptr(), _lib.stream_handle()) == 0
    torch.cuda.synchronize()
else:
    B = 128 if prec == "bf16" else 170
    m = resnet.ResnetModel(seed=0, precision=prec); sc = resnet.ResnetScratch(B, precision=prec)
    X, y = resnet.synthetic_cifar(B, seed=0)
    x = torch.as_tensor(X, device="cuda"); yl = torch.as_tensor(y, device="cuda")
    g = torch.zeros(m.P, device="cuda"); loss = torch.zeros(1, device="cuda")
    for _ in range(2): resnet.forward_backward(m, sc, x, yl, g, loss)
    torch.cuda.synchronize()
    resnet.forward_backward(m, sc, x, yl, g, loss)
    torch.cuda.synchronize()
