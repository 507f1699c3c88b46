"""Dev probe: per-kernel-phase timing of one ResNet-18 worker iteration (CUDA events)."""
import sys, time, torch
from paper_2007_11831_b200 import resnet, _lib
B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
m = resnet.ResnetModel(seed=0); sc = resnet.ResnetScratch(B)
X, y = resnet.synthetic_cifar(B, seed=0)
x = torch.as_tensor(X, device="cuda"); yl = torch.as_tensor(y, device="cuda")
g = torch.zeros(m.P, device="cuda"); loss = torch.zeros(1, device="cuda")
for _ in range(3): resnet.forward_backward(m, sc, x, yl, g, loss)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(10): resnet.forward_backward(m, sc, x, yl, g, loss)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"B={B}: {ms:.3f} ms / fwd+bwd  -> {B/ms*1e3:,.0f} samples/s  ({3.33e9*B/ms/1e9:,.1f} TFLOP/s)", flush=True)
