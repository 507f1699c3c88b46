"""Debug: ResNet-50 device loss / gradients vs torch fp32 and bf16-storage torch."""
import sys, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from test_resnet50_gpu import torch_resnet50, tame_residual_branches
from paper_2007_11831_b200 import resnet
dev = torch.device("cuda:0")
image, classes, B = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
scale = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
model = resnet.ResnetModel(classes, depth=50, image=image,
                           params=tame_residual_branches(resnet.init_params(classes, 1, depth=50, image=image), scale))
sc = resnet.ResnetScratch(B + 3, classes, depth=50, image=image)
X, y = resnet.synthetic_imagenet(B, image=image, classes=classes, seed=3)
x = torch.as_tensor(X, device=dev); yl = torch.as_tensor(y, device=dev)
grad = torch.zeros(model.P, device=dev); loss = torch.zeros(1, device=dev)
resnet.forward_backward(model, sc, x, yl, grad, loss); torch.cuda.synchronize()
tensors = model.host_tensors()
xr = (x.float() - 128.0) / 64.0
b1, p1 = torch_resnet50(torch, tensors); l1 = torch.nn.functional.cross_entropy(b1(xr), yl.long()); l1.backward()
b2, p2 = torch_resnet50(torch, tensors, True); l2 = torch.nn.functional.cross_entropy(b2(xr), yl.long()); l2.backward()
print("loss dev", float(loss), "torch fp32", float(l1), "torch bf16", float(l2))
got = model.layout.unpack(grad.cpu().numpy())
for i, (a, b, g) in enumerate(zip(p1, p2, got)):
    r, r2 = a.grad.double().cpu().numpy(), b.grad.double().cpu().numpy()
    n = np.linalg.norm(r2 - r) / (np.linalg.norm(r) + 1e-30)
    e = np.linalg.norm(g - r) / (np.linalg.norm(r) + 1e-30)
    print(i, r.shape, "rel %.4f noise %.4f %s" % (e, n, "BAD" if e > 1.5 * n + 0.02 else ""))
