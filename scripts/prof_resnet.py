"""Dev probe: kernel-time breakdown (torch.profiler/CUPTI) of ResNet-18 worker iterations."""
import sys, collections, torch
sys.path.insert(0, ".")
from torch.profiler import profile, ProfilerActivity
from paper_2007_11831_b200 import resnet, cluster
from paper_2007_11831_b200.trainer import SimulatedTrainer
mode = sys.argv[1]
def summarize(prof, title):
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            k = e.name[:90]
            agg[k][0] += 1; agg[k][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    tot = sum(v[1] for v in agg.values())
    print(f"== {title}: total kernel time {tot/1e3:.2f} ms")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
        print(f"{t/1e3:9.3f} ms {c:6d}x  {k}")
if mode == "single50":
    B = 64
    m = resnet.ResnetModel(1000, seed=0, depth=50, image=224); sc = resnet.ResnetScratch(B, 1000, depth=50, image=224)
    X, y = resnet.synthetic_imagenet(B, 224, 1000, seed=0)
    x = torch.as_tensor(X, device="cuda"); yl = torch.as_tensor(y, device="cuda")
    g = torch.zeros(m.P, device="cuda"); loss = torch.zeros(1, device="cuda")
    for _ in range(3): resnet.forward_backward(m, sc, x, yl, g, loss)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(2): resnet.forward_backward(m, sc, x, yl, g, loss)
        torch.cuda.synchronize()
    summarize(prof, "ResNet-50 single worker B=64 x2")
    sys.exit(0)
if mode == "single":
    B = 128
    m = resnet.ResnetModel(seed=0); sc = resnet.ResnetScratch(B)
    X, y = resnet.synthetic_cifar(B, seed=0)
    x = torch.as_tensor(X, device="cuda"); yl = torch.as_tensor(y, device="cuda")
    g = torch.zeros(m.P, device="cuda"); loss = torch.zeros(1, device="cuda")
    for _ in range(3): resnet.forward_backward(m, sc, x, yl, g, loss)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(2): resnet.forward_backward(m, sc, x, yl, g, loss)
        torch.cuda.synchronize()
    summarize(prof, "single worker B=128 x2")
elif mode == "part":
    # the bench layout: 3 workers on disjoint 48-SM partitions, 170 samples each
    X, y = resnet.synthetic_cifar(8000, seed=0)
    tr = SimulatedTrainer(X, y, n_workers=3, model="resnet18", partition=True, graphs=False, max_batch=210)
    tr.run(cluster.StrategyConfig("fixed_ssgd", 510), n_epochs=1, max_iters=2)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        r = tr.run(cluster.StrategyConfig("fixed_ssgd", 510), n_epochs=1, max_iters=4)
        torch.cuda.synchronize()
    summarize(prof, "trainer 3 workers x 48 SMs, 4 iterations")
else:
    X, y = resnet.synthetic_cifar(8000, seed=0)
    tr = SimulatedTrainer(X, y, n_workers=4, model="resnet18", partition=False, graphs=False, max_batch=512)
    tr.run(cluster.StrategyConfig("fixed_ssgd", 512), n_epochs=1, max_iters=2)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        r = tr.run(cluster.StrategyConfig("fixed_ssgd", 512), n_epochs=1, max_iters=2)
        torch.cuda.synchronize()
    print("epoch wall", r.stats[0].epoch_wall_time, "gpu", r.stats[0].per_worker_gpu)
    summarize(prof, "trainer 4 workers x 2 iterations")
