"""Dev probe: concurrency of worker streams, graphs, and the spin disturbance."""
import sys, time, torch
from paper_2007_11831_b200 import cluster, resnet, _lib
from paper_2007_11831_b200.trainer import SimulatedTrainer
X, y = resnet.synthetic_cifar(20000, seed=0)
def run(tag, **kw):
    prof = kw.pop("prof", None)
    tr = SimulatedTrainer(X, y, n_workers=4, model="resnet18", seed=0, max_batch=512, **kw)
    r = tr.run(cluster.StrategyConfig("fixed_ssgd", 512), n_epochs=1, profiles=prof, record_loss=False, max_iters=8)
    r = tr.run(cluster.StrategyConfig("fixed_ssgd", 512), n_epochs=1, profiles=prof, record_loss=False, max_iters=16)
    s = r.stats[-1]
    print(f"{tag:34s} ms/iter {s.epoch_wall_time/16*1e3:7.2f}  gpu/iter {[round(g/16*1e3,2) for g in s.per_worker_gpu]}", flush=True)
run("eager, shared SMs", partition=False, graphs=False)
run("graph, shared SMs", partition=False, graphs=True)
run("eager, green 4x32", partition=True, graphs=False)
run("graph, green 4x32", partition=True, graphs=True)
p2 = [cluster.WorkerProfile(0, 1.0, disturbances=(cluster.DisturbanceEvent(0, cost_multiplier=2.0),))] + [cluster.WorkerProfile(i,1.0) for i in range(1,4)]
run("eager, shared SMs, spin x2", partition=False, graphs=False, prof=p2)
run("eager, green 4x32, spin x2", partition=True, graphs=False, prof=p2)
# single worker with / without a co-running spin on another stream
m = resnet.ResnetModel(seed=0); sc = resnet.ResnetScratch(128)
x = torch.as_tensor(X[:128], device="cuda"); yl = torch.as_tensor(y[:128], device="cuda")
g = torch.zeros(m.P, device="cuda"); loss = torch.zeros(1, device="cuda")
for _ in range(3): resnet.forward_backward(m, sc, x, yl, g, loss)
stop = torch.zeros(1, dtype=torch.int32, device="cuda")
for ctas in (0, 37, 74, 111):
    side = torch.cuda.Stream()
    _lib.lib().dbs_dev_set_flag(stop.data_ptr(), 0, _lib.stream_handle())
    torch.cuda.synchronize()
    if ctas: _lib.lib().dbs_dev_spin_until(ctas, stop.data_ptr(), int(side.cuda_stream))
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): resnet.forward_backward(m, sc, x, yl, g, loss)
    e1.record()
    _lib.lib().dbs_dev_set_flag(stop.data_ptr(), 1, _lib.stream_handle())
    torch.cuda.synchronize()
    print(f"single worker B=128 with spin ctas={ctas:3d}: {e0.elapsed_time(e1)/10:.2f} ms/iter", flush=True)
