"""Dev probe: library green-context partitions -- concurrency and per-worker disturbance."""
import sys, time, torch
from paper_2007_11831_b200 import cluster, resnet
from paper_2007_11831_b200.trainer import SimulatedTrainer
X, y = resnet.synthetic_cifar(20000, seed=0)
def run(tag, prof, **kw):
    tr = SimulatedTrainer(X, y, n_workers=4, model="resnet18", seed=0, max_batch=512, **kw)
    for strat in ("fixed_ssgd", "dbs"):
        r = tr.run(cluster.StrategyConfig(strat, 512), n_epochs=3, profiles=prof, record_loss=False, max_iters=3*24)
        s = r.stats[-1]; it = cluster.iterations_for_plan(s.plan)
        it = min(it, 24)
        print(f"{tag:28s} {strat:10s} ms/iter {s.epoch_wall_time/it*1e3:7.2f} gpu/iter {[round(g/it*1e3,2) for g in s.per_worker_gpu]} b={s.plan.int_batches}", flush=True)
p2 = [cluster.WorkerProfile(0, 1.0, disturbances=(cluster.DisturbanceEvent(0, cost_multiplier=2.0),))] + [cluster.WorkerProfile(i,1.0) for i in range(1,4)]
run("green 4x32 clean", None, partition=True)
run("green 4x32 spin x2 (pin)", p2, partition=True)
run("shared graph slow x2", p2, partition=False)
