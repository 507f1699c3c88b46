"""Dev probe: ResNet-18 epoch slices with / without the spin disturbance."""
import sys, time, torch
from paper_2007_11831_b200 import cluster, resnet
from paper_2007_11831_b200.trainer import SimulatedTrainer
part = int(sys.argv[1]); nw = 4
X, y = resnet.synthetic_cifar(50000, seed=0)
tr = SimulatedTrainer(X, y, n_workers=nw, model="resnet18", seed=0, partition=bool(part), graphs=True, max_batch=512)
print("sms", [w.sm_count for w in tr.workers], flush=True)
for name, mult in [("clean", None), ("x1.5", 1.5), ("x2", 2.0), ("x4", 4.0), ("clean", None)]:
    prof = None if mult is None else [cluster.WorkerProfile(0, 1.0, disturbances=(cluster.DisturbanceEvent(0, cost_multiplier=mult),))] + [cluster.WorkerProfile(i,1.0) for i in range(1,nw)]
    for strat in ("fixed_ssgd", "dbs"):
        r = tr.run(cluster.StrategyConfig(strat, 512), n_epochs=3, profiles=prof, record_loss=False, max_iters=3*20)
        s = r.stats[-1]
        it = min(20, cluster.iterations_for_plan(s.plan))
        print(f"{name:6s} {strat:10s} ms/iter {s.epoch_wall_time/it*1e3:7.2f} gpu/iter {[round(g/it*1e3,2) for g in s.per_worker_gpu]} b={s.plan.int_batches}", flush=True)
