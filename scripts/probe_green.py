"""Probe: green-context SM partitions + spin disturbance on the MLP epoch (dev tool)."""
import time, sys
import numpy as np
import torch
from paper_2007_11831_b200 import cluster, mlp
from paper_2007_11831_b200.trainer import SimulatedTrainer, make_workers, _green_supported

print("green supported", _green_supported(), flush=True)
X, y = mlp.synthetic_mnist(60000, seed=0)
for partition in (False, True):
    try:
        tr = SimulatedTrainer(X, y, n_workers=3, seed=0, partition=partition)
    except Exception as e:
        print("partition", partition, "failed:", repr(e)); continue
    print("partition", partition, "sms", [w.sm_count for w in tr.workers], flush=True)
    for kind, prof in [("none", None),
                       ("sm75", [cluster.WorkerProfile(0, 1.0, disturbances=(cluster.DisturbanceEvent(0, cost_multiplier=4.0),)), cluster.WorkerProfile(1,1.0), cluster.WorkerProfile(2,1.0)]),
                       ("extra", [cluster.WorkerProfile(0, 1.0, disturbances=(cluster.DisturbanceEvent(0, extra_epoch_seconds=0.02),)), cluster.WorkerProfile(1,1.0), cluster.WorkerProfile(2,1.0)])]:
        for strat in ("fixed_ssgd", "dbs"):
            t0 = time.time()
            res = tr.run(cluster.StrategyConfig(strat, 384), n_epochs=4, profiles=prof, record_loss=False)
            s = res.stats[-1]
            print(f"{kind:6s} {strat:10s} wall/epoch {s.epoch_wall_time*1e3:8.2f} ms  gpu {[round(g*1e3,2) for g in s.per_worker_gpu]} "
                  f"b={s.plan.int_batches} samples/s {sum(s.plan.int_batches)*cluster.iterations_for_plan(s.plan)/s.epoch_wall_time:,.0f} host {time.time()-t0:.2f}s", flush=True)
