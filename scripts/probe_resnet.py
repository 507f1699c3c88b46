"""Dev probe: ResNet-18 DBS epochs with simulated workers (each variant in a subprocess)."""
import os, subprocess, sys
VARIANT = r'''
import sys, time, torch, faulthandler
faulthandler.dump_traceback_later(170, exit=True)
from paper_2007_11831_b200 import cluster, resnet
from paper_2007_11831_b200.trainer import SimulatedTrainer
part, graphs, nw = [int(x) for x in sys.argv[1:4]]
X, y = resnet.synthetic_cifar(50000, seed=0)
t0 = time.time()
tr = SimulatedTrainer(X, y, n_workers=nw, model="resnet18", seed=0, partition=bool(part), graphs=bool(graphs), max_batch=512)
print("init", round(time.time()-t0,2), "sms", [w.sm_count for w in tr.workers], flush=True)
prof = [cluster.WorkerProfile(0, 1.0, disturbances=(cluster.DisturbanceEvent(0, cost_multiplier=2.0),))] + [cluster.WorkerProfile(i,1.0) for i in range(1,nw)]
for strat in ("fixed_ssgd", "dbs"):
    t = time.time()
    r = tr.run(cluster.StrategyConfig(strat, 512), n_epochs=4, profiles=prof, record_loss=True)
    for s in r.stats:
        print(strat, s.epoch, "wall", round(s.epoch_wall_time*1e3,1), "ms gpu", [round(g*1e3,1) for g in s.per_worker_gpu], "b", s.plan.int_batches, "sps", round(sum(s.plan.int_batches)*cluster.iterations_for_plan(s.plan)/s.epoch_wall_time), flush=True)
    print(strat, "loss", [round(float(v),3) for v in r.losses[::40]], "host", round(time.time()-t,1), flush=True)
'''
for v in [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]]:
    p = subprocess.run([sys.executable, "-c", VARIANT, *map(str, v)], capture_output=True, text=True, timeout=200, env=dict(os.environ, PYTHONPATH="."))
    print("=== variant part,graphs,nw", v, "rc", p.returncode, flush=True)
    print("\n".join((p.stdout + p.stderr).strip().splitlines()[-24:]), flush=True)
