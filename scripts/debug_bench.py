import faulthandler, sys, time
faulthandler.dump_traceback_later(150, exit=True)
sys.argv = ["bench.py", "--steps", "2", "--warmup", "3", "--no-e2e", "--no-cpu"]
import bench
import torch
t0 = time.time()
def log(*a): print(f"[{time.time()-t0:7.2f}]", *a, file=sys.stderr, flush=True)
from paper_2007_11831_b200 import cluster
from paper_2007_11831_b200.mlp import synthetic_mnist
from paper_2007_11831_b200.trainer import SimulatedTrainer
X, y = synthetic_mnist(60000, 784, 10, seed=0); log("data")
tr = SimulatedTrainer(X, y, n_workers=3, seed=0, partition=True, max_batch=512); log("trainer", [w.sm_count for w in tr.workers])
prof = bench.disturbance_profiles(3)
for kind in ("fixed_ssgd", "dbs"):
    cfg = cluster.StrategyConfig(kind, 384)
    r = tr.run(cfg, n_epochs=3, profiles=prof, record_loss=False); log(kind, "warm", r.stats[-1].epoch_wall_time)
    s = bench.ClockSampler(0); s.start()
    r = tr.run(cfg, n_epochs=5, profiles=prof, record_loss=True); log(kind, "timed", r.stats[-1].epoch_wall_time)
    log(s.stop())
log("roof", bench.kernel_roofline(tr, bench.load_peaks()))
