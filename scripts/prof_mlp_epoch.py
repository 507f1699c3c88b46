"""Dev probe: where the time of one C1 (MLP, 3 shared-GPU workers) epoch goes --
kernel time by name (torch.profiler / CUPTI) and the epoch's wall time."""
import collections
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2007_11831_b200 import cluster  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

tr, _ = bench.make_trainer("mlp", 0)
w = bench.WL["mlp"]
prof = bench.profiles(w["workers"], None) if hasattr(bench, "profiles") else None
cfg = cluster.StrategyConfig("fixed_ssgd", w["workers"] * w["per_worker"])
profs = [cluster.WorkerProfile(0, 1.0, disturbances=(cluster.DisturbanceEvent(0, cost_multiplier=2.0),)),
         cluster.WorkerProfile(1, 1.0), cluster.WorkerProfile(2, 1.0)]
tr.run(cfg, n_epochs=2, profiles=profs)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as p:
    r = tr.run(cfg, n_epochs=1, profiles=profs)
    torch.cuda.synchronize()
print("epoch wall", r.stats[0].epoch_wall_time, "per-worker", r.stats[0].per_worker_gpu)
agg = collections.defaultdict(lambda: [0, 0.0])
for e in p.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        agg[e.name[:80]][0] += 1
        agg[e.name[:80]][1] += e.device_time_total
tot = sum(v[1] for v in agg.values())
print(f"kernel time {tot / 1e3:.2f} ms")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{t / 1e3:9.3f} ms {c:6d}x  {k}")
cpu = collections.defaultdict(lambda: [0, 0.0])
for e in p.events():
    if e.device_type == torch.autograd.DeviceType.CPU:
        cpu[e.name[:60]][0] += 1
        cpu[e.name[:60]][1] += e.cpu_time_total
print("host:")
for k, (c, t) in sorted(cpu.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"{t / 1e3:9.3f} ms {c:6d}x  {k}")
