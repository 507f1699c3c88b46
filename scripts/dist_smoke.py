"""Multi-process smoke of DistributedTrainer: torchrun --nproc-per-node 2 (both ranks may share GPU 0).
Host collectives over gloo; the data path is the fused IPC/NVLink kernel."""
import os, sys, time, torch, torch.distributed as dist
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
ngpu = torch.cuda.device_count()
torch.cuda.set_device(rank % ngpu)
dist.init_process_group("gloo")
from paper_2007_11831_b200 import cluster
from paper_2007_11831_b200.trainer import DistributedTrainer
model = sys.argv[1] if len(sys.argv) > 1 else "mlp"
prec = sys.argv[3] if len(sys.argv) > 3 else "f32"
wpr = int(sys.argv[4]) if len(sys.argv) > 4 else 1  # workers per rank (> 1: SM partitions, per-worker graphs)
tr = DistributedTrainer(2000 if model == "mlp" else 1024, workers_per_rank=wpr, model=model, seed=0,
                        partition=wpr > 1, max_batch=256, precision=prec)
t = time.time()
avg = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else None  # model averaging every `avg` iterations
r = tr.run(cluster.StrategyConfig("dbs", 128 * world * wpr), n_epochs=2, max_iters=6, record_loss=True,
           averaging_interval=avg)
torch.cuda.synchronize()
p = tr.comm.params[:1024].double().sum().item()
ps = [None] * world
dist.all_gather_object(ps, p)
print(f"rank {rank}: plans {[pl.int_batches for pl in r.plans]} losses {[round(float(v),4) for v in r.losses]} "
      f"param-sum agree {len(set(ps)) == 1} ({time.time()-t:.1f}s)", flush=True)
dist.destroy_process_group()
