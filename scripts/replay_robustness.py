"""Replay the reference's `robustness` scenario on a B200 (the
paper's Fig. 4 experiment): 4 ResNet-18 workers (disjoint 32-SM partitions), 41
epochs, B = 512, D = 50000; background jobs start on workers 0 / 1 / 2 at epochs
10 / 21 / 31 and stay (scenarios.py:287-309 adds a flat 10 s of compute there;
here the background job is a co-running spin kernel that pins half of the
worker's SMs -- the hardware form of the same disturbance).  Fixed-batch S-SGD and
DBS run the same schedule; every epoch's MEASURED EpochStats are written in the
reference's report format and summarised next to the reference simulator's
prediction for the same shape of schedule.

    python scripts/replay_robustness.py [--epochs 41] [--out profiles/robustness_r1]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--epochs", type=int, default=41)
    ap.add_argument("--out", default=str(ROOT / "profiles" / "robustness_r1"))
    ap.add_argument("--dataset", type=int, default=50000)
    ap.add_argument("--starts", default="10,21,31", help="epochs at which workers 0, 1, 2 get a background job")
    args = ap.parse_args()

    import torch

    from paper_2007_11831_b200 import cluster, report
    from paper_2007_11831_b200.resnet import synthetic_cifar
    from paper_2007_11831_b200.trainer import SimulatedTrainer

    torch.cuda.set_device(0)
    X, y = synthetic_cifar(args.dataset, seed=0)
    tr = SimulatedTrainer(X, y, n_workers=4, model="resnet18", seed=0, partition=True, max_batch=384)
    starts = {w: int(e) for w, e in enumerate(args.starts.split(","))}
    profiles = [cluster.WorkerProfile(w, 1.0, disturbances=((cluster.DisturbanceEvent(starts[w], cost_multiplier=2.0),)
                                                             if w in starts else ()))
                for w in range(4)]
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    reports, summary = [], {}
    for kind in ("fixed_ssgd", "dbs"):
        res = tr.run(cluster.StrategyConfig(kind, 512), n_epochs=args.epochs, lr=0.05, momentum=0.9,
                     profiles=profiles, record_loss=False)
        rep = report.RunReport.from_stats("robustness_b200", kind, 0, res.stats)
        report.write_epoch_csv(rep, out / f"robustness_b200_{kind}.csv")
        reports.append(rep)
        walls = [s.epoch_wall_time for s in res.stats]
        summary[kind] = {"total_s": round(sum(walls), 3), "epoch_wall_s": [round(v, 4) for v in walls],
                         "plans": [list(s.plan.int_batches) for s in res.stats]}
    report.write_run_json(reports, [], out / "robustness_b200.json")
    fixed, dbs = summary["fixed_ssgd"]["total_s"], summary["dbs"]["total_s"]
    summary["saving_measured"] = round(1.0 - dbs / fixed, 4)
    # DBS re-balancing latency: epochs after each disturbance start until the plan moves
    lat = {}
    for w, e0 in starts.items():
        plans = summary["dbs"]["plans"]
        before = plans[e0 - 1][w] if e0 >= 1 else None
        lat[w] = next((e - e0 for e in range(e0, len(plans)) if before is not None and plans[e][w] < before), None)
    summary["rebalance_epochs_after_start"] = lat
    # the reference simulator on the same schedule shape (uniform workers, 2x cost from the start epochs)
    sim = {}
    for kind in ("fixed_ssgd", "dbs"):
        st = cluster.run_training([cluster.WorkerProfile(w, 1e-3, disturbances=p.disturbances)
                                   for w, p in enumerate(profiles)], cluster.StrategyConfig(kind, 512),
                                  args.dataset, args.epochs)
        sim[kind] = sum(s.epoch_wall_time for s in st)
    summary["saving_reference_simulator"] = round(1.0 - sim["dbs"] / sim["fixed_ssgd"], 4)
    (out / "summary.json").write_text(json.dumps(summary, indent=1))
    print(json.dumps({k: v for k, v in summary.items() if k not in ("fixed_ssgd", "dbs")} |
                     {"fixed_total_s": fixed, "dbs_total_s": dbs}), flush=True)


if __name__ == "__main__":
    main()
