"""Generate tests/golden/mlp_trajectories.json by running the REFERENCE's own
synchronous S-SGD loop on the config-1 MLP.

Build container only (imports /root/reference/pkg/src):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_mlp_golden.py

The loop is dbsim.sgdlab.run_parallel_sgd (sgdlab.py:343-396) itself -- its
permutation stream, epoch layout, aggregation and heavy-ball step -- driving
the duck-typed Problem boundary (sgdlab.py:162) with oracle.MlpProblem, the
784-256-10 MLP in float64 (NO bf16 emulation).  SgdConfig.initial_point
(sgdlab.py:174) carries the MLP's initial weights (oracle.mlp_init).  DBS plans
come from dbsim.allocation.plan_next_epoch.  Recorded per iteration:
  * squared_distances with optimum 0 (||x_t||^2) and with optimum x_0
    (||x_t - x_0||^2, the displacement), straight from the reference;
  * the batch-weighted loss of the iteration (the adapter records each worker's
    batch loss as run_parallel_sgd requests its gradient, workers in order).
Floats are stored with float.hex().
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
REF = Path("/root/reference/pkg/src")
for p in (str(REF), str(ROOT)):
    if p not in sys.path:
        sys.path.insert(0, p)

from dbsim import allocation, sgdlab  # noqa: E402

from oracle import oracle as O  # noqa: E402


class RecordingMlp(O.MlpProblem):
    """MlpProblem that logs (batch loss, batch size) of every gradient request."""

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.log = []

    def per_sample_gradients(self, x, indices):
        idx = np.asarray(indices)
        loss, g = self.loss_and_grad(x, idx)
        self.log.append((loss, len(idx)))
        return g[None, :]


def synthetic_mnist(n, seed=0, in_dim=784, classes=10):
    """Same generator as the package's config-1 data."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, in_dim), dtype=np.float32)
    y = rng.integers(0, classes, size=n).astype(np.int32)
    return X, y


def run_case(name, D, data_seed, init_seed, n_workers, plan_source, iters, step, mom, aggregation, seed):
    X, y = synthetic_mnist(D, data_seed)
    x0 = O.mlp_init(seed=init_seed).astype(np.float64)
    out = {"name": name, "D": D, "data_seed": data_seed, "init_seed": init_seed, "n_workers": n_workers,
           "iters": iters, "step": step, "momentum": mom, "aggregation": aggregation, "seed": seed}
    if plan_source and isinstance(plan_source[0], allocation.PartitionPlan):
        out["plans"] = [{"int_batches": list(p.int_batches),
                         "cum": [0] + list(np.cumsum(p.int_batches).tolist())} for p in plan_source]
    else:
        out["fixed_batches"] = list(plan_source)
    for key, opt in (("sq_norm", np.zeros_like(x0)), ("sq_disp", x0)):
        prob = RecordingMlp(X, y)
        prob.optimum = opt
        cfg = sgdlab.SgdConfig(step_size=step, n_iterations=iters, momentum=mom, aggregation=aggregation,
                               seed=seed, initial_point=x0)
        traj = sgdlab.run_parallel_sgd(prob, cfg, n_workers, plan_source)
        out[key] = [float(v).hex() for v in traj.squared_distances]
        if key == "sq_norm":
            log = prob.log
            losses = []
            for t in range(iters):
                chunk = log[t * n_workers:(t + 1) * n_workers]
                tot = sum(b for _, b in chunk)
                losses.append(sum(l * b for l, b in chunk) / tot)
            out["losses"] = [float(v).hex() for v in losses]
    return out


def main():
    cases = [
        run_case("fixed_bw", 6000, 0, 0, 3, [128, 128, 128], 60, 0.05, 0.5, "batch_weighted", 0),
        run_case("fixed_uniform", 6000, 0, 0, 3, [128, 128, 128], 60, 0.05, 0.5, "uniform_average", 0),
    ]
    # a DBS stream: epoch 0 even, then the plan for a worker twice as slow (times = shares * cost)
    p0 = allocation.plan_next_epoch([1 / 3] * 3, [1.0] * 3, 384, 4000, 0)
    shares = p0.shares()
    p1 = allocation.plan_next_epoch(shares, [shares[0] * 2.0, shares[1], shares[2]], 384, 4000, 1)
    cases.append(run_case("dbs_plans", 4000, 2, 1, 3, [p0, p1], 40, 0.05, 0.5, "batch_weighted", 5))
    (HERE / "mlp_trajectories.json").write_text(json.dumps({"cases": cases}, indent=1))
    for c in cases:
        print(c["name"], c.get("plans") or c.get("fixed_batches"), float.fromhex(c["losses"][-1]))


if __name__ == "__main__":
    main()
