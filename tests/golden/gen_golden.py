"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_golden.py

Every fixture is produced by the reference's own functions (dbsim.allocation,
dbsim.cluster, dbsim.sgdlab) and by numpy's Generator -- the reference's
pinned third-party dependency for sample assignment (sgdlab.py:358, 372-374).
Floats are stored with float.hex() so comparisons are bit-exact.
"""

from __future__ import annotations

import hashlib
import json
import math
import random
import sys
from fractions import Fraction
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg/src")
if str(REF) not in sys.path:
    sys.path.insert(0, str(REF))

from dbsim import allocation, cluster, errors, sgdlab  # noqa: E402
from dbsim.scenarios import builtin_scenarios  # noqa: E402


def hx(v: float) -> str:
    return float(v).hex()


def err_name(fn, *a):
    try:
        return None, fn(*a)
    except errors.DbsError as exc:
        return type(exc).__name__, None
    except (OverflowError, ValueError, IndexError) as exc:
        return type(exc).__name__, None


def plan_record(plan):
    total = plan.ranges[-1][1].denominator if plan.ranges else 1
    # ranges are Fraction(cum_i, sum b); store the un-normalised numerators
    sb = sum(plan.int_batches)
    cum = [0]
    for b in plan.int_batches:
        cum.append(cum[-1] + b)
    assert all(Fraction(cum[i], sb) == plan.ranges[i][0] for i in range(len(cum) - 1))
    del total
    return {
        "int_batches": list(plan.int_batches),
        "cum": cum,
        "spans": [list(s) for s in plan.sample_spans],
    }


def gen_plan_cases(rng: random.Random):
    cases = []
    fixed = [
        ([0.25] * 4, [1 / 13.7, 1 / 16.5, 1 / 19.6, 1 / 14.2], 64, 50000, 1),  # test_allocation.py:236
        ([0.25] * 4, [1.0, 1.0, 1.0, 1000.0], 8, 100, 1),  # zero lift, :264-268
        ([0.9, 0.01, 0.05, 0.04], [99.0, 1.0, 2.0, 3.0], 64, 50000, 0),  # epoch 0, :227
        ([0.25] * 4, [4.0] * 4, 64, 50000, 1),
        ([1 / 3] * 3, [1.0, 1.0, 1.0], 128, 60000, 0),  # C1 epoch 0 (43,43,42)
        ([1 / 7] * 7, [1.0] * 7, 512, 50000, 0),  # deficit 511
        ([0.5, 0.5], [1.0, -1.0], 8, 100, 1),  # InvalidMeasurement
        ([0.5, 0.5], [1.0, 1.0], 1, 100, 1),  # BudgetTooSmall
        ([0.5, 1.5], [1.0, 1.0], 8, 100, 1),  # share > 1
        ([0.5, 0.5], [1.0, float("inf")], 8, 100, 1),
        ([0.5, 0.5], [1.0, float("nan")], 8, 100, 1),
        ([0.5, 0.5], [1.0, 1.0], 8, 1, 1),  # DatasetTooSmall
        ([1.0], [3.0], 1, 1, 5),
        ([1.0], [3.0], 512, 50000, 7),
    ]
    for sh, tm, B, D, ep in fixed:
        cases.append((sh, tm, B, D, ep))
    for _ in range(700):
        n = rng.randint(1, 16)
        w = [rng.random() + 1e-3 for _ in range(n)]
        s = sum(w)
        shares = [x / s for x in w]
        style = rng.random()
        if style < 0.3:
            times = [s_ / (rng.lognormvariate(0, 0.5)) for s_ in shares]
        elif style < 0.6:
            times = [rng.uniform(0.01, 100.0) for _ in range(n)]
        else:
            times = [10 ** rng.uniform(-6, 3) for _ in range(n)]
        B = rng.choice([n, n + 1, rng.randint(n, 64), rng.randint(n, 4096), 128, 384, 512, 1024])
        D = rng.choice([n, rng.randint(n, 5000), 50000, 60000, 100000, rng.randint(n, 10**7)])
        ep = rng.choice([0, 1, 1, 1, 2, 9])
        cases.append((shares, times, B, D, ep))
    out = []
    for sh, tm, B, D, ep in cases:
        e, plan = err_name(allocation.plan_next_epoch, sh, tm, B, D, ep)
        rec = {
            "shares": [hx(x) for x in sh],
            "times": [hx(x) for x in tm],
            "B": B,
            "D": D,
            "epoch": ep,
            "error": e,
        }
        if plan is not None:
            rec.update(plan_record(plan))
        out.append(rec)
    return out


def gen_fraction_cases(rng: random.Random):
    out = []
    vals_list = [[13.7, 16.5, 19.6, 14.2], [1, 1, 1, 1], [0.025, 0.05, 0.025], [1.0, 0.0], [],
                 [1e308, 1e308], [1e-300, 1.0, 1e16], [float("nan"), 1.0], [-1.0, 2.0]]
    for _ in range(600):
        n = rng.randint(1, 12)
        kind = rng.random()
        if kind < 0.5:
            vals_list.append([rng.uniform(0.01, 100.0) for _ in range(n)])
        else:
            vals_list.append([10 ** rng.uniform(-30, 30) for _ in range(n)])
    for vals in vals_list:
        perfs = [allocation.PerfEstimate(i, float(v)) for i, v in enumerate(vals)]
        e, fr = err_name(allocation.compute_batch_fractions, perfs)
        naive = None
        if fr is not None:
            naive = 0.0
            for v in vals:  # plain left-to-right sum (builtin sum() is compensated in 3.12)
                naive += v
        out.append({
            "perfs": [hx(v) for v in vals],
            "error": e,
            "fractions": [hx(v) for v in fr] if fr is not None else None,
            "fsum": hx(math.fsum(vals)) if fr is not None else None,
            "fsum_differs_from_naive": (fr is not None and naive != math.fsum(vals)),
        })
    return out


def gen_round_cases(rng: random.Random):
    out = []
    fixed = [([13.7, 16.5, 19.6, 14.2], 64), ([8.0] * 4, 32), ([5.4, 5.3, 5.3], 16),
             ([3.5, 3.5, 4.0], 11), ([-0.1, 5.0], 5), ([0.5, 0.5, 0.5], 1), ([2.5, 2.5], 3)]
    for r, b in fixed:
        out.append((r, b))
    for _ in range(800):
        n = rng.randint(1, 10)
        budget = rng.randint(max(n, 1), 200)
        w = [rng.random() + 1e-3 for _ in range(n)]
        reals = [x * budget / sum(w) for x in w]
        if rng.random() < 0.2:  # exact halves to exercise ties
            reals = [math.floor(x) + 0.5 for x in reals]
        out.append((reals, budget))
    rec = []
    for reals, b in out:
        e, ints = err_name(allocation.round_twice, reals, b)
        rec.append({"reals": [hx(x) for x in reals], "budget": b, "error": e, "ints": ints})
    return rec


def gen_zero_lift_cases(rng: random.Random):
    rec = []
    for _ in range(300):
        n = rng.randint(1, 10)
        b = [rng.choice([0, 0, 1, 2, rng.randint(0, 50)]) for _ in range(n)]
        rec.append({"in": b, "out": allocation._raise_zero_batches(b)})
    return rec


def bound_json(x):
    if isinstance(x, Fraction):
        return {"kind": 0, "num": x.numerator, "den": x.denominator}
    if isinstance(x, int):
        return {"kind": 0, "num": x, "den": 1}
    return {"kind": 1, "value": hx(x)}


def gen_span_cases(rng: random.Random):
    cases = [([(0, 0.5), (0.5, 1)], 10), ([(0, 1)], 7), ([(0, 0.5), (0.5, 1)], 1)]
    cases.append((allocation.partition_ranges([14, 16, 20, 14]), 50000))
    cases.append((allocation.partition_ranges([1, 100, 1]), 3))
    for _ in range(600):
        n = rng.randint(1, 12)
        b = [rng.randint(0, 60) for _ in range(n)]
        if sum(b) == 0:
            b[0] = 1
        D = rng.choice([n, n + rng.randint(0, 10), rng.randint(n, 100000)])
        rngs = allocation.partition_ranges(b)
        if rng.random() < 0.15:
            rngs = [(float(lo), float(hi)) for lo, hi in rngs]
        cases.append((rngs, D))
    rec = []
    for rngs, D in cases:
        e, spans = err_name(allocation.spans_from_ranges, rngs, D)
        rec.append({
            "lo": [bound_json(lo) for lo, _ in rngs],
            "hi": [bound_json(hi) for _, hi in rngs],
            "D": D,
            "error": e,
            "spans": [list(s) for s in spans] if spans is not None else None,
        })
    return rec


def gen_plan_streams():
    """Epoch-by-epoch DBS plans of cluster.run_training (cluster.py:234-275)."""
    out = []
    scen = builtin_scenarios()
    runs = []
    for name in ("scale4", "scale8", "scale16", "robustness", "homogeneous"):
        cfg = scen[name]
        strat = next(s for s in cfg.strategies if s.kind == "dbs")
        runs.append((name, cfg.profiles(), strat, cfg.dataset_size, cfg.n_epochs))
    prof = [cluster.WorkerProfile(i, 1e-4 * 2 ** (i / 3)) for i in range(4)]
    runs.append(("smooth0.5", prof, cluster.StrategyConfig("dbs", 512, perf_smoothing=0.5), 50000, 30))
    prof3 = [cluster.WorkerProfile(i, c) for i, c in enumerate([1e-4, 1.7e-4, 2.9e-4])]
    runs.append(("c1_b128", prof3, cluster.StrategyConfig("dbs", 128), 60000, 12))
    prof8 = [cluster.WorkerProfile(i, 2e-4 if i < 2 else 1e-4) for i in range(8)]
    runs.append(("c3_2x_ranks01", prof8, cluster.StrategyConfig("dbs", 512), 50000, 8))
    for name, profiles, strat, D, E in runs:
        stats = cluster.run_training(profiles, strat, D, E)
        out.append({
            "name": name,
            "B": strat.total_budget,
            "D": D,
            "smoothing": hx(strat.perf_smoothing),
            "epochs": [
                dict(plan_record(s.plan), times=[hx(t) for t in s.per_worker_gpu],
                     iters=cluster.iterations_for_plan(s.plan))
                for s in stats
            ],
        })
    return out


def gen_permutations():
    out = []
    cases = [
        (0, [(0, 20000)]),
        (0, [(0, 20156), (20156, 40312), (40312, 60000)]),
        (1, [(0, 7)]),
        (42, [(0, 1), (1, 3), (3, 3), (3, 1000)]),
        (12345, [(0, 3613), (3613, 7226), (7226, 14355), (14355, 21484), (21484, 28613),
                 (28613, 35742), (35742, 42871), (42871, 50000)]),
        (7, [(0, 65536), (65536, 70000)]),
        (3, [(0, 513)] ),
    ]
    for seed, spans in cases:
        g = np.random.default_rng(seed)
        st0 = g.bit_generator.state
        epochs = []
        for _ in range(2):  # two epochs back to back from one generator
            perms = [start + g.permutation(end - start) for start, end in spans]
            flat = np.concatenate(perms).astype(np.int64) if perms else np.zeros(0, np.int64)
            epochs.append({
                "sha256": hashlib.sha256(flat.tobytes()).hexdigest(),
                "head": flat[:16].tolist(),
                "tail": flat[-16:].tolist(),
                "state_after": {k: str(v) for k, v in g.bit_generator.state["state"].items()},
                "has_uint32": int(g.bit_generator.state["has_uint32"]),
                "uinteger": int(g.bit_generator.state["uinteger"]),
            })
        out.append({
            "seed": seed,
            "spans": [list(s) for s in spans],
            "state0": {k: str(v) for k, v in st0["state"].items()},
            "epochs": epochs,
        })
    return out


def gen_sgd_trajectories():
    """run_parallel_sgd (sgdlab.py:343-396) on the reference's own problems."""
    recs = []
    quad = sgdlab.ConvexProblem.quadratic(dimension=8, mu=1.0, sample_noise_scale=0.5,
                                          sample_count=4096, seed=0)
    plans = __import__("dbsim.checks", fromlist=["x"]).adaptive_plan_stream(4, 64, 4096, 6)
    logit = sgdlab.LogisticProblem.synthetic(dimension=16, mu=0.1, sample_count=1000, seed=0)
    configs = [
        ("quad_fixed", quad, sgdlab.SgdConfig(step_size=0.02, n_iterations=200, momentum=0.5, seed=0), 4, [16] * 4),
        ("quad_dbs", quad, sgdlab.SgdConfig(step_size=0.02, n_iterations=200, momentum=0.5, seed=3), 4, plans),
        ("quad_uniform", quad, sgdlab.SgdConfig(step_size=0.05, n_iterations=150, momentum=0.0,
                                                aggregation="uniform_average", seed=1), 4, plans),
        ("logit_fixed", logit, sgdlab.SgdConfig(step_size=0.5, n_iterations=120, momentum=0.5, seed=4), 2, [16, 16]),
        ("logit_dbs", logit, sgdlab.SgdConfig(step_size=0.5, n_iterations=120, momentum=0.5, seed=4), 4,
         __import__("dbsim.checks", fromlist=["x"]).adaptive_plan_stream(4, 64, 1000, 8)),
    ]
    for name, prob, cfg, n, src in configs:
        traj = sgdlab.run_parallel_sgd(prob, cfg, n, src)
        recs.append({
            "name": name,
            "squared_distances": [hx(v) for v in traj.squared_distances],
            "final_loss": hx(traj.final_loss),
        })
    return recs


def gen_equivalence():
    """checks.check_dbs_equivalence (checks.py:185-244) at a small size."""
    from dbsim import checks

    quad = sgdlab.ConvexProblem.quadratic(dimension=8, mu=1.0, sample_noise_scale=0.5, sample_count=4096, seed=0)
    res = checks.check_dbs_equivalence(quad, n_workers=4, total_budget=64, n_seeds=6, n_iterations=200, seed=2)
    return {"args": {"n_workers": 4, "total_budget": 64, "n_seeds": 6, "n_iterations": 200, "seed": 2},
            "final_gap_fixed": hx(res.final_gap_fixed), "final_gap_dynamic": hx(res.final_gap_dynamic),
            "relative_gap_diff": hx(res.relative_gap_diff), "max_trajectory_z": hx(res.max_trajectory_z),
            "passed": bool(res.passed)}


def gen_reports():
    """The reference's report formats (report.py) for a simulated scenario: the
    scenario definition, the DBS run's long CSV, the run JSON of every strategy
    and the savings table against fixed S-SGD."""
    from dbsim import report

    scen = builtin_scenarios()["robustness"]
    profs = scen.profiles()
    reports = []
    for strat in scen.strategies:
        stats = cluster.run_training(profs, strat, scen.dataset_size, scen.n_epochs)
        reports.append(report.RunReport.from_stats(scen.name, strat.kind, 0, stats))
    csv_path = HERE / "report_robustness_dbs.csv"
    report.write_epoch_csv(next(r for r in reports if r.strategy == "dbs"), csv_path)
    json_path = HERE / "report_robustness.json"
    report.write_run_json(reports, [], json_path)
    table = report.compare_strategies(reports, "fixed_ssgd")
    definition = {
        "name": scen.name, "dataset_size": scen.dataset_size, "n_epochs": scen.n_epochs,
        "profiles": [{"worker_id": p.worker_id, "base_cost": hx(p.base_cost),
                      "per_iteration_overhead": hx(p.per_iteration_overhead),
                      "disturbances": [{"start_epoch": d.start_epoch, "end_epoch": d.end_epoch,
                                        "extra_epoch_seconds": None if d.extra_epoch_seconds is None
                                        else hx(d.extra_epoch_seconds),
                                        "cost_multiplier": None if d.cost_multiplier is None
                                        else hx(d.cost_multiplier)} for d in p.disturbances]}
                     for p in profs],
        "strategies": [{"kind": s.kind, "total_budget": s.total_budget, "sync_interval": s.sync_interval,
                        "sync_cost_per_round": hx(s.sync_cost_per_round),
                        "sync_cost_per_worker": hx(s.sync_cost_per_worker),
                        "perf_smoothing": hx(s.perf_smoothing)} for s in scen.strategies],
        "savings": [[k, hx(t), hx(v)] for k, t, v in table],
    }
    return definition


def main():
    rng = random.Random(20072011831)
    data = {
        "numpy_version": np.__version__,
        "plan_next_epoch": gen_plan_cases(rng),
        "compute_batch_fractions": gen_fraction_cases(rng),
        "round_twice": gen_round_cases(rng),
        "raise_zero_batches": gen_zero_lift_cases(rng),
        "spans_from_ranges": gen_span_cases(rng),
    }
    (HERE / "controller.json").write_text(json.dumps(data, separators=(",", ":")))
    (HERE / "plan_streams.json").write_text(json.dumps(gen_plan_streams(), separators=(",", ":")))
    (HERE / "permutation.json").write_text(json.dumps(gen_permutations(), indent=1))
    (HERE / "sgd_trajectories.json").write_text(json.dumps(gen_sgd_trajectories(), separators=(",", ":")))
    (HERE / "report_scenario.json").write_text(json.dumps(gen_reports(), indent=1))
    (HERE / "equivalence.json").write_text(json.dumps(gen_equivalence(), indent=1))
    for p in sorted(HERE.glob("*.json")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
