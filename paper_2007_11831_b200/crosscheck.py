"""Simulator-vs-measurement cross-check.

The reference predicts an epoch from a cost law (cluster.py:123-145, 192-220):

    gpu_w  = effective_cost_w(e) * T * b_w + per_iteration_overhead_w * T (+ extra_epoch_seconds)
    wall   = max_w gpu_w + rounds(e) * (sync_cost_per_round + sync_cost_per_worker * n)

This module fits that law to MEASURED EpochStats of the B200 trainer (least
squares per worker for base_cost and per_iteration_overhead, with the
scenario's declared disturbance multipliers; one sync cost per round), replays
every measured plan through the reference's own run_epoch with the fitted
profiles, and reports the per-epoch prediction error -- so a GPU run can be
compared line by line with what the reference's simulator says for the same
plans, and a whole DBS run can be re-simulated (run_training) with the fitted
profiles.  Host-side bookkeeping only: no device work.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import cluster
from .cluster import EpochStats, StrategyConfig, WorkerProfile
from .errors import ConfigurationError


@dataclass(frozen=True)
class FittedCosts:
    base_cost: tuple          # seconds per sample, per worker (undisturbed)
    per_iteration_overhead: tuple  # seconds per iteration, per worker
    sync_cost_per_round: float
    residual_rel: float       # RMS of (fit - measured) / measured over the fitted points
    multiplier: tuple = ()    # fit_multiplier: the MEASURED cost multiplier of each worker's disturbed epochs


def _multiplier(profile: Optional[WorkerProfile], epoch: int) -> float:
    if profile is None:
        return 1.0
    return cluster.effective_cost(profile, epoch) / profile.base_cost


def _extra(profile: Optional[WorkerProfile], epoch: int) -> float:
    if profile is None:
        return 0.0
    t = 0.0
    for d in profile.disturbances:
        if d.extra_epoch_seconds is not None and d.active(epoch):
            t += d.extra_epoch_seconds
    return t


def fit_costs(runs: Sequence[tuple], profiles: Optional[Sequence[WorkerProfile]] = None,
              skip_epochs: int = 1, fit_multiplier: bool = False) -> FittedCosts:
    """Least-squares fit of the reference's cost law to measured epochs.

    runs: (StrategyConfig, [EpochStats]) pairs measured on the same workers.
    profiles: the scenario's WorkerProfiles (disturbance schedule; base costs
    are ignored), or None for undisturbed workers.  The first `skip_epochs` of
    every run (warm-up: graph capture, lazy loading) are left out.
    fit_multiplier: the cost of a worker's disturbed epochs is a free parameter
    (reported as `multiplier`, measured / base) instead of the declared one --
    how much a co-running job that pins a fraction of the SMs really slows it."""
    if not runs:
        raise ConfigurationError("no runs to fit")
    n = len(runs[0][1][0].per_worker_gpu)
    rows = [[] for _ in range(n)]
    ys = [[] for _ in range(n)]
    sx, sy = [], []
    for config, stats in runs:
        for s in stats[skip_epochs:]:
            T = cluster.iterations_for_plan(s.plan)
            if T <= 0:
                continue
            for w in range(n):
                prof = profiles[w] if profiles is not None else None
                m = _multiplier(prof, s.epoch)
                tb = T * s.plan.int_batches[w]
                if fit_multiplier:  # [undisturbed samples, disturbed samples, iterations]
                    rows[w].append((tb if m == 1.0 else 0.0, tb if m != 1.0 else 0.0, T))
                else:
                    rows[w].append((m * tb, T))
                ys[w].append(s.per_worker_gpu[w] - _extra(prof, s.epoch))
            sx.append(cluster.sync_rounds_for_epoch(config, T, False))
            sy.append(s.sync_time)
    base, over, mult = [], [], []
    rel = []
    for w in range(n):
        A = np.asarray(rows[w], dtype=np.float64)
        y = np.asarray(ys[w], dtype=np.float64)
        live = [j for j in range(A.shape[1]) if np.any(A[:, j] != 0.0)]  # e.g. never disturbed
        coef = np.zeros(A.shape[1])
        coef[live] = np.linalg.lstsq(A[:, live], y, rcond=None)[0]
        if coef[-1] < 0.0:  # the law has no negative overhead: refit through the origin
            coef[-1] = 0.0
            lv = [j for j in live if j != A.shape[1] - 1]
            coef[lv] = np.linalg.lstsq(A[:, lv], y, rcond=None)[0]
        c = max(float(coef[0]), 1e-15)
        base.append(c)
        over.append(float(coef[-1]))
        if fit_multiplier:
            mult.append(float(coef[1]) / c if coef[1] != 0.0 else 1.0)
        rel.extend(((A @ coef) - y) / np.maximum(y, 1e-12))
    sxa, sya = np.asarray(sx, dtype=np.float64), np.asarray(sy, dtype=np.float64)
    a = float(sxa @ sya / (sxa @ sxa)) if sxa.size and sxa @ sxa > 0 else 0.0
    return FittedCosts(tuple(base), tuple(over), max(a, 0.0),
                       float(np.sqrt(np.mean(np.square(rel)))) if rel else 0.0, tuple(mult))


def fitted_profiles(fit: FittedCosts, profiles: Optional[Sequence[WorkerProfile]] = None) -> list:
    """WorkerProfiles with the fitted costs and the scenario's disturbance schedule
    (with measured multipliers, when fitted, in place of the declared ones)."""
    from dataclasses import replace as dc_replace

    out = []
    for w, (c, o) in enumerate(zip(fit.base_cost, fit.per_iteration_overhead)):
        dist = profiles[w].disturbances if profiles is not None else ()
        if fit.multiplier:
            dist = tuple(dc_replace(d, cost_multiplier=fit.multiplier[w]) if d.cost_multiplier is not None else d
                         for d in dist)
        out.append(WorkerProfile(w, c, per_iteration_overhead=o, disturbances=dist))
    return out


def fitted_config(config: StrategyConfig, fit: FittedCosts) -> StrategyConfig:
    return StrategyConfig(config.kind, config.total_budget, sync_interval=config.sync_interval,
                          sync_cost_per_round=fit.sync_cost_per_round, sync_cost_per_worker=0.0,
                          perf_smoothing=config.perf_smoothing)


def replay(stats: Sequence[EpochStats], config: StrategyConfig, fit: FittedCosts,
           profiles: Optional[Sequence[WorkerProfile]] = None) -> list:
    """The reference's run_epoch (cluster.py:192-220) on every measured plan, with
    the fitted profiles: the simulator's prediction for exactly these epochs."""
    prof = fitted_profiles(fit, profiles)
    cfg = fitted_config(config, fit)
    last = len(stats) - 1
    return [cluster.run_epoch(prof, s.plan, cfg, s.epoch, is_final_epoch=(i == last)) for i, s in enumerate(stats)]


def compare(measured: Sequence[EpochStats], predicted: Sequence[EpochStats], skip_epochs: int = 1) -> dict:
    """Per-epoch relative error of the slowest worker's compute and of the wall time."""
    gpu, wall = [], []
    for m, p in zip(measured[skip_epochs:], predicted[skip_epochs:]):
        gpu.append((max(p.per_worker_gpu) - max(m.per_worker_gpu)) / max(m.per_worker_gpu))
        wall.append((p.epoch_wall_time - m.epoch_wall_time) / m.epoch_wall_time)
    g, w = np.abs(np.asarray(gpu)), np.abs(np.asarray(wall))
    return {"epochs": len(gpu), "max_abs_rel_err_slowest_gpu": float(g.max()) if g.size else 0.0,
            "mean_abs_rel_err_slowest_gpu": float(g.mean()) if g.size else 0.0,
            "max_abs_rel_err_wall": float(w.max()) if w.size else 0.0,
            "mean_abs_rel_err_wall": float(w.mean()) if w.size else 0.0,
            "rel_err_wall": [round(float(v), 5) for v in wall]}


def simulate(fit: FittedCosts, config: StrategyConfig, dataset_size: int, n_epochs: int,
             profiles: Optional[Sequence[WorkerProfile]] = None) -> list:
    """A whole run of the reference simulator (run_training, with its own re-plans)
    under the fitted profiles."""
    return cluster.run_training(fitted_profiles(fit, profiles), fitted_config(config, fit), dataset_size, n_epochs)
