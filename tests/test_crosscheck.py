"""Simulator-vs-measured cross-check (crosscheck.py): the cost-law fit recovers the
reference's own parameters from epochs the reference's run_epoch produced, and the
replay reproduces them (CPU; host bookkeeping only)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2007_11831_b200 import allocation, cluster, crosscheck


def _plan(batches, D=50000, epoch=0):
    cum = [0] + list(np.cumsum(batches))
    total = cum[-1]
    starts = [c * D // total for c in cum]
    spans = []
    for i in range(len(batches)):
        spans += [starts[i], starts[i + 1] if i + 1 < len(batches) else D]
    return allocation.plan_from_arrays(batches, cum, spans, epoch)


PLANS = [(128, 128, 128, 128), (100, 140, 130, 142), (80, 150, 140, 142), (64, 160, 150, 138), (90, 120, 150, 152)]


@pytest.mark.parametrize("kind", ["fixed_ssgd", "dbs"])
def test_fit_recovers_the_cost_law(kind):
    truth = [cluster.WorkerProfile(0, 2e-5, per_iteration_overhead=3e-4,
                                   disturbances=(cluster.DisturbanceEvent(2, cost_multiplier=2.0),)),
             cluster.WorkerProfile(1, 3e-5, per_iteration_overhead=1e-4),
             cluster.WorkerProfile(2, 2.5e-5, per_iteration_overhead=2e-4,
                                   disturbances=(cluster.DisturbanceEvent(3, extra_epoch_seconds=0.05),)),
             cluster.WorkerProfile(3, 1e-5, per_iteration_overhead=5e-4)]
    cfg = cluster.StrategyConfig(kind, 512, sync_cost_per_round=2e-4, sync_cost_per_worker=0.0)
    stats = [cluster.run_epoch(truth, _plan(b, epoch=e), cfg, e) for e, b in enumerate(PLANS * 2)]
    fit = crosscheck.fit_costs([(cfg, stats)], truth, skip_epochs=0)
    np.testing.assert_allclose(fit.base_cost, [p.base_cost for p in truth], rtol=1e-9)
    np.testing.assert_allclose(fit.per_iteration_overhead, [p.per_iteration_overhead for p in truth], rtol=1e-6)
    assert fit.sync_cost_per_round == pytest.approx(2e-4, rel=1e-9)
    assert fit.residual_rel < 1e-9
    pred = crosscheck.replay(stats, cfg, fit, truth)
    cmp = crosscheck.compare(stats, pred, skip_epochs=0)
    assert cmp["max_abs_rel_err_wall"] < 1e-9 and cmp["max_abs_rel_err_slowest_gpu"] < 1e-9


def test_fit_with_noise_and_no_overhead():
    rng = np.random.default_rng(0)
    truth = [cluster.WorkerProfile(w, c) for w, c in enumerate((1e-5, 2e-5, 3e-5))]
    cfg = cluster.StrategyConfig("fixed_ssgd", 384)
    stats = []
    for e, b in enumerate([(128, 128, 128), (200, 100, 84), (150, 130, 104)] * 3):
        s = cluster.run_epoch(truth, _plan(b, D=60000, epoch=e), cfg, e)
        noisy = tuple(g * (1 + 0.01 * rng.standard_normal()) for g in s.per_worker_gpu)
        stats.append(cluster.EpochStats(e, noisy, tuple(max(noisy) - g for g in noisy), s.sync_time,
                                        max(noisy) + s.sync_time, s.plan))
    fit = crosscheck.fit_costs([(cfg, stats)], None, skip_epochs=0)
    np.testing.assert_allclose(fit.base_cost, [1e-5, 2e-5, 3e-5], rtol=0.05)
    assert all(o >= 0.0 for o in fit.per_iteration_overhead)
    cmp = crosscheck.compare(stats, crosscheck.replay(stats, cfg, fit), skip_epochs=0)
    assert cmp["max_abs_rel_err_wall"] < 0.05


def test_fit_measures_the_disturbance_multiplier():
    """fit_multiplier: a worker declared 2x slower but really 1.8x is measured as 1.8x."""
    real = [cluster.WorkerProfile(0, 2e-5, per_iteration_overhead=1e-4,
                                  disturbances=(cluster.DisturbanceEvent(3, cost_multiplier=1.8),)),
            cluster.WorkerProfile(1, 2e-5, per_iteration_overhead=1e-4)]
    declared = [cluster.WorkerProfile(0, 1.0, disturbances=(cluster.DisturbanceEvent(3, cost_multiplier=2.0),)),
                cluster.WorkerProfile(1, 1.0)]
    cfg = cluster.StrategyConfig("fixed_ssgd", 256)
    plans = [(128, 128), (100, 156), (90, 166), (150, 106), (110, 146), (70, 186)]
    stats = [cluster.run_epoch(real, _plan(b, epoch=e), cfg, e) for e, b in enumerate(plans)]
    fit = crosscheck.fit_costs([(cfg, stats)], declared, skip_epochs=0, fit_multiplier=True)
    assert fit.multiplier[0] == pytest.approx(1.8, rel=1e-9) and fit.multiplier[1] == 1.0
    cmp = crosscheck.compare(stats, crosscheck.replay(stats, cfg, fit, declared), skip_epochs=0)
    assert cmp["max_abs_rel_err_wall"] < 1e-9
