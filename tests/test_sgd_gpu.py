"""Variable-batch gradients, aggregation and the SGD loop on the device vs the
reference (golden trajectories produced by sgdlab.run_parallel_sgd) and the
oracle.  fp64 throughout: the quadratic gradient and the step are bit-exact,
the BLAS-ordered reductions (dgemv aggregation, ddot distance) agree to
rel 1e-12; trajectories to rel 1e-9."""

from __future__ import annotations

import itertools

import numpy as np
import pytest

from conftest import load_golden, unhex
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S(dev):
    from paper_2007_11831_b200 import sgdlab

    return sgdlab


@pytest.fixture(scope="module")
def quad(S):
    return S.ConvexProblem.quadratic(dimension=3, mu=2.0, sample_noise_scale=0.5, sample_count=12, seed=3)


def test_quadratic_minibatch_gradient_bit_exact(S, quad):
    x = np.array([0.7, 0.7, -0.2])
    for idx in ([0, 5], [1, 2, 3, 8, 9, 11], list(range(12)), [4]):
        want = (quad.mu * (x - quad.optimum - quad.offsets[idx])).mean(axis=0)  # sgdlab.py:82,205
        got = S.minibatch_gradient(quad, x, idx)
        np.testing.assert_array_equal(got, want)


def test_unbiased_over_exhaustive_batches(S, quad):
    x = np.array([0.2, -0.4, 0.9])
    for m in (1, 2, 3):
        batches = list(itertools.combinations(range(12), m))
        avg = np.mean([S.minibatch_gradient(quad, x, list(b)) for b in batches], axis=0)
        np.testing.assert_allclose(avg, quad.full_gradient(x), atol=1e-10)


def test_weighted_recombination_equals_union_batch(S, quad):
    x = np.array([0.7, 0.7, -0.2])
    a, b = [0, 5], [1, 2, 3, 8, 9, 11]
    merged = S.aggregate_gradients([S.minibatch_gradient(quad, x, a), S.minibatch_gradient(quad, x, b)],
                                   [2, 6], "batch_weighted")
    np.testing.assert_allclose(merged, S.minibatch_gradient(quad, x, a + b), rtol=1e-12)


def test_aggregate_modes_and_errors(S):
    from paper_2007_11831_b200 import errors

    rng = np.random.default_rng(0)
    grads = [rng.standard_normal(10000) for _ in range(8)]
    b = [37, 37, 73, 73, 73, 73, 73, 73]
    np.testing.assert_allclose(S.aggregate_gradients(grads, b, "batch_weighted"), O.aggregate(grads, b, 1),
                               rtol=1e-13, atol=1e-15)
    np.testing.assert_array_equal(S.aggregate_gradients(grads, b, "uniform_average"), np.stack(grads).mean(axis=0))
    g = np.array([0.5, -1.5])
    np.testing.assert_allclose(S.aggregate_gradients([g, g], [2, 9], "batch_weighted"), g)
    with pytest.raises(errors.ConfigurationError):
        S.aggregate_gradients([np.zeros(2)], [1, 2], "uniform_average")
    with pytest.raises(errors.ConfigurationError):
        S.aggregate_gradients([np.zeros(2)], [0], "uniform_average")
    with pytest.raises(errors.EmptyBatchError):
        S.minibatch_gradient(S.ConvexProblem.quadratic(3, 1.0, 0.1, 10), np.zeros(3), [])


def test_sgd_step_bit_exact(S):
    rng = np.random.default_rng(1)
    x, g, v = rng.standard_normal(4099), rng.standard_normal(4099), rng.standard_normal(4099)
    cfg = S.SgdConfig(step_size=0.1, n_iterations=1, momentum=0.5)
    xo, vo = S.sgd_step(x, g, cfg, v)
    np.testing.assert_array_equal(vo, 0.5 * v + g)
    np.testing.assert_array_equal(xo, x - 0.1 * (0.5 * v + g))
    # momentum recursion of test_sgdlab.py:106-112
    c = S.SgdConfig(step_size=0.1, n_iterations=1, momentum=0.5)
    x1, v1 = S.sgd_step(np.array([0.0]), np.array([1.0]), c, np.zeros(1))
    x2, v2 = S.sgd_step(x1, np.array([1.0]), c, v1)
    assert x1[0] == pytest.approx(-0.1) and v2[0] == pytest.approx(1.5) and x2[0] == pytest.approx(-0.25)


def _golden_problem(S, name):
    from paper_2007_11831_b200 import cluster

    quad = S.ConvexProblem.quadratic(dimension=8, mu=1.0, sample_noise_scale=0.5, sample_count=4096, seed=0)
    logit = S.LogisticProblem.synthetic(dimension=16, mu=0.1, sample_count=1000, seed=0)

    def stream(n, B, D, E):
        profiles = [cluster.WorkerProfile(i, 1e-4 * 2.0 ** (i / max(n - 1, 1))) for i in range(n)]
        return [s.plan for s in cluster.run_training(profiles, cluster.StrategyConfig("dbs", B), D, E)]

    plans = stream(4, 64, 4096, 6)
    table = {
        "quad_fixed": (quad, S.SgdConfig(step_size=0.02, n_iterations=200, momentum=0.5, seed=0), 4, [16] * 4),
        "quad_dbs": (quad, S.SgdConfig(step_size=0.02, n_iterations=200, momentum=0.5, seed=3), 4, plans),
        "quad_uniform": (quad, S.SgdConfig(step_size=0.05, n_iterations=150, momentum=0.0,
                                           aggregation="uniform_average", seed=1), 4, plans),
        "logit_fixed": (logit, S.SgdConfig(step_size=0.5, n_iterations=120, momentum=0.5, seed=4), 2, [16, 16]),
        "logit_dbs": (logit, S.SgdConfig(step_size=0.5, n_iterations=120, momentum=0.5, seed=4), 4,
                      stream(4, 64, 1000, 8)),
    }
    return table[name]


@pytest.mark.parametrize("name", ["quad_fixed", "quad_dbs", "quad_uniform", "logit_fixed", "logit_dbs"])
def test_run_parallel_sgd_golden(S, name):
    rec = next(r for r in load_golden("sgd_trajectories.json") if r["name"] == name)
    prob, cfg, n, src = _golden_problem(S, name)
    traj = S.run_parallel_sgd(prob, cfg, n, src)
    want = np.array([unhex(v) for v in rec["squared_distances"]])
    np.testing.assert_allclose(traj.squared_distances, want, rtol=1e-9, atol=0)
    assert traj.final_loss == pytest.approx(unhex(rec["final_loss"]), rel=1e-7, abs=1e-13)


def test_noiseless_geometric_decay(S):
    """test_sgdlab.py:133-141: (1 - gamma mu)^(2(j+1)) d0 at rel 1e-10."""
    q = S.ConvexProblem.quadratic(dimension=3, mu=2.0, sample_noise_scale=0.0, sample_count=12, seed=3)
    cfg = S.SgdConfig(step_size=0.1, n_iterations=20, seed=0)
    run = S.run_parallel_sgd(q, cfg, 1, [12])
    d0 = 3.0
    np.testing.assert_allclose(run.squared_distances, [(1 - 0.2) ** (2 * (j + 1)) * d0 for j in range(20)],
                               rtol=1e-10)


def test_deterministic_and_span_errors(S, quad):
    from paper_2007_11831_b200 import errors

    cfg = S.SgdConfig(step_size=0.1, n_iterations=30, seed=42)
    a = S.run_parallel_sgd(quad, cfg, 2, [3, 3])
    b = S.run_parallel_sgd(quad, cfg, 2, [3, 3])
    np.testing.assert_array_equal(a.squared_distances, b.squared_distances)
    with pytest.raises(errors.ConfigurationError):
        S.run_parallel_sgd(quad, S.SgdConfig(step_size=0.1, n_iterations=5), 2, [7, 7])
    with pytest.raises(errors.InvalidStepSizeError):
        S.run_parallel_sgd(quad, S.SgdConfig(step_size=1.5 / quad.mu, n_iterations=5), 1, [4])
