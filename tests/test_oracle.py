"""Pin the CPU oracle against the reference's golden vectors (no GPU).

The fixtures in tests/golden/ were produced by running the reference
(tests/golden/gen_golden.py).  If these pass, the oracle used by the GPU parity
tests restates the reference bit for bit on the controller, the sample
assignment and the reference-problem SGD loop.
"""

from __future__ import annotations

import hashlib
import json
import math
from fractions import Fraction

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, unhex
from oracle import oracle as O


def test_oracle_builds_and_loads():
    assert O.lib() is not None


def test_fsum_and_fractions_bit_exact():
    cases = load_golden("controller.json")["compute_batch_fractions"]
    checked = 0
    for c in cases:
        vals = [unhex(v) for v in c["perfs"]]
        if c["error"]:
            with pytest.raises(O.OracleError) as ei:
                O.compute_batch_fractions(vals)
            assert ei.value.name == c["error"]
            continue
        assert O.fsum(vals).hex() == c["fsum"]
        got = O.compute_batch_fractions(vals)
        assert [g.hex() for g in got] == c["fractions"]
        checked += 1
    assert checked > 500


def test_fsum_matches_math_fsum_adversarial():
    rng = np.random.default_rng(5)
    for _ in range(2000):
        n = int(rng.integers(1, 40))
        v = (rng.standard_normal(n) * 10.0 ** rng.integers(-20, 20, n)).tolist()
        if rng.random() < 0.3:
            v += [-x for x in v[: n // 2]]
        assert O.fsum(v).hex() == math.fsum(v).hex()


def test_round_twice_golden():
    for c in load_golden("controller.json")["round_twice"]:
        reals = [unhex(v) for v in c["reals"]]
        if c["error"]:
            with pytest.raises(O.OracleError) as ei:
                O.round_twice(reals, c["budget"])
            assert ei.value.name == c["error"]
        else:
            assert O.round_twice(reals, c["budget"]) == c["ints"]


def test_raise_zero_golden():
    for c in load_golden("controller.json")["raise_zero_batches"]:
        assert O.raise_zero_batches(c["in"]) == c["out"]


def _bound(b):
    if b["kind"] == 0:
        return Fraction(b["num"], b["den"])
    return unhex(b["value"])


def test_spans_golden():
    for c in load_golden("controller.json")["spans_from_ranges"]:
        rngs = [(_bound(lo), _bound(hi)) for lo, hi in zip(c["lo"], c["hi"])]
        if c["error"]:
            with pytest.raises(O.OracleError) as ei:
                O.spans_from_ranges(rngs, c["D"])
            assert ei.value.name == c["error"]
        else:
            assert O.spans_from_ranges(rngs, c["D"]) == [tuple(s) for s in c["spans"]]


def test_plan_next_epoch_golden():
    n_ok = 0
    for c in load_golden("controller.json")["plan_next_epoch"]:
        sh = [unhex(v) for v in c["shares"]]
        tm = [unhex(v) for v in c["times"]]
        if c["error"]:
            with pytest.raises(O.OracleError) as ei:
                O.plan_next_epoch(sh, tm, c["B"], c["D"], c["epoch"])
            assert ei.value.name == c["error"]
            continue
        b, cum, spans = O.plan_next_epoch(sh, tm, c["B"], c["D"], c["epoch"])
        assert b == c["int_batches"]
        assert cum == c["cum"]
        assert spans == [tuple(s) for s in c["spans"]]
        n_ok += 1
    assert n_ok > 600


def test_worked_example_known_answers():
    # PAPER.md:284 / test_allocation.py:101-102,113-114,107-111,194-197
    assert O.round_twice([13.7, 16.5, 19.6, 14.2], 64) == [14, 16, 20, 14]
    assert O.round_twice([3.5, 3.5, 4.0], 11) == [4, 3, 4]
    assert O.round_twice([5.4, 5.3, 5.3], 16) == [5, 5, 5]
    b, cum, spans = O.plan_next_epoch([0.25] * 4, [1 / 13.7, 1 / 16.5, 1 / 19.6, 1 / 14.2], 64, 50000, 1)
    assert b == [14, 16, 20, 14]
    assert spans == [(0, 10937), (10937, 23437), (23437, 39062), (39062, 50000)]


def test_replan_streams_golden():
    """cluster.run_training DBS chain (cluster.py:253-271) epoch by epoch."""
    for run in load_golden("plan_streams.json"):
        eps = run["epochs"]
        n = len(eps[0]["int_batches"])
        st = O.ReplanState(n)
        a = unhex(run["smoothing"])
        prev = None
        for e, ep in enumerate(eps):
            times_prev = [unhex(t) for t in eps[e - 1]["times"]] if e else [1.0] * n
            b, cum, spans = O.replan(prev if prev is not None else [(0, run["D"])] * n, times_prev,
                                     run["B"], run["D"], e, True, a, st)
            assert b == ep["int_batches"], (run["name"], e)
            assert spans == [tuple(s) for s in ep["spans"]], (run["name"], e)
            prev = spans


def test_pcg64_seed_and_permutation_golden():
    for c in load_golden("permutation.json"):
        g = O.pcg64_seed(c["seed"])
        assert g.state == int(c["state0"]["state"])
        assert g.inc == int(c["state0"]["inc"])
        for ep in c["epochs"]:
            flat = O.permute_spans(g, [tuple(s) for s in c["spans"]])
            assert hashlib.sha256(flat.astype(np.int64).tobytes()).hexdigest() == ep["sha256"]
            assert g.state == int(ep["state_after"]["state"])
            assert g.has_uint32 == ep["has_uint32"]
            if ep["has_uint32"]:
                assert g.uinteger == ep["uinteger"]


def test_permutation_matches_numpy_random_cases():
    rng = np.random.default_rng(11)
    for _ in range(30):
        seed = int(rng.integers(0, 2**63))
        spans, s = [], 0
        for _k in range(int(rng.integers(1, 6))):
            w = int(rng.integers(0, 3000))
            spans.append((s, s + w))
            s += w
        g = O.pcg64_seed(seed)
        ref = np.random.default_rng(seed)
        want = [st + ref.permutation(en - st) for st, en in spans]
        want = np.concatenate(want) if want else np.zeros(0, np.int64)
        got = O.permute_spans(g, spans)
        np.testing.assert_array_equal(got, want)


def test_aggregate_and_step_match_numpy():
    rng = np.random.default_rng(2)
    grads = [rng.standard_normal(1000) for _ in range(5)]
    b = [37, 73, 73, 1, 128]
    w = np.asarray(b, dtype=float)
    w /= w.sum()
    np.testing.assert_allclose(O.aggregate(grads, b, 1), w @ np.stack(grads), rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(O.aggregate(grads, b, 0), np.stack(grads).mean(axis=0), rtol=1e-13, atol=1e-15)
    x, v = rng.standard_normal(1000), rng.standard_normal(1000)
    xo, vo = O.sgd_step(x, grads[0], v, 0.1, 0.5)
    np.testing.assert_array_equal(vo, 0.5 * v + grads[0])
    np.testing.assert_array_equal(xo, x - 0.1 * (0.5 * v + grads[0]))


def test_mlp_adapter_gradient_is_batch_mean():
    X, y = O.synthetic_mnist(64, 20, 5, seed=1)
    p = O.MlpProblem(X, y, hidden=16, classes=5)
    x = O.mlp_init(20, 16, 5).astype(np.float64)
    _, g_all = p.loss_and_grad(x, np.arange(64))
    singles = np.mean([p.loss_and_grad(x, np.array([i]))[1] for i in range(64)], axis=0)
    np.testing.assert_allclose(g_all, singles, rtol=1e-10, atol=1e-14)
    # finite-difference check of one coordinate per block
    eps = 1e-6
    for k in (3, 16 * 20 + 2, 16 * 20 + 16 + 7, p.dimension - 1):
        e = np.zeros_like(x)
        e[k] = eps
        fd = (p.loss_and_grad(x + e, np.arange(64))[0] - p.loss_and_grad(x - e, np.arange(64))[0]) / (2 * eps)
        assert abs(fd - g_all[k]) < 1e-6


def test_model_averaging_every_iteration_without_momentum_is_ssgd():
    """Declared model-averaging semantics, pinned by a size-independent identity:
    averaging after every step with momentum 0 is exactly synchronous SGD."""
    X, y = O.synthetic_mnist(600, 20, 5, seed=3)
    p = O.MlpProblem(X, y, hidden=16, classes=5)
    x0 = O.mlp_init(20, 16, 5).astype(np.float64)
    plans = [{"int_batches": [30, 50, 40], "cum": [0, 30, 80, 120]}] * 4
    for agg in ("batch_weighted", "uniform_average"):
        ref = O.run_parallel_sgd(p, 0.05, 12, 0.0, agg, 0, 3, plans, initial_point=x0, record_loss=True)
        avg = O.run_parallel_sgd(p, 0.05, 12, 0.0, agg, 0, 3, plans, initial_point=x0, record_loss=True,
                                 averaging_interval=1)
        np.testing.assert_allclose(avg["x"], ref["x"], rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(avg["losses"], ref["losses"], rtol=1e-12)


def test_model_averaging_rounds_and_replicas():
    """k > 1: replicas diverge between rounds and coincide right after one
    (floor(T / k) rounds per epoch, cluster.sync_rounds_for_epoch)."""
    X, y = O.synthetic_mnist(600, 20, 5, seed=4)
    p = O.MlpProblem(X, y, hidden=16, classes=5)
    x0 = O.mlp_init(20, 16, 5).astype(np.float64)
    plans = [{"int_batches": [30, 50, 40], "cum": [0, 30, 80, 120]}] * 4
    # 5 iterations per epoch (spans 150 / 250 / 200): a round after the 4th
    at_round = O.run_parallel_sgd(p, 0.05, 4, 0.5, "batch_weighted", 0, 3, plans, initial_point=x0,
                                  averaging_interval=4)
    assert all(np.array_equal(r, at_round["replicas"][0]) for r in at_round["replicas"])
    between = O.run_parallel_sgd(p, 0.05, 6, 0.5, "batch_weighted", 0, 3, plans, initial_point=x0,
                                 averaging_interval=4)
    assert not np.array_equal(between["replicas"][0], between["replicas"][1])


def test_theorem1_bound_formula():
    """sgdlab.theorem1_bound (host formula, sgdlab.py:241-249) and its domain errors."""
    import pytest as _pt

    from paper_2007_11831_b200 import errors, sgdlab

    assert sgdlab.theorem1_bound(0, 0.1, 1.0, 2.0, 0.5) == 2.0 + 0.1 * 0.5
    assert sgdlab.theorem1_bound(3, 0.1, 1.0, 2.0, 0.0) == (0.9 ** 3) * 2.0
    with _pt.raises(errors.InvalidStepSizeError):
        sgdlab.theorem1_bound(1, 2.0, 1.0, 1.0, 1.0)
    with _pt.raises(errors.ConfigurationError):
        sgdlab.theorem1_bound(1, 0.1, 1.0, -1.0, 1.0)


def test_oracle_mlp_loop_pinned_to_reference_golden():
    """oracle.run_parallel_sgd + oracle.MlpProblem (fp64, no emulation) reproduce
    the reference's own run_parallel_sgd on the config-1 MLP
    (tests/golden/mlp_trajectories.json, gen_mlp_golden.py): squared distances and
    per-iteration losses to 1e-12 relative (same fp64 operations, BLAS order aside)."""
    from conftest import load_golden
    from oracle import oracle as O

    for case in load_golden("mlp_trajectories.json")["cases"]:
        rng = np.random.default_rng(case["data_seed"])
        X = rng.standard_normal((case["D"], 784), dtype=np.float32)
        y = rng.integers(0, 10, size=case["D"]).astype(np.int32)
        x0 = O.mlp_init(seed=case["init_seed"]).astype(np.float64)
        plans = case.get("plans") or case["fixed_batches"]
        ref = O.run_parallel_sgd(O.MlpProblem(X, y), case["step"], case["iters"], case["momentum"],
                                 case["aggregation"], case["seed"], case["n_workers"], plans, initial_point=x0,
                                 record_loss=True)
        want_sq = np.array([float.fromhex(v) for v in case["sq_norm"]])
        want_loss = np.array([float.fromhex(v) for v in case["losses"]])
        np.testing.assert_allclose(ref["squared_distances"], want_sq, rtol=1e-12)
        np.testing.assert_allclose(ref["losses"], want_loss, rtol=1e-12)
        disp = np.array([float.fromhex(v) for v in case["sq_disp"]])
        assert disp[-1] > 0 and np.all(np.diff(disp[:5]) > 0)


@pytest.mark.parametrize("seed", [0, 1, 42])
def test_oracle_numpy_integers_restatement(seed):
    """The bounded-integer / uniform draws of dbsim.checks (rng.integers, rng.random)
    restated exactly -- the algorithm theory.cu runs on the device."""
    for n, cnt in ((4096, 1000), (7, 500), (2 ** 32, 50), (1, 5), (100000, 333)):
        g = np.random.default_rng(seed)
        ref = O.Pcg64Ref(g.bit_generator.state)
        assert list(g.integers(0, n, size=cnt)) == ref.integers(n, cnt)
        np.testing.assert_array_equal(g.random(7), np.asarray(ref.random(7)))
