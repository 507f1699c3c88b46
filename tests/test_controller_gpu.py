"""Device controller parity: bit-exact against the reference's golden vectors
(tests/golden/controller.json, plan_streams.json) and the C oracle."""

from __future__ import annotations

import random
from fractions import Fraction

import numpy as np
import pytest

from conftest import load_golden, unhex
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A(dev):
    from paper_2007_11831_b200 import allocation

    return allocation


@pytest.fixture(scope="module")
def E():
    from paper_2007_11831_b200 import errors

    return errors


def _err_class(E, name):
    return {"OverflowError": OverflowError, "ValueError": ValueError, "IndexError": IndexError}.get(name) or getattr(E, name)


def test_plan_next_epoch_golden_bit_exact(A, E):
    cases = load_golden("controller.json")["plan_next_epoch"]
    for c in cases:
        sh = [unhex(v) for v in c["shares"]]
        tm = [unhex(v) for v in c["times"]]
        if c["error"]:
            with pytest.raises(_err_class(E, c["error"])):
                A.plan_next_epoch(sh, tm, c["B"], c["D"], c["epoch"])
            continue
        plan = A.plan_next_epoch(sh, tm, c["B"], c["D"], c["epoch"])
        assert list(plan.int_batches) == c["int_batches"]
        cum = c["cum"]
        assert [lo for lo, _ in plan.ranges] == [Fraction(cum[i], cum[-1]) for i in range(len(cum) - 1)]
        assert [list(s) for s in plan.sample_spans] == c["spans"]
        assert plan.epoch == c["epoch"]


def test_fractions_bit_exact(A, E):
    for c in load_golden("controller.json")["compute_batch_fractions"]:
        perfs = [A.PerfEstimate(i, unhex(v)) for i, v in enumerate(c["perfs"])]
        if c["error"]:
            with pytest.raises(_err_class(E, c["error"])):
                A.compute_batch_fractions(perfs)
        else:
            assert [f.hex() for f in A.compute_batch_fractions(perfs)] == c["fractions"]


def test_round_twice_and_zero_lift_golden(A, E):
    g = load_golden("controller.json")
    for c in g["round_twice"]:
        reals = [unhex(v) for v in c["reals"]]
        if c["error"]:
            with pytest.raises(_err_class(E, c["error"])):
                A.round_twice(reals, c["budget"])
        else:
            assert A.round_twice(reals, c["budget"]) == c["ints"]
    for c in g["raise_zero_batches"]:
        assert A._raise_zero_batches(c["in"]) == c["out"]


def test_spans_golden(A, E):
    for c in load_golden("controller.json")["spans_from_ranges"]:
        def b(x):
            return Fraction(x["num"], x["den"]) if x["kind"] == 0 else unhex(x["value"])
        rngs = [(b(lo), b(hi)) for lo, hi in zip(c["lo"], c["hi"])]
        if c["error"]:
            with pytest.raises(_err_class(E, c["error"])):
                A.spans_from_ranges(rngs, c["D"])
        else:
            assert [list(s) for s in A.spans_from_ranges(rngs, c["D"])] == c["spans"]


def test_known_answers(A, E):
    # PAPER.md:284, test_allocation.py worked examples
    assert A.round_twice([13.7, 16.5, 19.6, 14.2], 64) == [14, 16, 20, 14]
    assert A.round_twice([3.5, 3.5, 4.0], 11) == [4, 3, 4]
    assert A.round_twice([5.4, 5.3, 5.3], 16) == [5, 5, 5]
    assert A.partition_ranges([14, 16, 20, 14])[1] == (Fraction(14, 64), Fraction(30, 64))
    assert A.spans_from_ranges(A.partition_ranges([14, 16, 20, 14]), 50000) == [
        (0, 10937), (10937, 23437), (23437, 39062), (39062, 50000)]
    assert A.spans_from_ranges([(0, 0.5), (0.5, 1)], 10) == [(0, 5), (5, 10)]
    assert A.spans_from_ranges(A.partition_ranges([1, 100, 1]), 3) == [(0, 1), (1, 2), (2, 3)]
    assert A.evaluate_performance(0.25, 10.0) == 0.025
    with pytest.raises(E.InvalidMeasurementError):
        A.evaluate_performance(0.25, 0.0)
    with pytest.raises(E.EmptyPartitionError):
        A.partition_ranges([0, 0])
    with pytest.raises(E.DatasetTooSmallError):
        A.spans_from_ranges([(0, 0.5), (0.5, 1)], 1)
    plan = A.plan_next_epoch([0.25] * 4, [1.0, 1.0, 1.0, 1000.0], 8, 100, 1)
    assert min(plan.int_batches) >= 1 and sum(plan.int_batches) <= 8


def test_random_plans_match_oracle(A):
    rng = random.Random(7)
    for _ in range(300):
        n = rng.randint(1, 24)
        w = [rng.random() + 1e-4 for _ in range(n)]
        shares = [x / sum(w) for x in w]
        times = [10 ** rng.uniform(-7, 4) for _ in range(n)]
        B = rng.randint(n, 5000)
        D = rng.randint(n, 2_000_000)
        plan = A.plan_next_epoch(shares, times, B, D, 1)
        b, cum, spans = O.plan_next_epoch(shares, times, B, D, 1)
        assert list(plan.int_batches) == b
        assert list(plan.sample_spans) == spans


def test_large_worker_count(A):
    rng = np.random.default_rng(3)
    n = 1500
    shares = rng.random(n) + 0.01
    shares = (shares / shares.sum()).tolist()
    times = (rng.random(n) * 5 + 0.1).tolist()
    plan = A.plan_next_epoch(shares, times, 100_000, 5_000_000, 3)
    b, cum, spans = O.plan_next_epoch(shares, times, 100_000, 5_000_000, 3)
    assert list(plan.int_batches) == b
    assert list(plan.sample_spans) == spans


def test_run_training_plan_streams_golden(dev):
    """cluster.run_training DBS chain epoch by epoch (cluster.py:253-271)."""
    from paper_2007_11831_b200 import cluster as C

    for run in load_golden("plan_streams.json"):
        eps = run["epochs"]
        n = len(eps[0]["int_batches"])
        cfg = C.StrategyConfig("dbs", run["B"], perf_smoothing=unhex(run["smoothing"]))
        prev, sm = None, None
        for e, ep in enumerate(eps):
            plan, sm = C.next_plan(cfg, e, n, run["D"], prev, sm)
            assert list(plan.int_batches) == ep["int_batches"], (run["name"], e)
            assert [list(s) for s in plan.sample_spans] == ep["spans"], (run["name"], e)
            assert C.iterations_for_plan(plan) == ep["iters"]
            times = tuple(unhex(t) for t in ep["times"])
            prev = C.EpochStats(e, times, tuple(0.0 for _ in times), 0.0, max(times), plan)


def test_device_replan_chain_matches_streams(dev):
    """dbs_dev_replan: the whole re-plan on the device, no host round trip."""
    import torch

    from paper_2007_11831_b200 import _lib

    for run in load_golden("plan_streams.json"):
        eps = run["epochs"]
        n = len(eps[0]["int_batches"])
        a = unhex(run["smoothing"])
        prev_spans = torch.zeros(2 * n, dtype=torch.int64, device=dev)
        times = torch.zeros(n, dtype=torch.float64, device=dev)
        smoothed = torch.zeros(n, dtype=torch.float64, device=dev)
        flags = torch.zeros(2, dtype=torch.int32, device=dev)
        b = torch.zeros(n, dtype=torch.int64, device=dev)
        cum = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        spans = torch.zeros(2 * n, dtype=torch.int64, device=dev)
        iters = torch.zeros(1, dtype=torch.int64, device=dev)
        s = _lib.stream_handle()
        for e, ep in enumerate(eps):
            if e:
                times.copy_(torch.tensor([unhex(t) for t in eps[e - 1]["times"]], dtype=torch.float64))
            st = _lib.lib().dbs_dev_replan(prev_spans.data_ptr(), times.data_ptr(), n, run["B"], run["D"], e, 1, a,
                                           smoothed.data_ptr(), flags.data_ptr(), b.data_ptr(), cum.data_ptr(),
                                           spans.data_ptr(), iters.data_ptr(), s)
            assert st == 0
            torch.cuda.synchronize()
            assert int(flags[1]) == 0
            assert b.tolist() == ep["int_batches"], (run["name"], e)
            assert spans.view(n, 2).tolist() == ep["spans"], (run["name"], e)
            assert int(iters) == ep["iters"]
            prev_spans.copy_(spans)
