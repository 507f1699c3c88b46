"""The named model (784-H-10 MLP) on tcgen05: gradients and loss curves vs the
reference's own S-SGD loop and the CPU oracle.

precision "f32" (the product default; 3xTF32 GEMMs on S32 operands, fp32
master parameters): pinned to tests/golden/mlp_trajectories.json, produced by
the REFERENCE's run_parallel_sgd (sgdlab.py:343-396) driving the fp64 MLP
Problem adapter with no operand emulation.  Stated fp32 tolerances:
  * per-block gradient vs the fp64 oracle: relative L2 <= 1e-5;
  * per-iteration batch loss: relative <= 1e-5 (60 iterations, 3 workers);
  * ||x_t||^2: relative <= 1e-6; ||x_t - x_0||^2: relative <= 2e-4 (fp32
    parameter storage rounds each update, ~60 * 2^-24 |x| of a small displacement).
precision "bf16": bf16 operands, checked against the oracle with the same
operands rounded to bf16 (relative 2e-2)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("b", [128, 37, 173, 512])
def test_forward_backward_matches_oracle(dev, b):
    import torch

    from paper_2007_11831_b200 import mlp

    X, y = mlp.synthetic_mnist(2048, seed=1)
    model = mlp.MlpModel(seed=3, precision="bf16")
    sc = mlp.MlpScratch(model.layout, 512)
    idx = np.random.default_rng(b).permutation(2048)[:b]
    xb = mlp.operand_rows(model.layout, torch.as_tensor(X[idx], device=dev))
    yb = torch.as_tensor(y[idx], device=dev)
    grad = torch.zeros(model.P, device=dev)
    loss = torch.zeros(1, device=dev)
    mlp.forward_backward(model, sc, xb, yb, grad, loss)
    torch.cuda.synchronize()
    prob = O.MlpProblem(X, y, emulate_bf16=True)
    ref_loss, ref_g = prob.loss_and_grad(model.host_params().astype(np.float64), idx)
    g = model.layout.unpad(grad.cpu().numpy()).astype(np.float64)
    L = model.layout
    H, I, C = L.hidden, L.in_dim, L.classes
    blocks = [(0, H * I), (H * I, H * I + H), (H * I + H, H * I + H + C * H), (H * I + H + C * H, L.dimension)]
    for lo, hi in blocks:
        assert _rel(g[lo:hi], ref_g[lo:hi]) < 2e-2, (lo, hi, _rel(g[lo:hi], ref_g[lo:hi]))
    assert float(loss) == pytest.approx(ref_loss, rel=5e-3)


def test_padding_layout_roundtrip():
    from paper_2007_11831_b200.mlp import MlpLayout, init_params

    p = init_params()
    for prec in ("bf16", "f32"):
        L = MlpLayout(784, 256, 10, precision=prec)
        assert L.P % (8 if prec == "bf16" else 32) == 0 and L.P >= L.dimension
        np.testing.assert_array_equal(L.unpad(L.pad(p)), p)
    assert MlpLayout(784, 256, 10, precision="f32").in_ld == 800


@pytest.mark.parametrize("aggregation", ["batch_weighted", "uniform_average"])
def test_training_loss_curve_matches_oracle(dev, aggregation):
    """3 simulated workers, B=384 (128 each), the reference loop on both sides."""
    from paper_2007_11831_b200 import cluster, mlp
    from paper_2007_11831_b200.trainer import SimulatedTrainer

    X, y = mlp.synthetic_mnist(6000, seed=0)
    tr = SimulatedTrainer(X, y, n_workers=3, seed=0, partition=False, precision="bf16")
    p0 = tr.model.host_params().copy()
    res = tr.run(cluster.StrategyConfig("fixed_ssgd", 384), n_epochs=8, lr=0.05, momentum=0.5,
                 aggregation=aggregation, seed=0, max_iters=60)
    plans = [{"int_batches": list(p.int_batches),
              "cum": [0] + list(np.cumsum(p.int_batches))} for p in res.plans]
    prob = O.MlpProblem(X, y, emulate_bf16=True)
    ref = O.run_parallel_sgd(prob, 0.05, 60, 0.5, aggregation, 0, 3, plans, initial_point=p0.astype(np.float64),
                             record_loss=True)
    assert len(res.losses) == 60
    np.testing.assert_allclose(res.losses, ref["losses"], rtol=2e-2)
    # parameters after 60 steps
    assert _rel(tr.model.host_params().astype(np.float64), ref["x"]) < 1e-2


def test_dbs_plans_feed_identical_batches(dev):
    """Unequal DBS batches (different per worker) keep the loss curve on the oracle's."""
    from paper_2007_11831_b200 import cluster, mlp
    from paper_2007_11831_b200.trainer import SimulatedTrainer

    X, y = mlp.synthetic_mnist(4000, seed=2)
    tr = SimulatedTrainer(X, y, n_workers=3, seed=1, partition=False, precision="bf16")
    p0 = tr.model.host_params().copy()
    prof = [cluster.WorkerProfile(0, 1.0, disturbances=(cluster.DisturbanceEvent(0, extra_epoch_seconds=0.02),)),
            cluster.WorkerProfile(1, 1.0), cluster.WorkerProfile(2, 1.0)]
    res = tr.run(cluster.StrategyConfig("dbs", 384), n_epochs=3, lr=0.05, momentum=0.5, seed=5, profiles=prof)
    assert res.plans[0].int_batches == (128, 128, 128)
    assert res.plans[1].int_batches[0] < 128  # the disturbed worker got a smaller batch
    plans = [{"int_batches": list(p.int_batches), "cum": [0] + list(np.cumsum(p.int_batches))} for p in res.plans]
    n_it = len(res.losses)
    prob = O.MlpProblem(X, y, emulate_bf16=True)
    ref = O.run_parallel_sgd(prob, 0.05, n_it, 0.5, "batch_weighted", 5, 3, plans,
                             initial_point=p0.astype(np.float64), record_loss=True)
    np.testing.assert_allclose(res.losses, ref["losses"], rtol=2e-2)


@pytest.mark.parametrize("prec", ["bf16", "f32"])
@pytest.mark.parametrize("kind,interval", [("model_averaging", None), ("dbs", 4), ("one_shot", None)])
def test_model_averaging_matches_oracle(dev, kind, interval, prec):
    """Local SGD on per-worker replicas with periodic averaging (BASELINE config
    4 semantics; the reference only counts the rounds) against the oracle."""
    from paper_2007_11831_b200 import cluster, mlp
    from paper_2007_11831_b200.trainer import SimulatedTrainer

    X, y = mlp.synthetic_mnist(6000, seed=0)
    tr = SimulatedTrainer(X, y, n_workers=3, seed=0, partition=False, precision=prec)
    p0 = tr.model.host_params().copy()
    cfg = cluster.StrategyConfig(kind, 384, sync_interval=4 if kind == "model_averaging" else 1)
    prof = None
    if kind == "dbs":
        prof = [cluster.WorkerProfile(0, 1.0, disturbances=(cluster.DisturbanceEvent(0, extra_epoch_seconds=0.02),)),
                cluster.WorkerProfile(1, 1.0), cluster.WorkerProfile(2, 1.0)]
    res = tr.run(cfg, n_epochs=3, lr=0.05, momentum=0.5, seed=0, max_iters=40, profiles=prof,
                 averaging_interval=interval)
    plans = [{"int_batches": list(p.int_batches), "cum": [0] + list(np.cumsum(p.int_batches))} for p in res.plans]
    prob = O.MlpProblem(X, y, emulate_bf16=(prec == "bf16"))
    k = 4 if kind != "one_shot" else 1 << 30
    ref = O.run_parallel_sgd(prob, 0.05, 40, 0.5, "batch_weighted", 0, 3, plans,
                             initial_point=p0.astype(np.float64), record_loss=True, averaging_interval=k)
    assert len(res.losses) == 40
    np.testing.assert_allclose(res.losses, ref["losses"], rtol=2e-2 if prec == "bf16" else 1e-5)
    if kind == "one_shot":  # one average at the very end of the run
        w = np.asarray(plans[-1]["int_batches"], dtype=float)
        want = (w / w.sum()) @ np.stack(ref["replicas"])
    else:  # the trainer hands worker 0's replica back to the shared model
        want = ref["replicas"][0]
    # f32: fp32 master replicas vs the fp64 oracle after 40 local steps (measured 6.9e-6
    # one-shot; 2e-5..3.7e-5 for DBS, whose measured-time plans differ run to run and
    # can leave the disturbed worker a small, noisier batch)
    assert _rel(tr.model.host_params().astype(np.float64), want) < (1e-2 if prec == "bf16" else 1e-4)


# ----------------------------- fp32-class (default) -----------------------------

@pytest.mark.parametrize("b", [128, 37, 173, 512])
def test_f32_forward_backward_matches_fp64_oracle(dev, b):
    import torch

    from paper_2007_11831_b200 import mlp

    X, y = mlp.synthetic_mnist(2048, seed=1)
    model = mlp.MlpModel(seed=3, precision="f32")
    sc = mlp.MlpScratch(model.layout, 512)
    idx = np.random.default_rng(b).permutation(2048)[:b]
    xb = mlp.operand_rows(model.layout, torch.as_tensor(X[idx], device=dev))
    yb = torch.as_tensor(y[idx], device=dev)
    grad = torch.zeros(model.P, device=dev)
    loss = torch.zeros(1, device=dev)
    mlp.forward_backward(model, sc, xb, yb, grad, loss)
    torch.cuda.synchronize()
    prob = O.MlpProblem(X, y)  # fp64, no operand emulation
    ref_loss, ref_g = prob.loss_and_grad(model.host_params().astype(np.float64), idx)
    g = model.layout.unpad(grad.cpu().numpy()).astype(np.float64)
    L = model.layout
    H, I, C = L.hidden, L.in_dim, L.classes
    blocks = [(0, H * I), (H * I, H * I + H), (H * I + H, H * I + H + C * H), (H * I + H + C * H, L.dimension)]
    for lo, hi in blocks:
        assert _rel(g[lo:hi], ref_g[lo:hi]) < 1e-5, (lo, hi, _rel(g[lo:hi], ref_g[lo:hi]))
    assert float(loss) == pytest.approx(ref_loss, rel=1e-5)


def _golden_case(name):
    from conftest import load_golden

    return next(c for c in load_golden("mlp_trajectories.json")["cases"] if c["name"] == name)


def _run_f32(case, iters):
    """The device S-SGD loop from the golden's initial point for `iters` iterations."""
    from paper_2007_11831_b200 import allocation, cluster, mlp
    from paper_2007_11831_b200.trainer import SimulatedTrainer

    X, y = mlp.synthetic_mnist(case["D"], seed=case["data_seed"])
    x0 = O.mlp_init(seed=case["init_seed"])
    tr = SimulatedTrainer(X, y, n_workers=case["n_workers"], seed=0, partition=False, params=x0, precision="f32")
    plans = None
    if "plans" in case:
        p0 = allocation.plan_next_epoch([1 / 3] * 3, [1.0] * 3, 384, case["D"], 0)
        sh = p0.shares()
        p1 = allocation.plan_next_epoch(sh, [sh[0] * 2.0, sh[1], sh[2]], 384, case["D"], 1)
        plans = [p0, p1]
        assert [list(p.int_batches) for p in plans] == [q["int_batches"] for q in case["plans"]]
    cfg = cluster.StrategyConfig("fixed_ssgd", sum(case.get("fixed_batches") or case["plans"][0]["int_batches"]))
    res = tr.run(cfg, n_epochs=8, lr=case["step"], momentum=case["momentum"], aggregation=case["aggregation"],
                 seed=case["seed"], max_iters=iters, plan_source=plans)
    xt = tr.model.host_params().astype(np.float64)
    return res, xt, x0.astype(np.float64)


@pytest.mark.parametrize("name", ["fixed_bw", "fixed_uniform", "dbs_plans"])
def test_f32_trajectory_matches_reference_golden(dev, name):
    """C1 on the device in the fp32 class against the reference's own loop."""
    case = _golden_case(name)
    want_loss = np.array([float.fromhex(v) for v in case["losses"]])
    want_sq = np.array([float.fromhex(v) for v in case["sq_norm"]])
    want_disp = np.array([float.fromhex(v) for v in case["sq_disp"]])
    n = case["iters"]
    res, xt, x0 = _run_f32(case, n)
    assert len(res.losses) == n
    np.testing.assert_allclose(res.losses, want_loss, rtol=1e-5)
    assert float(xt @ xt) == pytest.approx(want_sq[-1], rel=1e-6)
    d = xt - x0
    assert float(d @ d) == pytest.approx(want_disp[-1], rel=2e-4)
    for k in (1, 10):  # intermediate points of the same trajectory
        _, xk, _ = _run_f32(case, k)
        assert float(xk @ xk) == pytest.approx(want_sq[k - 1], rel=1e-6)
        dk = xk - x0
        assert float(dk @ dk) == pytest.approx(want_disp[k - 1], rel=2e-4)
