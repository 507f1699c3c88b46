"""The fused NVLink all-reduce + SGD kernel, exercised with simulated ranks on
one GPU (Communicator.local: the same kernel, peer pointers = local blocks),
against a plain PyTorch fp32 reference:  g = sum_j (b_j / sum b) g_j,
v' = m v + g, x' = x - lr v' on every rank (rel/abs 1e-6)."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu


def _launch_all(torch, comms, fn):
    streams = [torch.cuda.Stream() for _ in comms]
    cur = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(cur)
    for c, s in zip(comms, streams):
        fn(c, s)
    for s in streams:
        cur.wait_stream(s)
    torch.cuda.synchronize()


@pytest.mark.parametrize("world,P", [(2, 1000), (3, 203530), (4, 65536 * 3 + 7), (8, 11173962), (8, 4099)])
def test_fused_allreduce_sgd_matches_torch(dev, world, P):
    import torch

    from paper_2007_11831_b200.comm import Communicator

    comms = Communicator.local(world, P)
    Pp = comms[0].P
    g = torch.Generator(device=dev).manual_seed(world)
    x0 = torch.randn(Pp, device=dev, generator=g)
    grads = [torch.randn(Pp, device=dev, generator=g) for _ in range(world)]
    for c, gr in zip(comms, grads):
        c.params.copy_(x0)
        c.grad.copy_(gr)
    batches = ([37, 73, 73, 128] if world <= 4 else [37, 37, 73, 73, 73, 73, 73, 73])[:world]  # SURVEY 8(d) C2 weights
    lr, mom = 0.05, 0.9
    w = torch.tensor(batches, dtype=torch.float64, device=dev)
    w = (w / w.sum()).float()
    v = torch.zeros(Pp, device=dev)
    x = x0.clone()
    for it in range(3):
        _launch_all(torch, comms, lambda c, s: c.allreduce_sgd(batches, lr, mom, stream=s))
        gsum = sum(wj * gj for wj, gj in zip(w, grads))
        v = mom * v + gsum
        x = x - lr * v
        for c in comms:
            assert torch.allclose(c.params, x, rtol=1e-5, atol=1e-6), it
            assert torch.equal(c.params_bf16, c.params.to(torch.bfloat16))
        for r, c in enumerate(comms):
            assert torch.allclose(c.velocity, v[r * c.shard:(r + 1) * c.shard], rtol=1e-5, atol=1e-6)
    for c in comms:
        c.close()


def test_model_averaging_round(dev):
    import torch

    from paper_2007_11831_b200.comm import Communicator

    world, P = 4, 50000
    comms = Communicator.local(world, P)
    xs = [torch.randn(comms[0].P, device=dev) for _ in range(world)]
    for c, x in zip(comms, xs):
        c.params.copy_(x)
    batches = [10, 20, 30, 40]
    _launch_all(torch, comms, lambda c, s: c.average_params(batches, stream=s))
    want = sum((b / 100.0) * x for b, x in zip(batches, xs))
    for c in comms:
        assert torch.allclose(c.params, want, rtol=1e-5, atol=1e-6)
    for c in comms:
        c.close()


def test_uniform_mode(dev):
    import torch

    from paper_2007_11831_b200.comm import Communicator

    comms = Communicator.local(2, 4096)
    grads = [torch.randn(comms[0].P, device=dev) for _ in range(2)]
    for c, gr in zip(comms, grads):
        c.params.zero_()
        c.grad.copy_(gr)
    _launch_all(torch, comms, lambda c, s: c.allreduce_sgd([1, 99], 1.0, 0.0, mode=0, stream=s))
    want = -(grads[0] + grads[1]) / 2
    for c in comms:
        assert torch.allclose(c.params, want, rtol=1e-6, atol=1e-6)
