"""Host-side logic of the multi-GPU path on CPU (gloo, world_size 2).

Covers what runs between the device kernels of DistributedTrainer:
* every rank learns every worker's measured time (Alg. 2 step 1)
  in the same rank-major order;
* with those times every rank computes the IDENTICAL plan (here through the
  CPU oracle, which is bit-exact with the device controller), so no plan
  broadcast is needed;
* the epoch time reported is the max over ranks;
* the IPC handle bytes of every rank reach every rank intact.
"""

from __future__ import annotations

import os
import socket

import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2007_11831_b200 import comm, trainer

        # 2 local workers per rank with rank-dependent measured times
        local = [0.5 + rank + 0.25 * w for w in range(2)]
        times = trainer.gather_worker_times(local)
        handles = comm.exchange_handles(bytes([rank]) * 64)
        wall = comm.max_over_ranks(1.0 + rank)
        # previous plan: even split over the 4 global workers
        b, cum, spans = O.plan_next_epoch([0.25] * 4, [1.0] * 4, 512, 50000, 0)
        shares = [(e - s) / 50000 for s, e in spans]
        plan = O.plan_next_epoch(shares, times, 512, 50000, 1)
        q.put((rank, times, [h[0] for h in handles], len(handles[1]), wall, plan))
    finally:
        dist.destroy_process_group()


def test_two_rank_host_protocol():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    (r0, t0, h0, n0, w0, p0), (r1, t1, h1, n1, w1, p1) = out
    assert t0 == t1 == [0.5, 0.75, 1.5, 1.75]
    assert h0 == h1 == [0, 1] and n0 == n1 == 64
    assert w0 == w1 == 2.0
    assert p0 == p1  # identical plans on every rank without a broadcast
    assert p0[0][0] > p0[0][3]  # the fastest worker gets the largest batch
