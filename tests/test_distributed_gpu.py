"""Two real processes (torchrun, gloo host collectives) driving DistributedTrainer:
CUDA IPC handle exchange, the fused weighted all-reduce + SGD kernel across
process boundaries, identical plans and identical parameters on every rank.
Both ranks may share one GPU (the kernels time-slice; the in-kernel barrier
has a timeout so a missing peer can never wedge the device)."""

from __future__ import annotations

import os
import re
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("extra", [["0", "f32"], ["2", "f32"], ["0", "bf16"], ["2", "bf16"], ["0", "f32", "2"]],
                         ids=["ssgd_f32", "model_averaging_k2_f32", "ssgd_bf16", "model_averaging_k2_bf16",
                              "ssgd_f32_2_partitioned_workers_per_rank"])
def test_two_process_distributed_trainer(dev, extra):
    """S-SGD through the fused all-reduce + SGD kernel, and model averaging every 2
    iterations (local replica average, then the NVLink parameter average across
    ranks): both must leave identical parameters on the two ranks (6 iterations end
    on a sync round)."""
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    port = str(29531 + 2 * (int(extra[0]) + 4 * (extra[1] == "bf16")) + 20 * (len(extra) > 2))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", port, str(ROOT / "scripts" / "dist_smoke.py"), "mlp",
           *extra]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=240, env=env, cwd=str(ROOT))
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-3000:]
    lines = re.findall(r"rank (\d): plans (.*?) losses (.*?) param-sum agree (True|False)", out)
    assert len(lines) == 2, out[-2000:]
    assert all(agree == "True" for _, _, _, agree in lines)
    assert lines[0][1] == lines[1][1]  # same plan on both ranks
