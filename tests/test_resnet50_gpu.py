"""ResNet-50 (ImageNet-shaped, config 5) on tcgen05: convolutions at the 224x224
network's feature-map sizes (56/28/14/7 -- tiles that cross rows and images,
read through the im2col TMA path) against torch.nn.functional.conv2d, same
tolerances as tests/test_resnet_gpu.py (1e-2 of the operand scale for bf16
outputs, 1e-3 for the fp32 weight gradient)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

from test_resnet_gpu import test_conv_fwd_dgrad_wgrad as _conv_case

pytestmark = pytest.mark.gpu

SHAPES_R50 = [  # N, H, Cin, Cout, k, stride
    (2, 56, 64, 64, 3, 1),
    (2, 56, 64, 256, 1, 1),
    (2, 56, 256, 128, 1, 1),
    (2, 56, 128, 128, 3, 2),
    (2, 56, 256, 512, 1, 2),
    (3, 28, 256, 256, 3, 2),
    (4, 14, 256, 256, 3, 1),
    (2, 14, 1024, 2048, 1, 2),
    (4, 7, 512, 512, 3, 1),
    (3, 7, 2048, 512, 1, 1),
    (5, 14, 128, 64, 3, 1),
]


@pytest.mark.parametrize("N,H,Cin,Cout,k,stride", SHAPES_R50)
def test_conv_im2col_shapes(dev, N, H, Cin, Cout, k, stride):
    _conv_case(dev, N, H, Cin, Cout, k, stride)


def test_conv_im2col_forced_on_cifar_shapes(dev):
    """The im2col TMA path also on the ResNet-18 shapes that normally take the
    4-D box path (DBS_CONV_IM2COL=1 is read once per process: run in a child)."""
    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, DBS_CONV_IM2COL="1", DBS_CONV_HALO="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        str(root / "tests" / "test_resnet_gpu.py"), "-k", "conv_fwd_dgrad_wgrad"],
                       env=env, cwd=str(root), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
