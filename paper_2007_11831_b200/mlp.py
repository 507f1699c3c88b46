"""The named model of config 1: a 784-H-C MLP trained by synchronous DBS S-SGD.

Plugs into the reference's model boundary -- the duck-typed ``Problem`` of
sgdlab.py:162 (``mu``, ``dimension``, ``sample_count``, the batch-mean gradient
of minibatch_gradient sgdlab.py:200-205) -- but every step runs in
libdbs_b200: the forward/backward is 5 tcgen05 GEMMs + 2 small kernels
(csrc/mlp.cu), the update is the fused aggregate+SGD kernel.

Parameter layout (flat, fp32 master + bf16 shadow for the GEMMs):
    [ W1 (H x IN) | b1 (H) | W2 (C x H) | b2 (C) ]
each block padded to a multiple of 8 elements (16-byte TMA alignment).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib


def _pad8(x: int) -> int:
    return (x + 7) & ~7


class MlpLayout:
    def __init__(self, in_dim: int = 784, hidden: int = 256, classes: int = 10):
        self.in_dim, self.hidden, self.classes = in_dim, hidden, classes
        self.off_w1 = 0
        self.off_b1 = _pad8(hidden * in_dim)
        self.off_w2 = self.off_b1 + _pad8(hidden)
        self.off_b2 = self.off_w2 + _pad8(classes * hidden)
        self.P = self.off_b2 + _pad8(classes)
        self.dimension = hidden * in_dim + hidden + classes * hidden + classes  # unpadded (reference view)

    def pad(self, flat):
        """Unpadded [W1|b1|W2|b2] (the reference/oracle layout) -> padded device layout."""
        flat = np.asarray(flat, dtype=np.float32).reshape(-1)
        H, I, C = self.hidden, self.in_dim, self.classes
        out = np.zeros(self.P, dtype=np.float32)
        o = 0
        for off, n in ((self.off_w1, H * I), (self.off_b1, H), (self.off_w2, C * H), (self.off_b2, C)):
            out[off:off + n] = flat[o:o + n]
            o += n
        return out

    def unpad(self, padded):
        padded = np.asarray(padded).reshape(-1)
        H, I, C = self.hidden, self.in_dim, self.classes
        return np.concatenate([padded[self.off_w1:self.off_w1 + H * I], padded[self.off_b1:self.off_b1 + H],
                               padded[self.off_w2:self.off_w2 + C * H], padded[self.off_b2:self.off_b2 + C]])


def init_params(in_dim=784, hidden=256, classes=10, seed=0) -> np.ndarray:
    """Uniform(+-1/sqrt(fan_in)) init, unpadded reference layout (host set-up)."""
    rng = np.random.default_rng(seed + 1)
    b1 = 1.0 / math.sqrt(in_dim)
    b2 = 1.0 / math.sqrt(hidden)
    W1 = rng.uniform(-b1, b1, (hidden, in_dim)).astype(np.float32)
    c1 = rng.uniform(-b1, b1, hidden).astype(np.float32)
    W2 = rng.uniform(-b2, b2, (classes, hidden)).astype(np.float32)
    c2 = rng.uniform(-b2, b2, classes).astype(np.float32)
    return np.concatenate([W1.ravel(), c1, W2.ravel(), c2]).astype(np.float32)


def synthetic_mnist(n_samples=60000, in_dim=784, classes=10, seed=0):
    """Config-1 data: X ~ N(0,1) fp32, labels integers(0, classes), host seed 0."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n_samples, in_dim), dtype=np.float32)
    y = rng.integers(0, classes, size=n_samples).astype(np.int32)
    return X, y


class MlpModel:
    """Device parameters (fp32 master, bf16 shadow, momentum) of one replica."""

    def __init__(self, in_dim=784, hidden=256, classes=10, seed=0, device=None, params=None):
        import torch

        _lib.require_device()
        self.layout = L = MlpLayout(in_dim, hidden, classes)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        flat = init_params(in_dim, hidden, classes, seed) if params is None else np.asarray(params, np.float32)
        self.params = torch.as_tensor(L.pad(flat), device=self.device)
        self.params_bf16 = self.params.to(torch.bfloat16)
        self.velocity = torch.zeros_like(self.params)

    @property
    def P(self) -> int:
        return self.layout.P

    def refresh_shadow(self):
        self.params_bf16.copy_(self.params.to(self.params_bf16.dtype))

    def host_params(self) -> np.ndarray:
        return self.layout.unpad(self.params.cpu().numpy())


class MlpScratch:
    """Per-worker activation scratch (dbs_mlp) sized for the largest batch."""

    def __init__(self, layout: MlpLayout, max_batch: int):
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().dbs_mlp_create(layout.in_dim, layout.hidden, layout.classes, int(max_batch),
                                             ctypes.byref(h)), "mlp_create")
        self.handle = h
        self.max_batch = int(max_batch)
        p = ctypes.c_int64()
        _lib.check(_lib.lib().dbs_mlp_param_count(h, ctypes.byref(p)), "mlp_param_count")
        assert p.value == layout.P

    def __del__(self):
        try:
            if self.handle:
                _lib.lib().dbs_mlp_destroy(self.handle)
        except Exception:
            pass


def forward_backward(model: MlpModel, scratch: MlpScratch, x_bf16, labels, grad, loss, stream=None):
    """One worker's batch: flat fp32 gradient of the batch-mean CE loss."""
    b = int(x_bf16.shape[0])
    st = _lib.lib().dbs_mlp_forward_backward(scratch.handle, model.params_bf16.data_ptr(), model.params.data_ptr(),
                                             x_bf16.data_ptr(), labels.data_ptr(), b, grad.data_ptr(), loss.data_ptr(),
                                             _lib.stream_handle(stream))
    _lib.check(st, "mlp_forward_backward")
