"""The named model of config 1: a 784-H-C MLP trained by synchronous DBS S-SGD.

Plugs into the reference's model boundary -- the duck-typed ``Problem`` of
sgdlab.py:162 (``mu``, ``dimension``, ``sample_count``, the batch-mean gradient
of minibatch_gradient sgdlab.py:200-205) -- but every step runs in
libdbs_b200: the forward/backward is 5 tcgen05 GEMMs + 2 small kernels
(csrc/mlp.cu), the update is the fused aggregate+SGD kernel.

Parameter layout (flat, fp32 master + an operand shadow for the GEMMs):
    [ W1 (H x IN) | b1 (H) | W2 (C x H) | b2 (C) ]
precision "f32" (default; the fp32 class of the reference's numpy fp64 loop):
3xTF32 GEMMs on S32 operands, W1 rows padded to IN rounded up to 32, every
block starting on a 32-element boundary (the flat S32 shadow, 2P floats);
precision "bf16": bf16 operands, blocks padded to multiples of 8.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib


def _pad8(x: int) -> int:
    return (x + 7) & ~7


def _pad32(x: int) -> int:
    return (x + 31) & ~31


class MlpLayout:
    def __init__(self, in_dim: int = 784, hidden: int = 256, classes: int = 10, precision="f32"):
        self.in_dim, self.hidden, self.classes = in_dim, hidden, classes
        self.precision = _lib.precision_code(precision)
        f32 = self.precision == _lib.PREC_F32
        pad = _pad32 if f32 else _pad8
        self.in_ld = _pad32(in_dim) if f32 else in_dim  # W1 row length (and S32 input row length)
        self.off_w1 = 0
        self.off_b1 = pad(hidden * self.in_ld)
        self.off_w2 = self.off_b1 + pad(hidden)
        self.off_b2 = self.off_w2 + pad(classes * hidden)
        self.P = self.off_b2 + pad(classes)
        self.dimension = hidden * in_dim + hidden + classes * hidden + classes  # unpadded (reference view)

    def pad(self, flat):
        """Unpadded [W1|b1|W2|b2] (the reference/oracle layout) -> padded device layout."""
        flat = np.asarray(flat, dtype=np.float32).reshape(-1)
        H, I, C = self.hidden, self.in_dim, self.classes
        out = np.zeros(self.P, dtype=np.float32)
        out[self.off_w1:self.off_w1 + H * self.in_ld].reshape(H, self.in_ld)[:, :I] = flat[:H * I].reshape(H, I)
        o = H * I
        for off, n in ((self.off_b1, H), (self.off_w2, C * H), (self.off_b2, C)):
            out[off:off + n] = flat[o:o + n]
            o += n
        return out

    def unpad(self, padded):
        padded = np.asarray(padded).reshape(-1)
        H, I, C = self.hidden, self.in_dim, self.classes
        w1 = padded[self.off_w1:self.off_w1 + H * self.in_ld].reshape(H, self.in_ld)[:, :I].reshape(-1)
        return np.concatenate([w1, padded[self.off_b1:self.off_b1 + H],
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
    """Device parameters (fp32 master, operand shadow, momentum) of one replica.
    ``params_op`` is the GEMM operand copy (S32 for "f32", bf16 for "bf16");
    ``params_bf16`` names it for the bf16 precision."""

    def __init__(self, in_dim=784, hidden=256, classes=10, seed=0, device=None, params=None, precision="f32"):
        import torch

        _lib.require_device()
        self.layout = L = MlpLayout(in_dim, hidden, classes, precision)
        self.precision = L.precision
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        flat = init_params(in_dim, hidden, classes, seed) if params is None else np.asarray(params, np.float32)
        self.params = torch.as_tensor(L.pad(flat), device=self.device)
        self.params_op = _lib.new_shadow(self.params, self.precision)
        self.velocity = torch.zeros_like(self.params)

    @property
    def params_bf16(self):
        return self.params_op if self.precision == _lib.PREC_BF16 else None

    @property
    def P(self) -> int:
        return self.layout.P

    def refresh_shadow(self):
        _lib.refresh_shadow(self.params, self.params_op, self.precision)

    def host_params(self) -> np.ndarray:
        return self.layout.unpad(self.params.cpu().numpy())


class MlpScratch:
    """Per-worker activation scratch (dbs_mlp) sized for the largest batch."""

    def __init__(self, layout: MlpLayout, max_batch: int):
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().dbs_mlp_create_ex(layout.in_dim, layout.hidden, layout.classes, int(max_batch),
                                                layout.precision, ctypes.byref(h)), "mlp_create")
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


def operand_rows(layout: MlpLayout, x):
    """Input rows fp32 [b][in] on the device -> the GEMM operand form (S32 [b][in_ld]
    for "f32", bf16 for "bf16")."""
    import torch

    if layout.precision == _lib.PREC_BF16:
        return x.to(torch.bfloat16).contiguous()
    x = x.float().contiguous()
    out = torch.empty((x.shape[0], 2 * layout.in_ld), dtype=torch.float32, device=x.device)
    _lib.check(_lib.lib().dbs_dev_split_s32(x.data_ptr(), x.shape[0], layout.in_dim, layout.in_dim, out.data_ptr(),
                                            layout.in_ld, _lib.stream_handle()), "split_s32")
    return out


def forward_backward(model: MlpModel, scratch: MlpScratch, x_op, labels, grad, loss, stream=None):
    """One worker's batch (x_op from operand_rows): flat fp32 gradient of the batch-mean CE loss."""
    b = int(x_op.shape[0])
    st = _lib.lib().dbs_mlp_forward_backward(scratch.handle, model.params_op.data_ptr(), model.params.data_ptr(),
                                             x_op.data_ptr(), labels.data_ptr(), b, grad.data_ptr(), loss.data_ptr(),
                                             _lib.stream_handle(stream))
    _lib.check(st, "mlp_forward_backward")
