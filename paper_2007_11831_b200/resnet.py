"""ResNet-18 (CIFAR variant; configs 3/4) and ResNet-50 (ImageNet stem,
torchvision v1.5 bottlenecks; config 5) on tcgen05.

Host side of csrc/resnet.cu: the flat parameter layout (queried from the
library's parameter table, torchvision order), host initialisation
(kaiming-normal fan-out for convolutions, BN gamma=1 beta=0, PyTorch-default
uniform for the classifier), conversion to / from PyTorch OIHW tensors for the
parity tests, and per-worker activation scratch.

Data: synthetic CIFAR-shaped samples, fp32 [D][3][32][32] rows, labels 0..9
(SURVEY.md 8d, C3/C4 inputs); synthetic ImageNet-shaped samples, uint8
[D][3][224][224] rows (pixel value (u - 128) / 64), labels 0..999 (C5).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib

KIND_CONV, KIND_BN_G, KIND_BN_B, KIND_FC_W, KIND_FC_B = 0, 1, 2, 3, 4


class ResnetLayout:
    """Offsets of every parameter tensor in the flat vector (torchvision order)."""

    _cache = {}

    def __init__(self, classes: int = 10, depth: int = 18, image: int = 32):
        key = (classes, depth, image)
        if key not in ResnetLayout._cache:
            h = ctypes.c_void_p()
            _lib.check(_lib.lib().dbs_resnet_create_ex(depth, image, 1, classes, ctypes.byref(h)), "resnet_create")
            try:
                P = ctypes.c_int64()
                _lib.check(_lib.lib().dbs_resnet_param_count(h, ctypes.byref(P)), "resnet_param_count")
                cap = 512
                off = (ctypes.c_int64 * cap)()
                ln = (ctypes.c_int64 * cap)()
                kd = (ctypes.c_int32 * cap)()
                cnt = ctypes.c_int32()
                _lib.check(_lib.lib().dbs_resnet_param_table(h, off, ln, kd, cap, ctypes.byref(cnt)), "param_table")
                rb, sk = ctypes.c_int64(), ctypes.c_int32()
                _lib.check(_lib.lib().dbs_resnet_info(h, None, None, ctypes.byref(rb), ctypes.byref(sk)), "info")
                ResnetLayout._cache[key] = (P.value, [(off[i], ln[i], kd[i]) for i in range(cnt.value)], rb.value,
                                            sk.value)
            finally:
                _lib.lib().dbs_resnet_destroy(h)
        self.P, self.table, self.row_bytes, self.stem_k = ResnetLayout._cache[key]
        self.classes, self.depth, self.image = classes, depth, image
        self.shapes = self._shapes()

    def _shapes(self):
        """PyTorch (OIHW) shape of each table entry, in torchvision order."""
        shapes = []
        if self.depth == 18:
            convs = [(3, 64, 3)]
            cin = 64
            for L, w in enumerate((64, 128, 256, 512)):
                for b in range(2):
                    stride = 2 if (L > 0 and b == 0) else 1
                    convs.append((cin, w, 3))
                    convs.append((w, w, 3))
                    if stride != 1 or cin != w:
                        convs.append((cin, w, 1))
                    cin = w
        else:
            convs = [(3, 64, 7)]
            cin = 64
            for L, (w, n) in enumerate(zip((64, 128, 256, 512), (3, 4, 6, 3))):
                for b in range(n):
                    stride = 2 if (L > 0 and b == 0) else 1
                    convs += [(cin, w, 1), (w, w, 3), (w, 4 * w, 1)]
                    if stride != 1 or cin != 4 * w:
                        convs.append((cin, 4 * w, 1))
                    cin = 4 * w
        for ci, co, k in convs:
            shapes += [(co, ci, k, k), (co,), (co,)]
        shapes += [(self.classes, cin), (self.classes,)]
        assert len(shapes) == len(self.table), (len(shapes), len(self.table))
        return shapes

    @property
    def feat_dim(self) -> int:
        return self.shapes[-2][1]

    @property
    def n_weights(self) -> int:
        return int(sum(int(np.prod(s)) for s in self.shapes))

    def pack(self, tensors) -> np.ndarray:
        """PyTorch-layout arrays (torchvision order) -> flat device layout (fp32)."""
        flat = np.zeros(self.P, dtype=np.float32)
        for (off, ln, kind), shp, t in zip(self.table, self.shapes, tensors):
            a = np.asarray(t, dtype=np.float32).reshape(shp)
            if kind == KIND_CONV:
                w = a.transpose(0, 2, 3, 1)  # OIHW -> OHWI (c fastest)
                if shp[1] == 3:  # stem: [64][k*k*3] padded to [64][stem_k]
                    kk = shp[2] * shp[3] * 3
                    w2 = np.zeros((shp[0], self.stem_k), dtype=np.float32)
                    w2[:, :kk] = w.reshape(shp[0], kk)
                    w = w2
                flat[off:off + ln] = w.reshape(-1)
            else:
                flat[off:off + ln] = a.reshape(-1)
        return flat

    def unpack(self, flat) -> list:
        """Flat device layout -> PyTorch-layout arrays (torchvision order)."""
        flat = np.asarray(flat).reshape(-1)
        out = []
        for (off, ln, kind), shp in zip(self.table, self.shapes):
            v = flat[off:off + ln]
            if kind == KIND_CONV:
                if shp[1] == 3:
                    v = v.reshape(shp[0], self.stem_k)[:, :shp[2] * shp[3] * 3]
                out.append(v.reshape(shp[0], shp[2], shp[3], shp[1]).transpose(0, 3, 1, 2).copy())
            else:
                out.append(v.reshape(shp).copy())
        return out


def init_params(classes: int = 10, seed: int = 0, depth: int = 18, image: int = 32) -> list:
    """Host initialisation in torchvision order (kaiming fan-out / BN 1, 0 / FC uniform)."""
    rng = np.random.default_rng(seed)
    L = ResnetLayout(classes, depth, image)
    out = []
    for shp, (_, _, kind) in zip(L.shapes, L.table):
        if kind == KIND_CONV:
            fan_out = shp[0] * shp[2] * shp[3]
            out.append(rng.normal(0.0, math.sqrt(2.0 / fan_out), shp).astype(np.float32))
        elif kind == KIND_BN_G:
            out.append(np.ones(shp, dtype=np.float32))
        elif kind == KIND_BN_B:
            out.append(np.zeros(shp, dtype=np.float32))
        else:
            bound = 1.0 / math.sqrt(L.feat_dim)
            out.append(rng.uniform(-bound, bound, shp).astype(np.float32))
    return out


def synthetic_imagenet(n_samples=20000, image=224, classes=1000, seed=0, device=None):
    """C5 inputs: uint8 [D][3][image][image] uniform pixels, labels integers(0, classes).
    device=None: numpy arrays on the host; else torch tensors generated on that device."""
    if device is None:
        rng = np.random.default_rng(seed)
        X = rng.integers(0, 256, size=(n_samples, 3, image, image), dtype=np.uint8)
        y = rng.integers(0, classes, size=n_samples).astype(np.int32)
        return X, y
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    X = torch.randint(0, 256, (n_samples, 3, image, image), generator=g, device=device, dtype=torch.uint8)
    y = torch.randint(0, classes, (n_samples,), generator=g, device=device, dtype=torch.int32)
    return X, y


def synthetic_cifar(n_samples=50000, classes=10, seed=0):
    """C3 inputs: fp32 [D][3][32][32] ~ N(0,1), labels integers(0, classes)."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n_samples, 3, 32, 32), dtype=np.float32)
    y = rng.integers(0, classes, size=n_samples).astype(np.int32)
    return X, y


class ResnetModel:
    """Device parameters (fp32 master, operand shadow, momentum) of one replica.
    precision "f32" (default): 3xTF32 GEMMs, ``params_op`` = the S32 shadow (2P
    floats); "bf16": bf16 operands, ``params_op`` = ``params_bf16``."""

    def __init__(self, classes=10, seed=0, device=None, params=None, depth=18, image=32, precision="f32"):
        import torch

        _lib.require_device()
        self.layout = L = ResnetLayout(classes, depth, image)
        self.precision = _lib.precision_code(precision)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        tensors = init_params(classes, seed, depth, image) if params is None else params
        self.params = torch.as_tensor(L.pack(tensors), device=self.device)
        self.params_op = _lib.new_shadow(self.params, self.precision)
        self.velocity = torch.zeros_like(self.params)

    @property
    def params_bf16(self):
        return self.params_op if self.precision == _lib.PREC_BF16 else None

    def refresh_shadow(self):
        _lib.refresh_shadow(self.params, self.params_op, self.precision)

    @property
    def P(self) -> int:
        return self.layout.P

    def host_tensors(self) -> list:
        return self.layout.unpack(self.params.cpu().numpy())


class ResnetScratch:
    """Per-worker activation scratch (dbs_resnet) sized for the largest batch."""

    def __init__(self, max_batch: int, classes: int = 10, depth: int = 18, image: int = 32, precision="f32"):
        h = ctypes.c_void_p()
        self.precision = _lib.precision_code(precision)
        _lib.check(_lib.lib().dbs_resnet_create_ex2(depth, image, int(max_batch), classes, self.precision,
                                                    ctypes.byref(h)), "resnet_create")
        self.handle = h
        self.max_batch = int(max_batch)

    def running_stats(self, conv: int):
        """(mean, variance) numpy arrays of conv `conv`'s BatchNorm running statistics (f32 mode)."""
        import torch

        ptr, ch = ctypes.c_void_p(), ctypes.c_int32()
        _lib.check(_lib.lib().dbs_resnet_running_stats(self.handle, int(conv), ctypes.byref(ptr), ctypes.byref(ch)),
                   "running_stats")
        from .comm import _wrap

        t = _wrap(ptr.value, 2 * ch.value, "<f4", torch.device("cuda", torch.cuda.current_device())).cpu().numpy()
        return t[:ch.value].copy(), t[ch.value:].copy()

    def __del__(self):
        try:
            if self.handle:
                _lib.lib().dbs_resnet_destroy(self.handle)
        except Exception:
            pass


def forward_backward(model: ResnetModel, scratch: ResnetScratch, x, labels, grad, loss, stream=None, d_iter=None):
    """One worker's batch: flat fp32 gradient of the batch-mean cross-entropy."""
    b = int(labels.shape[0]) if d_iter is None else int(scratch.max_batch)
    if model.precision != scratch.precision:
        raise ValueError("model and scratch precisions differ")
    st = _lib.lib().dbs_resnet_forward_backward(
        scratch.handle, model.params_op.data_ptr(), model.params.data_ptr(), x.data_ptr(), labels.data_ptr(), b,
        d_iter.data_ptr() if d_iter is not None else None, grad.data_ptr(), loss.data_ptr() if loss is not None else None,
        _lib.stream_handle(stream))
    _lib.check(st, "resnet_forward_backward")
