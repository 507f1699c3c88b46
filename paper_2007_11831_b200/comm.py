"""NVLink peer-memory communicator for the fused weighted all-reduce + SGD.

One process per GPU.  ``Communicator`` allocates this rank's symmetric block
(gradient | fp32 params | bf16 params | signal words) in HBM, exchanges CUDA
IPC handles through torch.distributed (the ONLY use of the process group --
no NCCL collective touches the data path) and maps every peer's block.
``allreduce_sgd`` then runs csrc/comm.cu's single kernel per iteration:
reduce-scatter of sum_j (b_j / sum b) g_j over NVLink, momentum SGD on the
local shard, push of the updated shard into every peer (aggregate_gradients +
sgd_step, sgdlab.py:208-238).  ``average_params`` is the model-averaging round
(cluster.py:185-186).

``Communicator.local(world, P)`` builds ``world`` simulated ranks inside one
process on one device (plain local blocks instead of IPC) for testing the same
kernel on a single GPU.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


class _CudaArray:
    """__cuda_array_interface__ view of raw device memory (torch.as_tensor-able)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


def _wrap(ptr: int, n: int, typestr: str, device):
    import torch

    return torch.as_tensor(_CudaArray(ptr, n, typestr), device=device)


class Communicator:
    def __init__(self, handle: ctypes.c_void_p, rank: int, world: int, device, ipc: bool):
        import torch

        self.h = handle
        self.rank, self.world, self.ipc = rank, world, ipc
        P, shard = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.lib().dbs_comm_info(self.h, ctypes.byref(P), ctypes.byref(shard)), "comm_info")
        self.P, self.shard = P.value, shard.value
        g, p, pb = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(_lib.lib().dbs_comm_buffers(self.h, ctypes.byref(g), ctypes.byref(p), ctypes.byref(pb)), "buffers")
        self.device = device
        self.grad = _wrap(g.value, self.P, "<f4", device)
        self.params = _wrap(p.value, self.P, "<f4", device)
        self.params_bf16 = _wrap(pb.value, self.P, "<u2", device).view(torch.bfloat16)
        self.velocity = torch.zeros(self.shard, dtype=torch.float32, device=device)

    # -- construction --------------------------------------------------------
    @classmethod
    def create(cls, P: int, group=None):
        """IPC communicator across the ranks of a torch.distributed group."""
        import torch
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        dev = torch.device("cuda", torch.cuda.current_device())
        hsz = _lib.lib().dbs_comm_handle_size()
        buf = (ctypes.c_char * hsz)()
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().dbs_comm_alloc(rank, world, int(P), ctypes.byref(h), buf), "comm_alloc")
        handles = exchange_handles(bytes(buf), group)
        allh = (ctypes.c_char * (hsz * world)).from_buffer_copy(b"".join(handles))
        _lib.check(_lib.lib().dbs_comm_open(h, allh), "comm_open")
        return cls(h, rank, world, dev, ipc=True)

    @classmethod
    def local(cls, world: int, P: int):
        """``world`` simulated ranks in this process (tests on one GPU)."""
        import torch

        dev = torch.device("cuda", torch.cuda.current_device())
        arr = (ctypes.c_void_p * world)()
        _lib.check(_lib.lib().dbs_comm_create_local(world, int(P), arr), "comm_create_local")
        return [cls(ctypes.c_void_p(arr[r]), r, world, dev, ipc=False) for r in range(world)]

    def set_shadow(self, shadow, precision):
        """Register the parameter operand copy: precision "bf16" = the block's bf16
        region (pushed to every peer), "f32" = a local S32 tensor of 2 P floats that
        the iteration driver refreshes after each update."""
        code = _lib.precision_code(precision)
        st = _lib.lib().dbs_comm_set_shadow(self.h, shadow.data_ptr() if shadow is not None else None, code)
        _lib.check(st, "comm_set_shadow")

    # -- data path -------------------------------------------------------------
    def allreduce_sgd(self, batch_sizes, lr: float, momentum: float, mode: int = 1, stream=None):
        b = np.ascontiguousarray(np.asarray([int(x) for x in batch_sizes], dtype=np.int64))
        st = _lib.lib().dbs_comm_allreduce_sgd(self.h, b.ctypes.data_as(_lib.P_i64), int(mode), float(lr),
                                               float(momentum), self.velocity.data_ptr(), _lib.stream_handle(stream))
        _lib.check(st, "comm_allreduce_sgd")

    def average_params(self, batch_sizes, mode: int = 1, stream=None):
        b = np.ascontiguousarray(np.asarray([int(x) for x in batch_sizes], dtype=np.int64))
        st = _lib.lib().dbs_comm_average_params(self.h, b.ctypes.data_as(_lib.P_i64), int(mode),
                                                _lib.stream_handle(stream))
        _lib.check(st, "comm_average_params")

    def close(self):
        if self.h:
            if self.ipc:
                _lib.lib().dbs_comm_close_peers(self.h)
            _lib.lib().dbs_comm_destroy(self.h)
            self.h = None


def exchange_handles(mine: bytes, group=None) -> list:
    """All-gather of the per-rank IPC handle bytes (host metadata only)."""
    import torch.distributed as dist

    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, mine, group=group)
    return out


def gather_times(seconds: float, group=None) -> list:
    """Alg. 2 step 1: every rank learns every rank's compute time,
    so each rank runs the identical (deterministic, bit-exact) controller."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(seconds)], dtype=torch.float64, device=dev)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [float(x.item()) for x in out]


def max_over_ranks(value: float, group=None) -> float:
    import torch
    import torch.distributed as dist

    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
