"""ctypes binding of libdbs_b200.so (the C ABI declared in include/dbs_b200.h).

The shared library is built in-tree by ``paper_2007_11831_b200.build`` and is
the ONLY compute path of this package: there is no CPU fallback.  If the
library is missing or no sm_100 device is visible, every compute call raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from . import errors

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libdbs_b200.so"

c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_dbl = ctypes.c_double
c_flt = ctypes.c_float
c_vp = ctypes.c_void_p
P_dbl = ctypes.POINTER(ctypes.c_double)
P_i64 = ctypes.POINTER(ctypes.c_int64)
P_i32 = ctypes.POINTER(ctypes.c_int32)
P_u32 = ctypes.POINTER(ctypes.c_uint32)


class Bound(ctypes.Structure):
    """dbs_bound: exact rational (kind 0) or IEEE double (kind 1)."""

    _fields_ = [("kind", ctypes.c_int32), ("reserved", ctypes.c_int32), ("num", ctypes.c_int64),
                ("den", ctypes.c_int64), ("value", ctypes.c_double)]


class Pcg64(ctypes.Structure):
    """dbs_pcg64: numpy PCG64 state (128-bit state/inc + next_uint32 buffer)."""

    _fields_ = [("state_hi", ctypes.c_uint64), ("state_lo", ctypes.c_uint64),
                ("inc_hi", ctypes.c_uint64), ("inc_lo", ctypes.c_uint64),
                ("has_uint32", ctypes.c_uint32), ("uinteger", ctypes.c_uint32)]

    @property
    def state(self) -> int:
        return (self.state_hi << 64) | self.state_lo

    @property
    def inc(self) -> int:
        return (self.inc_hi << 64) | self.inc_lo

    def numpy_state(self) -> dict:
        """The dict numpy's ``Generator.bit_generator.state`` would report."""
        return {"bit_generator": "PCG64", "state": {"state": self.state, "inc": self.inc},
                "has_uint32": int(self.has_uint32), "uinteger": int(self.uinteger)}


class WorkerSlot(ctypes.Structure):
    """dbs_worker_slot (include/dbs_b200.h)."""

    _fields_ = [("model", ctypes.c_void_p), ("stream", ctypes.c_void_p), ("x_shard", ctypes.c_void_p),
                ("y_shard", ctypes.c_void_p), ("batch", ctypes.c_int64), ("grad", ctypes.c_void_p),
                ("loss", ctypes.c_void_p), ("loss_scratch", ctypes.c_void_p), ("stamps", ctypes.c_void_p),
                ("seconds", ctypes.c_void_p), ("worker_index", ctypes.c_int64), ("spin_ns", ctypes.c_int64),
                ("spin_ctas", ctypes.c_int32), ("model_kind", ctypes.c_int32), ("slow_scale", ctypes.c_float),
                ("slow_ctas", ctypes.c_int32), ("ctx", ctypes.c_void_p)]


# name -> (restype, argtypes)
SIGNATURES = {
    "dbs_last_error": (ctypes.c_char_p, []),
    "dbs_version": (c_i32, [P_i32, P_i32, P_i32]),
    "dbs_device_ok": (c_i32, []),
    "dbs_launch_count": (c_i64, []),
    "dbs_host_launch_count": (c_i64, []),
    "dbs_evaluate_performance": (c_i32, [P_dbl, P_dbl, c_i64, P_dbl, P_i64]),
    "dbs_compute_batch_fractions": (c_i32, [P_dbl, c_i64, P_dbl, P_i64]),
    "dbs_scale_to_real_batches": (c_i32, [P_dbl, c_i64, c_i64, P_dbl]),
    "dbs_round_twice": (c_i32, [P_dbl, c_i64, c_i64, P_i64]),
    "dbs_raise_zero_batches": (c_i32, [P_i64, c_i64, P_i64]),
    "dbs_partition_ranges": (c_i32, [P_i64, c_i64, P_i64]),
    "dbs_spans_from_ranges": (c_i32, [ctypes.POINTER(Bound), ctypes.POINTER(Bound), c_i64, c_i64, P_i64]),
    "dbs_plan_next_epoch": (c_i32, [P_dbl, P_dbl, c_i64, c_i64, c_i64, c_i64, P_i64, P_i64, P_i64, P_i64]),
    "dbs_dev_replan": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i32, c_dbl, c_vp, c_vp, c_vp, c_vp,
                               c_vp, c_vp, c_vp]),
    "dbs_pcg64_seed": (c_i32, [P_u32, c_i32, ctypes.POINTER(Pcg64)]),
    "dbs_permute_spans": (c_i32, [ctypes.POINTER(Pcg64), P_i64, c_i64, P_i64]),
    "dbs_dev_permute_spans": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "dbs_dev_gather_rows": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "dbs_dev_gather_rows_f32_bf16": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "dbs_dev_gather_rows_f32_s32": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp]),
    "dbs_dev_gather_i32": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "dbs_dev_aggregate_f64": (c_i32, [ctypes.POINTER(c_vp), P_i64, c_i64, c_i32, c_i64, c_vp, c_vp]),
    "dbs_dev_sgd_step_f64": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_dbl, c_dbl, c_vp, c_vp, c_vp]),
    "dbs_dev_aggregate_sgd_f64": (c_i32, [ctypes.POINTER(c_vp), P_i64, c_i64, c_i32, c_i64, c_dbl, c_dbl, c_vp,
                                          c_vp, c_vp]),
    "dbs_dev_aggregate_sgd_f32": (c_i32, [ctypes.POINTER(c_vp), P_i64, c_i64, c_i32, c_i64, c_flt, c_flt, c_vp,
                                          c_vp, c_vp, c_vp]),
    "dbs_dev_aggregate_sgd_f32_ex": (c_i32, [ctypes.POINTER(c_vp), P_i64, c_i64, c_i32, c_i64, c_flt, c_flt, c_vp,
                                             c_vp, c_vp, c_i32, c_vp]),
    "dbs_dev_refresh_shadow": (c_i32, [c_vp, c_i64, c_vp, c_i32, c_vp]),
    "dbs_comm_set_shadow": (c_i32, [c_vp, c_vp, c_i32]),
    "dbs_comm_shadow": (c_i32, [c_vp, ctypes.POINTER(c_vp), P_i32]),
    "dbs_comm_handle_size": (c_i32, []),
    "dbs_comm_alloc": (c_i32, [c_i32, c_i32, c_i64, ctypes.POINTER(c_vp), c_vp]),
    "dbs_comm_open": (c_i32, [c_vp, c_vp]),
    "dbs_comm_buffers": (c_i32, [c_vp, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_vp)]),
    "dbs_comm_destroy": (c_i32, [c_vp]),
    "dbs_comm_info": (c_i32, [c_vp, P_i64, P_i64]),
    "dbs_comm_close_peers": (c_i32, [c_vp]),
    "dbs_comm_create_local": (c_i32, [c_i32, c_i64, ctypes.POINTER(c_vp)]),
    "dbs_comm_allreduce_sgd": (c_i32, [c_vp, P_i64, c_i32, c_flt, c_flt, c_vp, c_vp]),
    "dbs_comm_average_params": (c_i32, [c_vp, P_i64, c_i32, c_vp]),
    "dbs_dev_quadratic_grads": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_dbl, c_vp, c_vp]),
    "dbs_dev_logistic_grads": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_dbl, c_vp, c_vp]),
    "dbs_dev_sgd_epoch": (c_i32, [c_i32, c_vp, c_vp, c_vp, c_i64, c_dbl, c_vp, P_i64, P_i64, c_i64, c_i32, c_i64,
                                  c_dbl, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dbs_dev_sq_dist": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "dbs_dev_gemm_bf16": (c_i32, [c_vp, c_i32, c_i64, c_vp, c_i32, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, c_i32,
                                  c_vp, c_vp, c_vp]),
    "dbs_dev_gemm_tf32x3": (c_i32, [c_vp, c_i32, c_i64, c_vp, c_i32, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, c_i32,
                                    c_vp, c_vp, c_vp]),
    "dbs_dev_split_s32": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp]),
    "dbs_dev_join_s32": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp]),
    "dbs_mlp_create": (c_i32, [c_i64, c_i64, c_i64, c_i64, ctypes.POINTER(c_vp)]),
    "dbs_mlp_create_ex": (c_i32, [c_i64, c_i64, c_i64, c_i64, c_i32, ctypes.POINTER(c_vp)]),
    "dbs_mlp_info": (c_i32, [c_vp, P_i32, P_i64]),
    "dbs_mlp_destroy": (c_i32, [c_vp]),
    "dbs_mlp_param_count": (c_i32, [c_vp, P_i64]),
    "dbs_mlp_forward_backward": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "dbs_mlp_run_iterations": (c_i32, [ctypes.POINTER(WorkerSlot), c_i32, c_i64, c_i64, c_i32, c_flt, c_flt, c_vp,
                                       c_vp, c_vp, c_i32, c_vp]),
    "dbs_run_iterations": (c_i32, [ctypes.POINTER(WorkerSlot), c_i32, c_i64, c_i64, c_i32, c_flt, c_flt, c_vp, c_vp,
                                   c_vp, c_i32, c_vp, c_vp]),
    "dbs_dev_iter_increment": (c_i32, [c_vp, c_vp]),
    "dbs_dev_bn_apply_s32": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i32, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "dbs_dev_bn_backward_s32": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp,
                                        c_vp]),
    "dbs_run_iterations_graphed": (c_i32, [ctypes.POINTER(WorkerSlot), c_i32, c_i64, c_i64, c_i32, c_flt, c_flt,
                                           c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "dbs_worker_graphs_capture": (c_i32, [ctypes.POINTER(WorkerSlot), c_i32, c_i32, c_flt, c_flt, c_vp, c_vp, c_vp,
                                          c_i32, c_vp, c_vp, c_vp]),
    "dbs_run_iterations_local_graphed": (c_i32, [ctypes.POINTER(WorkerSlot), c_i32, c_i64, c_i64, c_i32, c_flt,
                                                 c_flt, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32]),
    "dbs_run_iterations_comm_graphed": (c_i32, [ctypes.POINTER(WorkerSlot), c_i32, c_i64, c_i64, c_i32, c_flt, c_flt,
                                                c_vp, P_i64, c_vp, c_vp, c_vp, c_vp, c_i32]),
    "dbs_epoch_graph_create": (c_i32, [ctypes.POINTER(WorkerSlot), c_i32, c_i32, c_flt, c_flt, c_vp, c_vp, c_vp, c_i32,
                                       c_vp, c_vp, c_vp, ctypes.POINTER(c_vp)]),
    "dbs_epoch_graph_launch": (c_i32, [c_vp, c_i64, c_vp]),
    "dbs_epoch_graph_destroy": (c_i32, [c_vp]),
    "dbs_worker_graphs_create": (c_i32, [c_i32, ctypes.POINTER(c_vp)]),
    "dbs_worker_graphs_destroy": (c_i32, [c_vp]),
    "dbs_run_iterations_comm": (c_i32, [ctypes.POINTER(WorkerSlot), c_i32, c_i64, c_i64, c_i32, c_flt, c_flt, c_vp,
                                        P_i64, c_vp, c_vp, c_vp]),
    "dbs_dev_aggregate_f32": (c_i32, [ctypes.POINTER(c_vp), P_i64, c_i64, c_i32, c_i64, c_vp, c_vp]),
    "dbs_run_iterations_local": (c_i32, [ctypes.POINTER(WorkerSlot), c_i32, c_i64, c_i64, c_i32, c_flt, c_flt, c_i32,
                                         ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), c_vp]),
    "dbs_dev_average_replicas_f32": (c_i32, [ctypes.POINTER(c_vp), P_i64, c_i64, c_i32, c_i64, ctypes.POINTER(c_vp),
                                             c_vp]),
    "dbs_run_iterations_local_comm": (c_i32, [ctypes.POINTER(WorkerSlot), c_i32, c_i64, c_i64, c_i32, c_flt, c_flt,
                                              c_i32, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_vp),
                                              c_vp, P_i64, c_vp]),
    "dbs_resnet_create": (c_i32, [c_i64, c_i32, ctypes.POINTER(c_vp)]),
    "dbs_resnet_create_ex": (c_i32, [c_i32, c_i32, c_i64, c_i32, ctypes.POINTER(c_vp)]),
    "dbs_resnet_create_ex2": (c_i32, [c_i32, c_i32, c_i64, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "dbs_resnet_precision": (c_i32, [c_vp, P_i32]),
    "dbs_resnet_running_stats": (c_i32, [c_vp, c_i32, ctypes.POINTER(c_vp), P_i32]),
    "dbs_resnet_info": (c_i32, [c_vp, P_i32, P_i32, P_i64, P_i32]),
    "dbs_resnet_destroy": (c_i32, [c_vp]),
    "dbs_resnet_param_count": (c_i32, [c_vp, P_i64]),
    "dbs_resnet_param_table": (c_i32, [c_vp, P_i64, P_i64, P_i32, c_i32, P_i32]),
    "dbs_resnet_forward_backward": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "dbs_dev_conv2d_fwd": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "dbs_dev_conv2d_dgrad": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp,
                                     c_vp]),
    "dbs_dev_conv2d_wgrad": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "dbs_dev_conv2d_fwd_s32": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "dbs_dev_conv2d_dgrad_s32": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp,
                                         c_vp]),
    "dbs_dev_conv2d_wgrad_s32": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp,
                                         c_vp]),
    "dbs_dev_average_replicas_f32_ex": (c_i32, [ctypes.POINTER(c_vp), P_i64, c_i64, c_i32, c_i64,
                                                ctypes.POINTER(c_vp), c_i32, c_vp]),
    "dbs_dev_spin_until": (c_i32, [c_i32, c_vp, c_vp]),
    "dbs_dev_spin_until_ctx": (c_i32, [c_i32, c_vp, c_vp, c_vp]),
    "dbs_partition_create": (c_i32, [c_i32, c_i32, ctypes.POINTER(c_vp), P_i32]),
    "dbs_partition_get": (c_i32, [c_vp, c_i32, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_vp)]),
    "dbs_dev_pcg64_integers": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_vp]),
    "dbs_dev_pcg64_random": (c_i32, [c_vp, c_i64, c_vp, c_vp]),
    "dbs_dev_theorem1_trajectories": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_i64, c_dbl, c_vp, c_i32, c_vp,
                                              c_vp, c_vp, c_vp]),
    "dbs_dev_row_moments": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "dbs_dev_minibatch_sqnorms": (c_i32, [c_i32, c_vp, c_vp, c_vp, c_i64, c_dbl, c_vp, c_vp, c_i64, c_i64, c_vp,
                                          c_vp]),
    "dbs_dev_sample_values": (c_i32, [c_i32, c_vp, c_vp, c_vp, c_i64, c_dbl, c_vp, c_i64, c_vp, c_vp]),
    "dbs_dev_gather_means": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "dbs_partition_push": (c_i32, [c_vp]),
    "dbs_partition_pop": (c_i32, [c_vp]),
    "dbs_dev_spin_for": (c_i32, [c_i32, c_i64, c_vp]),
    "dbs_dev_stamp": (c_i32, [c_vp, c_i64, c_vp]),
    "dbs_dev_set_flag": (c_i32, [c_vp, c_i32, c_vp]),
    "dbs_dev_accumulate_time": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp]),
}

_LIB = None


def lib() -> ctypes.CDLL:
    """Load the CUDA library (raises if it was not built -- no fallback)."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2007_11831_b200.build` "
                "(the DBS hot path has no CPU fallback)")
        L = ctypes.CDLL(str(LIB_PATH), mode=ctypes.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def exported_symbols():
    return list(SIGNATURES)


def last_error() -> str:
    msg = lib().dbs_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(status: int, what: str = "", detail: str | None = None) -> None:
    """Raise the reference exception class mapped from a dbs_status code."""
    if status == 0:
        return
    raise errors.from_status(status, detail or f"{what}: {last_error()}")


def stream_handle(stream=None) -> int:
    """cudaStream_t of a torch stream (current stream when None)."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def require_device():
    """Fail loudly unless an sm_100 device is present."""
    if not lib().dbs_device_ok():
        raise RuntimeError("no CUDA device with compute capability 10.x (B200) is visible; "
                           "the DBS hot path runs only on sm_100a")


def ptr(t) -> int:
    return int(t.data_ptr())


PREC_BF16, PREC_F32 = 0, 1
PRECISIONS = {"bf16": PREC_BF16, "f32": PREC_F32}


def precision_code(precision) -> int:
    """'f32' (3xTF32 tensor-core GEMMs on S32 operands, the fp32 class) or 'bf16'."""
    if isinstance(precision, int) and precision in (PREC_BF16, PREC_F32):
        return precision
    if precision not in PRECISIONS:
        raise ValueError(f"precision must be 'f32' or 'bf16', got {precision!r}")
    return PRECISIONS[precision]


def new_shadow(params, precision):
    """Operand copy of flat fp32 params on the device: bf16 [P] or S32 [2P] floats."""
    import torch

    code = precision_code(precision)
    if code == PREC_BF16:
        return params.to(torch.bfloat16)
    out = torch.empty(2 * params.numel(), dtype=torch.float32, device=params.device)
    refresh_shadow(params, out, code)
    return out


def refresh_shadow(params, shadow, precision, stream=None):
    code = precision_code(precision)
    st = lib().dbs_dev_refresh_shadow(params.data_ptr(), int(params.numel()), shadow.data_ptr(), code,
                                      stream_handle(stream))
    check(st, "refresh_shadow")


def env_flag(name: str) -> bool:
    return os.environ.get(name, "") not in ("", "0", "false", "False")
