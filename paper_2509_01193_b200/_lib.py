"""Thin ctypes binding of the C ABI in ``include/lobra.h`` (argument marshalling only).

Every compute step runs inside ``liblobra.so`` (hand-written sm_100a kernels); this
module only converts Python / torch arguments to the ABI's plain pointers and sizes.
PyTorch is used by callers for device memory, streams and process groups.  There is no
fallback: if the library is missing, ``load()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblobra.so")

LOBRA_OK, LOBRA_ERR_INPUT, LOBRA_ERR_INFEASIBLE, LOBRA_ERR_BUDGET = 0, 1, 2, 3
LOBRA_ERR_CUDA, LOBRA_ERR_NCCL, LOBRA_ERR_UNSUPPORTED = 4, 5, 6
LOBRA_BF16, LOBRA_FP32 = 0, 1
LOBRA_TP_NONE, LOBRA_TP_COLUMN, LOBRA_TP_ROW = 0, 1, 2

EXPORTED = [
    "lobra_last_error", "lobra_version", "lobra_lora_workspace_bytes", "lobra_lora_saved_bytes",
    "lobra_lora_fwd", "lobra_lora_bwd", "lobra_dispatch", "lobra_nccl_unique_id",
    "lobra_comm_init", "lobra_comm_destroy", "lobra_comm_tp_info", "lobra_adapter_allreduce",
    "lobra_shutdown", "lobra_profile_enable", "lobra_profile_read", "lobra_launch_count",
    "lobra_adamw_step", "lobra_plan_deployment", "lobra_propose_configs",
    "lobra_lora_group_workspace_bytes", "lobra_lora_group_saved_bytes", "lobra_lora_group_fwd",
    "lobra_lora_group_bwd", "lobra_rmsnorm_fwd", "lobra_rmsnorm_bwd", "lobra_rope", "lobra_swiglu_fwd",
    "lobra_swiglu_bwd", "lobra_add", "lobra_symm_create", "lobra_symm_open", "lobra_symm_destroy",
    "lobra_symm_data", "lobra_symm_allreduce", "lobra_comm_from_symm", "lobra_comm_attach_symm",
    "lobra_attn_workspace_bytes", "lobra_attn_fwd", "lobra_attn_bwd_workspace_bytes", "lobra_attn_bwd", "lobra_replica_time",
]
K_NAMES = ["gemm_fwd", "gemm_bwd", "rowproj", "segred", "finalize", "pad", "fp32", "optim", "layer", "comm"]

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f32p = C.POINTER(C.c_float)


class Batch(C.Structure):
    _fields_ = [("num_seqs", C.c_int32), ("seq_lens", _i32p), ("seq_task", _i32p)]


class Adapters(C.Structure):
    _fields_ = [("num_tasks", C.c_int32), ("ranks", _i32p), ("scales", _f32p),
                ("A", C.c_void_p), ("B", C.c_void_p)]


class Problem(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("in_", C.c_int64), ("out", C.c_int64),
                ("tp_kind", C.c_int32), ("tp", C.c_void_p), ("dA_ld", C.c_int64)]


class GroupProblem(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("in_", C.c_int64), ("num_proj", C.c_int32), ("out", _i64p),
                ("tp_kind", C.c_int32), ("tp", C.c_void_p), ("dA_ld", C.c_int64)]


class GroupAdapters(C.Structure):
    _fields_ = [("num_tasks", C.c_int32), ("ranks", _i32p), ("scales", _f32p),
                ("A", C.POINTER(C.c_void_p)), ("B", C.POINTER(C.c_void_p))]


class Deployment(C.Structure):
    _fields_ = [("num_groups", C.c_int32), ("tp", _i32p), ("replicas", _i32p),
                ("max_tokens", _i32p), ("cost", _i64p)]


class DispatchOut(C.Structure):
    _fields_ = [("num_buckets", C.c_int32), ("boundaries", _i32p), ("d", _i64p),
                ("seq_bucket", _i32p), ("seq_replica", _i32p), ("seq_chunk", _i32p),
                ("pack_order", _i32p), ("replica_cost", _i64p), ("t_hat", C.c_int64),
                ("nodes", C.c_int64)]


class Candidates(C.Structure):
    _fields_ = [("num_configs", C.c_int32), ("tp", _i32p), ("max_tokens", _i32p), ("cost", _i64p)]


class ThruputTable(C.Structure):
    _fields_ = [("num_configs", C.c_int32), ("tp", _i32p), ("pp", _i32p), ("num_lens", C.c_int32),
                ("seq_len", _i32p), ("thruput", C.POINTER(C.c_double)), ("num_gpu_counts", C.c_int32),
                ("gpu_counts", _i32p)]


class PlanOut(C.Structure):
    _fields_ = [("replicas", _i32p), ("boundaries", _i32p), ("demands", _i64p),
                ("num_buckets", C.c_int32), ("plans_total", C.c_int32), ("plans_solved", C.c_int32),
                ("gpus_used", C.c_int32), ("t_hat", C.c_int64)]


class AdamHP(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float), ("step", C.c_int64)]


class Profile(C.Structure):
    _fields_ = [("count", C.c_int64 * len(K_NAMES)), ("ms", C.c_double * len(K_NAMES))]


_LIB = None


class LobraError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"lobra status {status}: {msg}")
        self.status = status


def load() -> C.CDLL:
    """Loads the in-tree ``liblobra.so`` (built by ``__graft_entry__.build()``)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(LIB_PATH)
    lib.lobra_last_error.restype = C.c_char_p
    lib.lobra_version.restype = C.c_char_p
    lib.lobra_lora_workspace_bytes.restype = C.c_size_t
    lib.lobra_lora_workspace_bytes.argtypes = [C.POINTER(Problem), C.POINTER(Batch), C.POINTER(Adapters)]
    lib.lobra_lora_saved_bytes.restype = C.c_size_t
    lib.lobra_lora_saved_bytes.argtypes = [C.POINTER(Problem), C.POINTER(Batch), C.POINTER(Adapters)]
    lib.lobra_lora_fwd.restype = C.c_int
    lib.lobra_lora_fwd.argtypes = [C.POINTER(Problem), C.POINTER(Batch), C.POINTER(Adapters),
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_size_t, C.c_void_p]
    lib.lobra_lora_bwd.restype = C.c_int
    lib.lobra_lora_bwd.argtypes = [C.POINTER(Problem), C.POINTER(Batch), C.POINTER(Adapters),
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                   C.c_size_t, C.c_void_p]
    _gp, _gb, _ga = C.POINTER(GroupProblem), C.POINTER(Batch), C.POINTER(GroupAdapters)
    _vpp = C.POINTER(C.c_void_p)
    lib.lobra_lora_group_workspace_bytes.restype = C.c_size_t
    lib.lobra_lora_group_workspace_bytes.argtypes = [_gp, _gb, _ga]
    lib.lobra_lora_group_saved_bytes.restype = C.c_size_t
    lib.lobra_lora_group_saved_bytes.argtypes = [_gp, _gb, _ga]
    lib.lobra_lora_group_fwd.restype = C.c_int
    lib.lobra_lora_group_fwd.argtypes = [_gp, _gb, _ga, C.c_void_p, _vpp, _vpp, C.c_void_p,
                                         C.c_void_p, C.c_size_t, C.c_void_p]
    lib.lobra_lora_group_bwd.restype = C.c_int
    lib.lobra_lora_group_bwd.argtypes = [_gp, _gb, _ga, C.c_void_p, _vpp, C.c_void_p, _vpp,
                                         C.c_void_p, C.c_int, _vpp, _vpp, C.c_int, C.c_void_p,
                                         C.c_size_t, C.c_void_p]
    _vp_ = C.c_void_p
    lib.lobra_rmsnorm_fwd.restype = C.c_int
    lib.lobra_rmsnorm_fwd.argtypes = [C.c_int64, C.c_int64, _vp_, _vp_, _vp_, _vp_, C.c_float, _vp_, _vp_, _vp_]
    lib.lobra_rmsnorm_bwd.restype = C.c_int
    lib.lobra_rmsnorm_bwd.argtypes = [C.c_int64, C.c_int64, _vp_, _vp_, _vp_, _vp_, _vp_, _vp_, _vp_]
    lib.lobra_rope.restype = C.c_int
    lib.lobra_rope.argtypes = [C.c_int32, _vp_, C.c_int64, C.c_int32, C.c_int32, C.c_float, _vp_, C.c_int64,
                               _vp_, C.c_int64, C.c_int, _vp_]
    lib.lobra_swiglu_fwd.restype = C.c_int
    lib.lobra_swiglu_fwd.argtypes = [C.c_int64, _vp_, _vp_, _vp_, _vp_]
    lib.lobra_swiglu_bwd.restype = C.c_int
    lib.lobra_swiglu_bwd.argtypes = [C.c_int64, _vp_, _vp_, _vp_, _vp_, _vp_, _vp_]
    lib.lobra_symm_create.restype = C.c_int
    lib.lobra_symm_create.argtypes = [C.c_int32, C.c_int32, C.c_size_t, C.POINTER(C.c_void_p), C.c_void_p]
    lib.lobra_symm_open.restype = C.c_int
    lib.lobra_symm_open.argtypes = [C.c_void_p, C.c_void_p]
    lib.lobra_symm_destroy.restype = C.c_int
    lib.lobra_symm_destroy.argtypes = [C.c_void_p]
    lib.lobra_symm_data.restype = C.c_void_p
    lib.lobra_symm_data.argtypes = [C.c_void_p]
    lib.lobra_symm_allreduce.restype = C.c_int
    lib.lobra_symm_allreduce.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
    lib.lobra_comm_from_symm.restype = C.c_int
    lib.lobra_comm_from_symm.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    lib.lobra_comm_attach_symm.restype = C.c_int
    lib.lobra_comm_attach_symm.argtypes = [C.c_void_p, C.c_void_p]
    lib.lobra_attn_workspace_bytes.restype = C.c_size_t
    lib.lobra_attn_workspace_bytes.argtypes = [C.c_int32, _i32p, C.c_int32]
    lib.lobra_attn_fwd.restype = C.c_int
    lib.lobra_attn_fwd.argtypes = [C.c_int32, _i32p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
    lib.lobra_attn_bwd_workspace_bytes.restype = C.c_size_t
    lib.lobra_attn_bwd_workspace_bytes.argtypes = [C.c_int32, _i32p, C.c_int32, C.c_int32]
    lib.lobra_attn_bwd.restype = C.c_int
    lib.lobra_attn_bwd.argtypes = [C.c_int32, _i32p, C.c_int32, C.c_int32, C.c_int32] + [C.c_void_p] * 10 + \
        [C.c_size_t, C.c_void_p]
    lib.lobra_add.restype = C.c_int
    lib.lobra_add.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.lobra_dispatch.restype = C.c_int
    lib.lobra_dispatch.argtypes = [C.POINTER(Deployment), C.POINTER(Batch), C.c_int32, C.c_int32,
                                   C.c_int32, C.c_int32, C.c_int32, C.c_int64,
                                   C.POINTER(DispatchOut)]
    lib.lobra_nccl_unique_id.restype = C.c_int
    lib.lobra_nccl_unique_id.argtypes = [C.c_void_p]
    lib.lobra_comm_init.restype = C.c_int
    lib.lobra_comm_init.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]
    lib.lobra_comm_destroy.restype = C.c_int
    lib.lobra_comm_destroy.argtypes = [C.c_void_p]
    lib.lobra_comm_tp_info.restype = C.c_int
    lib.lobra_comm_tp_info.argtypes = [C.c_void_p, _i32p, _i32p]
    lib.lobra_adapter_allreduce.restype = C.c_int
    lib.lobra_adapter_allreduce.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
    lib.lobra_shutdown.restype = C.c_int
    lib.lobra_profile_enable.restype = C.c_int
    lib.lobra_profile_enable.argtypes = [C.c_int]
    lib.lobra_profile_read.restype = C.c_int
    lib.lobra_profile_read.argtypes = [C.POINTER(Profile), C.c_int]
    lib.lobra_launch_count.restype = C.c_int64
    lib.lobra_replica_time.restype = C.c_int
    lib.lobra_replica_time.argtypes = [C.c_int32, _i32p, _i32p, C.c_int64, C.c_int32, C.c_double,
                                       C.c_double, C.c_double, C.POINTER(C.c_double)]
    lib.lobra_propose_configs.restype = C.c_int
    lib.lobra_propose_configs.argtypes = [C.POINTER(ThruputTable), _i32p, _i32p]
    lib.lobra_plan_deployment.restype = C.c_int
    lib.lobra_plan_deployment.argtypes = [C.POINTER(Candidates), C.c_int32, _i32p, C.c_int32,
                                          C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double,
                                          C.c_int64, C.POINTER(PlanOut)]
    lib.lobra_adamw_step.restype = C.c_int
    lib.lobra_adamw_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_size_t, C.POINTER(AdamHP), C.c_int32,
                                     C.c_int64, C.c_float, C.c_void_p]
    _LIB = lib
    return lib


def _check(st: int):
    if st != LOBRA_OK:
        raise LobraError(st, load().lobra_last_error().decode())


def version() -> str:
    return load().lobra_version().decode()


# ---------------------------------------------------------------------------- marshalling
def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(x) -> int:
    """Device (or host) address of a torch tensor / int."""
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    return int(x.data_ptr())


def _stream(stream) -> int:
    if stream is None:
        import torch
        return int(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


class _Args:
    """Keeps the numpy arrays alive while their pointers are inside ctypes structs."""

    def __init__(self, dtype, d_in, d_out, seq_lens, seq_task, ranks, scales, A=None, B=None,
                 tp_kind=LOBRA_TP_NONE, comm=None, dA_ld=0):
        self.lens = _i32(seq_lens)
        self.tasks = _i32(seq_task)
        self.ranks = _i32(ranks)
        self.scales = np.ascontiguousarray(np.asarray(scales, dtype=np.float32))
        self.batch = Batch(len(self.lens), self.lens.ctypes.data_as(_i32p),
                           self.tasks.ctypes.data_as(_i32p))
        self.ad = Adapters(len(self.ranks), self.ranks.ctypes.data_as(_i32p),
                           self.scales.ctypes.data_as(_f32p), _ptr(A) or 1, _ptr(B) or 1)
        self.prob = Problem(dtype, d_in, d_out, tp_kind, comm.handle if comm is not None else None,
                            dA_ld)


def _vp(ptrs):
    arr = (C.c_void_p * len(ptrs))(*[_ptr(p) or None for p in ptrs])
    return arr


class _GroupArgs:
    """Projection-group structs (include/lobra.h); keeps every array alive."""

    def __init__(self, dtype, d_in, outs, seq_lens, seq_task, ranks, scales, A=None, B=None,
                 tp_kind=LOBRA_TP_NONE, comm=None, dA_ld=0):
        n = len(outs)
        self.lens = _i32(seq_lens)
        self.tasks = _i32(seq_task)
        self.ranks = _i32(ranks)
        self.scales = np.ascontiguousarray(np.asarray(scales, dtype=np.float32))
        self.outs = np.ascontiguousarray(np.asarray(outs, dtype=np.int64))
        self.batch = Batch(len(self.lens), self.lens.ctypes.data_as(_i32p),
                           self.tasks.ctypes.data_as(_i32p))
        self.A = _vp(A if A is not None else [1] * n)
        self.B = _vp(B if B is not None else [1] * n)
        self.ad = GroupAdapters(len(self.ranks), self.ranks.ctypes.data_as(_i32p),
                                self.scales.ctypes.data_as(_f32p), self.A, self.B)
        self.prob = GroupProblem(dtype, d_in, n, self.outs.ctypes.data_as(_i64p), tp_kind,
                                 comm.handle if comm is not None else None, dA_ld)


def lobra_lora_group_workspace_bytes(dtype: int, d_in: int, outs, seq_lens, seq_task, ranks,
                                     scales) -> int:
    a = _GroupArgs(dtype, d_in, outs, seq_lens, seq_task, ranks, scales)
    n = load().lobra_lora_group_workspace_bytes(C.byref(a.prob), C.byref(a.batch), C.byref(a.ad))
    if n == 0:
        raise LobraError(LOBRA_ERR_INPUT, load().lobra_last_error().decode())
    return int(n)


def lobra_lora_group_saved_bytes(dtype: int, d_in: int, outs, seq_lens, seq_task, ranks,
                                 scales) -> int:
    a = _GroupArgs(dtype, d_in, outs, seq_lens, seq_task, ranks, scales)
    n = load().lobra_lora_group_saved_bytes(C.byref(a.prob), C.byref(a.batch), C.byref(a.ad))
    if n == 0:
        raise LobraError(LOBRA_ERR_INPUT, load().lobra_last_error().decode())
    return int(n)


def lobra_lora_group_fwd(X, Ws, As, Bs, ranks, scales, seq_lens, seq_task, Ys, Hs, ws,
                         ws_bytes=None, tp_kind=LOBRA_TP_NONE, comm=None, stream=None, dtype=None):
    """Projection group sharing X (include/lobra.h): Y_p = X W_p^T + s_t (X A_p,t^T) B_p,t^T."""
    dt = dtype_code(X.dtype) if dtype is None else dtype
    outs = [int(W.shape[0]) for W in Ws]
    a = _GroupArgs(dt, int(X.shape[1]), outs, seq_lens, seq_task, ranks, scales, As, Bs, tp_kind, comm)
    W, Y = _vp(Ws), _vp(Ys)
    nb = ws.numel() * ws.element_size() if ws_bytes is None else ws_bytes
    _check(load().lobra_lora_group_fwd(C.byref(a.prob), C.byref(a.batch), C.byref(a.ad), _ptr(X), W, Y,
                                       _ptr(Hs), _ptr(ws), nb, _stream(stream)))


def lobra_lora_group_bwd(X, Ws, As, Bs, ranks, scales, seq_lens, seq_task, Hs, dYs, dX, dAs, dBs, ws,
                         accumulate_dx=False, accumulate_dadb=False, ws_bytes=None, dA_ld=0,
                         tp_kind=LOBRA_TP_NONE, comm=None, stream=None, dtype=None):
    """dX (+)= sum_p [dY_p W_p + s_t (dY_p B_p,t) A_p,t]; dA_p, dB_p (+)= token sums."""
    dt = dtype_code(X.dtype) if dtype is None else dtype
    outs = [int(W.shape[0]) for W in Ws]
    a = _GroupArgs(dt, int(X.shape[1]), outs, seq_lens, seq_task, ranks, scales, As, Bs, tp_kind, comm,
                   dA_ld)
    W, dY, dA, dB = _vp(Ws), _vp(dYs), _vp(dAs), _vp(dBs)
    nb = ws.numel() * ws.element_size() if ws_bytes is None else ws_bytes
    _check(load().lobra_lora_group_bwd(C.byref(a.prob), C.byref(a.batch), C.byref(a.ad), _ptr(X), W,
                                       _ptr(Hs), dY, _ptr(dX), int(bool(accumulate_dx)), dA, dB,
                                       int(bool(accumulate_dadb)), _ptr(ws), nb, _stream(stream)))


def dtype_code(torch_dtype) -> int:
    import torch
    if torch_dtype == torch.bfloat16:
        return LOBRA_BF16
    if torch_dtype == torch.float32:
        return LOBRA_FP32
    raise ValueError(f"unsupported dtype {torch_dtype}")


def lobra_lora_workspace_bytes(dtype: int, d_in: int, d_out: int, seq_lens, seq_task, ranks,
                               scales) -> int:
    a = _Args(dtype, d_in, d_out, seq_lens, seq_task, ranks, scales)
    n = load().lobra_lora_workspace_bytes(C.byref(a.prob), C.byref(a.batch), C.byref(a.ad))
    if n == 0:
        raise LobraError(LOBRA_ERR_INPUT, load().lobra_last_error().decode())
    return int(n)


def lobra_lora_saved_bytes(dtype: int, d_in: int, d_out: int, seq_lens, seq_task, ranks,
                           scales) -> int:
    a = _Args(dtype, d_in, d_out, seq_lens, seq_task, ranks, scales)
    n = load().lobra_lora_saved_bytes(C.byref(a.prob), C.byref(a.batch), C.byref(a.ad))
    if n == 0:
        raise LobraError(LOBRA_ERR_INPUT, load().lobra_last_error().decode())
    return int(n)


def lobra_lora_fwd(X, W, A, B, ranks, scales, seq_lens, seq_task, Y, Hs, ws, ws_bytes=None,
                   tp_kind=LOBRA_TP_NONE, comm=None, stream=None, dtype=None):
    """Y = X W^T + s_t (X A_t^T) B_t^T per task segment (include/lobra.h)."""
    dt = dtype_code(X.dtype) if dtype is None else dtype
    d_out, d_in = int(W.shape[0]), int(W.shape[1])
    a = _Args(dt, d_in, d_out, seq_lens, seq_task, ranks, scales, A, B, tp_kind, comm)
    nb = ws.numel() * ws.element_size() if ws_bytes is None else ws_bytes
    _check(load().lobra_lora_fwd(C.byref(a.prob), C.byref(a.batch), C.byref(a.ad), _ptr(X), _ptr(W),
                                 _ptr(Y), _ptr(Hs), _ptr(ws), nb, _stream(stream)))


def lobra_lora_bwd(X, W, A, B, ranks, scales, seq_lens, seq_task, Hs, dY, dX, dA, dB, ws,
                   accumulate_dx=False, accumulate_dadb=False, ws_bytes=None, dA_ld=0,
                   tp_kind=LOBRA_TP_NONE, comm=None, stream=None, dtype=None):
    """dX (+)= dY W + s_t (dY B_t) A_t ; dA_t, dB_t (+)= token sums (include/lobra.h)."""
    dt = dtype_code(X.dtype) if dtype is None else dtype
    d_out, d_in = int(W.shape[0]), int(W.shape[1])
    a = _Args(dt, d_in, d_out, seq_lens, seq_task, ranks, scales, A, B, tp_kind, comm, dA_ld)
    nb = ws.numel() * ws.element_size() if ws_bytes is None else ws_bytes
    _check(load().lobra_lora_bwd(C.byref(a.prob), C.byref(a.batch), C.byref(a.ad), _ptr(X), _ptr(W),
                                 _ptr(Hs), _ptr(dY), _ptr(dX), int(bool(accumulate_dx)), _ptr(dA),
                                 _ptr(dB), int(bool(accumulate_dadb)), _ptr(ws), nb, _stream(stream)))


def lobra_dispatch(tp, replicas, max_tokens, cost, seq_lens, seq_task, grid_step=256,
                   grid_max=16384, R=16, mode=0, node_cap=0, chunking=0, allow_budget=False):
    """Per-step dispatch (host).  Returns a dict of numpy arrays; raises LobraError on
    input / infeasibility errors and, unless ``allow_budget``, when the exact Eq. 3 solver
    exhausted its node budget (LOBRA_ERR_BUDGET: the returned d would be the length-based
    one, not the Eq. 3 optimum)."""
    tp, replicas, max_tokens = _i32(tp), _i32(replicas), _i32(max_tokens)
    cost = np.ascontiguousarray(np.asarray(cost, dtype=np.int64))
    G = len(tp)
    lens, tasks = _i32(seq_lens), _i32(seq_task)
    n = len(lens)
    dep = Deployment(G, tp.ctypes.data_as(_i32p), replicas.ctypes.data_as(_i32p),
                     max_tokens.ctypes.data_as(_i32p), cost.ctypes.data_as(_i64p))
    batch = Batch(n, lens.ctypes.data_as(_i32p), tasks.ctypes.data_as(_i32p))
    out = {"boundaries": np.zeros(R, np.int32), "d": np.zeros(G * R, np.int64),
           "seq_bucket": np.zeros(n, np.int32), "seq_replica": np.zeros(n, np.int32),
           "seq_chunk": np.zeros(n, np.int32), "pack_order": np.zeros(n, np.int32),
           "replica_cost": np.zeros(max(int(replicas.sum()), 1), np.int64)}
    o = DispatchOut(0, out["boundaries"].ctypes.data_as(_i32p), out["d"].ctypes.data_as(_i64p),
                    out["seq_bucket"].ctypes.data_as(_i32p), out["seq_replica"].ctypes.data_as(_i32p),
                    out["seq_chunk"].ctypes.data_as(_i32p), out["pack_order"].ctypes.data_as(_i32p),
                    out["replica_cost"].ctypes.data_as(_i64p), 0, 0)
    st = load().lobra_dispatch(C.byref(dep), C.byref(batch), grid_step, grid_max, R, mode,
                               chunking, node_cap, C.byref(o))
    if st != LOBRA_OK and not (st == LOBRA_ERR_BUDGET and allow_budget):
        raise LobraError(st, load().lobra_last_error().decode())
    nb = o.num_buckets
    out["status"] = st
    out["boundaries"] = out["boundaries"][:nb]
    out["d"] = out["d"].reshape(G, R)[:, :nb]
    out["t_hat"] = int(o.t_hat)
    out["nodes"] = int(o.nodes)
    return out


# ---------------------------------------------------------------------------- comm
class Comm:
    """World NCCL communicator + this rank's TP sub-communicator (lobra_comm)."""

    def __init__(self, handle: int, world: int, rank: int, replica_id: int):
        self.handle = handle
        self.world, self.rank, self.replica_id = world, rank, replica_id
        ts, tr = C.c_int32(0), C.c_int32(0)
        _check(load().lobra_comm_tp_info(C.c_void_p(handle), C.byref(ts), C.byref(tr)))
        self.tp_size, self.tp_rank = ts.value, tr.value

    def destroy(self):
        if self.handle:
            load().lobra_comm_destroy(C.c_void_p(self.handle))
            self.handle = 0


def lobra_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(load().lobra_nccl_unique_id(buf))
    return buf.raw


def lobra_comm_init(uid: bytes, world: int, rank: int, replica_id: int) -> Comm:
    h = C.c_void_p(0)
    buf = C.create_string_buffer(uid, 128)
    _check(load().lobra_comm_init(buf, world, rank, replica_id, C.byref(h)))
    return Comm(h.value, world, rank, replica_id)


def lobra_adapter_allreduce(comm: Comm, flat, stream=None):
    _check(load().lobra_adapter_allreduce(C.c_void_p(comm.handle), _ptr(flat), int(flat.numel()),
                                          _stream(stream)))


def lobra_shutdown():
    _check(load().lobra_shutdown())


# ---------------------------------------------------------------------------- tracing
def lobra_profile_enable(on: bool = True):
    _check(load().lobra_profile_enable(int(bool(on))))


def lobra_profile_read(reset: bool = True) -> dict:
    """{kernel class: (launches, device ms)} since the last reset (synchronises)."""
    p = Profile()
    _check(load().lobra_profile_read(C.byref(p), int(bool(reset))))
    return {K_NAMES[k]: (int(p.count[k]), float(p.ms[k])) for k in range(len(K_NAMES))}


def lobra_launch_count() -> int:
    return int(load().lobra_launch_count())


# ---------------------------------------------------------------------------- optimizer
def lobra_adamw_step(params, grads, m, v, hparams, step, group=None, params_bf16=None,
                     grad_scale=1.0, stream=None):
    """One multi-tenant AdamW step (include/lobra.h).  hparams: list of dicts with keys
    lr, beta1, beta2, eps, weight_decay and optionally step (the group's own step count,
    else `step`), one per group; group: uint8 tensor or None."""
    hp = (AdamHP * len(hparams))(*[AdamHP(h["lr"], h["beta1"], h["beta2"], h["eps"],
                                          h["weight_decay"], int(h.get("step", 0))) for h in hparams])
    _check(load().lobra_adamw_step(_ptr(params), _ptr(params_bf16), _ptr(grads), _ptr(m), _ptr(v),
                                   _ptr(group), int(params.numel()), hp, len(hparams), int(step),
                                   float(grad_scale), _stream(stream)))


# ---------------------------------------------------------------------------- planner
def lobra_plan_deployment(tp, max_tokens, cost, n_gpus, lens, batch_size=0, grid_step=256,
                          grid_max=16384, R=16, threshold=0.15, node_cap=0, allow_budget=False):
    """Stage-1 deployment planning (include/lobra.h).  Returns a dict; raises LobraError
    on input/infeasible errors and, unless ``allow_budget``, when a per-plan Eq. 3 solve
    exhausted its node budget (LOBRA_ERR_BUDGET)."""
    tp, max_tokens, lens = _i32(tp), _i32(max_tokens), _i32(lens)
    cost = np.ascontiguousarray(np.asarray(cost, dtype=np.int64))
    S = len(tp)
    reps = np.zeros(S, np.int32)
    bnd = np.zeros(R, np.int32)
    dem = np.zeros(R, np.int64)
    cand = Candidates(S, tp.ctypes.data_as(_i32p), max_tokens.ctypes.data_as(_i32p),
                      cost.ctypes.data_as(_i64p))
    o = PlanOut(reps.ctypes.data_as(_i32p), bnd.ctypes.data_as(_i32p), dem.ctypes.data_as(_i64p),
                0, 0, 0, 0, 0)
    st = load().lobra_plan_deployment(C.byref(cand), n_gpus, lens.ctypes.data_as(_i32p), len(lens),
                                      batch_size, grid_step, grid_max, R, threshold, node_cap,
                                      C.byref(o))
    if st != LOBRA_OK and not (st == LOBRA_ERR_BUDGET and allow_budget):
        raise LobraError(st, load().lobra_last_error().decode())
    nb = o.num_buckets
    return {"status": st, "replicas": reps, "boundaries": bnd[:nb], "demands": dem[:nb],
            "plans_total": o.plans_total, "plans_solved": o.plans_solved, "gpus_used": o.gpus_used,
            "t_hat": int(o.t_hat)}


def lobra_replica_time(d, s, max_tokens, pp_stages, c0, c1, c2) -> float:
    """App. D replica time with 1F1B bubble (include/lobra.h): buckets (d[j] sequences of
    length s[j]), micro-batch token limit max_tokens, t(b, s) = c0 + c1 b s + c2 b s^2."""
    d, s = _i32(d), _i32(s)
    out = C.c_double(0.0)
    st = load().lobra_replica_time(len(d), d.ctypes.data_as(_i32p), s.ctypes.data_as(_i32p), int(max_tokens),
                                   int(pp_stages), float(c0), float(c1), float(c2), C.byref(out))
    if st != LOBRA_OK:
        raise LobraError(st, load().lobra_last_error().decode())
    return out.value


def lobra_propose_configs(tp, pp, seq_lens, thruput, gpu_counts):
    """Configuration proposal from a throughput table (include/lobra.h).  Returns
    (winner [K, L] int32 with -1 for empty groups, keep [C] int32)."""
    tp, pp, sl, gc = _i32(tp), _i32(pp), _i32(seq_lens), _i32(gpu_counts)
    th = np.ascontiguousarray(np.asarray(thruput, dtype=np.float64).reshape(len(tp), len(sl)))
    win = np.zeros((len(gc), len(sl)), np.int32)
    keep = np.zeros(len(tp), np.int32)
    t = ThruputTable(len(tp), tp.ctypes.data_as(_i32p), pp.ctypes.data_as(_i32p), len(sl),
                     sl.ctypes.data_as(_i32p), th.ctypes.data_as(C.POINTER(C.c_double)), len(gc),
                     gc.ctypes.data_as(_i32p))
    st = load().lobra_propose_configs(C.byref(t), win.ctypes.data_as(_i32p), keep.ctypes.data_as(_i32p))
    if st != LOBRA_OK:
        raise LobraError(st, load().lobra_last_error().decode())
    return win, keep


# ------------------------------------------------------------------ decoder-layer ops
def lobra_rmsnorm_fwd(X, g, eps, Y, rstd, R=None, S_out=None, stream=None):
    """Y = rmsnorm(X (+ R)) * g; S_out = X + R when R is given (include/lobra.h)."""
    T, h = int(X.shape[0]), int(X.shape[1])
    _check(load().lobra_rmsnorm_fwd(T, h, _ptr(X), _ptr(R) or None, _ptr(S_out) or None, _ptr(g), float(eps),
                                    _ptr(Y), _ptr(rstd), _stream(stream)))


def lobra_rmsnorm_bwd(dY, S, g, rstd, dS, dRes=None, stream=None):
    T, h = int(S.shape[0]), int(S.shape[1])
    _check(load().lobra_rmsnorm_bwd(T, h, _ptr(dY), _ptr(S), _ptr(g), _ptr(rstd), _ptr(dRes) or None, _ptr(dS),
                                    _stream(stream)))


def lobra_rope(cu_seqlens, T, n_heads, head_dim, theta, Q, K=None, inverse=False, stream=None):
    """In-place rotary embedding on Q (and K), positions restarted per packed sequence."""
    ldq = int(Q.stride(0))
    ldk = int(K.stride(0)) if K is not None else 0
    _check(load().lobra_rope(int(cu_seqlens.numel()) - 1, _ptr(cu_seqlens), int(T), int(n_heads), int(head_dim),
                             float(theta), _ptr(Q), ldq, _ptr(K) or None, ldk, int(bool(inverse)), _stream(stream)))


def lobra_swiglu_fwd(gate, up, act, stream=None):
    _check(load().lobra_swiglu_fwd(int(gate.numel()), _ptr(gate), _ptr(up), _ptr(act), _stream(stream)))


def lobra_swiglu_bwd(d, gate, up, d_gate, d_up, stream=None):
    _check(load().lobra_swiglu_bwd(int(gate.numel()), _ptr(d), _ptr(gate), _ptr(up), _ptr(d_gate), _ptr(d_up),
                                   _stream(stream)))


def lobra_add(A, B, C_, stream=None):
    _check(load().lobra_add(int(A.numel()), _ptr(A), _ptr(B), _ptr(C_), _stream(stream)))


# ------------------------------------------------------------------ own peer-memory collectives
class Symm:
    """Symmetric device buffer of one rank of a TP group (include/lobra.h lobra_symm_*).
    Usage: s = Symm(rank, world, nbytes); handles = all_gather(s.handle); s.open(handles)."""

    def __init__(self, rank: int, world: int, nbytes: int):
        h = C.c_void_p(0)
        buf = C.create_string_buffer(64)
        _check(load().lobra_symm_create(rank, world, nbytes, C.byref(h), buf))
        self.ptr, self.handle = h.value, buf.raw
        self.rank, self.world, self.nbytes = rank, world, nbytes

    def open(self, handles):
        blob = b"".join(handles)
        assert len(blob) == 64 * self.world
        _check(load().lobra_symm_open(C.c_void_p(self.ptr), C.create_string_buffer(blob, len(blob))))

    def data_ptr(self) -> int:
        return int(load().lobra_symm_data(C.c_void_p(self.ptr)))

    def allreduce(self, src, dst=None, stream=None):
        dst = src if dst is None else dst
        _check(load().lobra_symm_allreduce(C.c_void_p(self.ptr), dtype_code(src.dtype), _ptr(src), _ptr(dst),
                                           int(src.numel()), _stream(stream)))

    def destroy(self):
        if self.ptr:
            load().lobra_symm_destroy(C.c_void_p(self.ptr))
            self.ptr = 0


def lobra_comm_from_symm(symm: Symm) -> Comm:
    h = C.c_void_p(0)
    _check(load().lobra_comm_from_symm(C.c_void_p(symm.ptr), C.byref(h)))
    return Comm(h.value, symm.world, symm.rank, 0)


def lobra_comm_attach_symm(comm: Comm, symm: Symm | None):
    _check(load().lobra_comm_attach_symm(C.c_void_p(comm.handle), C.c_void_p(symm.ptr if symm else 0)))


# ------------------------------------------------------------------ attention (NEXT-3)
def lobra_attn_workspace_bytes(seq_lens, n_heads) -> int:
    lens = _i32(seq_lens)
    return int(load().lobra_attn_workspace_bytes(len(lens), lens.ctypes.data_as(_i32p), int(n_heads)))


def lobra_attn_bwd_workspace_bytes(seq_lens, n_heads, n_kv_heads) -> int:
    lens = _i32(seq_lens)
    return int(load().lobra_attn_bwd_workspace_bytes(len(lens), lens.ctypes.data_as(_i32p), int(n_heads),
                                                     int(n_kv_heads)))


def lobra_attn_bwd(seq_lens, Q, K, V, O, dO, lse, dQ, dK, dV, ws, stream=None):
    """Gradients of lobra_attn_fwd (tcgen05): dQ [T, H, 128], dK, dV [T, Hkv, 128] (include/lobra.h)."""
    lens = _i32(seq_lens)
    H, D, Hkv = int(Q.shape[-2]), int(Q.shape[-1]), int(K.shape[-2])
    _check(load().lobra_attn_bwd(len(lens), lens.ctypes.data_as(_i32p), H, Hkv, D, _ptr(Q), _ptr(K), _ptr(V),
                                 _ptr(O), _ptr(dO), _ptr(lse), _ptr(dQ), _ptr(dK), _ptr(dV), _ptr(ws),
                                 ws.numel() * ws.element_size(), _stream(stream)))


def lobra_attn_fwd(seq_lens, Q, K, V, O, lse, ws, stream=None):
    """Causal attention per packed sequence (tcgen05): Q [T, H, 128], K, V [T, Hkv, 128],
    O [T, H, 128], lse [H, T] (include/lobra.h)."""
    lens = _i32(seq_lens)
    H, D, Hkv = int(Q.shape[-2]), int(Q.shape[-1]), int(K.shape[-2])
    _check(load().lobra_attn_fwd(len(lens), lens.ctypes.data_as(_i32p), H, Hkv, D, _ptr(Q), _ptr(K), _ptr(V),
                                 _ptr(O), _ptr(lse), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))
