"""ctypes declarations of include/ac.h and include/ac_kernels.h.

Argument marshalling only: every step of the path runs inside libautochunk.so.
Importing fails loudly if the library has not been built (no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AC_LIB_PATH") or os.path.join(HERE, "libautochunk.so")  # (override: A/B variants)

AC_OK, AC_ERR_ARG, AC_ERR_GRAPH, AC_ERR_BUDGET, AC_ERR_PLAN, AC_ERR_UNSUPPORTED, AC_ERR_BIND, \
    AC_ERR_CUDA, AC_ERR_NCCL, AC_ERR_WORKSPACE = range(10)
STATUS_NAMES = ["AC_OK", "AC_ERR_ARG", "AC_ERR_GRAPH", "AC_ERR_BUDGET", "AC_ERR_PLAN", "AC_ERR_UNSUPPORTED",
                "AC_ERR_BIND", "AC_ERR_CUDA", "AC_ERR_NCCL", "AC_ERR_WORKSPACE"]
AC_F32, AC_BF16, AC_F64 = 0, 1, 2
AC_BLOCK_TRANSFORMER, AC_BLOCK_ATTN_ONLY, AC_BLOCK_TRI_ATTN_PAIR = 0, 1, 2
AC_BLOCK_TRANSFORMER_FA, AC_BLOCK_ATTN_ONLY_FA, AC_BLOCK_EVOFORMER_PAIR = 3, 4, 5
AC_FLAG_NO_HOIST, AC_FLAG_NO_DENSITY, AC_FLAG_NO_STRIDE, AC_FLAG_NO_NODES, AC_FLAG_NO_FLOPS, \
    AC_FLAG_CONTIGUITY, AC_FLAG_NORMALIZE = 1, 2, 4, 8, 16, 32, 64


class ACError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 10 else status}: {msg}")
        self.status = status


class BlockDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("N", C.c_int64), ("d", C.c_int64), ("h", C.c_int64), ("f", C.c_int64),
                ("causal", C.c_int32), ("dtype", C.c_int32), ("ln_eps", C.c_double), ("name", C.c_char_p),
                ("layers", C.c_int32)]


class MemProfile(C.Structure):
    _fields_ = [("peak_bytes", C.c_int64), ("peak_step", C.c_int32), ("n_steps", C.c_int32),
                ("x_bytes", C.c_int64), ("y_bytes", C.c_int64), ("a_bytes", C.c_int64)]


class CostParams(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("gamma", C.c_double), ("lambda_", C.c_double),
                ("beam", C.c_int32), ("window", C.c_int32), ("max_passes", C.c_int32), ("max_chunks", C.c_int32),
                ("flags", C.c_uint32), ("allowed_dims_mask", C.c_uint32)]


class Tensor(C.Structure):
    _fields_ = [("tensor_id", C.c_char_p), ("dtype", C.c_int32), ("ndim", C.c_int32),
                ("shape", C.c_int64 * 6), ("stride", C.c_int64 * 6), ("data", C.c_void_p)]


class RunStats(C.Structure):
    _fields_ = [("workspace_high_water", C.c_int64), ("planned_peak", C.c_int64), ("caller_bytes", C.c_int64),
                ("launches", C.c_int32), ("chunks_run", C.c_int32), ("arena_live_peak", C.c_int64),
                ("control_bytes", C.c_int64), ("exchanges", C.c_int32), ("pipelined_chunks", C.c_int32)]


class ExchangeOp(C.Structure):
    _fields_ = [("kind", C.c_int32), ("before_node", C.c_int32), ("region", C.c_int32), ("eager", C.c_int32),
                ("group", C.c_int64), ("c_first", C.c_int64), ("dim", C.c_int32), ("root", C.c_int32),
                ("outer", C.c_int64), ("run_bytes", C.c_int64), ("ext_bytes", C.c_int64), ("offset", C.c_int64),
                ("tensor", C.c_char * 48)]


class KernelTime(C.Structure):
    _fields_ = [("node", C.c_char * 48), ("kind", C.c_char * 16), ("ms", C.c_double), ("launches", C.c_int32)]


class GemmDesc(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("M", C.c_int32), ("N", C.c_int32), ("K", C.c_int32),
                ("B1", C.c_int32), ("B2", C.c_int32),
                ("a", C.c_void_p), ("a_srow", C.c_int64), ("a_sb1", C.c_int64), ("a_sb2", C.c_int64),
                ("a_use_b1", C.c_int32), ("a_use_b2", C.c_int32),
                ("b", C.c_void_p), ("b_srow", C.c_int64), ("b_sb1", C.c_int64), ("b_sb2", C.c_int64),
                ("b_use_b1", C.c_int32), ("b_use_b2", C.c_int32),
                ("scale", C.c_float), ("act", C.c_int32), ("causal", C.c_int32),
                ("row_off", C.c_int64), ("col_off", C.c_int64),
                ("causal_tiles", C.c_int32), ("causal_k", C.c_int32), ("k_row_off", C.c_int64),
                ("bias", C.c_void_p), ("bias_along_m", C.c_int32),
                ("add", C.c_void_p), ("add_sb1", C.c_int64), ("add_sb2", C.c_int64), ("add_sm", C.c_int64),
                ("add_sn", C.c_int64),
                ("gate", C.c_void_p), ("res", C.c_void_p),
                ("out", C.c_void_p), ("out_sb1", C.c_int64), ("out_sb2", C.c_int64), ("out_sm", C.c_int64),
                ("out_sn", C.c_int64), ("bn", C.c_int32), ("cta_pair", C.c_int32)]


# (name, restype, argtypes) for every symbol declared in include/*.h
P = C.c_void_p
SIGNATURES = [
    ("ac_last_error", C.c_char_p, []),
    ("ac_version", C.c_char_p, []),
    ("ac_graph_parse", C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(P)]),
    ("ac_graph_block", C.c_int, [C.POINTER(BlockDesc), C.POINTER(P)]),
    ("ac_graph_serialize", C.c_int, [P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("ac_graph_free", None, [P]),
    ("ac_graph_num_nodes", C.c_int32, [P]),
    ("ac_estimate_memory", C.c_int, [P, P, C.POINTER(MemProfile), C.POINTER(C.c_int64)]),
    ("ac_cost_params_default", None, [C.POINTER(CostParams)]),
    ("ac_plan", C.c_int, [P, C.c_int64, C.POINTER(CostParams), C.POINTER(P)]),
    ("ac_plan_parse", C.c_int, [P, C.c_char_p, C.c_size_t, C.POINTER(P)]),
    ("ac_plan_serialize", C.c_int, [P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("ac_plan_free", None, [P]),
    ("ac_plan_num_regions", C.c_int32, [P]),
    ("ac_plan_workspace_bytes", C.c_int64, [P, C.c_int32, C.c_int32]),
    ("ac_max_length", C.c_int, [C.POINTER(BlockDesc), C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("ac_plan_arena_profile", C.c_int, [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("ac_plan_rank_chunks", C.c_int, [P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.c_int32,
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64)]),
    ("ac_plan_rank_schedule", C.c_int, [P, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                        C.POINTER(ExchangeOp), C.c_int32, C.POINTER(C.c_int32)]),
    ("ac_comm_get_unique_id", C.c_int, [C.c_char_p]),
    ("ac_comm_init", C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(P)]),
    ("ac_comm_init_local", C.c_int, [C.c_int32, C.POINTER(P)]),
    ("ac_comm_check", C.c_int, [P]),
    ("ac_comm_free", None, [P]),
    ("ac_exec_create", C.c_int, [P, P, C.c_int64, P, C.POINTER(P)]),
    ("ac_exec_free", None, [P]),
    ("ac_run", C.c_int, [P, C.POINTER(Tensor), C.c_int32, C.POINTER(Tensor), C.c_int32, P]),
    ("ac_exec_stats", C.c_int, [P, C.POINTER(RunStats)]),
    ("ac_plan_chunk_pipeline", C.c_int, [P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    ("ac_exec_set_profiling", C.c_int, [P, C.c_int32]),
    ("ac_exec_kernel_times", C.c_int, [P, C.POINTER(KernelTime), C.c_int32, C.POINTER(C.c_int32)]),
    ("ac_kernel_gemm", C.c_int, [C.POINTER(GemmDesc), P]),
    ("ac_kernel_layernorm", C.c_int, [P, P, P, P, C.c_int64, C.c_int32, C.c_float, C.c_int32, P]),
    ("ac_kernel_softmax", C.c_int, [P, P, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int64, C.c_int64,
                                    C.c_int32, P]),
]

_lib = None


def lib():
    """Load libautochunk.so (built by paper_2401_10652_b200.build); raise if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2401_10652_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int):
    if status != AC_OK:
        raise ACError(status, lib().ac_last_error().decode())
    return status
