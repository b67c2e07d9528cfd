"""ctypes binding of the C-ABI in include/adasgd.h (argument marshalling only).

Every step of the hot path runs inside libadasgd.so (CUDA kernels for sm_100a +
NCCL).  There is no CPU fallback: if the library cannot be loaded this module
raises, and so does every call on a box without a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ADASGD_LIB", os.path.join(HERE, "libadasgd.so"))

AS_OK, AS_E_INVALID, AS_E_CUDA, AS_E_NCCL, AS_E_OOM, AS_E_STATE = 0, -1, -2, -3, -4, -5
AS_FP32, AS_BF16 = 0, 1
AS_ALGO_ADAPTIVE, AS_ALGO_ELASTIC, AS_ALGO_SYNC = 0, 1, 2
AS_MERGE_NCCL, AS_MERGE_P2P = 0, 1
MERGE_BACKENDS = {"nccl": AS_MERGE_NCCL, "p2p": AS_MERGE_P2P}
AS_MAX_WORLD = 64
AS_P2P_EXPORT_BYTES = 128
ALGOS = {"adaptive": AS_ALGO_ADAPTIVE, "elastic": AS_ALGO_ELASTIC, "sync": AS_ALGO_SYNC}
AS_FLAG_DEBUG_GRADS, AS_FLAG_NORM_UB = 1, 2
AS_NORM_UPDATES, AS_NORM_UB, AS_NORM_R14_LITERAL = 0, 1, 2
AS_FLAG_R14_LITERAL = 16
AS_NORM_METRIC_SHIFT = 2
METRICS = {"l2/P": 0, "l2^2/P": 1, "l2/sqrt(P)": 2, "l2": 3}
AS_PARAMS_REPLICA, AS_PARAMS_GLOBAL, AS_PARAMS_GLOBAL_PREV = 0, 1, 2
(AS_DBG_H, AS_DBG_LSE, AS_DBG_LOSS, AS_DBG_DA, AS_DBG_DB1, AS_DBG_DW2T, AS_DBG_DB2, AS_DBG_DW1,
 AS_DBG_FSEG, AS_DBG_LSEG, AS_DBG_BATCH, AS_DBG_LOGITS, AS_DBG_DHSOFT) = range(13)

# every exported symbol of include/adasgd.h (checked by tests/test_abi.py)
EXPORTS = [
    "as_workspace_size", "as_nccl_unique_id", "as_init", "as_destroy", "as_last_error",
    "as_load_batch_csr", "as_dataset_bytes", "as_dataset_upload", "as_load_batch_stream",
    "as_train_step", "as_merge", "as_group_merge", "as_set_batch_sizes", "as_get_params",
    "as_set_params", "as_debug_get", "as_tc_selftest", "as_sched_route_replay", "as_sched_alg1",
    "as_sched_alg2", "as_sched_permutation", "as_live_open", "as_live_claim", "as_live_reset",
    "as_live_close", "as_profile", "as_profile_read", "as_tc_bench", "as_trace_dump", "as_tc_selftest2",
    "as_eval_top1", "as_sched_route_static", "as_sched_alg2_ex", "as_sched_fit_cost",
    "as_sched_scale_period", "as_replica_norm", "as_merge_weighted", "as_p2p_export", "as_p2p_open",
]
AS_PH_NAMES = ["batch", "transpose", "spmm", "out_fwd", "combine", "out_bwd", "dw1", "merge"]


class ASError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("adasgd error %d: %s" % (code, msg))
        self.code = code


class Config(C.Structure):
    _fields_ = [
        ("n_features", C.c_int64), ("n_labels", C.c_int64), ("hidden", C.c_int32),
        ("b_max", C.c_int32), ("b_min", C.c_int32), ("beta", C.c_int32), ("megabatch", C.c_int64),
        ("max_row_nnz", C.c_int32), ("max_row_labels", C.c_int32), ("lr0", C.c_double),
        ("gamma", C.c_double), ("delta", C.c_double), ("pert_thr", C.c_double),
        ("precision", C.c_int32), ("flags", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
        ("nccl_unique_id", C.c_void_p), ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
        ("stream", C.c_void_p), ("device", C.c_int32), ("algo", C.c_int32),
        ("merge_backend", C.c_int32),
    ]


class CostModel(C.Structure):
    _fields_ = [("c0", C.c_int64), ("c_row", C.c_int64), ("c_nnz", C.c_int64),
                ("num", C.c_int64), ("den", C.c_int64)]


class Route(C.Structure):
    _fields_ = [("replica", C.c_int32), ("rows", C.c_int32), ("start", C.c_int64)]


_LIB = None


def load():
    """Load libadasgd.so (building it first if the sources are newer)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if os.environ.get("ADASGD_NO_BUILD") != "1":
        from . import build as _build
        try:
            _build.build()
        except Exception:
            if not os.path.exists(LIB_PATH):
                raise
    if not os.path.exists(LIB_PATH):
        raise ImportError("libadasgd.so not built: run __graft_entry__.build()")
    lib = C.CDLL(LIB_PATH)
    P, I32, I64, VP, D, F = C.POINTER, C.c_int32, C.c_int64, C.c_void_p, C.c_double, C.c_float
    sig = {
        "as_workspace_size": [P(Config), P(C.c_size_t)],
        "as_nccl_unique_id": [VP],
        "as_init": [P(Config), P(F), P(VP)],
        "as_destroy": [VP],
        "as_load_batch_csr": [VP, I32, P(I64), P(I32), P(F), P(I64), P(I32)],
        "as_eval_top1": [VP, I32, P(I64), P(I32), P(F), P(I64), P(I32), P(I32), P(I64)],
        "as_dataset_bytes": [I64, I64, I64, P(C.c_size_t)],
        "as_dataset_upload": [VP, VP, C.c_size_t, I64, P(I64), P(I32), P(F), P(I64), P(I32), P(I64)],
        "as_load_batch_stream": [VP, I64, I32],
        "as_train_step": [VP, P(F)],
        "as_merge": [VP, P(I32), P(I32), P(D), P(I32)],
        "as_group_merge": [P(VP), I32, P(I32), P(I32), P(D), P(I32)],
        "as_set_batch_sizes": [VP, P(I32), P(F)],
        "as_get_params": [VP, I32, P(F)],
        "as_set_params": [VP, I32, P(F)],
        "as_debug_get": [VP, I32, VP, C.c_size_t, P(C.c_size_t)],
        "as_tc_selftest": [VP, VP, P(F), P(F), P(F)],
        "as_sched_route_replay": [I32, P(CostModel), P(I32), I64, P(I64), P(Route), I64, P(I64),
                                  P(I32), P(I64)],
        "as_sched_route_static": [I32, P(CostModel), P(I32), I64, P(I64), P(Route), I64, P(I64),
                                  P(I32), P(I64)],
        "as_sched_alg1": [I32, P(I32), P(I32), I32, I32, I32, D, P(I32), P(F)],
        "as_sched_alg2": [I32, P(I32), P(I32), P(D), D, D, P(D), P(I32)],
        "as_sched_alg2_ex": [I32, P(I32), P(I32), P(D), D, D, I32, P(D), P(I32)],
        "as_sched_scale_period": [I32, P(I32), P(I32), P(I32), I32, I32, P(I32)],
        "as_sched_fit_cost": [I64, P(I32), P(I64), P(I64), P(CostModel)],
        "as_sched_permutation": [I64, C.c_uint64, P(I64)],
        "as_live_open": [C.c_char_p, I32, P(VP)],
        "as_live_claim": [VP, I64, I32, P(I64), P(I32)],
        "as_live_reset": [VP],
        "as_live_close": [VP, I32],
        "as_profile": [VP, I32],
        "as_tc_bench": [I32, I32, P(I64)],
        "as_tc_selftest2": [VP, VP, P(F), P(F)],
        "as_trace_dump": [P(I64), I32],
        "as_profile_read": [VP, P(D), P(I64), P(I64)],
        "as_replica_norm": [VP, I32, P(D)],
        "as_merge_weighted": [VP, P(D)],
        "as_p2p_export": [VP, VP],
        "as_p2p_open": [VP, VP],
    }
    for name, args in sig.items():
        if not hasattr(lib, name):          # an older experiment build (A/B runs); the product
            continue                        # library exports everything (tests/test_abi.py)
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.as_last_error.argtypes = []
    lib.as_last_error.restype = C.c_char_p
    _LIB = lib
    return lib


def check(rc):
    if rc != AS_OK:
        raise ASError(rc, _LIB.as_last_error().decode(errors="replace"))


def ptr(a, ctype):
    """Pointer to the data of a C-contiguous numpy array (None -> NULL)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))


def as_np(a, dtype):
    return np.ascontiguousarray(np.asarray(a), dtype=dtype)
