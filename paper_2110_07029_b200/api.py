"""Python face of the C-ABI: one Replica per GPU process.

PyTorch provides only device memory (the workspace arena, the resident
dataset buffer) and the CUDA stream; every step of the path runs inside
libadasgd.so.  Names follow include/adasgd.h.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2110_07029_b200 needs a CUDA device (no CPU fallback)")
    return torch


class Replica:
    """One model replica = one as_ctx (include/adasgd.h)."""

    def __init__(self, d, C_labels, h, b_max, init_params, *, b_min=None, beta=None, megabatch=None,
                 max_row_nnz=1024, max_row_labels=64, lr0=0.1, gamma=0.9, delta=0.1, pert_thr=0.1,
                 precision="bf16", rank=0, world=1, nccl_id=None, device=0, stream=None,
                 debug_grads=False, algo="adaptive", merge_norm="u", norm_metric="l2/P",
                 merge_backend="nccl", merge_ties="lex"):
        torch = _torch()
        self.lib = L.load()
        b_min = b_max // 8 if b_min is None else b_min
        beta = max(b_min // 2, 0) if beta is None else beta
        megabatch = 100 * b_max if megabatch is None else megabatch
        torch.cuda.set_device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        cfg = L.Config()
        cfg.n_features, cfg.n_labels, cfg.hidden = d, C_labels, h
        cfg.b_max, cfg.b_min, cfg.beta, cfg.megabatch = b_max, max(b_min, 1), beta, megabatch
        cfg.algo = L.ALGOS[algo]
        cfg.max_row_nnz, cfg.max_row_labels = max_row_nnz, max_row_labels
        cfg.lr0, cfg.gamma, cfg.delta, cfg.pert_thr = lr0, gamma, delta, pert_thr
        cfg.precision = L.AS_BF16 if precision == "bf16" else L.AS_FP32
        cfg.flags = ((L.AS_FLAG_DEBUG_GRADS if debug_grads else 0) | (L.AS_FLAG_NORM_UB if merge_norm == "ub" else 0)
                     | (L.METRICS[norm_metric] << L.AS_NORM_METRIC_SHIFT)
                     | (L.AS_FLAG_R14_LITERAL if merge_ties == "literal" else 0))
        cfg.rank, cfg.world, cfg.device = rank, world, device
        cfg.merge_backend = L.MERGE_BACKENDS[merge_backend]
        self._nccl_buf = None
        if nccl_id is not None:
            self._nccl_buf = C.create_string_buffer(bytes(nccl_id), 128)
            cfg.nccl_unique_id = C.cast(self._nccl_buf, C.c_void_p)
        cfg.stream = C.c_void_p(self.stream.cuda_stream)
        nbytes = C.c_size_t()
        L.check(self.lib.as_workspace_size(C.byref(cfg), C.byref(nbytes)))
        self.workspace = torch.empty(nbytes.value, dtype=torch.uint8, device="cuda:%d" % device)
        cfg.workspace, cfg.workspace_bytes = self.workspace.data_ptr(), nbytes.value
        self.cfg = cfg
        self.d, self.C, self.h, self.rank, self.world = d, C_labels, h, rank, world
        self.P = d * h + h + C_labels * h + C_labels
        init = L.as_np(init_params, np.float32)
        assert init.size == self.P, "init_params must hold P = %d floats" % self.P
        ctx = C.c_void_p()
        L.check(self.lib.as_init(C.byref(cfg), L.ptr(init, C.c_float), C.byref(ctx)))
        self.ctx = ctx
        self.dataset_buf = None

    # ---- batches ---------------------------------------------------------
    def load_batch_csr(self, rows, row_ptr, col, val, lab_ptr, lab):
        rp, cl, vl = L.as_np(row_ptr, np.int64), L.as_np(col, np.int32), L.as_np(val, np.float32)
        lp, lb = L.as_np(lab_ptr, np.int64), L.as_np(lab, np.int32)
        L.check(self.lib.as_load_batch_csr(self.ctx, int(rows), L.ptr(rp, C.c_int64), L.ptr(cl, C.c_int32),
                                           L.ptr(vl, C.c_float), L.ptr(lp, C.c_int64),
                                           L.ptr(lb, C.c_int32)))

    def eval_top1(self, rows, row_ptr, col, val, lab_ptr, lab):
        """as_eval_top1: (top1 class ids [rows] int32, hits) of the current model."""
        rp, cl, vl = L.as_np(row_ptr, np.int64), L.as_np(col, np.int32), L.as_np(val, np.float32)
        lp, lb = L.as_np(lab_ptr, np.int64), L.as_np(lab, np.int32)
        top1 = np.empty(int(rows), np.int32)
        hits = C.c_int64()
        L.check(self.lib.as_eval_top1(self.ctx, int(rows), L.ptr(rp, C.c_int64), L.ptr(cl, C.c_int32),
                                      L.ptr(vl, C.c_float), L.ptr(lp, C.c_int64), L.ptr(lb, C.c_int32),
                                      L.ptr(top1, C.c_int32), C.byref(hits)))
        return top1, int(hits.value)

    def evaluate(self, ds, batch=None):
        """Top-1 accuracy of the current model over a whole CSR dataset, in
        batches of at most b_max rows (the paper's per-mega-batch test metric)."""
        b = int(batch or self.cfg.b_max)
        n = len(ds.row_ptr) - 1
        hits = 0
        for a in range(0, n, b):
            r = min(b, n - a)
            c0, c1 = ds.row_ptr[a], ds.row_ptr[a + r]
            l0, l1 = ds.lab_ptr[a], ds.lab_ptr[a + r]
            _, h = self.eval_top1(r, ds.row_ptr[a:a + r + 1] - c0, ds.col[c0:c1], ds.val[c0:c1],
                                  ds.lab_ptr[a:a + r + 1] - l0, ds.lab[l0:l1])
            hits += h
        return hits / max(n, 1)

    def upload_dataset(self, ds, order=None):
        torch = _torch()
        rp, cl, vl = L.as_np(ds.row_ptr, np.int64), L.as_np(ds.col, np.int32), L.as_np(ds.val, np.float32)
        lp, lb = L.as_np(ds.lab_ptr, np.int64), L.as_np(ds.lab, np.int32)
        n = len(rp) - 1
        nb = C.c_size_t()
        L.check(self.lib.as_dataset_bytes(n, len(cl), len(lb), C.byref(nb)))
        self.dataset_buf = torch.empty(nb.value, dtype=torch.uint8, device=self.workspace.device)
        od = None if order is None else L.as_np(order, np.int64)
        L.check(self.lib.as_dataset_upload(self.ctx, C.c_void_p(self.dataset_buf.data_ptr()), nb.value, n,
                                           L.ptr(rp, C.c_int64), L.ptr(cl, C.c_int32), L.ptr(vl, C.c_float),
                                           L.ptr(lp, C.c_int64), L.ptr(lb, C.c_int32), L.ptr(od, C.c_int64)))

    def load_batch_stream(self, pos, rows):
        L.check(self.lib.as_load_batch_stream(self.ctx, int(pos), int(rows)))

    # ---- step / merge ----------------------------------------------------
    def train_step(self, want_loss=False):
        if want_loss:
            out = C.c_float()
            L.check(self.lib.as_train_step(self.ctx, C.byref(out)))
            return out.value
        L.check(self.lib.as_train_step(self.ctx, None))
        return None

    def merge(self, u, b, want_alpha=True):
        u = L.as_np(u, np.int32); b = L.as_np(b, np.int32)
        if want_alpha:
            alpha = np.zeros(self.world, np.float64); pert = C.c_int32()
            L.check(self.lib.as_merge(self.ctx, L.ptr(u, C.c_int32), L.ptr(b, C.c_int32),
                                      L.ptr(alpha, C.c_double), C.byref(pert)))
            return alpha, pert.value
        L.check(self.lib.as_merge(self.ctx, L.ptr(u, C.c_int32), L.ptr(b, C.c_int32), None, None))
        return None, None

    def merge_weighted(self, alpha):
        """as_merge_weighted: steps a11-a13 with caller-given weights alpha[world]."""
        a = L.as_np(alpha, np.float64)
        L.check(self.lib.as_merge_weighted(self.ctx, L.ptr(a, C.c_double)))

    def replica_norm(self, metric="l2/P"):
        """as_replica_norm: the Alg. 2 line-7 metric of this replica (step a9), fp64."""
        out = C.c_double()
        L.check(self.lib.as_replica_norm(self.ctx, L.METRICS[metric], C.byref(out)))
        return out.value

    def p2p_export(self):
        """as_p2p_export: this rank's peer-mapping record (bytes, AS_P2P_EXPORT_BYTES)."""
        buf = C.create_string_buffer(L.AS_P2P_EXPORT_BYTES)
        L.check(self.lib.as_p2p_export(self.ctx, buf))
        return buf.raw

    def p2p_open(self, records):
        """as_p2p_open: records = the export records of all ranks, rank order."""
        blob = b"".join(bytes(r) for r in records)
        assert len(blob) == L.AS_P2P_EXPORT_BYTES * self.world
        buf = C.create_string_buffer(blob, len(blob))
        L.check(self.lib.as_p2p_open(self.ctx, buf))

    def set_batch_sizes(self, b, lr):
        b = L.as_np(b, np.int32); lr = L.as_np(lr, np.float32)
        L.check(self.lib.as_set_batch_sizes(self.ctx, L.ptr(b, C.c_int32), L.ptr(lr, C.c_float)))

    # ---- inspection --------------------------------------------------------
    def get_params(self, which=L.AS_PARAMS_REPLICA):
        out = np.empty(self.P, np.float32)
        L.check(self.lib.as_get_params(self.ctx, which, L.ptr(out, C.c_float)))
        return out

    def set_params(self, p, which=L.AS_PARAMS_REPLICA):
        p = L.as_np(p, np.float32)
        L.check(self.lib.as_set_params(self.ctx, which, L.ptr(p, C.c_float)))

    def debug_get(self, which, nbytes):
        buf = np.empty(nbytes, np.uint8)
        w = C.c_size_t()
        L.check(self.lib.as_debug_get(self.ctx, which, buf.ctypes.data_as(C.c_void_p), nbytes, C.byref(w)))
        return buf[:w.value]

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.as_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def group_merge(replicas, u, b):
    """as_group_merge over replicas living in this process."""
    lib = L.load()
    u = L.as_np(u, np.int32); b = L.as_np(b, np.int32)
    n = len(replicas)
    arr = (C.c_void_p * n)(*[r.ctx.value for r in replicas])
    alpha = np.zeros(n, np.float64); pert = C.c_int32()
    L.check(lib.as_group_merge(arr, n, L.ptr(u, C.c_int32), L.ptr(b, C.c_int32),
                               L.ptr(alpha, C.c_double), C.byref(pert)))
    return alpha, pert.value


def nccl_unique_id():
    lib = L.load()
    buf = C.create_string_buffer(128)
    L.check(lib.as_nccl_unique_id(buf))
    return buf.raw


def tc_selftest(A, B):
    """A, B: torch bf16 [128,128] cuda tensors -> (S, O, T) fp32 tensors."""
    torch = _torch()
    lib = L.load()
    S = torch.empty(128, 128, dtype=torch.float32, device=A.device)
    O = torch.empty_like(S); T = torch.empty_like(S)
    torch.cuda.synchronize()
    L.check(lib.as_tc_selftest(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()),
                               C.cast(C.c_void_p(S.data_ptr()), C.POINTER(C.c_float)),
                               C.cast(C.c_void_p(O.data_ptr()), C.POINTER(C.c_float)),
                               C.cast(C.c_void_p(T.data_ptr()), C.POINTER(C.c_float))))
    return S, O, T


def tc_selftest2(A, B):
    """A, B: torch bf16 [128,128] -> (V = A B^T, U = bf16(A/4) B) via TMEM-A MMAs."""
    torch = _torch()
    lib = L.load()
    V = torch.empty(128, 128, dtype=torch.float32, device=A.device)
    U = torch.empty_like(V)
    torch.cuda.synchronize()
    L.check(lib.as_tc_selftest2(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()),
                                C.cast(C.c_void_p(V.data_ptr()), C.POINTER(C.c_float)),
                                C.cast(C.c_void_p(U.data_ptr()), C.POINTER(C.c_float))))
    return V, U
