"""Scheduler calls of the C-ABI (pure host functions in libadasgd.so):
replay routing, Alg. 1, Alg. 2 weights,
stream permutation (R10) and the live shared cursor."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L


def route_replay(costs, b, M, nnz_prefix, static=False):
    """costs: sequence of (c0, c_row, c_nnz, num, den); b: batch sizes;
    nnz_prefix: int64[M+1].  Returns (log [(replica, start, rows)], u, clocks).
    static=True: as_sched_route_static (batch k -> replica k mod N)."""
    lib = L.load()
    N = len(b)
    cm = (L.CostModel * N)(*[L.CostModel(*[int(v) for v in c]) for c in costs])
    bb = L.as_np(b, np.int32)
    pre = L.as_np(nnz_prefix, np.int64)
    assert len(pre) == M + 1
    cap = int(M // max(1, min(b))) + N + 2
    log = (L.Route * cap)()
    nlog = C.c_int64()
    u = np.zeros(N, np.int32)
    clk = np.zeros(N, np.int64)
    fn = lib.as_sched_route_static if static else lib.as_sched_route_replay
    L.check(fn(N, cm, L.ptr(bb, C.c_int32), int(M), L.ptr(pre, C.c_int64), log, cap,
               C.byref(nlog), L.ptr(u, C.c_int32), L.ptr(clk, C.c_int64)))
    return [(log[k].replica, int(log[k].start), log[k].rows) for k in range(nlog.value)], u.tolist(), clk.tolist()


def alg1(u, b, beta, b_min, b_max, lr0):
    lib = L.load()
    N = len(u)
    uu, bb = L.as_np(u, np.int32), L.as_np(b, np.int32)
    bo = np.zeros(N, np.int32)
    lo = np.zeros(N, np.float32)
    L.check(lib.as_sched_alg1(N, L.ptr(uu, C.c_int32), L.ptr(bb, C.c_int32), beta, b_min, b_max, float(lr0),
                              L.ptr(bo, C.c_int32), L.ptr(lo, C.c_float)))
    return bo.tolist(), [float(x) for x in lo]



def scale_period(b_prev, b_next, dir_state, period, p_max):
    """as_sched_scale_period (R27): returns (next interval in
    mega-batches, updated direction state)."""
    lib = L.load()
    N = len(b_prev)
    bp, bn = L.as_np(b_prev, np.int32), L.as_np(b_next, np.int32)
    ds = np.array(dir_state, np.int32)
    po = C.c_int32()
    L.check(lib.as_sched_scale_period(N, L.ptr(bp, C.c_int32), L.ptr(bn, C.c_int32), L.ptr(ds, C.c_int32),
                                      int(period), int(p_max), C.byref(po)))
    return po.value, ds.tolist()


def alg2(u, b, norms, delta, pert_thr, norm="u", ties="lex"):
    """norm: "u" (Alg. 2 line 5 as printed) or "ub" (the P:175 alternative);
    ties: "lex" (reading R14: lexicographic (u, b), skip when all equal) or
    "literal" (line 8 as printed: argmax / argmin of u, lowest id, no skip)."""
    lib = L.load()
    N = len(u)
    uu, bb, nn = L.as_np(u, np.int32), L.as_np(b, np.int32), L.as_np(norms, np.float64)
    a = np.zeros(N, np.float64)
    p = C.c_int32()
    L.check(lib.as_sched_alg2_ex(N, L.ptr(uu, C.c_int32), L.ptr(bb, C.c_int32), L.ptr(nn, C.c_double),
                                 float(delta), float(pert_thr),
                                 (L.AS_NORM_UB if norm == "ub" else L.AS_NORM_UPDATES)
                                 | (L.AS_NORM_R14_LITERAL if ties == "literal" else 0),
                                 L.ptr(a, C.c_double), C.byref(p)))
    return a.tolist(), p.value


def fit_cost(rows, nnz, ps):
    """as_sched_fit_cost: replay cost model (c0, c_row, c_nnz, 1, 1) of one
    replica from a live trace of (rows, nnz, picoseconds) per batch."""
    lib = L.load()
    r, z, t = L.as_np(rows, np.int32), L.as_np(nnz, np.int64), L.as_np(ps, np.int64)
    out = L.CostModel()
    L.check(lib.as_sched_fit_cost(len(r), L.ptr(r, C.c_int32), L.ptr(z, C.c_int64), L.ptr(t, C.c_int64),
                                  C.byref(out)))
    return (out.c0, out.c_row, out.c_nnz, out.num, out.den)


def permutation(n, seed):
    lib = L.load()
    out = np.zeros(n, np.int64)
    L.check(lib.as_sched_permutation(int(n), C.c_uint64(seed & ((1 << 64) - 1)), L.ptr(out, C.c_int64)))
    return out


class LiveCursor:
    """Cross-process batch cursor of one mega-batch (live dynamic scheduling)."""

    def __init__(self, name, create):
        self.lib = L.load()
        h = C.c_void_p()
        L.check(self.lib.as_live_open(name.encode(), 1 if create else 0, C.byref(h)))
        self.h, self.owner = h, create

    def claim(self, M, b):
        s = C.c_int64(); r = C.c_int32()
        L.check(self.lib.as_live_claim(self.h, int(M), int(b), C.byref(s), C.byref(r)))
        return s.value, r.value

    def reset(self):
        L.check(self.lib.as_live_reset(self.h))

    def close(self):
        if self.h:
            self.lib.as_live_close(self.h, 1 if self.owner else 0)
            self.h = None
