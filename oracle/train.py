"""Oracle: the whole Adaptive SGD run, step by step in the paper's order.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Per mega-batch (section 3.1, section 4, reading R18):
  1. every replica restarts from the global model  w_i <- wbar
  2. batches are routed to the earliest-free replica (replay, oracle.sched)
     and each replica runs SGD steps with its own b_i, lr_i
  3. Alg. 2: norms, weights, merge + momentum
  4. Alg. 1: batch sizes and learning rates for the next one
"""
from __future__ import annotations

import dataclasses
import numpy as np

from . import csr as ocsr
from . import merge as omerge
from . import model as omodel
from . import sched as osched


@dataclasses.dataclass
class RunConfig:
    d: int
    C: int
    h: int
    b_max: int
    b_min: int
    beta: int
    M: int                 # mega-batch size in samples
    lr0: float
    gamma: float = 0.9
    delta: float = 0.1
    pert_thr: float = 0.1
    world: int = 2
    # "adaptive" (the paper's method) or the comparison methods of P:215:
    # "elastic" (elastic model averaging, Fig. 3) and "sync" (gradient
    # aggregation, Fig. 2; callers set M = N * b_max): static equal
    # batches, alpha_i = 1/N, no perturbation, no batch scaling
    algo: str = "adaptive"
    # adaptive scaling frequency (R27): the interval between Alg. 1
    # runs doubles up to scale_pmax mega-batches; 1 = every mega-batch
    scale_pmax: int = 1


def unpack(p, d, C, h):
    o = 0
    W1 = p[o:o + d * h].reshape(d, h); o += d * h
    b1 = p[o:o + h]; o += h
    W2T = p[o:o + C * h].reshape(C, h); o += C * h
    b2 = p[o:o + C]
    return {"W1": W1, "b1": b1, "W2T": W2T, "b2": b2}


def pack(params):
    return np.concatenate([np.asarray(params[k], np.float32).ravel()
                           for k in ("W1", "b1", "W2T", "b2")])


def batch_of(dataset, ids):
    rp, col, val, lp, lab = ocsr.batch_csr(dataset, ids)

    class _B:
        pass
    bt = _B()
    bt.row_ptr, bt.col, bt.val, bt.lab_ptr, bt.lab = rp, col, val, lp, lab
    return bt


def run(dataset, init, cfg: RunConfig, costs, total_samples, order=None, log_steps=False, logs=None):
    """Adaptive SGD over ``total_samples`` stream samples.  Returns a list of
    per-mega-batch records (routing log, u, b, lr, norms, alpha, perturbed,
    wbar) and the final global model.

    logs (optional): the dispatch log [(replica, start, rows)] of every
    mega-batch as a LIVE run observed it ("dispatched one-by-one based
    on GPU availability"); the oracle then follows it instead of replaying the
    cost models, and u_i counts the batches dispatched to replica i."""
    N = cfg.world
    wbar = np.asarray(init, np.float32).copy()
    wbar_p = wbar.copy()                                   # reading R17
    b = [cfg.b_max] * N                                    # P:228 initial b = b_max
    lr = [float(np.float32(cfg.lr0))] * N
    pos = 0
    records = []
    period, since, dirs = 1, 0, [0] * N                   # reading R27
    rp = dataset.row_ptr
    while pos < total_samples:
        Mm = min(cfg.M, total_samples - pos)
        replicas = [wbar.copy() for _ in range(N)]

        def nnz_of(start, rows, _pos=pos):
            ids = ocsr.stream_ids(_pos + start, rows, dataset.n, order)
            return int(np.sum(rp[ids + 1] - rp[ids]))

        if logs is not None:
            log = [tuple(x) for x in logs[len(records)]]
            u, clocks = [sum(1 for x in log if x[0] == i) for i in range(N)], None
            assert sorted(x for (_, s0, r0) in log for x in range(s0, s0 + r0)) == list(range(Mm))
        elif cfg.algo == "adaptive":
            log, u, clocks = osched.route_replay(costs, b, Mm, nnz_of)
        else:
            log, u, clocks = osched.route_static(costs, b, Mm, nnz_of)
        losses = []
        for (i, start, rows) in log:
            bt = batch_of(dataset, ocsr.stream_ids(pos + start, rows, dataset.n, order))
            new, loss, _ = omodel.sgd_step(bt, unpack(replicas[i], cfg.d, cfg.C, cfg.h), lr[i])
            replicas[i] = pack(new)
            losses.append(loss)
        if cfg.algo == "adaptive":
            norms = [omerge.replica_norm(w) for w in replicas]
            alpha, pert = osched.alg2(u, b, norms, cfg.delta, cfg.pert_thr)
        else:                                              # plain model average
            norms, alpha, pert = None, [1.0 / N] * N, False
        b_used, lr_used = list(b), list(lr)
        wbar, wbar_p = omerge.merge(replicas, alpha, wbar, wbar_p, cfg.gamma)
        since += 1
        if cfg.algo == "adaptive" and since >= period:
            b, lr = osched.alg1(u, b, cfg.beta, cfg.b_min, cfg.b_max, cfg.lr0)
            period, dirs = osched.scale_period(b_used, b, dirs, period, cfg.scale_pmax)
            since = 0
        records.append({"log": log, "u": u, "clocks": clocks, "b": b_used, "lr": lr_used,
                        "norms": norms, "alpha": alpha, "perturbed": pert,
                        "b_next": list(b), "lr_next": list(lr), "losses": losses,
                        "period": period,
                        "wbar": wbar.copy(), "replicas": replicas if log_steps else None})
        pos += Mm
    return records, wbar
