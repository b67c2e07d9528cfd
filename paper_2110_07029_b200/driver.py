"""The Adaptive SGD mega-batch loop on top of the C-ABI.

Per mega-batch: route batches (replay: identical pure function on every rank),
run the SGD steps of this rank's batches on the device, merge (Alg. 2), then
rescale batch sizes (Alg. 1).  Replicas restart from the global model inside
the merge.
"""
from __future__ import annotations

import numpy as np

from . import sched


def stream_nnz_prefix(row_ptr, n, pos, M, order=None):
    """Cumulative nnz of stream positions [pos, pos+M) (input to replay routing)."""
    p = (np.arange(M, dtype=np.int64) + int(pos)) % int(n)
    ids = p if order is None else np.asarray(order, np.int64)[p]
    rl = row_ptr[ids + 1] - row_ptr[ids]
    out = np.zeros(M + 1, np.int64)
    np.cumsum(rl, out=out[1:])
    return out


class ReplayState:
    """Host scheduler state shared (identically) by every rank."""

    def __init__(self, world, b_max, b_min, beta, lr0, costs, algo="adaptive", scale_pmax=1):
        """algo: "adaptive" (P:105 dynamic routing + Alg. 1) or a comparison
        method of P:215 ("elastic", "sync": static equal batches, no scaling;
        the replicas' as_config.algo must match).  scale_pmax: adaptive
        scaling frequency (R27) -- Alg. 1 runs every `period`
        mega-batches, period in [1, scale_pmax] set by as_sched_scale_period;
        1 = the paper's default (every mega-batch)."""
        self.world, self.b_max, self.b_min, self.beta, self.lr0 = world, b_max, b_min, beta, lr0
        self.algo = algo
        self.costs = [tuple(int(v) for v in (c.c0, c.c_row, c.c_nnz, c.num, c.den)) if hasattr(c, "c0")
                      else tuple(c) for c in costs]
        self.b = [b_max] * world
        self.lr = [float(np.float32(lr0))] * world
        self.scale_pmax, self.period, self.since, self.dirs = int(scale_pmax), 1, 0, [0] * world

    def route(self, row_ptr, n, pos, M, order=None):
        pre = stream_nnz_prefix(row_ptr, n, pos, M, order)
        return sched.route_replay(self.costs, self.b, M, pre, static=self.algo != "adaptive")

    def rescale(self, u):
        b_used = list(self.b)
        self.since += 1
        if self.algo == "adaptive" and self.since >= self.period:
            self.b, self.lr = sched.alg1(u, self.b, self.beta, self.b_min, self.b_max, self.lr0)
            self.period, self.dirs = sched.scale_period(b_used, self.b, self.dirs, self.period, self.scale_pmax)
            self.since = 0
        return b_used


def run_local(replicas, ds, state, total, order=None, resident=True, want_loss=False):
    """All replicas in this process (local-group merge).  Returns per-mega-batch
    records (log, u, b, alpha, perturbed, losses)."""
    from .api import group_merge
    n = len(ds.row_ptr) - 1
    M = replicas[0].cfg.megabatch
    pos, recs = 0, []
    if resident:
        for r in replicas:
            if r.dataset_buf is None:
                r.upload_dataset(ds, order)
    while pos < total:
        Mm = int(min(M, total - pos))
        log, u, clocks = state.route(ds.row_ptr, n, pos, Mm, order)
        losses = []
        for (i, start, rows) in log:
            rep = replicas[i]
            if resident:
                rep.load_batch_stream(pos + start, rows)
            else:
                p = (np.arange(rows) + pos + start) % n
                ids = p if order is None else np.asarray(order)[p]
                sub = ds.rows(ids)
                rep.load_batch_csr(rows, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
            losses.append(rep.train_step(want_loss))
        b_used = list(state.b)
        alpha, pert = group_merge(replicas, u, b_used)
        state.rescale(u)
        for rep in replicas:
            rep.set_batch_sizes(state.b, state.lr)
        recs.append({"log": log, "u": u, "clocks": clocks, "b": b_used, "alpha": list(alpha),
                     "perturbed": pert, "b_next": list(state.b), "lr_next": list(state.lr),
                     "losses": losses})
        pos += Mm
    return recs


def run_rank(rep, ds_row_ptr, n, state, total, order=None, want_alpha=False):
    """One rank of a torchrun job (NCCL merge).  The dataset must be resident."""
    M = rep.cfg.megabatch
    pos, recs = 0, []
    while pos < total:
        Mm = int(min(M, total - pos))
        log, u, _ = state.route(ds_row_ptr, n, pos, Mm, order)
        for (i, start, rows) in log:
            if i == rep.rank:
                rep.load_batch_stream(pos + start, rows)
                rep.train_step(False)
        b_used = list(state.b)
        alpha, pert = rep.merge(u, b_used, want_alpha=want_alpha)
        state.rescale(u)
        rep.set_batch_sizes(state.b, state.lr)
        recs.append({"u": u, "b": b_used, "alpha": alpha, "perturbed": pert, "samples": Mm})
        pos += Mm
    return recs


def broadcast_nccl_id(dist, rank, device=None, make_id=None):
    """Rank 0 draws the 128-byte ncclUniqueId and every rank receives it over
    the torch.distributed process group (plumbing only)."""
    import torch
    if make_id is None:
        from .api import nccl_unique_id as make_id
    buf = torch.zeros(128, dtype=torch.uint8, device=device or "cpu")
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(make_id()), dtype=torch.uint8))
    dist.broadcast(buf, src=0)
    return bytes(buf.cpu().numpy().tobytes())


def open_p2p(rep, dist):
    """AS_MERGE_P2P setup: all-gather every rank's export record over the
    torch.distributed group (plumbing) and map the peers' workspaces."""
    import torch
    mine = torch.frombuffer(bytearray(rep.p2p_export()), dtype=torch.uint8)
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    parts = [torch.zeros_like(mine, device=dev) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, mine.to(dev))
    rep.p2p_open([bytes(p.cpu().numpy().tobytes()) for p in parts])


# ---------------------------------------------------------------------------
# Live event-timed routing ("batches are dispatched one-by-one based on
# GPU availability. Whenever a GPU finishes an epoch, it is assigned the next
# batch"; P:193-195 the scheduler counts u_i at dispatch).  One process per
# replica: a rank claims its next min(b_i, M - claimed) samples from the shared
# cursor (as_live_claim) as soon as its previous batch has COMPLETED on its
# device; the first dispatch of a mega-batch goes in id order (R8).  Every
# batch's device time is recorded, giving the trace (replica, rows, nnz, ps)
# from which the replay cost models are fitted (R9, as_sched_fit_cost).
# ---------------------------------------------------------------------------
def run_live(rank, world, dist, cursor, row_ptr, n, state, M, total, train_fn, merge_fn=None, order=None):
    """train_fn(gpos, rows) -> picoseconds the batch took (it returns after the
    batch completed).  merge_fn(u, b_used) runs the merge (steps a9-a13).
    Returns per-mega-batch records: log [(replica, start, rows)] in dispatch
    (cursor) order, u, b, and trace [(replica, start, rows, nnz, ps)]."""
    pos, recs = 0, []
    while pos < total:
        Mm = int(min(M, total - pos))
        pre = stream_nnz_prefix(row_ptr, n, pos, Mm, order)
        if rank == 0:
            cursor.reset()
        dist.barrier()
        b_me = int(state.b[rank])
        mine = []
        claim = None
        for k in range(world):                 # first dispatch in id order (R8)
            if k == rank:
                claim = cursor.claim(Mm, b_me)
            dist.barrier()
        start, rows = claim
        while rows > 0:
            ps = int(train_fn(pos + start, rows))
            mine.append((rank, int(start), int(rows), int(pre[start + rows] - pre[start]), ps))
            start, rows = cursor.claim(Mm, b_me)
        every = [None] * world
        dist.all_gather_object(every, mine)
        trace = sorted([t for part in every for t in part], key=lambda t: t[1])
        log = [(t[0], t[1], t[2]) for t in trace]
        u = [sum(1 for t in trace if t[0] == i) for i in range(world)]
        assert sum(t[2] for t in trace) == Mm          # samples conserved (R8)
        b_used = list(state.b)
        if merge_fn is not None:
            merge_fn(u, b_used)
        state.rescale(u)
        recs.append({"log": log, "u": u, "b": b_used, "trace": trace, "samples": Mm, "pos": pos})
        pos += Mm
    return recs


def fit_live_costs(recs, world):
    """Replay cost model of every replica fitted to the live trace (R9)."""
    out = []
    for i in range(world):
        tr = [t for r in recs for t in r["trace"] if t[0] == i]
        out.append(sched.fit_cost([t[2] for t in tr], [t[3] for t in tr], [t[4] for t in tr]))
    return out


def replay_live(recs, costs, row_ptr, n, order=None):
    """Replay every recorded mega-batch with the given cost models and the
    batch sizes that were in force: the logs the replay scheduler produces."""
    out = []
    for r in recs:
        pre = stream_nnz_prefix(row_ptr, n, r["pos"], r["samples"], order)
        log, u, _ = sched.route_replay(costs, r["b"], r["samples"], pre)
        out.append(log)
    return out


def gpu_train_fn(rep, stream=None):
    """train_fn for run_live on a replica: load the stream batch, run the SGD
    step and time it with CUDA events on the replica stream (returns ps)."""
    import torch
    s = stream or rep.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def fn(gpos, rows):
        e0.record(s)
        rep.load_batch_stream(gpos, rows)
        rep.train_step(False)
        e1.record(s)
        e1.synchronize()
        return int(round(e0.elapsed_time(e1) * 1e9))
    return fn
