"""World-size-2 host logic over torch.distributed gloo on CPU (the N > 1 path
without a GPU): identical replay routing on every rank (no collective
needed), a conserving live cursor shared by two processes, and the
ncclUniqueId broadcast plumbing."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

import synthgen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2110_07029_b200 import driver, sched
        ds = synthgen.tiny_dataset(n=500, d=50, C=30, seed=11)
        costs = synthgen.make_cost_models(world, hetero=True)
        st = driver.ReplayState(world, 16, 2, 1, 0.1, costs)
        logs, mine = [], []
        pos = 0
        for mb in range(4):
            log, u, clk = st.route(ds.row_ptr, ds.n, pos, 160)
            logs.append((log, u, clk, list(st.b)))
            mine.extend([(pos + s, r) for (i, s, r) in log if i == rank])
            st.rescale(u)
            pos += 160
        allx = [None] * world
        dist.all_gather_object(allx, (logs, mine))
        # live cursor shared by both processes
        name = "/adasgd_mp_%d" % port
        if rank == 0:
            cur = sched.LiveCursor(name, create=True)
        dist.barrier()
        if rank != 0:
            cur = sched.LiveCursor(name, create=False)
        dist.barrier()
        claims = []
        while True:
            s, r = cur.claim(997, 13 + 7 * rank)
            if r == 0:
                break
            claims.append((s, r))
        allc = [None] * world
        dist.all_gather_object(allc, claims)
        dist.barrier()
        cur.close()
        nid = driver.broadcast_nccl_id(dist, rank, make_id=lambda: bytes(range(128)))
        if rank == 0:
            q.put((allx, allc, nid))
    finally:
        dist.destroy_process_group()


def test_two_ranks_route_identically_and_share_cursor():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    allx, allc, nid = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (logs0, mine0), (logs1, mine1) = allx
    assert logs0 == logs1                          # replay routing identical on every rank
    covered = sorted(mine0 + mine1)
    flat = [x for s, r in covered for x in range(s, s + r)]
    assert flat == list(range(4 * 160))            # each sample processed exactly once
    flat = sorted(x for c in allc for s, r in c for x in range(s, s + r))
    assert flat == list(range(997))                # live cursor conserves samples across processes
    assert nid == bytes(range(128))


def _merge_worker(rank, world, port, q):
    """as_merge's host protocol (a9-a13) with the collectives over gloo: local
    norm, all-gather of the norms, Alg. 2 on every rank via the C++ scheduler
    (must agree bit-exactly), all-reduce of alpha_i w_i, momentum."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        from oracle import merge as omerge
        from paper_2110_07029_b200 import sched
        P = 4099
        reps = [np.random.default_rng(100 + i).normal(0, 0.01, P).astype(np.float32) for i in range(world)]
        wbar = np.random.default_rng(7).normal(0, 0.01, P).astype(np.float32)
        wbar_p = np.random.default_rng(8).normal(0, 0.01, P).astype(np.float32)
        u, b = [5, 3, 4][:world], [64, 60, 48][:world]
        out = {}
        for norm_mode in ("u", "ub"):
            n_me = torch.tensor([omerge.replica_norm(reps[rank])], dtype=torch.float64)
            norms = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(norms, n_me)
            norms = [float(t.item()) for t in norms]
            alpha, pert = sched.alg2(u, b, norms, 0.1, 0.1, norm=norm_mode)
            acc = torch.tensor(alpha[rank] * reps[rank].astype(np.float64))
            dist.all_reduce(acc)
            merged = (acc.numpy() + 0.9 * (wbar.astype(np.float64) - wbar_p.astype(np.float64))).astype(np.float32)
            out[norm_mode] = (alpha, pert, merged)
        allo = [None] * world
        dist.all_gather_object(allo, out)
        if rank == 0:
            q.put((allo, reps, wbar, wbar_p, u, b))
    finally:
        dist.destroy_process_group()


def test_two_ranks_merge_protocol_matches_oracle():
    from oracle import merge as omerge
    from oracle import sched as osched
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_merge_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    allo, reps, wbar, wbar_p, u, b = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for mode in ("u", "ub"):
        (a0, p0, m0), (a1, p1, m1) = allo[0][mode], allo[1][mode]
        assert a0 == a1 and p0 == p1                     # Alg. 2 identical on every rank (R13-R16)
        assert np.array_equal(m0, m1)
        oa, op = osched.alg2(u, b, [omerge.replica_norm(w) for w in reps], 0.1, 0.1, norm=mode)
        assert a0 == oa and p0 == op
        ow, _ = omerge.merge(reps, oa, wbar, wbar_p, 0.9)
        np.testing.assert_allclose(m0, ow, rtol=0, atol=1e-7)


# true per-replica speeds of the simulated "devices" (R9 integer model, ps):
# replica 0: 2 ms + 2 ms per row; replica 1 the same x 7/4 (a 75% slower GPU)
LIVE_COSTS = [(2_000_000_000, 2_000_000_000, 0, 1, 1), (2_000_000_000, 2_000_000_000, 0, 7, 4)]


def _live_worker(rank, world, port, q):
    """Live event-timed routing over the shared cursor: each
    rank claims its next batch when its previous one has completed; the batch
    'runs' by sleeping its true cost; per-batch durations are recorded."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import time
        from paper_2110_07029_b200 import driver, sched
        ds = synthgen.tiny_dataset(n=200, d=50, C=30, seed=12)
        name = "/adasgd_live_%d" % port
        if rank == 0:
            cur = sched.LiveCursor(name, create=True)
        dist.barrier()
        if rank != 0:
            cur = sched.LiveCursor(name, create=False)
        st = driver.ReplayState(world, 8, 2, 2, 0.1, LIVE_COSTS)
        c0, cr, cz, num, den = LIVE_COSTS[rank]
        row_ptr = ds.row_ptr

        def train_fn(gpos, rows):
            ids = (np.arange(rows) + gpos) % ds.n
            nnz = int(np.sum(row_ptr[ids + 1] - row_ptr[ids]))
            t0 = time.perf_counter_ns()
            time.sleep(((c0 + cr * rows + cz * nnz) * num // den) * 1e-12)
            return (time.perf_counter_ns() - t0) * 1000        # ns -> ps
        recs = driver.run_live(rank, world, dist, cur, row_ptr, ds.n, st, 60, 120, train_fn)
        dist.barrier()
        cur.close()
        if rank == 0:
            q.put(recs)
    finally:
        dist.destroy_process_group()


def test_live_routing_trace_fit_replays_bit_exactly():
    """Live dispatch on completion with a shared cursor across two processes,
    the per-batch trace fitted to replay cost models (as_sched_fit_cost), and
    the replay scheduler (as_sched_route_replay) on the fitted models
    reproducing the live dispatch log of every mega-batch exactly (the
    simulated speeds keep every dispatch decision >= 2 ms from a tie)."""
    from paper_2110_07029_b200 import driver
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_live_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    recs = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ds = synthgen.tiny_dataset(n=200, d=50, C=30, seed=12)
    assert len(recs) == 2
    for r in recs:
        cover = sorted(x for (_, s, rows) in r["log"] for x in range(s, s + rows))
        assert cover == list(range(60))                     # every sample of the mega-batch once
        assert r["u"][1] < r["u"][0]                        # the slower replica takes fewer batches
    fitted = driver.fit_live_costs(recs, 2)
    for i, f in enumerate(fitted):                          # fitted speeds close to the true ones
        c0, cr, _, num, den = LIVE_COSTS[i]
        true8 = (c0 + 8 * cr) * num // den
        fit8 = f[0] + 8 * f[1]
        assert abs(fit8 - true8) <= 0.1 * true8, (i, f)
    replayed = driver.replay_live(recs, fitted, ds.row_ptr, ds.n)
    for r, log in zip(recs, replayed):
        assert [tuple(x) for x in log] == [tuple(x) for x in r["log"]]
