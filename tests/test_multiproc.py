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
