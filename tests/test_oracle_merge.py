"""Pins for oracle/merge.py and oracle/train.py (CPU only).

* norm of a constant vector: |c| / sqrt(P)
* equal speeds -> plain model averaging (north star)
* one batch per replica per mega-batch, gamma = 0 -> exactly one synchronous
  SGD step on the union batch ("gradient and model averaging are
  equivalent in this case", "a mega-batch of 4 batches on 4 GPUs
  corresponds to gradient aggregation")
* N = 1, gamma = 0 -> plain mini-batch SGD ("When the testing
  configuration has a single GPU, all the methods become mini-batch SGD")
* N = 1, one batch per mega-batch, gamma > 0 -> torch.optim.SGD with momentum
  (heavy-ball form; library routine)
"""
import numpy as np
import torch

import synthgen
from oracle import csr as ocsr
from oracle import merge as omerge
from oracle import model as om
from oracle import sched as osched
from oracle import train as otrain

D, C, H = 40, 24, 8


def _setup(n=64, seed=3):
    ds = synthgen.tiny_dataset(n=n, d=D, C=C, seed=seed)
    p = synthgen.make_init_params(D, C, H, seed)
    return ds, p


def _cfg(**kw):
    base = dict(d=D, C=C, h=H, b_max=16, b_min=2, beta=1, M=32, lr0=0.5, gamma=0.0,
                delta=0.1, pert_thr=0.1, world=2)
    base.update(kw)
    return otrain.RunConfig(**base)


def test_norm_constant_vector():
    for c, P in [(0.25, 1000), (-3.0, 7), (1e-3, 12345)]:
        w = np.full(P, c, np.float32)
        assert abs(omerge.replica_norm(w) - abs(np.float32(c)) / np.sqrt(P)) <= 1e-15 * abs(c)


def test_equal_speeds_is_plain_averaging():
    ds, p = _setup()
    cfg = _cfg(world=2, b_max=8, M=32)
    costs = [synthgen.CostModel(0, 10, 0)] * 2          # row-only equal costs: round robin
    recs, wbar = otrain.run(ds, p, cfg, costs, 32, log_steps=True)
    r = recs[0]
    assert r["u"] == [2, 2] and r["alpha"] == [0.5, 0.5] and r["perturbed"] == 0
    mean = (0.5 * r["replicas"][0].astype(np.float64) + 0.5 * r["replicas"][1]).astype(np.float32)
    assert np.array_equal(wbar, mean)


def test_one_batch_per_replica_equals_sync_sgd_on_union():
    ds, p = _setup()
    # b = (4, 6), M = 10: replica 0 takes samples 0..3, replica 1 takes 4..9
    cfg = _cfg(world=2, b_max=8, b_min=1, M=10, gamma=0.0, pert_thr=0.0)
    costs = [synthgen.CostModel(0, 10, 0)] * 2
    # force unequal batch sizes through a run with b set by hand
    N = 2
    b = [4, 6]
    lr = 0.5
    log, u, _ = osched.route_replay(costs, b, 10, lambda s, r: 0)
    assert log == [(0, 0, 4), (1, 4, 6)]
    reps = []
    for (i, s, rows) in log:
        bt = otrain.batch_of(ds, ocsr.stream_ids(s, rows, ds.n))
        new, _, _ = om.sgd_step(bt, otrain.unpack(p, D, C, H), lr)
        reps.append(otrain.pack(new))
    alpha, pert = osched.alg2(u, b, [1.0] * N, 0.1, 0.1)
    merged, _ = omerge.merge(reps, alpha, p, p, 0.0)
    union = otrain.batch_of(ds, ocsr.stream_ids(0, 10, ds.n))
    ref, _, _ = om.sgd_step(union, otrain.unpack(p, D, C, H), lr)
    np.testing.assert_allclose(merged, otrain.pack(ref), rtol=0, atol=1e-6)


def test_single_replica_is_minibatch_sgd():
    ds, p = _setup(n=48)
    cfg = _cfg(world=1, b_max=8, b_min=1, M=24, gamma=0.0)
    costs = [synthgen.CostModel(1, 1, 1)]
    recs, wbar = otrain.run(ds, p, cfg, costs, 48)
    w = p.copy()
    for s in range(0, 48, 8):
        bt = otrain.batch_of(ds, ocsr.stream_ids(s, 8, ds.n))
        new, _, _ = om.sgd_step(bt, otrain.unpack(w, D, C, H), 0.5)
        w = otrain.pack(new)
    assert all(r["alpha"] == [1.0] and r["perturbed"] == 0 for r in recs)
    assert np.array_equal(wbar, w)


def test_momentum_matches_torch_sgd_heavy_ball():
    ds, p = _setup(n=48)
    gamma, lr, bsz = 0.9, 0.3, 8
    cfg = _cfg(world=1, b_max=bsz, b_min=1, M=bsz, gamma=gamma, lr0=lr)
    recs, wbar = otrain.run(ds, p, cfg, [synthgen.CostModel(1, 1, 1)], 48)
    prm = otrain.unpack(p.astype(np.float64), D, C, H)
    ts = {k: torch.tensor(np.array(v), requires_grad=True) for k, v in prm.items()}
    opt = torch.optim.SGD(list(ts.values()), lr=float(np.float32(lr)), momentum=gamma)
    for s in range(0, 48, bsz):
        ids = ocsr.stream_ids(s, bsz, ds.n)
        sub = ds.rows(ids)
        X = torch.zeros(bsz, D, dtype=torch.float64)
        T = torch.zeros(bsz, C, dtype=torch.float64)
        for r in range(bsz):
            a, e = sub.row_ptr[r], sub.row_ptr[r + 1]
            X[r, torch.tensor(sub.col[a:e], dtype=torch.long)] = torch.tensor(sub.val[a:e], dtype=torch.float64)
            a, e = sub.lab_ptr[r], sub.lab_ptr[r + 1]
            T[r, torch.tensor(sub.lab[a:e], dtype=torch.long)] = 1.0 / (e - a)
        opt.zero_grad()
        Z = torch.relu(X @ ts["W1"] + ts["b1"]) @ ts["W2T"].T + ts["b2"]
        torch.nn.functional.cross_entropy(Z, T).backward()
        opt.step()
    ref = np.concatenate([ts[k].detach().numpy().ravel() for k in ("W1", "b1", "W2T", "b2")])
    np.testing.assert_allclose(wbar, ref, rtol=0, atol=2e-6)


def test_samples_conserved_over_run():
    ds, p = _setup(n=100)
    cfg = _cfg(world=3, b_max=8, b_min=1, beta=1, M=30)
    costs = synthgen.make_cost_models(3, hetero=True)
    recs, _ = otrain.run(ds, p, cfg, costs, 100)
    assert sum(sum(r for _, _, r in rec["log"]) for rec in recs) == 100
    assert [sum(r for _, _, r in rec["log"]) for rec in recs] == [30, 30, 30, 10]


# ------------------------------------------------ comparison methods (NEXT f2)
def test_sync_mode_is_sgd_on_union_batch_under_heterogeneous_speeds():
    """algo="sync" (gradient aggregation, Fig. 2): M = N b, so every
    merge follows exactly one batch per replica regardless of the replay
    speeds; with gamma = 0 every merge equals ONE mini-batch SGD step on the
    union batch ("gradient and model averaging are equivalent in this
    case").  A 32% slowdown does not change the result (static routing)."""
    ds, p = _setup(n=72)
    N, b, lr = 3, 8, 0.4
    cfg = _cfg(world=N, b_max=b, b_min=1, M=N * b, gamma=0.0, lr0=lr, algo="sync", pert_thr=1e9)
    costs = [synthgen.CostModel(5, 10, 1, 1, 1), synthgen.CostModel(5, 10, 1, 132, 100),
             synthgen.CostModel(5, 10, 1, 116, 100)]
    recs, wbar = otrain.run(ds, p, cfg, costs, 72)
    w = p.copy()
    for s in range(0, 72, N * b):
        union = otrain.batch_of(ds, ocsr.stream_ids(s, N * b, ds.n))
        new, _, _ = om.sgd_step(union, otrain.unpack(w, D, C, H), lr)
        w = otrain.pack(new)
    for r in recs:
        assert r["u"] == [1] * N and r["alpha"] == [1.0 / N] * N and not r["perturbed"]
        assert r["b_next"] == [b] * N
    np.testing.assert_allclose(wbar, w, rtol=0, atol=2e-6)


def test_elastic_equals_adaptive_at_equal_speeds():
    """With equal row-only costs dynamic routing is round-robin, Alg. 1 leaves
    b unchanged, Alg. 2 gives 1/N with no perturbation (R14): the paper's method
    reduces to elastic model averaging; the whole runs are identical."""
    ds, p = _setup(n=64)
    kw = dict(world=2, b_max=8, b_min=1, M=32, gamma=0.9, lr0=0.5)
    costs = [synthgen.CostModel(0, 10, 0, 1, 1)] * 2
    ra, wa = otrain.run(ds, p, _cfg(algo="adaptive", **kw), costs, 64)
    re, we = otrain.run(ds, p, _cfg(algo="elastic", **kw), costs, 64)
    for a, e in zip(ra, re):
        assert a["log"] == e["log"] and a["u"] == e["u"] and a["alpha"] == e["alpha"]
    assert np.array_equal(wa, we)


def test_elastic_static_split_ignores_speed():
    """Under a 32% slowdown the elastic split keeps equal batch counts (the
    straggler problem) while adaptive routing gives the fast GPU more."""
    ds, p = _setup(n=64)
    kw = dict(world=2, b_max=4, b_min=1, beta=1, M=64, gamma=0.0, lr0=0.5)
    costs = [synthgen.CostModel(0, 10, 0, 1, 1), synthgen.CostModel(0, 10, 0, 132, 100)]
    re, _ = otrain.run(ds, p, _cfg(algo="elastic", **kw), costs, 64)
    ra, _ = otrain.run(ds, p, _cfg(algo="adaptive", **kw), costs, 64)
    assert re[0]["u"] == [8, 8] and max(re[0]["clocks"]) == 8 * (40 * 132 // 100)
    assert ra[0]["u"][0] > ra[0]["u"][1] and max(ra[0]["clocks"]) < max(re[0]["clocks"])


def test_norm_metrics_closed_form():
    """R15's switchable regularisation metrics on a constant vector c (P entries):
    ||w|| = |c| sqrt(P): l2/P = |c|/sqrt(P), l2^2/P = c^2, l2/sqrt(P) = |c|, l2 = |c| sqrt(P)."""
    P, c = 10_000, -0.3
    w = np.full(P, c, np.float32)
    cc = float(np.float32(c))
    assert abs(omerge.replica_norm(w, "l2/P") - abs(cc) / np.sqrt(P)) < 1e-15
    assert abs(omerge.replica_norm(w, "l2^2/P") - cc * cc) < 1e-12
    assert abs(omerge.replica_norm(w, "l2/sqrt(P)") - abs(cc)) < 1e-12
    assert abs(omerge.replica_norm(w, "l2") - abs(cc) * np.sqrt(P)) < 1e-9
