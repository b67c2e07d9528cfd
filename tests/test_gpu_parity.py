"""GPU parity of the CUDA path (through the C-ABI) against the oracle.

Tolerances (north star, reading R22: per tensor
||a-o||_2/||o||_2 <= tol AND max|a-o| <= tol * max|o|):
  bit-exact  batch transposes (integer/index work), replay routing, b_i
  1e-4       AS_FP32 mode: logits (LSE), loss, gradients after one step
  2e-2       AS_BF16 mode (tcgen05 tensor-core output layer)
  1e-5       merged weights
"""
import math
import os
import struct

import numpy as np
import pytest

import _parity_log as plog

import synthgen
from oracle import csr as ocsr
from oracle import merge as omerge
from oracle import model as om
from oracle import sched as osched
from oracle import train as otrain

pytestmark = pytest.mark.gpu

LN2 = math.log(2.0)


def rel_err(a, o):
    a = np.asarray(a, np.float64); o = np.asarray(o, np.float64)
    n = np.linalg.norm(o)
    e1 = np.linalg.norm(a - o) / max(n, 1e-300)
    e2 = np.max(np.abs(a - o)) / max(np.max(np.abs(o)), 1e-300) if o.size else 0.0
    return max(e1, e2)


def _test_name():
    return os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]


def assert_close(name, a, o, tol):
    e = rel_err(a, o)
    plog.record(_test_name(), name, e, tol, "rel (R22)")
    assert e <= tol, "%s: rel err %.3e > %.1e" % (name, e, tol)
    return e


def assert_abs(name, a, o, tol):
    """max |a - o| <= tol (absolute): used for LSE, whose error in natural-log
    units is the relative error of the partition function sum_c exp(z_rc)."""
    a = np.asarray(a, np.float64); o = np.asarray(o, np.float64)
    e = float(np.max(np.abs(a - o))) if o.size else 0.0
    plog.record(_test_name(), name, e, tol, "abs")
    assert e <= tol, "%s: max abs err %.3e > %.1e" % (name, e, tol)
    return e


def check_softmax_terms(name, rep, sub, ref, C, h, tol):
    """The softmax parts of the gradients on their own, where the label term
    cannot hide them: pass 1's O / l (dHsoft, AS_DBG_DHSOFT) and the dW2T
    rows / db2 entries of classes with no label in the batch (pure softmax)."""
    B = len(sub.row_ptr) - 1
    assert_close(name + " dHsoft", _f32(rep.debug_get(12, 4 * B * h)).reshape(B, h), ref["dHsoft"], tol)
    unl = np.setdiff1d(np.arange(C), sub.lab)
    if len(unl):
        dW2T = _f32(rep.debug_get(5, 4 * C * h)).reshape(C, h)
        assert_close(name + " dW2T unlabelled", dW2T[unl], ref["dW2T"][unl], tol)
        assert_close(name + " db2 unlabelled", _f32(rep.debug_get(6, 4 * C))[unl], ref["db2"][unl], tol)


def _cfg(d, C, h, n, b_max, avg_nnz=20.0, avg_labels=3.0, seed=0):
    return synthgen.XMLConfig("t", d, C, n, avg_nnz, avg_labels, h, b_max, 1, seed)


def _params(cfg, seed=3, bias=0.2):
    p = synthgen.make_init_params(cfg.d, cfg.C, cfg.h, seed)
    lay = synthgen.param_layout(cfg.d, cfg.C, cfg.h)
    rng = np.random.default_rng(seed)
    for k in ("b1", "b2"):
        o, shp = lay[k]
        p[o:o + shp[0]] = rng.normal(0, bias, shp[0]).astype(np.float32)
    return p


def _replica(cfg, p, ds, precision, lr=0.5, debug=True, b_min=None, rank=0, world=1):
    from paper_2110_07029_b200.api import Replica
    return Replica(cfg.d, cfg.C, cfg.h, cfg.b_max, p, b_min=b_min or max(1, cfg.b_max // 8),
                   max_row_nnz=int(np.diff(ds.row_ptr).max()), max_row_labels=int(np.diff(ds.lab_ptr).max()),
                   lr0=lr, precision=precision, debug_grads=debug, rank=rank, world=world)


def _f32(buf):
    return np.frombuffer(buf.tobytes(), np.float32)


def _i32(buf):
    return np.frombuffer(buf.tobytes(), np.int32)


def test_tc_selftest_descriptors(gpu_lib):
    import torch
    from paper_2110_07029_b200.api import tc_selftest
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(128, 128, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(128, 128, device="cuda", generator=g).to(torch.bfloat16)
    S, O, T = tc_selftest(A, B)
    Af, Bf = A.double(), B.double()
    assert rel_err(S.cpu().numpy(), (Af @ Bf.T).cpu().numpy()) < 1e-5
    P = (S / 16).to(torch.bfloat16).double()
    assert rel_err(O.cpu().numpy(), (P @ Bf).cpu().numpy()) < 1e-5
    assert rel_err(T.cpu().numpy(), (Af.T @ P.T).cpu().numpy()) < 1e-5


def test_tc_selftest_tmem_a_operand(gpu_lib):
    import torch
    from paper_2110_07029_b200.api import tc_selftest2
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(128, 128, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(128, 128, device="cuda", generator=g).to(torch.bfloat16)
    V, U = tc_selftest2(A, B)
    Af, Bf = A.double(), B.double()
    assert rel_err(V.cpu().numpy(), (Af @ Bf.T).cpu().numpy()) < 1e-5
    P = (A.float() * 0.25).to(torch.bfloat16).double()
    assert rel_err(U.cpu().numpy(), (P @ Bf).cpu().numpy()) < 1e-5


CASES = [
    # d, C, h, n, B (rows of the batch), b_max
    (2000, 1000, 128, 600, 200, 256),    # ragged: 2 row tiles (72 rows in the 2nd), C % 128 = 104
    (3000, 700, 256, 400, 130, 192),     # h = 256
    (500, 50, 128, 64, 1, 64),           # a single row, C < 128
    (2000, 900, 128, 300, 100, 128),     # one row tile (pass-2 WGs walk alternate class blocks), 8 blocks
    (1500, 2048, 128, 700, 512, 512),    # exact tiles
    (4000, 30000, 128, 1200, 1024, 1024),  # multi-block pipelines: 13 class blocks per pass-1 CTA
    (3000, 20000, 256, 800, 512, 512),   # h = 256, W ring wraps (2 stages)
]
# seeded random shapes (ragged batches, small and odd C, both hidden widths; h = 256
# with C <= 128 SMs takes the one-block pass 2)
_rng = np.random.default_rng(20260)
RANDOM_CASES = []
for _k in range(8):
    _bm = int(_rng.choice([64, 128, 256, 512]))
    _B = int(_rng.integers(1, _bm + 1))
    RANDOM_CASES.append((int(_rng.integers(300, 5000)), int(_rng.integers(60, 6000)), int(_rng.choice([128, 256])),
                         max(_B + 16, 200), _B, _bm))


def _one_step(case, precision):
    d, C, h, n, B, b_max = case
    cfg = _cfg(d, C, h, n, b_max, seed=hash(case) % 97)
    ds = synthgen.make_dataset(cfg, n=n)
    p = _params(cfg)
    rep = _replica(cfg, p, ds, precision, lr=0.5)
    ids = np.arange(B) + 7
    sub = ds.rows(ids)
    rep.load_batch_csr(B, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
    loss = rep.train_step(want_loss=True)
    prm = otrain.unpack(p, d, C, h)
    ref = om.gradients_chunked(sub, prm, chunk=64)
    return cfg, ds, sub, rep, loss, ref, p


@pytest.mark.parametrize("case", CASES)
def test_transposes_bit_exact(gpu_lib, case):
    cfg, ds, sub, rep, loss, ref, p = _one_step(case, "fp32")
    keys, sptr, srow, sval = ocsr.transpose(sub.row_ptr, sub.col, sub.val)
    buf = rep.debug_get(8, 64 << 20)
    w = _i32(buf)
    U = int(w[0])
    nnz = len(sub.col)
    assert U == len(keys)
    got_ids = w[1:1 + U]; o = 1 + U
    got_ptr = w[o:o + U + 1]; o += U + 1
    got_row = w[o:o + nnz]; o += nnz
    got_val = w[o:o + nnz]
    assert np.array_equal(got_ids, keys) and np.array_equal(got_ptr, sptr)
    assert np.array_equal(got_row, srow)
    assert np.array_equal(got_val, sval.view(np.int32))            # bit-exact values
    lkeys, lptr, lrow, _ = ocsr.transpose(sub.lab_ptr, sub.lab)
    w = _i32(rep.debug_get(9, 64 << 20))
    V = int(w[0])
    assert V == len(lkeys)
    assert np.array_equal(w[1:1 + V], lkeys) and np.array_equal(w[1 + V:2 + 2 * V], lptr)
    assert np.array_equal(w[2 + 2 * V:2 + 2 * V + len(sub.lab)], lrow)


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-4), ("bf16", 2e-2)])
@pytest.mark.parametrize("case", CASES + RANDOM_CASES)
def test_one_step_parity(gpu_lib, case, precision, tol):
    cfg, ds, sub, rep, loss, ref, p = _one_step(case, precision)
    d, C, h, n, B, b_max = case
    H = _f32(rep.debug_get(0, 4 * B * h)).reshape(B, h)
    assert_close("H", H, ref["H"], 1e-5)                       # SpMM is fp32 in both modes
    lse = _f32(rep.debug_get(1, 4 * B)) * LN2
    assert_close("LSE", lse, ref["LSE"], tol)
    assert_abs("LSE abs", lse, ref["LSE"], tol)
    assert abs(loss - ref["loss"]) <= tol * abs(ref["loss"])
    check_softmax_terms("step", rep, sub, ref, C, h, tol)
    dA = _f32(rep.debug_get(3, 4 * B * h)).reshape(B, h)
    assert_close("dA", dA, ref["dA"], tol)
    db1 = _f32(rep.debug_get(4, 4 * h))
    assert_close("db1", db1, ref["db1"], tol)
    dW2T = _f32(rep.debug_get(5, 4 * C * h)).reshape(C, h)
    assert_close("dW2T", dW2T, ref["dW2T"], tol)
    db2 = _f32(rep.debug_get(6, 4 * C))
    assert_close("db2", db2, ref["db2"], tol)
    keys = np.unique(sub.col)
    dW1 = _f32(rep.debug_get(7, 4 * len(keys) * h)).reshape(len(keys), h)
    assert_close("dW1", dW1, ref["dW1"][keys], tol)
    # the SGD update applied the gradients with lr (P:51 third pass)
    new = rep.get_params()
    dnew = otrain.unpack(new.astype(np.float64) - p.astype(np.float64), d, C, h)
    assert_close("W2T update", dnew["W2T"], -0.5 * ref["dW2T"], max(tol, 1e-3))
    assert_close("W1 update", dnew["W1"][keys], -0.5 * ref["dW1"][keys], max(tol, 1e-3))
    untouched = np.setdiff1d(np.arange(d), keys)
    assert np.all(dnew["W1"][untouched] == 0)                  # untouched rows bit-identical


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("h,B,avg_nnz,d", [(128, 64, 400.0, 3000), (256, 96, 250.0, 2000), (128, 1, 600.0, 5000),
                                            (128, 700, 3.0, 900)])
def test_sparse_long_segments(gpu_lib, h, B, avg_nnz, d, precision):
    """SpMM rows and dW1 feature segments far longer than one CTA's entry range
    (every segment crosses warp and CTA ranges: the ordered shared-memory and
    last-arriver combines), plus many very short rows; twice for
    bit-identical results (deterministic sum order).  bf16 at h = 128 runs a7
    inside pass 2's idle warps (one warp per feature segment)."""
    tol = 1e-4 if precision == "fp32" else 2e-2
    cfg = _cfg(d, 300, h, 4 * B + 8, max(B, 8), avg_nnz=avg_nnz, seed=5)
    ds = synthgen.make_dataset(cfg, n=cfg.n)
    p = _params(cfg)
    sub = ds.rows(np.arange(B) + 3)
    ref = om.gradients_chunked(sub, otrain.unpack(p, d, cfg.C, h), chunk=64)
    keys = np.unique(sub.col)
    outs = []
    for _ in range(2):
        rep = _replica(cfg, p, ds, precision, lr=0.5)
        rep.load_batch_csr(B, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
        rep.train_step(want_loss=True)
        H = _f32(rep.debug_get(0, 4 * B * h)).reshape(B, h)
        assert_close("H", H, ref["H"], 1e-5)
        dW1 = _f32(rep.debug_get(7, 4 * len(keys) * h)).reshape(len(keys), h)
        assert_close("dW1", dW1, ref["dW1"][keys], tol)
        new = rep.get_params()
        dnew = otrain.unpack(new.astype(np.float64) - p.astype(np.float64), d, cfg.C, h)
        assert_close("W1 update", dnew["W1"][keys], -0.5 * ref["dW1"][keys], max(tol, 1e-3))
        untouched = np.setdiff1d(np.arange(d), keys)
        assert np.all(dnew["W1"][untouched] == 0)
        outs.append((H.copy(), new.copy()))
        rep.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("h", [128, 256])
def test_bf16_online_softmax_rescale_paths(gpu_lib, h):
    """b2 ramps up over the classes and the rows differ in scale, so the lazy
    online-softmax rescale (pass 1) fires at different class blocks for
    different rows of the same warp."""
    d, C, n, B = 2500, 12000, 600, 384
    cfg = _cfg(d, C, h, n, 512, seed=21)
    ds = synthgen.make_dataset(cfg, n=n)
    p = _params(cfg)
    lay = synthgen.param_layout(d, C, h)
    o, _ = lay["b2"]
    p[o:o + C] = np.linspace(0.0, 40.0, C, dtype=np.float32)
    o, _ = lay["W2T"]
    p[o:o + C * h] *= np.float32(8.0)
    rep = _replica(cfg, p, ds, "bf16")
    sub = ds.rows(np.arange(B))
    sub.val[:] = sub.val * np.repeat(np.linspace(0.2, 3.0, B), np.diff(sub.row_ptr)).astype(np.float32)
    rep.load_batch_csr(B, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
    loss = rep.train_step(want_loss=True)
    ref = om.gradients_chunked(sub, otrain.unpack(p, d, C, h), chunk=64)
    assert abs(loss - ref["loss"]) <= 2e-2 * abs(ref["loss"])
    assert_close("LSE", _f32(rep.debug_get(1, 4 * B)) * LN2, ref["LSE"], 2e-2)
    assert_abs("LSE abs", _f32(rep.debug_get(1, 4 * B)) * LN2, ref["LSE"], 2e-2)
    check_softmax_terms("rescale", rep, sub, ref, C, h, 2e-2)
    assert_close("dA", _f32(rep.debug_get(3, 4 * B * h)).reshape(B, h), ref["dA"], 2e-2)
    assert_close("dW2T", _f32(rep.debug_get(5, 4 * C * h)).reshape(C, h), ref["dW2T"], 2e-2)


def test_invalid_batch_is_rejected_without_state_change(gpu_lib):
    from paper_2110_07029_b200._lib import ASError
    cfg = _cfg(800, 300, 128, 100, 64)
    ds = synthgen.make_dataset(cfg, n=100)
    p = _params(cfg)
    rep = _replica(cfg, p, ds, "bf16")
    sub = ds.rows(np.arange(10))
    bad_col = sub.col.copy(); bad_col[1], bad_col[0] = bad_col[0], bad_col[1]
    for args in [(0, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab),
                 (65, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab),
                 (10, sub.row_ptr, bad_col, sub.val, sub.lab_ptr, sub.lab),
                 (10, sub.row_ptr, sub.col, sub.val, np.zeros(11, np.int64), sub.lab)]:
        with pytest.raises(ASError) as e:
            rep.load_batch_csr(*args)
        assert e.value.code == -1
    with pytest.raises(ASError):
        rep.train_step()                                       # nothing loaded yet
    assert np.array_equal(rep.get_params(), p)
    rep.load_batch_csr(10, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
    assert np.isfinite(rep.train_step(want_loss=True))


def test_large_host_batch_threaded_staging(gpu_lib):
    """Host batches with more than 32K entries are validated and packed by host
    threads (row ranges): a valid batch trains bit-identically to the same rows
    built on the device; an error in the first, a middle or the last row range
    (unsorted features, bad label id, empty label list) is rejected with no
    state change, and the next valid batch trains normally."""
    from paper_2110_07029_b200._lib import ASError
    cfg = _cfg(20000, 3000, 128, 1100, 1024, avg_nnz=60.0, avg_labels=4.0, seed=5)
    ds = synthgen.make_dataset(cfg, n=1100)
    p = _params(cfg)
    sub = ds.rows(np.arange(1024))
    assert sub.row_ptr[-1] > 32768
    r1 = _replica(cfg, p, ds, "bf16", debug=False)
    r2 = _replica(cfg, p, ds, "bf16", debug=False)
    r1.upload_dataset(ds)
    for row in (0, 500, 1023):
        a, e = int(sub.row_ptr[row]), int(sub.row_ptr[row + 1])
        bad_col = sub.col.copy(); bad_col[a], bad_col[a + 1] = bad_col[a + 1], bad_col[a]
        bad_lab = sub.lab.copy(); bad_lab[int(sub.lab_ptr[row])] = cfg.C
        bad_lp = sub.lab_ptr.copy(); bad_lp[row + 1:] -= bad_lp[row + 1] - bad_lp[row]
        bad_lp = np.ascontiguousarray(bad_lp)
        assert e - a >= 2
        for args in [(1024, sub.row_ptr, bad_col, sub.val, sub.lab_ptr, sub.lab),
                     (1024, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, bad_lab),
                     (1024, sub.row_ptr, sub.col, sub.val, bad_lp, sub.lab)]:
            with pytest.raises(ASError) as ex:
                r2.load_batch_csr(*args)
            assert ex.value.code == -1
    assert np.array_equal(r2.get_params(), p)
    r1.load_batch_stream(0, 1024)
    l1 = r1.train_step(True)
    r2.load_batch_csr(1024, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
    l2 = r2.train_step(True)
    assert l1 == l2
    assert np.array_equal(r1.get_params(), r2.get_params())


@pytest.mark.parametrize("shuffled,pos", [(True, 250), (False, 250), (False, 130)])
def test_resident_stream_batch_equals_host_batch(gpu_lib, shuffled, pos):
    """The device-built batch (a gather for a shuffled or wrapping stream, the
    in-place contiguous slice otherwise) trains bit-identically to the same
    samples loaded from host CSR."""
    cfg = _cfg(1200, 400, 128, 300, 128)
    ds = synthgen.make_dataset(cfg, n=300)
    p = _params(cfg)
    order = osched.permutation(300, 99) if shuffled else None
    r1 = _replica(cfg, p, ds, "bf16", debug=False)
    r2 = _replica(cfg, p, ds, "bf16", debug=False)
    r1.upload_dataset(ds, order)
    rows = 100                                                 # pos 250 wraps the data epoch
    r1.load_batch_stream(pos, rows)
    l1 = r1.train_step(True)
    sub = ds.rows(ocsr.stream_ids(pos, rows, 300, order))
    r2.load_batch_csr(rows, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
    l2 = r2.train_step(True)
    assert l1 == l2
    assert np.array_equal(r1.get_params(), r2.get_params())     # deterministic, bit-identical


def test_step_is_deterministic(gpu_lib):
    cfg = _cfg(3000, 2000, 128, 700, 512, avg_nnz=40)
    ds = synthgen.make_dataset(cfg, n=700)
    p = _params(cfg)
    outs = []
    for _ in range(2):
        rep = _replica(cfg, p, ds, "bf16", debug=False)
        sub = ds.rows(np.arange(512))
        rep.load_batch_csr(512, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
        rep.train_step()
        outs.append(rep.get_params())
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_group_merge_parity(gpu_lib, precision):
    from paper_2110_07029_b200.api import group_merge
    cfg = _cfg(1000, 500, 128, 200, 64)
    ds = synthgen.make_dataset(cfg, n=200)
    p = _params(cfg)
    reps = [_replica(cfg, p, ds, precision, debug=False, rank=i, world=3) for i in range(3)]
    for i, r in enumerate(reps):
        r.set_batch_sizes([64, 64, 64], [0.5, 0.5, 0.5])
        for k in range(i + 1):                                 # u = (1, 2, 3)
            sub = ds.rows(np.arange(32) + 40 * i + 8 * k)
            r.load_batch_csr(32, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
            r.train_step()
    ws = [r.get_params() for r in reps]
    u, b = [1, 2, 3], [64, 64, 64]
    alpha, pert = group_merge(reps, u, b)
    norms = [omerge.replica_norm(w) for w in ws]
    oa, op = osched.alg2(u, b, norms, 0.1, 0.1)
    assert list(alpha) == oa and pert == op == 1
    wbar, wbar_p = omerge.merge(ws, oa, p, p, 0.9)
    for r in reps:
        assert_close("wbar", r.get_params(1), wbar, 1e-5)
        assert np.array_equal(r.get_params(2), p)              # wbar_p <- wbar
        assert np.array_equal(r.get_params(0), r.get_params(1))  # replicas restart from wbar
    # second merge exercises the momentum term gamma (wbar - wbar_p)
    ws2 = [r.get_params() for r in reps]
    alpha2, _ = group_merge(reps, [2, 2, 2], b)
    oa2, _ = osched.alg2([2, 2, 2], b, [omerge.replica_norm(w) for w in ws2], 0.1, 0.1)
    wbar2, _ = omerge.merge(ws2, oa2, wbar, p, 0.9)
    assert_close("wbar2", reps[0].get_params(1), wbar2, 1e-5)


def test_group_merge_ub_normalisation(gpu_lib):
    """AS_FLAG_NORM_UB (P:175 alternative: alpha_i ~ u_i b_i): alpha bit-exact
    with oracle.sched.alg2(norm="ub"), merged model within 1e-5."""
    from paper_2110_07029_b200.api import Replica, group_merge
    cfg = _cfg(1000, 500, 128, 200, 64)
    ds = synthgen.make_dataset(cfg, n=200)
    p = _params(cfg)
    b = [64, 48, 32]
    reps = [Replica(cfg.d, cfg.C, cfg.h, cfg.b_max, p, b_min=8, max_row_nnz=int(np.diff(ds.row_ptr).max()),
                    max_row_labels=int(np.diff(ds.lab_ptr).max()), lr0=0.5, precision="fp32", rank=i, world=3,
                    merge_norm="ub") for i in range(3)]
    for i, r in enumerate(reps):
        r.set_batch_sizes(b, [0.5, 0.375, 0.25])
        for k in range(i + 1):
            sub = ds.rows(np.arange(b[i] // 2) + 40 * i + 8 * k)
            r.load_batch_csr(b[i] // 2, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
            r.train_step()
    ws = [r.get_params() for r in reps]
    alpha, pert = group_merge(reps, [1, 2, 3], b)
    oa, op = osched.alg2([1, 2, 3], b, [omerge.replica_norm(w) for w in ws], 0.1, 0.1, norm="ub")
    assert list(alpha) == oa and pert == op
    wbar, _ = omerge.merge(ws, oa, p, p, 0.9)
    assert_close("wbar", reps[0].get_params(1), wbar, 1e-5)


@pytest.mark.parametrize("u", [[2, 2, 1], [3, 3, 3]])
def test_group_merge_r14_literal(gpu_lib, u):
    """AS_FLAG_R14_LITERAL (Alg. 2 line 8 as printed): alpha bit-exact with
    oracle.sched.alg2(ties="literal") -- ties on u go to the lowest id, and with
    equal u the perturbation lands on replica 0 twice -- merged model within 1e-5."""
    from paper_2110_07029_b200.api import Replica, group_merge
    cfg = _cfg(1000, 500, 128, 200, 64)
    ds = synthgen.make_dataset(cfg, n=200)
    p = _params(cfg)
    b = [48, 64, 32]
    reps = [Replica(cfg.d, cfg.C, cfg.h, cfg.b_max, p, b_min=8, max_row_nnz=int(np.diff(ds.row_ptr).max()),
                    max_row_labels=int(np.diff(ds.lab_ptr).max()), lr0=0.5, precision="fp32", rank=i, world=3,
                    pert_thr=1e6, merge_ties="literal") for i in range(3)]
    for i, r in enumerate(reps):
        r.set_batch_sizes(b, [0.375, 0.5, 0.25])
        sub = ds.rows(np.arange(b[i] // 2) + 40 * i)
        r.load_batch_csr(b[i] // 2, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
        r.train_step()
    ws = [r.get_params() for r in reps]
    alpha, pert = group_merge(reps, u, b)
    oa, op = osched.alg2(u, b, [omerge.replica_norm(w) for w in ws], 0.1, 1e6, ties="literal")
    lex, _ = osched.alg2(u, b, [omerge.replica_norm(w) for w in ws], 0.1, 1e6)
    assert oa != lex                          # the case separates the two readings
    assert list(alpha) == oa and pert == op == 1
    wbar, _ = omerge.merge(ws, oa, p, p, 0.9)
    assert_close("wbar", reps[0].get_params(1), wbar, 1e-5)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_merge_one_replica_r14_literal(gpu_lib, precision):
    """One replica under AS_FLAG_R14_LITERAL: r = s = 0, so a regular replica
    gets alpha = (1 + delta)(1 - delta) = 0.99 through as_merge (norm pass and
    Alg. 2 on the device); irregular keeps 1.  Merged model vs oracle within 1e-5."""
    from paper_2110_07029_b200.api import Replica
    cfg = _cfg(1000, 500, 128, 200, 64)
    ds = synthgen.make_dataset(cfg, n=200)
    p = _params(cfg)
    for thr, want in ((1e6, 0.99), (0.0, 1.0)):
        r = Replica(cfg.d, cfg.C, cfg.h, cfg.b_max, p, b_min=8, max_row_nnz=int(np.diff(ds.row_ptr).max()),
                    max_row_labels=int(np.diff(ds.lab_ptr).max()), lr0=0.5, precision=precision,
                    pert_thr=thr, merge_ties="literal")
        sub = ds.rows(np.arange(32))
        r.load_batch_csr(32, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
        r.train_step()
        w = r.get_params()
        alpha, pert = r.merge([1], [64])
        oa, op = osched.alg2([1], [64], [omerge.replica_norm(w)], 0.1, thr, ties="literal")
        assert list(alpha) == oa and pert == op
        assert abs(oa[0] - want) < 1e-15
        wbar, _ = omerge.merge([w], oa, p, p, 0.9)
        assert_close("wbar", r.get_params(1), wbar, 1e-5)
        r.close()


@pytest.mark.parametrize("metric,thr", [("l2", 1.0), ("l2", 1e6), ("l2/sqrt(P)", 0.05), ("l2^2/P", 1e-3)])
def test_group_merge_norm_metrics(gpu_lib, metric, thr):
    """R15's metric switch: the perturbation decision of Alg. 2 line 7 with each
    metric (thresholds chosen on both sides of the replicas' values) matches the
    oracle bit-exactly, merged model within 1e-5."""
    from paper_2110_07029_b200.api import Replica, group_merge
    cfg = _cfg(1000, 500, 128, 200, 64)
    ds = synthgen.make_dataset(cfg, n=200)
    p = _params(cfg)
    reps = [Replica(cfg.d, cfg.C, cfg.h, cfg.b_max, p, b_min=8, max_row_nnz=int(np.diff(ds.row_ptr).max()),
                    max_row_labels=int(np.diff(ds.lab_ptr).max()), lr0=0.5, precision="fp32", rank=i, world=2,
                    pert_thr=thr, norm_metric=metric) for i in range(2)]
    for i, r in enumerate(reps):
        for k in range(i + 1):
            sub = ds.rows(np.arange(32) + 40 * i + 8 * k)
            r.load_batch_csr(32, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
            r.train_step()
    ws = [r.get_params() for r in reps]
    alpha, pert = group_merge(reps, [1, 2], [64, 64])
    oa, op = osched.alg2([1, 2], [64, 64], [omerge.replica_norm(w, metric) for w in ws], 0.1, thr)
    assert list(alpha) == oa and pert == op
    wbar, _ = omerge.merge(ws, oa, p, p, 0.9)
    assert_close("wbar", reps[0].get_params(1), wbar, 1e-5)


def test_end_to_end_tiny_two_replicas_replay(gpu_lib):
    """T5: config 'tiny' (BASELINE.json configs[0]): 2 replicas, replay with a
    32% slowdown, 1 epoch, 4 merges, fp32 mode.  Routing, b_i, lr_i and alpha
    are bit-exact; the global model matches the oracle after every merge."""
    from paper_2110_07029_b200 import driver
    cfg = synthgen.CONFIGS["tiny"]
    ds = synthgen.make_dataset(cfg)
    p = synthgen.make_init_params(cfg.d, cfg.C, cfg.h, cfg.seed)
    costs = synthgen.make_cost_models(2, hetero=True)
    lr0 = 0.5
    reps = []
    for rank in range(2):
        from paper_2110_07029_b200.api import Replica
        reps.append(Replica(cfg.d, cfg.C, cfg.h, cfg.b_max, p, b_min=cfg.b_min, beta=cfg.beta,
                            megabatch=1024, max_row_nnz=int(np.diff(ds.row_ptr).max()),
                            max_row_labels=int(np.diff(ds.lab_ptr).max()), lr0=lr0, precision="fp32",
                            rank=rank, world=2))
    st = driver.ReplayState(2, cfg.b_max, cfg.b_min, cfg.beta, lr0, costs)
    recs = driver.run_local(reps, ds, st, ds.n)
    ocfg = otrain.RunConfig(d=cfg.d, C=cfg.C, h=cfg.h, b_max=cfg.b_max, b_min=cfg.b_min, beta=cfg.beta,
                            M=1024, lr0=lr0, world=2)
    orecs, owbar = otrain.run(ds, p, ocfg, costs, ds.n)
    assert len(recs) == len(orecs) == 4
    for g, o in zip(recs, orecs):
        assert [tuple(x) for x in g["log"]] == [tuple(x) for x in o["log"]]
        assert g["u"] == o["u"] and g["b"] == o["b"] and g["b_next"] == o["b_next"]
        assert g["lr_next"] == o["lr_next"]
        assert g["alpha"] == o["alpha"] and g["perturbed"] == o["perturbed"]
    assert any(g["u"][0] != g["u"][1] for g in recs)           # heterogeneity exercised
    assert_close("wbar after 4 merges", reps[0].get_params(1), owbar, 1e-4)


@pytest.mark.parametrize("chunks", [None, "7"])
def test_rank_api_world1_matches_oracle(gpu_lib, chunks, monkeypatch):
    """The per-rank public path bench.py times (driver.run_rank: resident
    dataset, stream batches, as_merge with its N = 1 shortcut) against the
    oracle's whole run at N = 1: alpha = [1] every merge (Alg. 2 line 3, R14),
    momentum gamma = 0.9 across 4 merges, global model within 1e-4 (fp32).
    chunks="7": the partitioned merge's chunk bookkeeping (7 uneven chunks, the
    W2T shadow range crossing chunk borders) forced on one GPU."""
    if chunks:
        monkeypatch.setenv("ADASGD_MERGE_CHUNKS", chunks)
    from paper_2110_07029_b200 import driver
    from paper_2110_07029_b200.api import Replica
    cfg = synthgen.CONFIGS["tiny"]
    ds = synthgen.make_dataset(cfg)
    p = synthgen.make_init_params(cfg.d, cfg.C, cfg.h, cfg.seed)
    costs = synthgen.make_cost_models(1, hetero=False)
    lr0, M = 0.5, 256
    rep = Replica(cfg.d, cfg.C, cfg.h, cfg.b_max, p, b_min=cfg.b_min, beta=cfg.beta, megabatch=M,
                  max_row_nnz=int(np.diff(ds.row_ptr).max()), max_row_labels=int(np.diff(ds.lab_ptr).max()),
                  lr0=lr0, gamma=0.9, precision="fp32", rank=0, world=1)
    rep.upload_dataset(ds)
    st = driver.ReplayState(1, cfg.b_max, cfg.b_min, cfg.beta, lr0, costs)
    recs = driver.run_rank(rep, ds.row_ptr, ds.n, st, 4 * M, want_alpha=True)
    ocfg = otrain.RunConfig(d=cfg.d, C=cfg.C, h=cfg.h, b_max=cfg.b_max, b_min=cfg.b_min, beta=cfg.beta,
                            M=M, lr0=lr0, gamma=0.9, world=1)
    orecs, owbar = otrain.run(ds, p, ocfg, costs, 4 * M)
    assert len(recs) == len(orecs) == 4
    for g, o in zip(recs, orecs):
        assert list(g["alpha"]) == o["alpha"] == [1.0] and g["perturbed"] == o["perturbed"] == 0
    assert_close("wbar", rep.get_params(1), owbar, 1e-4)
    assert np.array_equal(rep.get_params(0), rep.get_params(1))
    rep.close()


@pytest.mark.parametrize("algo,M", [("elastic", 1024), ("sync", 128)])
def test_end_to_end_tiny_comparison_methods(gpu_lib, algo, M):
    """the comparison methods of P:215 under the same
    heterogeneous replay as T5: static equal batches (batch k -> replica k mod
    N), alpha = 1/N, no perturbation, no batch scaling.  "sync" merges after
    one batch per replica (M = N b_max).  Routing bit-exact, b_i
    trajectories constant, the global model matches the oracle."""
    from paper_2110_07029_b200 import driver
    from paper_2110_07029_b200.api import Replica
    cfg = synthgen.CONFIGS["tiny"]
    ds = synthgen.make_dataset(cfg)
    p = synthgen.make_init_params(cfg.d, cfg.C, cfg.h, cfg.seed)
    costs = synthgen.make_cost_models(2, hetero=True)
    lr0, gamma = 0.5, 0.0
    reps = [Replica(cfg.d, cfg.C, cfg.h, cfg.b_max, p, b_min=cfg.b_min, beta=cfg.beta, megabatch=M,
                    max_row_nnz=int(np.diff(ds.row_ptr).max()), max_row_labels=int(np.diff(ds.lab_ptr).max()),
                    lr0=lr0, gamma=gamma, precision="fp32", rank=rank, world=2, algo=algo) for rank in range(2)]
    st = driver.ReplayState(2, cfg.b_max, cfg.b_min, cfg.beta, lr0, costs, algo=algo)
    total = 1024
    recs = driver.run_local(reps, ds, st, total)
    ocfg = otrain.RunConfig(d=cfg.d, C=cfg.C, h=cfg.h, b_max=cfg.b_max, b_min=cfg.b_min, beta=cfg.beta,
                            M=M, lr0=lr0, gamma=gamma, world=2, algo=algo)
    orecs, owbar = otrain.run(ds, p, ocfg, costs, total)
    assert len(recs) == len(orecs) == total // M
    for g, o in zip(recs, orecs):
        assert [tuple(x) for x in g["log"]] == [tuple(x) for x in o["log"]]
        assert g["u"] == o["u"] == [M // (2 * cfg.b_max)] * 2
        assert g["b"] == o["b"] == [cfg.b_max] * 2 and g["b_next"] == [cfg.b_max] * 2
        assert g["alpha"] == o["alpha"] == [0.5, 0.5] and not g["perturbed"]
    assert_close("wbar", reps[0].get_params(1), owbar, 1e-4)


@pytest.mark.slow
@pytest.mark.parametrize("peaked", [False, True])
def test_full_size_amazon670k_sampled(gpu_lib, peaked):
    """Amazon-670K shape at b = 1024 in the bench's launch configuration
    (bf16, resident dataset, stream batch): the oracle recomputes the whole
    step in fp64 (chunked over rows) and every output is compared -- including
    the softmax terms on their own (pass 1's O / l and the ~668K unlabelled
    classes of pass 2), which the label term dominates in dA / dW2T / db2.
    peaked: W2T x 8 and a b2 ramp to 40 (as in the rescale test) so the softmax
    of every row is concentrated and the online rescale fires across blocks."""
    cfg = synthgen.CONFIGS["amazon670k"]
    ds = synthgen.make_dataset(cfg, n=40_000)
    p = synthgen.make_init_params(cfg.d, cfg.C, cfg.h, cfg.seed)
    if peaked:
        lay = synthgen.param_layout(cfg.d, cfg.C, cfg.h)
        o, _ = lay["b2"]
        p[o:o + cfg.C] = np.linspace(0.0, 40.0, cfg.C, dtype=np.float32)
        o, _ = lay["W2T"]
        p[o:o + cfg.C * cfg.h] *= np.float32(8.0)
    rep = _replica(cfg, p, ds, "bf16", lr=0.5)
    rep.upload_dataset(ds)
    rep.load_batch_stream(1000, 1024)
    loss = rep.train_step(True)
    sub = ds.rows(ocsr.stream_ids(1000, 1024, ds.n))
    ref = om.gradients_chunked(sub, otrain.unpack(p, cfg.d, cfg.C, cfg.h), chunk=128)
    tol = 2e-2
    assert abs(loss - ref["loss"]) <= tol * ref["loss"]
    lse = _f32(rep.debug_get(1, 4 * 1024)) * LN2
    assert_close("LSE", lse, ref["LSE"], tol)
    assert_abs("LSE abs", lse, ref["LSE"], tol)
    check_softmax_terms("full", rep, sub, ref, cfg.C, 128, tol)
    assert_close("dA", _f32(rep.debug_get(3, 4 * 1024 * 128)).reshape(1024, 128), ref["dA"], tol)
    dW2T = _f32(rep.debug_get(5, 4 * cfg.C * 128)).reshape(cfg.C, 128)
    assert_close("dW2T", dW2T, ref["dW2T"], tol)
    assert_close("db2", _f32(rep.debug_get(6, 4 * cfg.C)), ref["db2"], tol)
    keys = np.unique(sub.col)
    dW1 = _f32(rep.debug_get(7, 4 * len(keys) * 128)).reshape(len(keys), 128)
    assert_close("dW1", dW1, ref["dW1"][keys], tol)
    rep.close()


@pytest.mark.slow
@pytest.mark.parametrize("peaked", [False, True])
def test_full_size_amazoncat13k(gpu_lib, peaked):
    """AmazonCat-13K shape (h = 256, C = 13 330) at b = 1024 in the bench's
    launch configuration: one class block per CTA (pass 2 with the W2T block in
    shared memory and four S^T buffers, the last-block update through the H
    stages, bf16 shadow by TMA), the label terms in pass 1's idle warpgroup,
    the transposes forked before the SpMM, 16-warp sparse kernels.  Every
    output against the fp64 oracle, softmax terms on their own; peaked as in
    the Amazon-670K test."""
    cfg = synthgen.CONFIGS["amazoncat13k"]
    ds = synthgen.make_dataset(cfg, n=8_000)
    p = synthgen.make_init_params(cfg.d, cfg.C, cfg.h, cfg.seed)
    if peaked:
        lay = synthgen.param_layout(cfg.d, cfg.C, cfg.h)
        o, _ = lay["b2"]
        p[o:o + cfg.C] = np.linspace(0.0, 40.0, cfg.C, dtype=np.float32)
        o, _ = lay["W2T"]
        p[o:o + cfg.C * cfg.h] *= np.float32(8.0)
    h = cfg.h
    rep = _replica(cfg, p, ds, "bf16", lr=0.5)
    rep.upload_dataset(ds)
    rep.load_batch_stream(1000, 1024)
    loss = rep.train_step(True)
    sub = ds.rows(ocsr.stream_ids(1000, 1024, ds.n))
    ref = om.gradients_chunked(sub, otrain.unpack(p, cfg.d, cfg.C, h), chunk=128)
    tol = 2e-2
    assert abs(loss - ref["loss"]) <= tol * ref["loss"]
    lse = _f32(rep.debug_get(1, 4 * 1024)) * LN2
    assert_close("LSE", lse, ref["LSE"], tol)
    assert_abs("LSE abs", lse, ref["LSE"], tol)
    check_softmax_terms("full", rep, sub, ref, cfg.C, h, tol)
    assert_close("dA", _f32(rep.debug_get(3, 4 * 1024 * h)).reshape(1024, h), ref["dA"], tol)
    assert_close("dW2T", _f32(rep.debug_get(5, 4 * cfg.C * h)).reshape(cfg.C, h), ref["dW2T"], tol)
    assert_close("db2", _f32(rep.debug_get(6, 4 * cfg.C)), ref["db2"], tol)
    keys = np.unique(sub.col)
    dW1 = _f32(rep.debug_get(7, 4 * len(keys) * h)).reshape(len(keys), h)
    assert_close("dW1", dW1, ref["dW1"][keys], tol)
    new = otrain.unpack(rep.get_params(), cfg.d, cfg.C, h)
    old = otrain.unpack(p, cfg.d, cfg.C, h)
    assert_close("W2T update", new["W2T"] - old["W2T"], -0.5 * ref["dW2T"], tol)
    rep.close()


@pytest.mark.slow
def test_full_size_amazon670k_top1_sampled(gpu_lib):
    """Top-1 evaluation at the Amazon-670K shape (670 091 classes, 5236 class
    blocks over the pass-1 splits) on 1024 rows after one training step: 24
    sampled rows recomputed by the oracle from the updated parameters with the
    kernel's bf16 operands; argmax equal or a near-tie, hits consistent."""
    cfg = synthgen.CONFIGS["amazon670k"]
    ds = synthgen.make_dataset(cfg, n=20_000)
    p = synthgen.make_init_params(cfg.d, cfg.C, cfg.h, cfg.seed)
    rep = _replica(cfg, p, ds, "bf16", lr=0.5, debug=False)
    rep.upload_dataset(ds)
    rep.load_batch_stream(0, 1024)
    rep.train_step(False)
    ev = ds.rows(np.arange(5000, 6024))
    top, hits = rep.eval_top1(1024, ev.row_ptr, ev.col, ev.val, ev.lab_ptr, ev.lab)
    assert top.shape == (1024,) and np.all((top >= 0) & (top < cfg.C))
    new = otrain.unpack(rep.get_params(), cfg.d, cfg.C, cfg.h)
    rows = np.random.default_rng(0).choice(1024, 24, replace=False)
    sub = ds.rows(5000 + rows)
    otop, _, zmax, logit = om.top1(sub, new, operands="bf16")
    bad = 0
    for k, r in enumerate(rows):
        if top[r] != otop[k]:
            bad += 1
            assert zmax[k] - logit(k, int(top[r])) <= 1e-4 * (1.0 + abs(zmax[k])), r
    assert bad <= 2
    lab = [set(ev.lab[ev.lab_ptr[r]:ev.lab_ptr[r + 1]].tolist()) for r in range(1024)]
    assert hits == sum(int(top[r] in lab[r]) for r in range(1024))
    rep.close()


# ---------------------------------------------------------------- top-1 evaluation (NEXT f1)
TOP1_CASES = [
    (2000, 1000, 128, 600, 200, 256),     # ragged row tile, C % 128 = 104
    (3000, 700, 256, 400, 130, 192),      # h = 256
    (4000, 30000, 128, 1200, 1024, 1024), # many class blocks per split
    (500, 50, 128, 64, 1, 64),            # a single row, C < 128
]


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
@pytest.mark.parametrize("case", TOP1_CASES)
def test_eval_top1_parity(gpu_lib, case, precision):
    """as_eval_top1 vs oracle.model.top1 with the decision taken in the kernel's
    operand precision (bf16 operands for the tensor-core path).  The argmax is
    unique except at near-ties: a differing row must be a near-tie of the
    oracle's logits (both classes valid); hits agree up to those rows.  The
    training state is untouched (a following step matches the oracle)."""
    d, C, h, n, B, b_max = case
    cfg = _cfg(d, C, h, n, b_max, seed=hash(case) % 89)
    ds = synthgen.make_dataset(cfg, n=n)
    p = _params(cfg)
    rep = _replica(cfg, p, ds, precision, lr=0.5, debug=False)
    sub = ds.rows(np.arange(B) + 11)
    top, hits = rep.eval_top1(B, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
    prm = otrain.unpack(p, d, C, h)
    otop, ohits, zmax, logit = om.top1(sub, prm, operands="bf16" if precision == "bf16" else "fp64")
    diff = np.nonzero(top != otop)[0]
    assert len(diff) <= max(1, B // 50), (len(diff), B)
    for r in diff:
        assert 0 <= top[r] < C
        assert zmax[r] - logit(r, int(top[r])) <= 1e-4 * (1.0 + abs(zmax[r])), r
    assert abs(hits - ohits) <= len(diff)
    # the training batch path is unaffected by the evaluation
    tr = ds.rows(np.arange(B))
    rep.load_batch_csr(B, tr.row_ptr, tr.col, tr.val, tr.lab_ptr, tr.lab)
    loss = rep.train_step(want_loss=True)
    ref = om.gradients_chunked(tr, prm, chunk=64)
    assert abs(loss - ref["loss"]) <= (2e-2 if precision == "bf16" else 1e-4) * abs(ref["loss"])
    rep.close()


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_eval_top1_ties_lowest_class_across_splits(gpu_lib, precision):
    """W2T = 0: z = b2 exactly on both paths; the maximum is repeated at class
    5 and at class 29000 (different class blocks and pass-1 splits): the
    lowest id must win on every row (R21), bit-exact."""
    d, C, h, B = 3000, 30000, 128, 300
    cfg = _cfg(d, C, h, 400, 512, seed=2)
    ds = synthgen.make_dataset(cfg, n=400)
    p = _params(cfg)
    lay = synthgen.param_layout(d, C, h)
    o, shp = lay["W2T"]
    p[o:o + shp[0] * shp[1]] = 0.0
    o, _ = lay["b2"]
    b2 = np.linspace(-1, 1, C).astype(np.float32)
    b2[5] = b2[29000] = 3.0
    p[o:o + C] = b2
    rep = _replica(cfg, p, ds, precision, debug=False)
    sub = ds.rows(np.arange(B))
    top, hits = rep.eval_top1(B, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
    assert np.all(top == 5)
    otop, ohits, _, _ = om.top1(sub, otrain.unpack(p, d, C, h))
    assert np.all(otop == 5) and hits == ohits
    rep.close()


def _strip_features(sub, empty_rows):
    """The batch with the features of `empty_rows` removed (rows with no
    non-zero feature: H = ReLU(b1), no dW1 contribution)."""
    keep_rp, cols, vals = [0], [], []
    for r in range(len(sub.row_ptr) - 1):
        s, e = sub.row_ptr[r], sub.row_ptr[r + 1]
        if r not in empty_rows:
            cols.append(sub.col[s:e]); vals.append(sub.val[s:e])
        keep_rp.append(keep_rp[-1] + (0 if r in empty_rows else e - s))
    col = np.concatenate(cols) if cols else np.zeros(0, np.int32)
    val = np.concatenate(vals) if vals else np.zeros(0, np.float32)
    return synthgen.CSRDataset(sub.d, sub.C, np.asarray(keep_rp, np.int64), col.astype(np.int32),
                               val.astype(np.float32), sub.lab_ptr.copy(), sub.lab.copy())


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-4), ("bf16", 2e-2)])
@pytest.mark.parametrize("which", ["some", "all"])
def test_empty_feature_rows(gpu_lib, precision, tol, which):
    """Degenerate rows with no features (first, last, consecutive ones) and a
    batch with no features at all (nnz = 0: empty SpMM / transposes / dW1):
    one step against the oracle; W1 untouched when nnz = 0."""
    d, C, h, B = 2000, 1500, 128, 200
    cfg = _cfg(d, C, h, 400, 256, seed=9)
    ds = synthgen.make_dataset(cfg, n=400)
    p = _params(cfg)
    rep = _replica(cfg, p, ds, precision, lr=0.5)
    sub0 = ds.rows(np.arange(B))
    empty = set(range(B)) if which == "all" else {0, 1, 2, 77, 78, B - 1}
    sub = _strip_features(sub0, empty)
    rep.load_batch_csr(B, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
    loss = rep.train_step(want_loss=True)
    prm = otrain.unpack(p, d, C, h)
    ref = om.gradients_chunked(sub, prm, chunk=64)
    H = _f32(rep.debug_get(0, 4 * B * h)).reshape(B, h)
    assert_close("H", H, ref["H"], 1e-5)
    assert abs(loss - ref["loss"]) <= tol * abs(ref["loss"])
    assert_close("dA", _f32(rep.debug_get(3, 4 * B * h)).reshape(B, h), ref["dA"], tol)
    assert_close("dW2T", _f32(rep.debug_get(5, 4 * C * h)).reshape(C, h), ref["dW2T"], tol)
    new = rep.get_params()
    dnew = otrain.unpack(new.astype(np.float64) - p.astype(np.float64), d, C, h)
    keys = np.unique(sub.col)
    if len(keys):
        assert_close("W1 update", dnew["W1"][keys], -0.5 * ref["dW1"][keys], max(tol, 1e-3))
    untouched = np.setdiff1d(np.arange(d), keys)
    assert np.all(dnew["W1"][untouched] == 0)
    # the next step on a normal batch still matches (transpose state back to idle)
    nxt = ds.rows(np.arange(B) + 200)
    rep.load_batch_csr(B, nxt.row_ptr, nxt.col, nxt.val, nxt.lab_ptr, nxt.lab)
    loss2 = rep.train_step(want_loss=True)
    ref2 = om.gradients_chunked(nxt, otrain.unpack(new, d, C, h), chunk=64)
    assert abs(loss2 - ref2["loss"]) <= tol * abs(ref2["loss"])
    rep.close()


@pytest.mark.parametrize("h,C,avg_labels", [(128, 300, 40.0), (256, 200, 25.0), (128, 5000, 75.0)])
def test_label_heavy_batches(gpu_lib, h, C, avg_labels):
    """Delicious-like label density (tens of labels per row, Zipf-hot classes
    labelled in most rows): the pass-2 label term from the row bitmaps and the
    per-row weights, against the oracle (bf16 bar)."""
    d, B = 3000, 256
    cfg = _cfg(d, C, h, 300, 256, avg_labels=avg_labels, seed=21)
    ds = synthgen.make_dataset(cfg, n=300)
    p = _params(cfg)
    rep = _replica(cfg, p, ds, "bf16", lr=0.5)
    sub = ds.rows(np.arange(B))
    rep.load_batch_csr(B, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
    loss = rep.train_step(want_loss=True)
    ref = om.gradients_chunked(sub, otrain.unpack(p, d, C, h), chunk=64)
    assert abs(loss - ref["loss"]) <= 2e-2 * abs(ref["loss"])
    assert_close("dW2T", _f32(rep.debug_get(5, 4 * C * h)).reshape(C, h), ref["dW2T"], 2e-2)
    assert_close("db2", _f32(rep.debug_get(6, 4 * C)), ref["db2"], 2e-2)
    assert_close("dA", _f32(rep.debug_get(3, 4 * B * h)).reshape(B, h), ref["dA"], 2e-2)
    rep.close()


@pytest.mark.parametrize("metric", ["l2/P", "l2^2/P", "l2/sqrt(P)", "l2"])
def test_replica_norm_vs_oracle(gpu_lib, metric):
    """Step a9 (Alg. 2 line 7, R15): the device fp64 norm of a trained replica
    against oracle.merge.replica_norm of the same parameters, <= 1e-12 relative."""
    cfg = _cfg(3000, 2000, 128, 300, 128)
    ds = synthgen.make_dataset(cfg, n=300)
    p = _params(cfg)
    rep = _replica(cfg, p, ds, "bf16", debug=False)
    sub = ds.rows(np.arange(100))
    rep.load_batch_csr(100, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
    rep.train_step()
    w = rep.get_params()
    got = rep.replica_norm(metric)
    want = omerge.replica_norm(w, metric)
    e = abs(got - want) / abs(want)
    plog.record(_test_name(), "norm " + metric, e, 1e-12, "rel")
    assert e <= 1e-12, (got, want)
    rep.close()


@pytest.mark.parametrize("nccl_self,chunks", [(False, None), (True, "3"), (True, "7")])
def test_merge_weighted_forced_alpha(gpu_lib, monkeypatch, nccl_self, chunks):
    """Steps a11-a13 with a forced weight alpha = 0.7 at world = 1: the prescale
    kernel (no communicator), or with ADASGD_NCCL_SELF=1 the NCCL PreMulSum
    all-reduce on a one-rank communicator (the N > 1 code path: PreMulSum op,
    chunked all-reduce on the communication stream, momentum chasing the
    chunks).  Two merges (gamma = 0.9 momentum) against oracle.merge.merge,
    <= 1e-5; replicas restart from wbar; wbar_p rotation.  (NCCL 2.28.9's one-rank
    PreMulSum leaves a few tail elements unscaled for some counts, e.g. the whole
    308 228-float vector here -- scripts/nccl_premul_probe.py -- so the one-rank
    cases use chunked merges; multi-rank all-reduces go through NCCL's regular
    kernels, which this one-GPU box cannot run.)"""
    if nccl_self:
        monkeypatch.setenv("ADASGD_NCCL_SELF", "1")
    if chunks:
        monkeypatch.setenv("ADASGD_MERGE_CHUNKS", chunks)
    cfg = _cfg(1500, 900, 128, 300, 128)
    ds = synthgen.make_dataset(cfg, n=300)
    p = _params(cfg)
    rep = _replica(cfg, p, ds, "bf16", debug=False)
    wbar, wbar_p = p.copy(), p.copy()
    for m in range(2):
        sub = ds.rows(np.arange(100) + 50 * m)
        rep.load_batch_csr(100, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
        rep.train_step()
        w = rep.get_params()
        prev = rep.get_params(1)
        rep.merge_weighted([0.7])
        wbar, wbar_p = omerge.merge([w], [0.7], wbar, wbar_p, 0.9)
        assert_close("wbar merge %d" % m, rep.get_params(1), wbar, 1e-5)
        assert np.array_equal(rep.get_params(2), prev)             # wbar_p <- wbar (rotation)
        assert np.array_equal(rep.get_params(0), rep.get_params(1))
    rep.close()


def test_pass1_grid_more_row_tiles_than_sms(gpu_lib):
    """b = 18 945 rows = 149 row tiles > 148 SMs: pass 1 launches one CTA per
    row tile (several waves) instead of leaving tiles 148+ unwritten (advisor
    finding); one bf16 step against the oracle, plus top-1 on the same rows."""
    B = 148 * 128 + 1
    cfg = _cfg(2000, 300, 128, B + 10, B, avg_nnz=8.0, seed=4)
    ds = synthgen.make_dataset(cfg, n=B + 10)
    p = _params(cfg)
    rep = _replica(cfg, p, ds, "bf16", lr=0.5)
    sub = ds.rows(np.arange(B))
    rep.load_batch_csr(B, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
    loss = rep.train_step(want_loss=True)
    prm = otrain.unpack(p, cfg.d, cfg.C, cfg.h)
    ref = om.gradients_chunked(sub, prm, chunk=2048)
    assert abs(loss - ref["loss"]) <= 2e-2 * abs(ref["loss"])
    lse = _f32(rep.debug_get(1, 4 * B)) * LN2
    assert_abs("LSE abs", lse, ref["LSE"], 2e-2)
    assert_close("dA", _f32(rep.debug_get(3, 4 * B * 128)).reshape(B, 128), ref["dA"], 2e-2)
    assert_close("dW2T", _f32(rep.debug_get(5, 4 * cfg.C * 128)).reshape(cfg.C, 128), ref["dW2T"], 2e-2)
    rep.close()
    rep = _replica(cfg, p, ds, "bf16", debug=False)
    top, hits = rep.eval_top1(B, sub.row_ptr, sub.col, sub.val, sub.lab_ptr, sub.lab)
    otop, ohits, zmax, logit = om.top1(sub, prm, operands="bf16")
    diff = np.nonzero(top != otop)[0]
    assert len(diff) <= B // 50
    for r in diff[:50]:
        assert zmax[r] - logit(r, int(top[r])) <= 1e-4 * (1.0 + abs(zmax[r]))
    rep.close()
