"""Pins for oracle/model.py against things other than itself (CPU only).

* SpMM      vs a densified X and torch.matmul (textbook / library routine)
* loss      vs torch.nn.functional.cross_entropy with probability targets
* gradients vs torch autograd (fp64) AND central finite differences
* closed form: W2T = 0, b2 = 0  ->  loss = ln C, dH = 0, db2 = 1/C - T-colsum/B
"""
import math

import numpy as np
import pytest
import torch

import synthgen
from oracle import model as om
from oracle import train as otrain


def _tiny(seed=1, n=24, d=40, C=24, h=8, scale=1.0):
    ds = synthgen.tiny_dataset(n=n, d=d, C=C, seed=seed)
    p = synthgen.make_init_params(d, C, h, seed)
    p = (p * np.float32(scale)).astype(np.float32)
    rng = np.random.default_rng(seed + 100)
    lay = synthgen.param_layout(d, C, h)
    o, _ = lay["b1"]; p[o:o + h] = rng.normal(0, 0.3, h).astype(np.float32)
    o, _ = lay["b2"]; p[o:o + C] = rng.normal(0, 0.3, C).astype(np.float32)
    return ds, p


def _dense_x(ds):
    X = np.zeros((ds.n, ds.d))
    for r in range(ds.n):
        s, e = ds.row_ptr[r], ds.row_ptr[r + 1]
        X[r, ds.col[s:e]] = ds.val[s:e]
    T = np.zeros((ds.n, ds.C))
    for r in range(ds.n):
        s, e = ds.lab_ptr[r], ds.lab_ptr[r + 1]
        T[r, ds.lab[s:e]] = 1.0 / (e - s)
    return X, T


def _torch_loss(X, T, prm):
    W1 = torch.tensor(np.asarray(prm["W1"], np.float64), requires_grad=True)
    b1 = torch.tensor(np.asarray(prm["b1"], np.float64), requires_grad=True)
    W2T = torch.tensor(np.asarray(prm["W2T"], np.float64), requires_grad=True)
    b2 = torch.tensor(np.asarray(prm["b2"], np.float64), requires_grad=True)
    Xt = torch.tensor(X); Tt = torch.tensor(T)
    Z = torch.relu(Xt @ W1 + b1) @ W2T.T + b2
    loss = torch.nn.functional.cross_entropy(Z, Tt)       # probability targets, mean over rows
    loss.backward()
    return loss.item(), Z.detach().numpy(), {"W1": W1.grad.numpy(), "b1": b1.grad.numpy(),
                                              "W2T": W2T.grad.numpy(), "b2": b2.grad.numpy()}


def test_spmm_vs_dense_matmul():
    ds, p = _tiny()
    prm = otrain.unpack(p, ds.d, ds.C, 8)
    X, _ = _dense_x(ds)
    ref = (torch.tensor(X) @ torch.tensor(prm["W1"], dtype=torch.float64)
           + torch.tensor(prm["b1"], dtype=torch.float64)).numpy()
    got = om.spmm(ds.row_ptr, ds.col, ds.val, prm["W1"], prm["b1"])
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_loss_logits_grads_vs_torch(seed):
    ds, p = _tiny(seed=seed)
    prm = otrain.unpack(p, ds.d, ds.C, 8)
    X, T = _dense_x(ds)
    loss_t, Z_t, g_t = _torch_loss(X, T, prm)
    fwd = om.forward(ds, prm)
    g = om.gradients(ds, prm, fwd)
    assert abs(fwd["loss"] - loss_t) <= 1e-12 * abs(loss_t)
    np.testing.assert_allclose(fwd["Z"], Z_t, rtol=1e-12, atol=1e-13)
    for k in ("W1", "b1", "W2T", "b2"):
        np.testing.assert_allclose(g[k], g_t[k], rtol=1e-10, atol=1e-14)


def test_grads_vs_central_finite_differences():
    ds, p = _tiny(seed=5, n=12)
    prm = otrain.unpack(p.astype(np.float64), ds.d, ds.C, 8)
    g = om.gradients(ds, prm)
    A = om.forward(ds, prm)["A"]
    rng = np.random.default_rng(0)
    eps = 1e-6
    checked = 0
    touched = np.unique(ds.col)
    for key in ("W1", "b1", "W2T", "b2"):
        arr = prm[key]
        for _ in range(12):
            if key == "W1":
                idx = (int(rng.choice(touched)), int(rng.integers(arr.shape[1])))
            else:
                idx = tuple(int(rng.integers(s)) for s in arr.shape)
            # skip coordinates that move a pre-activation across the ReLU kink
            old = arr[idx]
            arr[idx] = old + eps; lp = om.forward(ds, prm)["loss"]; Ap = om.forward(ds, prm)["A"]
            arr[idx] = old - eps; lm = om.forward(ds, prm)["loss"]; Am = om.forward(ds, prm)["A"]
            arr[idx] = old
            if np.any(np.sign(Ap) != np.sign(Am)) or np.min(np.abs(A)) < 1e-9:
                continue
            fd = (lp - lm) / (2 * eps)
            assert abs(fd - g[key][idx]) <= 1e-6 * max(1e-3, abs(fd)), (key, idx, fd, g[key][idx])
            checked += 1
    assert checked >= 30


def test_closed_form_zero_output_layer():
    ds, p = _tiny(seed=7)
    prm = otrain.unpack(p.copy(), ds.d, ds.C, 8)
    prm["W2T"][:] = 0.0
    prm["b2"][:] = 0.0
    fwd = om.forward(ds, prm)
    g = om.gradients(ds, prm, fwd)
    assert abs(fwd["loss"] - math.log(ds.C)) < 1e-13            # softmax uniform -> ln C
    _, T = _dense_x(ds)
    np.testing.assert_allclose(g["b2"], 1.0 / ds.C - T.sum(0) / ds.n, atol=1e-15)
    H = fwd["H"]
    np.testing.assert_allclose(g["W2T"], (1.0 / ds.C - T).T @ H / ds.n, atol=1e-14)
    assert np.all(g["dH"] == 0) and np.all(g["W1"] == 0) and np.all(g["b1"] == 0)


def test_sgd_step_moves_against_gradient_and_lowers_loss():
    ds, p = _tiny(seed=9)
    prm = otrain.unpack(p, ds.d, ds.C, 8)
    new, loss0, _ = om.sgd_step(ds, prm, 0.5)
    loss1 = om.forward(ds, new)["loss"]
    assert loss1 < loss0
    # untouched W1 rows stay bit-identical
    untouched = np.setdiff1d(np.arange(ds.d), np.unique(ds.col))
    assert np.array_equal(new["W1"][untouched], np.asarray(prm["W1"])[untouched])


def test_chunked_gradients_equal_plain():
    ds, p = _tiny(seed=12, n=40)
    prm = otrain.unpack(p, ds.d, ds.C, 8)
    g = om.gradients(ds, prm)
    f = om.forward(ds, prm)
    gc = om.gradients_chunked(ds, prm, chunk=7)
    assert abs(gc["loss"] - f["loss"]) <= 1e-13
    np.testing.assert_allclose(gc["LSE"], f["LSE"], rtol=1e-14)
    for k, kc in (("W1", "dW1"), ("W2T", "dW2T"), ("b2", "db2"), ("b1", "db1"), ("dA", "dA")):
        np.testing.assert_allclose(gc[kc], g[k], rtol=1e-12, atol=1e-15)


# ---------------------------------------------------------------- top-1 (NEXT f1)
def test_top1_vs_torch_argmax_and_label_hits():
    """P:228 top-1 = class of highest probability; pinned to torch softmax +
    argmax on the densified batch (library routine) and a direct hit count."""
    ds, p = _tiny(seed=4, n=30, d=50, C=40, h=8)
    prm = otrain.unpack(p, ds.d, ds.C, 8)
    X, _ = _dense_x(ds)
    t = {k: torch.tensor(np.asarray(v, np.float64)) for k, v in prm.items()}
    prob = torch.softmax(torch.relu(torch.tensor(X) @ t["W1"] + t["b1"]) @ t["W2T"].T + t["b2"], dim=1)
    want = torch.argmax(prob, dim=1).numpy()
    top, hits, zmax, logit = om.top1(ds, prm)
    assert np.array_equal(top, want)
    h = sum(int(want[r] in set(ds.lab[ds.lab_ptr[r]:ds.lab_ptr[r + 1]].tolist())) for r in range(ds.n))
    assert hits == h
    assert all(abs(zmax[r] - logit(r, int(top[r]))) < 1e-12 for r in range(ds.n))


def test_top1_closed_form_zero_output_weights_ties_lowest_id():
    """W2T = 0: z_r = b2 for every row, so top-1 = argmax b2; with the maximum
    repeated at classes 3 and 7 the lowest id (3) wins (reading R21)."""
    ds, p = _tiny(seed=6, n=20, d=30, C=12, h=8)
    prm = otrain.unpack(p, ds.d, ds.C, 8)
    prm["W2T"] = np.zeros_like(prm["W2T"])
    b2 = np.linspace(-1.0, 0.5, ds.C).astype(np.float32)
    b2[3] = b2[7] = 2.0
    prm["b2"] = b2
    for ops in ("fp64", "bf16"):
        top, hits, _, _ = om.top1(ds, prm, operands=ops)
        assert np.all(top == 3)
        assert hits == sum(int(3 in ds.lab[ds.lab_ptr[r]:ds.lab_ptr[r + 1]]) for r in range(ds.n))


def test_bf16_round_matches_torch_bfloat16():
    """bf16_round (round to nearest even) vs torch's float32 -> bfloat16 cast,
    including exact halfway cases and signed zeros."""
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.normal(0, 3, 5000), rng.normal(0, 1e-3, 1000)]).astype(np.float32)
    half = np.array([0x3F808000, 0x3F818000, 0xBF808000, 0x00000000, 0x80000000], np.uint32).view(np.float32)
    x = np.concatenate([x, half])
    want = torch.tensor(x).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(om.bf16_round(x), want)


def test_dHsoft_closed_form_uniform_softmax():
    """H = 0 (W1 = 0, b1 < 0) and b2 = 0 make every logit 0, so softmax(z_r) =
    1/C exactly and the softmax part of dH is the mean row of W2T over B:
    dHsoft_r = (1/B) (1/C) sum_c W2T[c] for every row (both oracle routes)."""
    ds, p = _tiny(seed=5)
    d, C, h = ds.d, ds.C, 8
    lay = synthgen.param_layout(d, C, h)
    o, shp = lay["W1"]; p[o:o + shp[0] * shp[1]] = 0.0
    o, _ = lay["b1"]; p[o:o + h] = -1.0
    o, _ = lay["b2"]; p[o:o + C] = 0.0
    prm = otrain.unpack(p, d, C, h)
    B = ds.n
    want = np.tile(np.asarray(prm["W2T"], np.float64).mean(axis=0) / B, (B, 1))
    g = om.gradients(ds, prm)
    gc = om.gradients_chunked(ds, prm, chunk=5)
    assert np.allclose(g["dHsoft"], want, rtol=1e-12, atol=1e-18)
    assert np.allclose(gc["dHsoft"], want, rtol=1e-12, atol=1e-18)


def test_dHsoft_plus_label_part_is_dH_brute_force():
    """dH = dHsoft - (1/(k_r B)) sum_{y in Y_r} W2T[y] (the two terms of dz), with
    dHsoft recomputed here by explicit loops over rows and classes (math.exp,
    max-shifted) on a tiny case; dH from torch autograd w.r.t. H."""
    ds, p = _tiny(seed=6, n=6, C=7)
    h = 8
    prm = otrain.unpack(p, ds.d, ds.C, h)
    g = om.gradients(ds, prm)
    W2T = np.asarray(prm["W2T"], np.float64); b2 = np.asarray(prm["b2"], np.float64)
    X, T = _dense_x(ds)
    A = X @ np.asarray(prm["W1"], np.float64) + np.asarray(prm["b1"], np.float64)
    Hn = np.maximum(A, 0.0)
    B = ds.n
    brute = np.zeros((B, h))
    for r in range(B):
        z = [float(Hn[r] @ W2T[c] + b2[c]) for c in range(ds.C)]
        m = max(z)
        e = [math.exp(v - m) for v in z]
        tot = sum(e)
        for c in range(ds.C):
            brute[r] += (e[c] / tot) * W2T[c] / B
    assert np.allclose(g["dHsoft"], brute, rtol=1e-12, atol=1e-18)
    Ht = torch.tensor(Hn, requires_grad=True)
    Z = Ht @ torch.tensor(W2T).T + torch.tensor(b2)
    torch.nn.functional.cross_entropy(Z, torch.tensor(T)).backward()
    assert np.allclose(brute - (T @ W2T) / B, Ht.grad.numpy(), rtol=1e-10, atol=1e-15)
