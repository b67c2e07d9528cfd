"""Oracle: the sparse-input MLP of the paper, one SGD step, in fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Model (section 5.1 "3-layer Multi-Layer Perceptron (MLP) model having
ReLU layer activation, softmax multi-class probability, and cross-entropy
loss"; reading R1: input -> one ReLU hidden layer -> softmax output):

    a_r   = b1 + sum_{(f, v) in x_r} v * W1[f]          (sparse x_r)
    h_r   = max(a_r, 0)
    z_r   = W2T h_r + b2                                (length C)
    LSE_r = log sum_c exp(z_rc)
    loss  = (1/B) sum_r [LSE_r - (1/k_r) sum_{y in Y_r} z_ry]     (reading R3)

Backward ("the backward pass implements the chain rule"), all from the
pre-update parameters:

    dz_rc = (softmax(z_r)_c - [c in Y_r]/k_r) / B
    dW2T  = dz^T H,  db2 = sum_r dz_r,  dH = dz W2T,  dA = dH * [A > 0]  (R4)
    dW1[f] = sum_{r: f in x_r} v_rf dA_r,  db1 = sum_r dA_r

dH splits into its softmax part and its label part (the two terms of dz):
    dHsoft_r = (1/B) sum_c softmax(z_r)_c W2T[c],   dH_r = dHsoft_r - (1/(k_r B)) sum_{y in Y_r} W2T[y]

Update ("the third pass ... updates the model with the computed gradient
using the learning rate"):  theta <- theta - lr * dtheta, computed in
fp64 and stored in fp32 (parameters are fp32 in the packed layout, R2).
"""
from __future__ import annotations

import numpy as np


def spmm(row_ptr, col, val, W1, b1):
    """A = X W1 + b1 for a CSR batch X (P:51 forward pass, first layer)."""
    B = len(row_ptr) - 1
    W1 = np.asarray(W1, np.float64)
    A = np.empty((B, W1.shape[1]), np.float64)
    for r in range(B):
        s, e = int(row_ptr[r]), int(row_ptr[r + 1])
        A[r] = np.asarray(b1, np.float64) + np.asarray(val[s:e], np.float64) @ W1[col[s:e]]
    return A


def target_matrix_rows(lab_ptr, lab):
    """(rows, cols, weights) of the sparse target T_rc = [c in Y_r]/k_r (R3)."""
    B = len(lab_ptr) - 1
    rows, cols, w = [], [], []
    for r in range(B):
        s, e = int(lab_ptr[r]), int(lab_ptr[r + 1])
        k = e - s
        if k < 1:
            raise ValueError("row %d has no label (reading R3 rejects k_r = 0)" % r)
        for y in lab[s:e]:
            rows.append(r); cols.append(int(y)); w.append(1.0 / k)
    return np.array(rows, np.int64), np.array(cols, np.int64), np.array(w, np.float64)


def forward(batch, params):
    """Forward pass.  Returns dict with A, H, Z (logits), LSE, loss (fp64)."""
    W1, b1, W2T, b2 = (np.asarray(params[k], np.float64) for k in ("W1", "b1", "W2T", "b2"))
    A = spmm(batch.row_ptr, batch.col, batch.val, W1, b1)
    H = np.maximum(A, 0.0)
    Z = H @ W2T.T + b2
    zmax = Z.max(axis=1, keepdims=True)
    LSE = zmax[:, 0] + np.log(np.exp(Z - zmax).sum(axis=1))
    tr, tc, tw = target_matrix_rows(batch.lab_ptr, batch.lab)
    B = A.shape[0]
    label_term = np.zeros(B)
    np.add.at(label_term, tr, tw * Z[tr, tc])
    loss = float(np.mean(LSE - label_term))
    return {"A": A, "H": H, "Z": Z, "LSE": LSE, "loss": loss}


def gradients(batch, params, fwd=None):
    """All four gradients of the loss w.r.t. the packed parameters (fp64)."""
    if fwd is None:
        fwd = forward(batch, params)
    W2T = np.asarray(params["W2T"], np.float64)
    A, H, Z, LSE = fwd["A"], fwd["H"], fwd["Z"], fwd["LSE"]
    B = A.shape[0]
    G = np.exp(Z - LSE[:, None])                    # softmax(z_r)
    dHsoft = (G @ W2T) / B                          # softmax part of dH
    tr, tc, tw = target_matrix_rows(batch.lab_ptr, batch.lab)
    np.add.at(G, (tr, tc), -tw)                     # - T
    G /= B                                          # dz
    dW2T = G.T @ H
    db2 = G.sum(axis=0)
    dH = G @ W2T
    dA = dH * (A > 0)
    d = np.asarray(params["W1"]).shape[0]
    dW1 = np.zeros((d, A.shape[1]), np.float64)
    rid = np.repeat(np.arange(B), np.diff(np.asarray(batch.row_ptr)))
    np.add.at(dW1, np.asarray(batch.col, np.int64),
              np.asarray(batch.val, np.float64)[:, None] * dA[rid])
    db1 = dA.sum(axis=0)
    return {"W1": dW1, "b1": db1, "W2T": dW2T, "b2": db2, "dZ": G, "dH": dH, "dA": dA, "dHsoft": dHsoft}


def sgd_step(batch, params, lr):
    """One SGD step (P:51 three passes).  params: dict of fp32 arrays.
    Returns (new fp32 params dict, loss, grads)."""
    fwd = forward(batch, params)
    g = gradients(batch, params, fwd)
    lr = float(np.float32(lr))
    new = {}
    for k in ("W1", "b1", "W2T", "b2"):
        new[k] = (np.asarray(params[k], np.float64) - lr * g[k]).astype(np.float32)
    return new, fwd["loss"], g


def gradients_chunked(batch, params, chunk=64):
    """The same forward/backward as forward() + gradients(), evaluated `chunk`
    rows at a time so that the b x C logits never exist at once (memory only:
    every quantity is the same definition; used for the full-size sampled
    parity checks).  Returns dict with LSE, loss, dA, db1, dW1, dW2T, db2."""
    W1, b1, W2T, b2 = (np.asarray(params[k], np.float64) for k in ("W1", "b1", "W2T", "b2"))
    A = spmm(batch.row_ptr, batch.col, batch.val, W1, b1)
    H = np.maximum(A, 0.0)
    B = A.shape[0]
    tr, tc, tw = target_matrix_rows(batch.lab_ptr, batch.lab)
    LSE = np.empty(B)
    label_term = np.zeros(B)
    dH = np.empty_like(H)
    dHsoft = np.empty_like(H)
    dW2T = np.zeros_like(W2T)
    db2 = np.zeros_like(b2)
    for r0 in range(0, B, chunk):
        r1 = min(B, r0 + chunk)
        Z = H[r0:r1] @ W2T.T + b2
        zmax = Z.max(axis=1, keepdims=True)
        LSE[r0:r1] = zmax[:, 0] + np.log(np.exp(Z - zmax).sum(axis=1))
        sel = (tr >= r0) & (tr < r1)
        np.add.at(label_term, tr[sel], tw[sel] * Z[tr[sel] - r0, tc[sel]])
        G = np.exp(Z - LSE[r0:r1, None])
        dHsoft[r0:r1] = (G @ W2T) / B
        np.add.at(G, (tr[sel] - r0, tc[sel]), -tw[sel])
        G /= B
        dW2T += G.T @ H[r0:r1]
        db2 += G.sum(axis=0)
        dH[r0:r1] = G @ W2T
    dA = dH * (A > 0)
    d = W1.shape[0]
    dW1 = np.zeros((d, A.shape[1]), np.float64)
    rid = np.repeat(np.arange(B), np.diff(np.asarray(batch.row_ptr)))
    np.add.at(dW1, np.asarray(batch.col, np.int64), np.asarray(batch.val, np.float64)[:, None] * dA[rid])
    return {"A": A, "H": H, "LSE": LSE, "loss": float(np.mean(LSE - label_term)), "dA": dA,
            "db1": dA.sum(axis=0), "dW1": dW1, "dW2T": dW2T, "db2": db2, "dHsoft": dHsoft}


def bf16_round(x):
    """Round fp32 values to bfloat16 (round to nearest even), returned as fp64.
    Used only where an integer decision (an argmax) is taken in the kernel's
    operand precision (task rule: both sides decide in the same precision)."""
    x32 = np.ascontiguousarray(np.asarray(x, np.float32))
    u = x32.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def top1(batch, params, operands="fp64", chunk=256):
    """Top-1 prediction and hits ("top-1 accuracy – corresponding to the
    class with the highest probability"; softmax is monotone, so the class
    with the largest logit z_rc).  Ties -> lowest class id (reading R21); a hit
    when that class is one of the row's labels.

    operands="bf16" rounds h_r and W2T to bfloat16 before the product (the
    tensor-core path's operands; the products are still summed in fp64), so the
    argmax is decided in the kernel's operand precision.

    Returns (top1[B] int64, hits int, zmax[B] fp64, Z-accessor) where
    Z-accessor(r, c) gives the logit used for the decision (for near-tie checks)."""
    W1, b1, W2T, b2 = (np.asarray(params[k], np.float64) for k in ("W1", "b1", "W2T", "b2"))
    H = np.maximum(spmm(batch.row_ptr, batch.col, batch.val, W1, b1), 0.0)
    if operands == "bf16":
        H = bf16_round(H.astype(np.float32))
        W2T = bf16_round(np.asarray(params["W2T"], np.float32))
    B = H.shape[0]
    top = np.empty(B, np.int64)
    zmax = np.empty(B, np.float64)
    for r0 in range(0, B, chunk):
        Z = H[r0:r0 + chunk] @ W2T.T + b2
        top[r0:r0 + chunk] = np.argmax(Z, axis=1)          # numpy: first (lowest) index on ties
        zmax[r0:r0 + chunk] = Z[np.arange(Z.shape[0]), top[r0:r0 + chunk]]
    hits = 0
    for r in range(B):
        s, e = int(batch.lab_ptr[r]), int(batch.lab_ptr[r + 1])
        hits += int(top[r] in set(int(y) for y in batch.lab[s:e]))

    def logit(r, c):
        return float(H[r] @ W2T[c] + b2[c])
    return top, hits, zmax, logit
