"""Oracle: replica norm and the normalized weighted merge with momentum.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np


def replica_norm(w, metric="l2/P"):
    """||w_i||_2 / |w| over the packed parameter vector (Alg. 2 line 7;
    P:177 "L2-norm divided by model dimensionality"; reading R15), fp64.
    metric: "l2/P" (literal, default), "l2^2/P", "l2/sqrt(P)", "l2" -- the
    readings R15 keeps switchable (P:276 is in tension with the literal one)."""
    w = np.asarray(w, np.float64)
    S = float(np.sum(w * w))
    P = w.size
    return {"l2/P": np.sqrt(S) / P, "l2^2/P": S / P, "l2/sqrt(P)": np.sqrt(S / P), "l2": np.sqrt(S)}[metric]


def merge(replicas, alpha, wbar, wbar_p, gamma):
    """Alg. 2 lines 11-12:
        w' = sum_i alpha_i w_i + gamma (wbar - wbar_p);  wbar_p <- wbar;  wbar <- w'
    fp64 arithmetic, result stored in fp32.  Returns (new wbar, new wbar_p)."""
    acc = np.zeros(np.asarray(wbar).shape, np.float64)
    for a, w in zip(alpha, replicas):
        acc += float(a) * np.asarray(w, np.float64)
    acc += float(gamma) * (np.asarray(wbar, np.float64) - np.asarray(wbar_p, np.float64))
    return acc.astype(np.float32), np.asarray(wbar, np.float32).copy()
