"""Oracle: the scheduler -- replay routing, Alg. 1, Alg. 2 weights.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain Python integers and
doubles, written out in the paper's order and notation.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1


# --------------------------------------------------------------------------
# Stream order (reading R10: not in the paper).  Fisher-Yates driven by
# SplitMix64; the bounded draw is j = (r * (i + 1)) >> 64.
# --------------------------------------------------------------------------
def splitmix64(state):
    state = (state + 0x9E3779B97F4A7C15) & MASK64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return state, z ^ (z >> 31)


def permutation(n, seed):
    perm = list(range(n))
    s = seed & MASK64
    for i in range(n - 1, 0, -1):
        s, r = splitmix64(s)
        j = (r * (i + 1)) >> 64
        perm[i], perm[j] = perm[j], perm[i]
    return perm


# --------------------------------------------------------------------------
# Dynamic scheduling, replay mode (section 3.1: "batches are dispatched
# one-by-one based on GPU availability. Whenever a GPU finishes an epoch, it is
# assigned the next batch ... controlled by fixing the number of training
# samples processed between model merging stages -- we call these samples a
# mega-batch").  GPU availability is replayed from integer cost models
# (reading R9); ties go to the lowest id and the last batch is truncated
# (reading R8); u_i counts dispatched batches.
# --------------------------------------------------------------------------
def batch_cost(cm, rows, nnz):
    return ((cm.c0 + cm.c_row * rows + cm.c_nnz * nnz) * cm.num) // cm.den


def route_replay(costs, b, M, nnz_of):
    """costs: list of CostModel; b: batch sizes; M: samples in this mega-batch;
    nnz_of(start, rows) -> nnz of that slice of the mega-batch.
    Returns (log [(replica, start, rows)], u, clocks)."""
    N = len(costs)
    t = [0] * N
    u = [0] * N
    log = []
    assigned = 0
    while assigned < M:
        i = min(range(N), key=lambda k: (t[k], k))       # earliest free, lowest id
        rows = min(b[i], M - assigned)
        log.append((i, assigned, rows))
        t[i] += batch_cost(costs[i], rows, nnz_of(assigned, rows))
        u[i] += 1
        assigned += rows
    return log, u, t


def route_static(costs, b, M, nnz_of):
    """Static partitioning of the comparison methods that "do not consider
    heterogeneity": elastic model averaging (Fig. 3) and gradient
    aggregation (Fig. 2) give every GPU the same batches regardless of
    speed - batch k of the mega-batch goes to GPU k mod N, all batches of the
    same size (the last one truncated, R8).  Clocks advance with the same cost
    models as route_replay so the straggler time max_i t_i is comparable."""
    N = len(costs)
    assert all(x == b[0] for x in b), "static partitioning uses equal batch sizes"
    t = [0] * N
    u = [0] * N
    log = []
    assigned = 0
    k = 0
    while assigned < M:
        i = k % N
        rows = min(b[0], M - assigned)
        log.append((i, assigned, rows))
        t[i] += batch_cost(costs[i], rows, nnz_of(assigned, rows))
        u[i] += 1
        assigned += rows
        k += 1
    return log, u, t


# --------------------------------------------------------------------------
# Algorithm 1 "Batch Size Scaling", reading R11/R23 for the
# rounding of beta*(u_i - mu) and the bound check, and the linear scaling rule
# for lr.
# --------------------------------------------------------------------------
def alg1(u, b, beta, b_min, b_max, lr0):
    N = len(u)
    U = sum(u)                            # line 1: mu = U / N
    b_new = list(b)
    for i in range(N):                    # line 2: for all GPU_i
        D = N * u[i] - U                  # N * (u_i - mu), exact integer
        step = (2 * beta * abs(D) + N) // (2 * N)   # round(beta*|u_i - mu|), half away from 0
        if D > 0 and b[i] + step <= b_max:          # lines 2-4 (faster GPU)
            b_new[i] = b[i] + step
        elif D < 0 and b[i] - step >= b_min:        # lines 5-7 (slower GPU)
            b_new[i] = b[i] - step
    lr_new = [float(_f32(float(lr0) * bi / b_max)) for bi in b_new]
    return b_new, lr_new



# --------------------------------------------------------------------------
# Adaptive scaling frequency ("By default, the algorithm is executed
# after every mega-batch. However, if stability is achieved or the system
# enters an oscillatory state, the frequency at which scaling is performed can
# be increased"), reading R27: the quantity adapted is the interval between
# Alg. 1 runs, in mega-batches.  Written as the two states the sentence names.
# --------------------------------------------------------------------------
def scale_period(b_prev, b_next, dir_prev, period, p_max):
    """Returns (next interval, this run's direction of each b_i)."""
    directions = []
    for before, after in zip(b_prev, b_next):
        if after > before:
            directions.append(1)
        elif after < before:
            directions.append(-1)
        else:
            directions.append(0)
    # "stability is achieved": Alg. 1 left every batch size where it was
    stable = all(d == 0 for d in directions)
    # "an oscillatory state": the batch sizes that move now move back (at
    # least one reverses its previous change, none continues in its direction)
    reversing = [d != 0 and p != 0 and d != p for d, p in zip(directions, dir_prev)]
    continuing = [d != 0 and d == p for d, p in zip(directions, dir_prev)]
    oscillatory = any(reversing) and not any(continuing)
    if stable or oscillatory:
        return min(2 * period, p_max), directions
    return 1, directions


def _f32(x):
    import numpy as np
    return np.float32(x)


# --------------------------------------------------------------------------
# Algorithm 2 "Normalized Model Merging", weights part; readings
# R13 (exact equality), R14 (lexicographic argmax/argmin of (u_i, b_i), skip
# when identical), R15 (strict <), R16 (no renormalisation).
# --------------------------------------------------------------------------
def alg2(u, b, norms, delta, pert_thr, norm="u", ties="lex"):
    """norm="ub": line 5 normalises by u_i b_i instead ("an alternative
    for later stages is to normalize based on the product between the number
    of updates and the batch size").  ties="literal": line 8 exactly as printed
    ("r <- argmax_i {u_i}, s <- argmin_i {u_i}"): the first index of the
    largest / smallest u, and lines 8-9 applied even when r = s."""
    N = len(u)
    if all(x == u[0] for x in u):                 # line 2
        sb = float(sum(b))
        alpha = [float(bi) / sb for bi in b]      # line 3
    elif norm == "u":
        su = float(sum(u))
        alpha = [float(ui) / su for ui in u]      # line 5
    else:
        sub = float(sum(ui * bi for ui, bi in zip(u, b)))
        alpha = [float(ui * bi) / sub for ui, bi in zip(u, b)]
    perturbed = 0
    if ties == "literal" and all(nrm < pert_thr for nrm in norms):   # line 7
        r = u.index(max(u))                       # line 8 as printed
        s = u.index(min(u))
        alpha[r] = alpha[r] * (1.0 + delta)       # line 9 (r = s: both on alpha_r)
        alpha[s] = alpha[s] * (1.0 - delta)
        perturbed = 1
    elif all(nrm < pert_thr for nrm in norms):    # line 7
        keys = [(u[i], b[i]) for i in range(N)]
        r = max(range(N), key=lambda i: (keys[i], -i))    # argmax, lowest id on ties
        s = min(range(N), key=lambda i: (keys[i], i))     # argmin, lowest id on ties
        if keys[r] != keys[s]:
            alpha[r] = alpha[r] * (1.0 + delta)   # line 9
            alpha[s] = alpha[s] * (1.0 - delta)
            perturbed = 1
    return alpha, perturbed


def fit_cost(rows, nnz, ps):
    """Replay cost model from a live trace (reading R9): least
    squares of ps = c0 + c_row rows + c_nnz nnz (numpy lstsq), rounded to the
    nearest integer and clamped at 0; num = den = 1."""
    X = np.stack([np.ones(len(rows)), np.asarray(rows, np.float64), np.asarray(nnz, np.float64)], axis=1)
    coef, *_ = np.linalg.lstsq(X, np.asarray(ps, np.float64), rcond=None)
    c = [max(0, int(np.rint(v))) for v in coef]
    return (c[0], c[1], c[2], 1, 1)
