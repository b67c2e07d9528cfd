"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no forward, gradient, routing,
scaling or merge).  It only draws inputs:

* sparse XML datasets in CSR form shaped like the paper's Table 1
  ("Table 1: Experimental datasets for XML classification"),
* initial parameters (the paper's init sentence at PAPER.md:228 is garbled;
  DESIGN.md reading R5 fixes Glorot-normal, biases 0),
* per-replica integer cost models for deterministic replay (reading R9).

Recipe:
  nnz/row   lognormal(sigma=0.7) mean-matched to the target average, rounded,
            clamped to [1, 8*avg]
  features  Zipf(s=1.0) over a fixed random permutation of [0, d), drawn
            without replacement inside a row (duplicates redrawn), sorted
  values    U(0, 1], then each row L2-normalised (tf-idf-like)
  labels/row 1 + Poisson(avg - 1), clamped to [1, min(C, 8*avg)]
  label ids Zipf(s=1.1) over a random permutation of [0, C), unique, sorted
Everything is drawn from numpy's PCG64 generator seeded with
``seed = 0x211007029 + config_index``.
"""
from __future__ import annotations

import dataclasses
import numpy as np

BASE_SEED = 0x211007029


@dataclasses.dataclass(frozen=True)
class XMLConfig:
    """Shape of one BASELINE.json config."""
    name: str
    d: int            # features
    C: int            # labels (classes)
    n: int            # training samples
    avg_nnz: float
    avg_labels: float
    h: int            # hidden width
    b_max: int
    world: int        # replicas in the config
    index: int        # config index -> seed

    @property
    def b_min(self) -> int:      # PAPER.md:228 "b_min ... 8 times smaller than b_max"
        return self.b_max // 8

    @property
    def beta(self) -> int:       # PAPER.md:228 "beta to half of b_min"
        return self.b_min // 2

    @property
    def megabatch(self) -> int:  # PAPER.md:242,266 "100 batches"; reading R7: M = 100*b_max
        return 100 * self.b_max

    @property
    def seed(self) -> int:
        return BASE_SEED + self.index

    @property
    def n_params(self) -> int:
        return self.d * self.h + self.h + self.C * self.h + self.C


CONFIGS = {
    # BASELINE.json configs[0..4]; sizes per SURVEY.md section 8(d).
    "tiny": XMLConfig("tiny", 10_000, 1_000, 4_096, 20.0, 3.0, 128, 64, 2, 0),
    "amazoncat13k": XMLConfig("amazoncat13k", 203_882, 13_330, 1_186_239, 71.0, 5.04, 256, 1024, 1, 1),
    "delicious200k": XMLConfig("delicious200k", 782_585, 205_443, 196_606, 302.0, 75.0, 128, 1024, 4, 2),
    "amazon670k": XMLConfig("amazon670k", 135_909, 670_091, 490_449, 76.0, 5.0, 128, 1024, 8, 3),
    "wikilshtc325k": XMLConfig("wikilshtc325k", 1_617_899, 325_056, 1_778_351, 42.0, 3.19, 128, 1024, 8, 4),
}


@dataclasses.dataclass
class CSRDataset:
    """Sparse dataset: row r has features col[row_ptr[r]:row_ptr[r+1]] (sorted,
    unique) with values val[...] and labels lab[lab_ptr[r]:lab_ptr[r+1]]
    (sorted, unique, at least one)."""
    d: int
    C: int
    row_ptr: np.ndarray   # int64 [n+1]
    col: np.ndarray       # int32 [nnz]
    val: np.ndarray       # float32 [nnz]
    lab_ptr: np.ndarray   # int64 [n+1]
    lab: np.ndarray       # int32 [L]

    @property
    def n(self) -> int:
        return len(self.row_ptr) - 1

    def rows(self, ids: np.ndarray) -> "CSRDataset":
        """Plain row gather (input plumbing, not part of the method)."""
        ids = np.asarray(ids, dtype=np.int64)
        rl = self.row_ptr[ids + 1] - self.row_ptr[ids]
        ll = self.lab_ptr[ids + 1] - self.lab_ptr[ids]
        rp = np.zeros(len(ids) + 1, np.int64); rp[1:] = np.cumsum(rl)
        lp = np.zeros(len(ids) + 1, np.int64); lp[1:] = np.cumsum(ll)
        src = np.concatenate([np.arange(self.row_ptr[i], self.row_ptr[i + 1]) for i in ids]) \
            if len(ids) else np.zeros(0, np.int64)
        lsrc = np.concatenate([np.arange(self.lab_ptr[i], self.lab_ptr[i + 1]) for i in ids]) \
            if len(ids) else np.zeros(0, np.int64)
        return CSRDataset(self.d, self.C, rp, self.col[src].copy(), self.val[src].copy(),
                          lp, self.lab[lsrc].copy())


def _lognormal_counts(rng, n, avg, sigma, lo, hi):
    mu = np.log(avg) - 0.5 * sigma * sigma           # E[lognormal] = avg
    x = np.rint(rng.lognormal(mu, sigma, size=n))
    return np.clip(x, lo, hi).astype(np.int64)


def _zipf_cdf(n_items, s):
    w = 1.0 / np.arange(1, n_items + 1, dtype=np.float64) ** s
    c = np.cumsum(w)
    return c / c[-1]


def _draw_sets(rng, counts, n_items, s, perm, max_rounds=32):
    """Per row r draw counts[r] distinct items ~ Zipf(s) over perm (sequential
    draws, duplicates skipped = sampling without replacement); returns
    (ptr, items) with items sorted inside each row."""
    n = len(counts)
    counts = np.minimum(counts, n_items).astype(np.int64)
    cdf = _zipf_cdf(n_items, s)
    chosen_keys = []
    have = np.zeros(n, np.int64)
    finished = np.zeros(n, bool)
    prev = np.zeros(0, np.int64)          # keys already chosen for rows still short
    for rnd in range(max_rounds):
        need = np.where(finished, 0, counts - have)
        rows = np.nonzero(need > 0)[0]
        if len(rows) == 0:
            break
        m = np.ceil(need[rows] * (1.6 if rnd == 0 else 3.0)).astype(np.int64) + 2
        rr = np.repeat(rows, m)
        it = perm[np.minimum(np.searchsorted(cdf, rng.random(len(rr)), side="right"), n_items - 1)]
        key = rr * np.int64(n_items) + it
        # draw order: previously chosen keys first, then new draws in order
        allk = np.concatenate([prev, key])
        _, first = np.unique(allk, return_index=True)
        first.sort()                       # first occurrences in draw order
        k = allk[first]
        krow = k // n_items
        order = np.argsort(krow, kind="stable")
        k, krow = k[order], krow[order]
        # rank inside row; keep the first counts[r]
        start = np.searchsorted(krow, krow, side="left")
        rank = np.arange(len(k)) - start
        keep = rank < counts[krow]
        k, krow = k[keep], krow[keep]
        done = (np.bincount(krow, minlength=n) >= counts) & ~finished
        fin = done[krow]
        chosen_keys.append(k[fin])
        finished |= done
        prev = k[~fin]
        have = np.bincount(prev // n_items, minlength=n)
    if len(prev):                           # rows still short keep what they have
        chosen_keys.append(prev)
    keys = np.sort(np.concatenate(chosen_keys)) if chosen_keys else np.zeros(0, np.int64)
    got = np.bincount(keys // n_items, minlength=n)
    ptr = np.zeros(n + 1, np.int64)
    ptr[1:] = np.cumsum(got)
    return ptr, (keys % n_items).astype(np.int32)


def make_dataset(cfg: XMLConfig, n: int | None = None, seed: int | None = None) -> CSRDataset:
    """Draw a CSR dataset with cfg's shape (optionally fewer rows n)."""
    n = cfg.n if n is None else int(n)
    rng = np.random.default_rng(cfg.seed if seed is None else seed)
    fperm = rng.permutation(cfg.d).astype(np.int64)
    lperm = rng.permutation(cfg.C).astype(np.int64)
    nnz = _lognormal_counts(rng, n, cfg.avg_nnz, 0.7, 1, int(8 * cfg.avg_nnz))
    nlab = np.clip(1 + rng.poisson(max(cfg.avg_labels - 1.0, 0.0), size=n),
                   1, min(cfg.C, int(8 * cfg.avg_labels))).astype(np.int64)
    row_ptr, col = _draw_sets(rng, nnz, cfg.d, 1.0, fperm)
    lab_ptr, lab = _draw_sets(rng, nlab, cfg.C, 1.1, lperm)
    val = (1.0 - rng.random(len(col))).astype(np.float64)      # U(0, 1]
    # row L2 normalisation (input preprocessing, tf-idf-like)
    rid = np.repeat(np.arange(n), np.diff(row_ptr))
    ss = np.bincount(rid, weights=val * val, minlength=n)
    val = (val / np.sqrt(ss)[rid]).astype(np.float32)
    return CSRDataset(cfg.d, cfg.C, row_ptr, col, val, lab_ptr, lab)


def make_planted_dataset(cfg: XMLConfig, n: int | None = None, seed: int | None = None, signal: float = 0.6,
                         proto: int = 6) -> CSRDataset:
    """Like make_dataset, but with a learnable label signal (for the synthetic
    time-to-accuracy harness only; the paper's data are real): class
    c owns `proto` fixed prototype features, and about `signal` of a row's
    features are drawn from the prototypes of its labels (the rest is the
    Zipf noise of make_dataset).  Labels are drawn exactly as in make_dataset."""
    n = cfg.n if n is None else int(n)
    rng = np.random.default_rng((cfg.seed if seed is None else seed) ^ 0xA11CE)
    base = make_dataset(cfg, n=n, seed=(cfg.seed if seed is None else seed))
    protos = rng.integers(0, cfg.d, size=(cfg.C, proto))
    rp, cols = [0], []
    for r in range(n):
        noise = base.col[base.row_ptr[r]:base.row_ptr[r + 1]]
        labs = base.lab[base.lab_ptr[r]:base.lab_ptr[r + 1]]
        k = max(1, int(round(signal * len(noise))))
        sig = protos[labs].ravel()
        sig = sig[rng.integers(0, len(sig), size=k)]
        keep = noise[: max(0, len(noise) - k)]
        row = np.unique(np.concatenate([sig, keep]).astype(np.int32))
        cols.append(row)
        rp.append(rp[-1] + len(row))
    col = np.concatenate(cols).astype(np.int32)
    row_ptr = np.asarray(rp, np.int64)
    val = (1.0 - rng.random(len(col))).astype(np.float64)
    rid = np.repeat(np.arange(n), np.diff(row_ptr))
    ss = np.bincount(rid, weights=val * val, minlength=n)
    val = (val / np.sqrt(ss)[rid]).astype(np.float32)
    return CSRDataset(cfg.d, cfg.C, row_ptr, col, val, base.lab_ptr.copy(), base.lab.copy())


def param_layout(d: int, C: int, h: int) -> dict:
    """Offsets (in floats) of the packed parameter vector [W1 | b1 | W2T | b2]
    (reading R2).  W1 is [d][h], W2T is [C][h] (label-major)."""
    o_w1 = 0
    o_b1 = d * h
    o_w2 = o_b1 + h
    o_b2 = o_w2 + C * h
    return {"W1": (o_w1, (d, h)), "b1": (o_b1, (h,)), "W2T": (o_w2, (C, h)),
            "b2": (o_b2, (C,)), "P": o_b2 + C}


def make_init_params(d: int, C: int, h: int, seed: int) -> np.ndarray:
    """Packed fp32 init (reading R5): Glorot-normal sigma = sqrt(2/(fan_in+fan_out)),
    biases 0."""
    lay = param_layout(d, C, h)
    rng = np.random.default_rng(seed ^ 0x5EED)
    p = np.zeros(lay["P"], np.float32)
    o, _ = lay["W1"]
    p[o:o + d * h] = rng.standard_normal(d * h, dtype=np.float32) * np.float32(np.sqrt(2.0 / (d + h)))
    o, _ = lay["W2T"]
    p[o:o + C * h] = rng.standard_normal(C * h, dtype=np.float32) * np.float32(np.sqrt(2.0 / (h + C)))
    return p


def split_params(p: np.ndarray, d: int, C: int, h: int) -> dict:
    lay = param_layout(d, C, h)
    out = {}
    for k in ("W1", "b1", "W2T", "b2"):
        o, shp = lay[k]
        out[k] = p[o:o + int(np.prod(shp))].reshape(shp)
    return out


@dataclasses.dataclass(frozen=True)
class CostModel:
    """Integer replay cost of one batch on replica i, in picoseconds
    (reading R9): cost = (c0 + c_row*rows + c_nnz*nnz) * num // den."""
    c0: int
    c_row: int
    c_nnz: int
    num: int = 1
    den: int = 1


def make_cost_models(world: int, hetero: bool, seed: int = 7) -> list:
    """Cost models for replay.  hetero=True injects per-GPU slowdowns spread
    over [1, 1.32] -- the 32% fastest/slowest gap of PAPER.md:27 (Fig. 1)."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(world):
        num = 100 + (int(round(32 * i / max(world - 1, 1))) if hetero else 0)
        jitter = int(rng.integers(0, 3)) if hetero else 0
        out.append(CostModel(c0=2_000_000, c_row=40_000 + 1000 * jitter, c_nnz=500, num=num, den=100))
    return out


def tiny_dataset(n=96, d=40, C=24, avg_nnz=5.0, avg_labels=2.0, seed=1) -> CSRDataset:
    """Small dataset for exhaustive oracle checks (finite differences etc.)."""
    cfg = XMLConfig("t", d, C, n, avg_nnz, avg_labels, 8, 16, 2, 0)
    return make_dataset(cfg, n=n, seed=seed)
