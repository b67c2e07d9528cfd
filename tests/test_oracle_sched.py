"""Pins for oracle/sched.py and oracle/csr.py (CPU only).

Golden cases under tests/golden/ are worked by hand from the paper's
Algorithms 1-2 and section 3.1 (citations inside each file)."""
import json
import os
from fractions import Fraction

import numpy as np
from hypothesis import given, settings, strategies as st

import synthgen
from oracle import csr as ocsr
from oracle import sched as osched

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _cm(c):
    return synthgen.CostModel(*c)


def test_routing_golden():
    for case in _load("routing_cases.json")["cases"]:
        costs = [_cm(c) for c in case["costs"]]
        log, u, t = osched.route_replay(costs, case["b"], case["M"], lambda s, r: 0)
        assert [list(x) for x in log] == case["log"]
        assert u == case["u"] and t == case["clocks"]


@settings(max_examples=60, deadline=None)
@given(st.integers(1, 6), st.integers(1, 400), st.data())
def test_routing_conserves_samples(N, M, data):
    b = [data.draw(st.integers(1, 40)) for _ in range(N)]
    costs = [synthgen.CostModel(data.draw(st.integers(0, 50)), data.draw(st.integers(0, 9)),
                                data.draw(st.integers(0, 3)), data.draw(st.integers(1, 5)), 1)
             for _ in range(N)]
    log, u, _ = osched.route_replay(costs, b, M, lambda s, r: 3 * r)
    covered = []
    for i, s, r in log:
        assert 1 <= r <= b[i]
        covered.extend(range(s, s + r))
    assert covered == list(range(M))              # every sample exactly once, in stream order
    assert sum(u) == len(log)
    # only the last batch may be truncated
    for i, s, r in log[:-1]:
        assert r == b[i]


def test_alg1_golden():
    for case in _load("alg1_cases.json")["cases"]:
        b, lr = osched.alg1(case["u"], case["b"], case["beta"], case["b_min"], case["b_max"], 0.1)
        assert b == case["b_out"], case["why"]
        for bi, li in zip(b, lr):
            assert li == float(np.float32(0.1 * bi / case["b_max"]))


@settings(max_examples=100, deadline=None)
@given(st.integers(1, 8), st.data())
def test_alg1_invariants(N, data):
    b_max = data.draw(st.sampled_from([16, 64, 1024]))
    b_min = b_max // 8
    beta = max(1, b_min // 2)
    b = [data.draw(st.integers(b_min, b_max)) for _ in range(N)]
    u = [data.draw(st.integers(0, 30)) for _ in range(N)]
    bn, lr = osched.alg1(u, b, beta, b_min, b_max, 0.5)
    assert all(b_min <= x <= b_max for x in bn)
    mu = Fraction(sum(u), N)
    for i in range(N):
        if u[i] > mu:
            assert bn[i] >= b[i]
        elif u[i] < mu:
            assert bn[i] <= b[i]
        else:
            assert bn[i] == b[i]
        assert abs(lr[i] - 0.5 * bn[i] / b_max) <= 1e-7 * lr[i]


def test_alg2_golden():
    for case in _load("alg2_cases.json")["cases"]:
        norms = [0.0 if case["norms_below"] else 1.0] * len(case["u"])
        alpha, pert = osched.alg2(case["u"], case["b"], norms, 0.1, 0.1)
        exp = [Fraction(a) for a in case["alpha"]]
        for a, e in zip(alpha, exp):
            assert abs(Fraction(a) - e) <= Fraction(1, 10**15) * e
        assert abs(Fraction(sum(alpha)) - Fraction(case["sum"])) <= Fraction(1, 10**14)
        assert pert == case["perturbed"]


@settings(max_examples=100, deadline=None)
@given(st.integers(1, 8), st.data())
def test_alg2_invariants(N, data):
    u = [data.draw(st.integers(0, 20)) for _ in range(N)]
    if sum(u) == 0:
        u[0] = 1
    b = [data.draw(st.integers(1, 64)) for _ in range(N)]
    a0, p0 = osched.alg2(u, b, [1.0] * N, 0.1, 0.1)          # not regularised: no perturbation
    assert p0 == 0 and abs(sum(a0) - 1.0) <= 1e-15 * N
    a1, p1 = osched.alg2(u, b, [0.0] * N, 0.1, 0.1)
    if p1:
        r = max(range(N), key=lambda i: ((u[i], b[i]), -i))
        s = min(range(N), key=lambda i: ((u[i], b[i]), i))
        assert abs(sum(a1) - (1.0 + 0.1 * (a0[r] - a0[s]))) <= 1e-14
    a2, p2 = osched.alg2(u, b, [0.0] * N, 0.1, 0.0)          # pert_thr = 0: never perturb
    assert p2 == 0 and a2 == a0


def test_splitmix64_reference_vector():
    # SplitMix64 (Steele, Lea, Flood 2014) from state 0: first output 0xE220A8397B1DCDAF
    _, z = osched.splitmix64(0)
    assert z == 0xE220A8397B1DCDAF


def test_splitmix64_reference_stream():
    # the first five outputs of the published SplitMix64 reference generator from
    # state 0 (Vigna, splitmix64.c; the same constants as Steele et al. 2014)
    ref = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC,
           0x1B39896A51A8749B]
    s, out = 0, []
    for _ in range(5):
        s, z = osched.splitmix64(s)
        out.append(z)
    assert out == ref


def test_permutation_hand_derived_n5():
    """Reading R10 worked by hand for n = 5, seed 0: Fisher-Yates from the top,
    i = 4, 3, 2, 1, with j = floor(r (i + 1) / 2^64) and r the reference
    SplitMix64 outputs above (their leading bytes give r / 2^64):
      i = 4: r = 0xE220.. (0.883) -> j = floor(4.41) = 4  swap(4, 4): [0 1 2 3 4]
      i = 3: r = 0x6E78.. (0.431) -> j = floor(1.73) = 1  swap(3, 1): [0 3 2 1 4]
      i = 2: r = 0x06C4.. (0.026) -> j = floor(0.08) = 0  swap(2, 0): [2 3 0 1 4]
      i = 1: r = 0xF88B.. (0.971) -> j = floor(1.94) = 1  swap(1, 1): [2 3 0 1 4]"""
    assert osched.permutation(5, 0) == [2, 3, 0, 1, 4]


def test_permutation_is_permutation():
    for n, seed in [(1, 0), (2, 5), (100, 7), (1000, 123)]:
        p = osched.permutation(n, seed)
        assert sorted(p) == list(range(n))
    assert osched.permutation(100, 1) != osched.permutation(100, 2)


def test_transpose_against_lexsort_and_roundtrip():
    ds = synthgen.tiny_dataset(n=50, d=30, C=20, seed=4)
    keys, sptr, srow, sval = ocsr.transpose(ds.row_ptr, ds.col, ds.val)
    rid = np.repeat(np.arange(ds.n), np.diff(ds.row_ptr))
    order = np.lexsort((rid, ds.col))            # library sort by (feature, row)
    assert np.array_equal(srow, rid[order]) and np.array_equal(sval, ds.val[order])
    assert np.array_equal(keys, np.unique(ds.col))
    assert sptr[-1] == len(ds.col) and np.all(np.diff(sptr) > 0)
    # transpose of the transpose is the original CSR
    k2, p2, r2, v2 = ocsr.transpose(sptr, srow, sval)
    assert np.array_equal(k2, np.arange(ds.n)) and np.array_equal(p2, ds.row_ptr)
    assert np.array_equal(keys[r2], ds.col)
    assert np.array_equal(v2, ds.val)


def test_stream_ids_and_batch_csr():
    ds = synthgen.tiny_dataset(n=10, d=30, C=20, seed=4)
    ids = ocsr.stream_ids(8, 5, ds.n)
    assert list(ids) == [8, 9, 0, 1, 2]
    rp, col, val, lp, lab = ocsr.batch_csr(ds, ids)
    ref = ds.rows(ids)
    assert np.array_equal(rp, ref.row_ptr) and np.array_equal(col, ref.col)
    assert np.array_equal(lp, ref.lab_ptr) and np.array_equal(lab, ref.lab)


def test_routing_static_golden():
    """as hand-worked in tests/golden/routing_static_cases.json (R26)."""
    cases = json.load(open(os.path.join(GOLD, "routing_static_cases.json")))["cases"]
    for c in cases:
        costs = [synthgen.CostModel(*x) for x in c["costs"]]
        log, u, t = osched.route_static(costs, c["b"], c["M"], lambda s, r: 0)
        assert [list(x) for x in log] == c["log"] and u == c["u"] and t == c["clocks"]


def test_alg2_ub_normalisation_hand_worked():
    """P:175 variant (u_i b_i normalisation), hand-worked: u = (5, 3), b = (64, 60)
    -> u b = (320, 180), alpha = (0.64, 0.36); all norms regular -> perturbed
    (0.704, 0.324), sum = 1 + delta (0.64 - 0.36) = 1.028 (R16).  Equal u keeps
    line 3 (b normalisation) in both modes."""
    a, p = osched.alg2([5, 3], [64, 60], [0.0, 0.0], 0.1, 0.1, norm="ub")
    assert p == 1
    assert [Fraction(x).limit_denominator(10**6) for x in a] == [Fraction(704, 1000), Fraction(324, 1000)]
    a0, _ = osched.alg2([5, 3], [64, 60], [1.0, 1.0], 0.1, 0.1, norm="ub")
    assert [Fraction(x).limit_denominator(10**6) for x in a0] == [Fraction(16, 25), Fraction(9, 25)]
    assert osched.alg2([4, 4], [64, 48], [1.0, 1.0], 0.1, 0.1, norm="ub") == \
        osched.alg2([4, 4], [64, 48], [1.0, 1.0], 0.1, 0.1, norm="u")


def test_alg2_r14_literal_hand_worked():
    """Line 8 as printed (reading R14 "literal"): r / s are the FIRST
    indices of max u / min u, and lines 8-9 apply even when r = s.
    u = (3, 3, 1), b = (100, 200, 50): line 5 alpha = (3/7, 3/7, 1/7); literal
    r = 0, s = 2 -> (33/70, 3/7, 9/70), where the lexicographic reading picks
    r = 1 (larger b) -> (3/7, 33/70, 9/70).  Equal u = (4, 4), b = (64, 48):
    line 3 alpha = (4/7, 3/7); literal r = s = 0 -> (0.99 * 4/7, 3/7) =
    (99/175, 3/7); lexicographic r = 0, s = 1 -> (22/35, 27/70).  One replica:
    literal (0.99,), lexicographic (1.0,) unperturbed."""
    F = lambda a: [Fraction(x).limit_denominator(10**6) for x in a]
    a, p = osched.alg2([3, 3, 1], [100, 200, 50], [0.0] * 3, 0.1, 0.1, ties="literal")
    assert p == 1 and F(a) == [Fraction(33, 70), Fraction(3, 7), Fraction(9, 70)]
    a, p = osched.alg2([3, 3, 1], [100, 200, 50], [0.0] * 3, 0.1, 0.1)
    assert p == 1 and F(a) == [Fraction(3, 7), Fraction(33, 70), Fraction(9, 70)]
    a, p = osched.alg2([4, 4], [64, 48], [0.0] * 2, 0.1, 0.1, ties="literal")
    assert p == 1 and F(a) == [Fraction(99, 175), Fraction(3, 7)]
    a, p = osched.alg2([4, 4], [64, 48], [0.0] * 2, 0.1, 0.1)
    assert p == 1 and F(a) == [Fraction(22, 35), Fraction(27, 70)]
    a, p = osched.alg2([2], [64], [0.0], 0.1, 0.1, ties="literal")
    assert p == 1 and F(a) == [Fraction(99, 100)]
    assert osched.alg2([2], [64], [0.0], 0.1, 0.1) == ([1.0], 0)
    # not regular: no perturbation in either reading
    assert osched.alg2([3, 3, 1], [100, 200, 50], [1.0] * 3, 0.1, 0.1, ties="literal") == \
        osched.alg2([3, 3, 1], [100, 200, 50], [1.0] * 3, 0.1, 0.1)


def test_fit_cost_recovers_integer_model():
    """R9 replay model from a live trace: noiseless times generated by a known
    integer model are recovered exactly; with +-0.4 ps of noise too."""
    rng = np.random.default_rng(3)
    rows = rng.integers(64, 1025, 40)
    nnz = rows * 70 + rng.integers(-2000, 2000, 40)
    t = 2_000_000 + 40_000 * rows + 500 * nnz
    assert osched.fit_cost(rows, nnz, t) == (2_000_000, 40_000, 500, 1, 1)
    assert osched.fit_cost(rows, nnz, t + rng.uniform(-0.4, 0.4, 40)) == (2_000_000, 40_000, 500, 1, 1)


def test_scale_period_golden():
    for case in _load("scale_period_cases.json")["cases"]:
        p, d = osched.scale_period(case["b_prev"], case["b_next"], case["dir"], case["period"], case["p_max"])
        assert (p, d) == (case["period_out"], case["dir_out"]), case["why"]


def test_scale_period_equal_speeds_doubles_interval():
    """Equal speeds (P:105 replay with one cost model): every GPU gets the same
    number of batches, Alg. 1 is a no-op (stable), so with R27 Alg. 1 runs
    after mega-batches 1, 3, 7 (interval 1, 2, 4) and the interval saturates
    at p_max; the trajectory of b is the default's (b_max throughout)."""
    from oracle import train as otrain
    cfg_x = synthgen.XMLConfig("sp", 300, 40, 60, 6.0, 2.0, 32, 16, 1, 5)
    ds = synthgen.make_dataset(cfg_x, n=200)
    p0 = synthgen.make_init_params(cfg_x.d, cfg_x.C, cfg_x.h, 3)
    costs = [synthgen.CostModel(c0=0, c_row=10, c_nnz=0, num=1, den=1)] * 2
    rc = otrain.RunConfig(cfg_x.d, cfg_x.C, cfg_x.h, b_max=16, b_min=2, beta=1, M=64, lr0=0.1,
                          world=2, scale_pmax=4)
    recs, _ = otrain.run(ds, p0, rc, costs, 64 * 9)
    assert [r["period"] for r in recs] == [2, 2, 4, 4, 4, 4, 4, 4, 4]
    assert all(r["b_next"] == [16, 16] for r in recs)


def test_scale_period_pure_oscillation_saturates():
    """Two GPUs whose batch sizes swing back and forth every Alg. 1 run (the
    "oscillatory state" of P:141): the first move resets to 1, every later
    reversal doubles the interval (R27) until p_max."""
    b = [[48, 40], [44, 44], [48, 40], [44, 44], [48, 40], [44, 44], [48, 40]]
    period, dirs, seen = 1, [0, 0], []
    for prev, nxt in zip(b, b[1:]):
        period, dirs = osched.scale_period(prev, nxt, dirs, period, 8)
        seen.append(period)
    assert seen == [1, 2, 4, 8, 8, 8]
