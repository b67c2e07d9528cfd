"""CPU tests of the C-ABI library (no GPU needed):

* libadasgd.so loads and exports every symbol include/adasgd.h declares;
* the C++ scheduler is bit-exact with the oracle's scheduler (routing logs,
  batch sizes, lr bits, alpha bits, permutations) on the golden cases and on
  random cases;
* config validation returns AS_E_INVALID;
* the live cursor conserves samples.
"""
import ctypes as C
import json
import os
import re
import struct
import subprocess

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import synthgen
from oracle import sched as osched
from paper_2110_07029_b200 import _lib as L
from paper_2110_07029_b200 import sched as psched

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def _header_functions():
    txt = open(os.path.join(ROOT, "include", "adasgd.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(as_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = L.load()
    declared = _header_functions()
    assert declared, "no declarations parsed"
    assert sorted(L.EXPORTS) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (as_[a-z0-9_]+)\b", out))
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:
        assert hasattr(lib, s)


def _f32bits(x):
    return struct.unpack("<I", struct.pack("<f", x))[0]


def test_routing_golden_cpp():
    for case in json.load(open(os.path.join(GOLD, "routing_cases.json")))["cases"]:
        log, u, t = psched.route_replay(case["costs"], case["b"], case["M"], [0] * (case["M"] + 1))
        assert [list(x) for x in log] == case["log"] and u == case["u"] and t == case["clocks"]


@settings(max_examples=80, deadline=None)
@given(st.integers(1, 8), st.integers(1, 500), st.data())
def test_routing_bit_exact_vs_oracle(N, M, data):
    b = [data.draw(st.integers(1, 64)) for _ in range(N)]
    costs = [(data.draw(st.integers(0, 10**6)), data.draw(st.integers(0, 10**5)),
              data.draw(st.integers(0, 10**3)), data.draw(st.integers(1, 140)), data.draw(st.integers(1, 100)))
             for _ in range(N)]
    nnz = np.array([data.draw(st.integers(1, 50)) for _ in range(M)], np.int64)
    pre = np.zeros(M + 1, np.int64); pre[1:] = np.cumsum(nnz)
    log, u, t = psched.route_replay(costs, b, M, pre)
    ocosts = [synthgen.CostModel(*c) for c in costs]
    olog, ou, ot = osched.route_replay(ocosts, b, M, lambda s, r: int(pre[s + r] - pre[s]))
    assert log == olog and u == ou and t == ot


def test_routing_static_golden_cpp():
    for case in json.load(open(os.path.join(GOLD, "routing_static_cases.json")))["cases"]:
        log, u, t = psched.route_replay(case["costs"], case["b"], case["M"], [0] * (case["M"] + 1), static=True)
        assert [list(x) for x in log] == case["log"] and u == case["u"] and t == case["clocks"]


@settings(max_examples=60, deadline=None)
@given(st.integers(1, 8), st.integers(1, 500), st.integers(1, 64), st.data())
def test_routing_static_bit_exact_vs_oracle(N, M, b0, data):
    costs = [(data.draw(st.integers(0, 10**6)), data.draw(st.integers(0, 10**5)),
              data.draw(st.integers(0, 10**3)), data.draw(st.integers(1, 140)), data.draw(st.integers(1, 100)))
             for _ in range(N)]
    nnz = np.array([data.draw(st.integers(1, 50)) for _ in range(M)], np.int64)
    pre = np.zeros(M + 1, np.int64); pre[1:] = np.cumsum(nnz)
    log, u, t = psched.route_replay(costs, [b0] * N, M, pre, static=True)
    olog, ou, ot = osched.route_static([synthgen.CostModel(*c) for c in costs], [b0] * N, M,
                                       lambda s, r: int(pre[s + r] - pre[s]))
    assert log == olog and u == ou and t == ot
    assert sum(r for (_, _, r) in log) == M


@settings(max_examples=60, deadline=None)
@given(st.integers(1, 8), st.data())
def test_alg2_ub_bit_exact_vs_oracle(N, data):
    u = [data.draw(st.integers(0, 40)) for _ in range(N)]
    if sum(u) == 0:
        u[0] = 1
    b = [data.draw(st.integers(1, 1024)) for _ in range(N)]
    norms = [data.draw(st.floats(0.0, 0.2)) for _ in range(N)]
    a, p = psched.alg2(u, b, norms, 0.1, 0.1, norm="ub")
    oa, op = osched.alg2(u, b, norms, 0.1, 0.1, norm="ub")
    assert a == oa and p == op


@settings(max_examples=60, deadline=None)
@given(st.integers(1, 8), st.sampled_from(["u", "ub"]), st.data())
def test_alg2_r14_literal_bit_exact_vs_oracle(N, norm, data):
    """AS_NORM_R14_LITERAL (line 8 as printed) in the C++ export against the oracle."""
    u = [data.draw(st.integers(0, 6)) for _ in range(N)]
    if sum(u) == 0:
        u[0] = 1
    b = [data.draw(st.integers(1, 1024)) for _ in range(N)]
    norms = [data.draw(st.floats(0.0, 0.2)) for _ in range(N)]
    a, p = psched.alg2(u, b, norms, 0.1, 0.1, norm=norm, ties="literal")
    oa, op = osched.alg2(u, b, norms, 0.1, 0.1, norm=norm, ties="literal")
    assert a == oa and p == op


def test_fit_cost_cpp_vs_oracle():
    rng = np.random.default_rng(11)
    for trial in range(20):
        n = int(rng.integers(3, 60))
        rows = rng.integers(1, 1025, n)
        nnz = rng.integers(1, 80_000, n)
        c = (int(rng.integers(0, 10**7)), int(rng.integers(0, 10**5)), int(rng.integers(0, 10**3)))
        t = c[0] + c[1] * rows + c[2] * nnz
        assert psched.fit_cost(rows, nnz, t) == osched.fit_cost(rows, nnz, t) == c + (1, 1)


def test_alg1_golden_cpp():
    for case in json.load(open(os.path.join(GOLD, "alg1_cases.json")))["cases"]:
        b, lr = psched.alg1(case["u"], case["b"], case["beta"], case["b_min"], case["b_max"], 0.1)
        ob, olr = osched.alg1(case["u"], case["b"], case["beta"], case["b_min"], case["b_max"], 0.1)
        assert b == case["b_out"] == ob
        assert [_f32bits(x) for x in lr] == [_f32bits(x) for x in olr]


@settings(max_examples=150, deadline=None)
@given(st.integers(1, 8), st.data())
def test_alg1_bit_exact_vs_oracle(N, data):
    b_max = data.draw(st.sampled_from([64, 512, 1024, 2048]))
    b_min = b_max // 8
    beta = data.draw(st.integers(0, b_min))
    lr0 = data.draw(st.floats(1e-4, 10.0))
    b = [data.draw(st.integers(b_min, b_max)) for _ in range(N)]
    u = [data.draw(st.integers(0, 100)) for _ in range(N)]
    cb, clr = psched.alg1(u, b, beta, b_min, b_max, lr0)
    ob, olr = osched.alg1(u, b, beta, b_min, b_max, lr0)
    assert cb == ob and [_f32bits(x) for x in clr] == [_f32bits(x) for x in olr]


def test_alg2_golden_cpp():
    for case in json.load(open(os.path.join(GOLD, "alg2_cases.json")))["cases"]:
        norms = [0.0 if case["norms_below"] else 1.0] * len(case["u"])
        a, p = psched.alg2(case["u"], case["b"], norms, 0.1, 0.1)
        oa, op = osched.alg2(case["u"], case["b"], norms, 0.1, 0.1)
        assert a == oa and p == op == case["perturbed"]       # bit-identical doubles


@settings(max_examples=150, deadline=None)
@given(st.integers(1, 8), st.data())
def test_alg2_bit_exact_vs_oracle(N, data):
    u = [data.draw(st.integers(0, 30)) for _ in range(N)]
    if sum(u) == 0:
        u[0] = 1
    b = [data.draw(st.integers(1, 2048)) for _ in range(N)]
    norms = [data.draw(st.floats(0.0, 0.2)) for _ in range(N)]
    delta = data.draw(st.floats(0.0, 0.5))
    thr = data.draw(st.floats(0.0, 0.2))
    assert psched.alg2(u, b, norms, delta, thr) == tuple(osched.alg2(u, b, norms, delta, thr))


@pytest.mark.parametrize("n,seed", [(1, 0), (7, 3), (1000, 0x211007029), (4096, 12345678901234)])
def test_permutation_bit_exact_vs_oracle(n, seed):
    assert psched.permutation(n, seed).tolist() == osched.permutation(n, seed)


def _cfg(**kw):
    c = L.Config()
    base = dict(n_features=1000, n_labels=100, hidden=128, b_max=64, b_min=8, beta=4, megabatch=6400,
                max_row_nnz=32, max_row_labels=8, lr0=0.1, gamma=0.9, delta=0.1, pert_thr=0.1,
                precision=L.AS_BF16, flags=0, rank=0, world=1, device=0)
    base.update(kw)
    for k, v in base.items():
        setattr(c, k, v)
    return c


def test_workspace_size_and_validation():
    lib = L.load()
    n = C.c_size_t()
    assert lib.as_workspace_size(C.byref(_cfg()), C.byref(n)) == L.AS_OK and n.value > 0
    n32 = C.c_size_t()
    assert lib.as_workspace_size(C.byref(_cfg(precision=L.AS_FP32)), C.byref(n32)) == L.AS_OK
    for bad in [dict(hidden=64), dict(b_min=128), dict(world=2, rank=2), dict(precision=7),
                dict(lr0=0.0), dict(n_labels=0), dict(max_row_nnz=0)]:
        assert lib.as_workspace_size(C.byref(_cfg(**bad)), C.byref(n)) == L.AS_E_INVALID, bad
        assert lib.as_last_error()
    assert lib.as_sched_alg1(0, None, None, 1, 1, 1, 0.1, None, None) == L.AS_E_INVALID
    # init with a too-small workspace fails before touching the device
    c = _cfg()
    c.workspace, c.workspace_bytes = 256, 16
    ctx = C.c_void_p()
    p = np.zeros(10, np.float32)
    assert lib.as_init(C.byref(c), L.ptr(p, C.c_float), C.byref(ctx)) == L.AS_E_OOM


def test_live_cursor_conserves_samples():
    name = "/adasgd_test_%d" % os.getpid()
    cur = psched.LiveCursor(name, create=True)
    try:
        M, got = 1000, []
        for k in range(40):
            s, r = cur.claim(M, [64, 48, 40][k % 3])
            if r == 0:
                break
            got.extend(range(s, s + r))
        assert got == list(range(M))
        cur.reset()
        assert cur.claim(M, 10) == (0, 10)
    finally:
        cur.close()


def test_scale_period_golden_cpp():
    from paper_2110_07029_b200 import sched as psched
    with open(os.path.join(os.path.dirname(__file__), "golden", "scale_period_cases.json")) as f:
        cases = json.load(f)["cases"]
    for case in cases:
        p, d = psched.scale_period(case["b_prev"], case["b_next"], case["dir"], case["period"], case["p_max"])
        assert (p, d) == (case["period_out"], case["dir_out"]), case["why"]


@settings(max_examples=200, deadline=None)
@given(st.integers(1, 6), st.data())
def test_scale_period_bit_exact_vs_oracle(N, data):
    from paper_2110_07029_b200 import sched as psched
    bp = [data.draw(st.integers(8, 64)) for _ in range(N)]
    bn = [x + data.draw(st.integers(-3, 3)) for x in bp]
    dirs = [data.draw(st.integers(-1, 1)) for _ in range(N)]
    p_max = data.draw(st.integers(1, 16))
    period = data.draw(st.integers(1, p_max))
    assert psched.scale_period(bp, bn, dirs, period, p_max) == osched.scale_period(bp, bn, dirs, period, p_max)


def test_scale_period_validation_no_state_change():
    lib = L.load()
    b = np.array([8, 8], np.int32)
    d = np.array([1, -1], np.int32)
    out = C.c_int32(77)
    for period, p_max in ((0, 4), (5, 4), (1, 0)):
        assert lib.as_sched_scale_period(2, L.ptr(b, C.c_int32), L.ptr(b, C.c_int32), L.ptr(d, C.c_int32),
                                         period, p_max, C.byref(out)) == L.AS_E_INVALID
    assert d.tolist() == [1, -1] and out.value == 77


def test_replay_state_scaling_period_vs_oracle():
    """driver.ReplayState with scale_pmax (host logic through the C-ABI) follows
    the oracle's mega-batch loop (oracle/train.py, R27) on a scripted u
    sequence: converging, oscillating, then stable."""
    from paper_2110_07029_b200 import driver
    us = [[6, 2], [5, 3], [3, 5], [5, 3], [3, 5], [4, 4], [4, 4], [4, 4], [6, 2], [4, 4]]
    st_ = driver.ReplayState(2, 64, 8, 4, 0.1, [(0, 1, 0, 1, 1)] * 2, scale_pmax=4)
    b, lr, period, since, dirs = [64, 64], None, 1, 0, [0, 0]
    for u in us:
        used = st_.rescale(u)
        assert used == b
        since += 1
        if since >= period:
            nb, lr = osched.alg1(u, b, 4, 8, 64, 0.1)
            period, dirs = osched.scale_period(b, nb, dirs, period, 4)
            b, since = nb, 0
        assert (st_.b, st_.period) == (b, period)


def test_binding_constants_match_header():
    """The ctypes binding's enum values are the header's (include/adasgd.h is the
    contract; the binding only marshals)."""
    import re
    from paper_2110_07029_b200 import _lib as L
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                            "adasgd.h")).read()
    vals = {m.group(1): int(m.group(2)) for m in re.finditer(r"\b(AS_[A-Z0-9_]+)\s*=\s*(-?\d+)", hdr)}
    for name in ("AS_FLAG_DEBUG_GRADS", "AS_FLAG_NORM_UB", "AS_NORM_METRIC_SHIFT", "AS_FLAG_R14_LITERAL",
                 "AS_NORM_UPDATES", "AS_NORM_UB", "AS_NORM_R14_LITERAL"):
        assert name in vals, name
        assert getattr(L, name) == vals[name], name
    # the R14 flag does not collide with the metric bits (flags |= metric << 2)
    assert vals["AS_FLAG_R14_LITERAL"] & (3 << vals["AS_NORM_METRIC_SHIFT"]) == 0


def test_alg1_dynamics_two_replicas_hetero():
    """Replay routing + Alg. 1 over mega-batches (the C++ scheduler through
    driver.ReplayState) for two replicas, one 32% slower, at b_max = 1024:
    with the paper's beta = b_min / 2 = 64 the first correction overshoots and the
    literal bound check (R11) then refuses every step, leaving the batch sizes
    inverted; beta = 16 settles at equal update counts (DESIGN, R11)."""
    from paper_2110_07029_b200 import driver
    costs = synthgen.make_cost_models(2, hetero=True)
    n = 400_000
    rp = np.arange(n + 1, dtype=np.int64) * 41

    def run(beta, k):
        st = driver.ReplayState(2, 1024, 128, beta, 0.1, costs)
        pos, out = 0, []
        for _ in range(k):
            _, u, _ = st.route(rp, n, pos, 102_400)
            out.append((list(st.b), list(u)))
            st.rescale(u)
            pos += 102_400
        return out

    hi = run(64, 5)
    assert hi[0] == ([1024, 1024], [56, 44])
    assert hi[2:] == [([640, 1024], [90, 44])] * 3
    lo = run(16, 8)
    assert lo[-1][1][0] == lo[-1][1][1] and lo[-1][0][0] == 1024 and lo[-1][0][1] < 1024
