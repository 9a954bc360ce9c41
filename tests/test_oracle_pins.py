"""Pins for the CPU oracle (oracle/messi_oracle.c) against things other than itself:
textbook constants, independent library routines (scipy.special.ndtri / ndtr,
statistics.NormalDist, numpy.searchsorted, scipy.ndimage filters, numpy argmin),
paper invariants (Property 1; the LB_Keogh chain) and brute
force over all warping paths on tiny inputs.  CPU only (no gpu marker).
"""
import itertools
import json
import math
import os
from statistics import NormalDist

import numpy as np
import pytest
import scipy.ndimage as ndi
import scipy.special as sps

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_pins.json")))


def zwalks(rows, n, seed):
    """z-normalised random walks -- numpy, test-local."""
    rng = np.random.default_rng(seed)
    x = np.cumsum(rng.standard_normal((rows, n)), axis=1)
    x = (x - x.mean(1, keepdims=True)) / x.std(1, keepdims=True)
    return x.astype(np.float32)


# ------------------------------------------------------------------ breakpoints (O3)
def test_breakpoints_match_independent_quantile_routines():
    b64, b32 = oracle.breakpoints(256)
    k = np.arange(1, 256)
    ref = sps.ndtri(k / 256.0)
    assert np.allclose(b64, ref, rtol=4e-15, atol=1e-15)
    nd = NormalDist()
    ref2 = np.array([nd.inv_cdf(kk / 256.0) for kk in k])
    assert np.allclose(b64, ref2, rtol=4e-15, atol=1e-15)
    # the fp32 table the symbols use is the correctly rounded float of the quantile
    assert np.array_equal(b32, ref.astype(np.float32))
    assert np.all(np.diff(b64) > 0)


def test_breakpoints_closed_forms():
    b64, _ = oracle.breakpoints(256)
    q = GOLD["quartile_beta"]["value"]
    assert b64[127] == 0.0  # beta_128 = median
    assert abs(b64[191] - q) <= 2e-16 and abs(b64[63] + q) <= 2e-16
    assert np.allclose(b64[::-1], -b64, rtol=0, atol=1e-15)  # symmetry beta_{256-k} = -beta_k
    assert oracle.breakpoints(2)[0].tolist() == GOLD["card2_breakpoints"]["value"]
    assert np.allclose(oracle.breakpoints(4)[0], GOLD["card4_breakpoints"]["value"], atol=1e-4)
    for card in (2, 4, 8, 16, 32, 64, 128, 256):
        bb, _ = oracle.breakpoints(card)
        edges = np.concatenate([[-np.inf], bb, [np.inf]])
        probs = np.diff(sps.ndtr(edges))
        assert np.allclose(probs, 1.0 / card, atol=1e-14)  # equiprobable regions
    with pytest.raises(ValueError):
        oracle.breakpoints(3)


# ----------------------------------------------------------------------- symbols (O4)
def test_symbol_cases_and_prefix_property():
    _, b32 = oracle.breakpoints(256)
    for v, s in GOLD["symbols"]["cases"]:
        assert oracle.symbol(v, b32) == s
    # value exactly on a breakpoint goes to the region above; just below -> region below
    assert oracle.symbol(b32[191], b32) == 192
    assert oracle.symbol(np.nextafter(b32[191], np.float32(-np.inf)), b32) == 191
    _, b4 = oracle.breakpoints(4)
    assert oracle.symbol(0.2, b4, 4) == GOLD["symbols"]["card4_of_0.2"]
    assert oracle.symbol(-5.0, b4, 4) == 0 and oracle.symbol(5.0, b4, 4) == 3
    rng = np.random.default_rng(3)
    xs = np.concatenate([rng.standard_normal(4000), b32, np.nextafter(b32, -np.inf)]).astype(np.float32)
    tables = {c: oracle.breakpoints(c)[1] for c in (2, 4, 16, 256)}
    for x in xs:
        s256 = oracle.symbol(x, b32)
        # independent library routine: count of breakpoints <= x
        assert s256 == int(np.searchsorted(b32, x, side="right"))
        for c, tb in tables.items():
            # prefix soundness: the card-c symbol is the bit prefix of the 8-bit one
            assert oracle.symbol(x, tb, c) == s256 >> (8 - int(math.log2(c)))


# --------------------------------------------------------------------------- PAA (O2)
def test_paa_examples():
    g = GOLD["paa_spec"]
    assert oracle.paa32(g["x"], g["w"]).tolist() == g["paa"]
    assert np.all(oracle.paa32(np.full(64, 0.375, np.float32), 16) == np.float32(0.375))
    g = GOLD["worked_isax"]
    p, s = oracle.isax(g["x"], g["w"])
    assert p.tolist() == g["paa"]
    assert s.tolist() == g["sym256"]
    # the symbols agree with floor(256 * Phi(paa)) from a normal table
    assert [int(256 * v) for v in g["phi_of_paa"]] == g["sym256"]
    assert (s >> 6).tolist() == g["card4_word"]
    with pytest.raises(ValueError):
        oracle.paa32(np.zeros(10, np.float32), 3)  # n % w != 0 rejected
    with pytest.raises(ValueError):
        oracle.paa32(np.zeros(4, np.float32), 8)  # w > n rejected


def test_paa_matches_numpy_mean():
    X = zwalks(200, 256, 7)
    for x in X:
        ref = x.astype(np.float64).reshape(16, 16).mean(1)
        assert np.allclose(oracle.paa64(x, 16), ref, rtol=1e-14, atol=1e-15)
        assert np.allclose(oracle.paa32(x, 16), ref.astype(np.float32), rtol=1e-6, atol=1e-7)


# ----------------------------------------------------------------------- mindist (O6)
def test_mindist_closed_form_and_zero_on_own_box():
    g = GOLD["mindist_closed_form"]
    rng = np.random.default_rng(5)
    x = zwalks(1, 256, 11)[0]
    qpaa = oracle.paa64(x, 16)
    _, sym = oracle.isax(x, 16)
    # a series' PAA lies inside its own boxes (up to the fp32 rounding of the PAA)
    assert oracle.mindist2(oracle.paa32(x, 16).astype(np.float64), sym, 256) == 0.0
    # closed form: query PAA 0 vs symbol 192 in segment 0, own boxes elsewhere
    sym2 = sym.copy()
    sym2[0] = g["sym_in_seg0"]
    q2 = oracle.paa32(x, 16).astype(np.float64)
    q2[0] = g["qpaa_seg0"]
    got = oracle.mindist2(q2, sym2, 256)
    # box edges are the fp32-rounded breakpoints (reading R5): 16 * fl32(z_0.75)^2 exactly
    edge = float(np.float32(GOLD["quartile_beta"]["value"]))
    assert math.isclose(got, 16.0 * edge * edge, rel_tol=1e-15)
    assert math.isclose(got, g["value"], rel_tol=2e-7)  # the real-valued closed form
    # worked example: zero query vs the worked iSAX word, m = 2: lower edges from a normal table
    nd = NormalDist()
    gw = GOLD["worked_isax"]
    exp = 2 * (nd.inv_cdf(41 / 256) ** 2 + nd.inv_cdf(177 / 256) ** 2 + nd.inv_cdf(238 / 256) ** 2)
    got = oracle.mindist2(np.zeros(4), np.array(gw["sym256"], np.uint8), 8)
    assert math.isclose(got, exp, rel_tol=1e-6)
    assert got <= oracle.ed2(gw["x"], np.zeros(8, np.float32))


def test_property1_lower_bound():
    """Property 1: mindist(PAA(q), iSAX(c)) <= ED^2(q, c), 10k pairs."""
    X = zwalks(100, 256, 1)
    Q = zwalks(100, 256, 2)
    P, S = oracle.isax_rows(X)
    for q in Q:
        qp = oracle.paa64(q, 16)
        d = oracle.ed2_rows(X, q)
        for k in range(X.shape[0]):
            assert oracle.mindist2(qp, S[k], 256) <= d[k]


# ------------------------------------------------------------------------------- ED (O7)
def test_ed_examples_and_library():
    g = GOLD["ed_spec"]
    assert oracle.ed2(g["a"], g["b"]) == g["ed2"]
    X = zwalks(50, 256, 4)
    assert oracle.ed2(X[0], X[0]) == 0.0
    for a, b in zip(X[:-1], X[1:]):
        ref = float(np.sum((a.astype(np.float64) - b.astype(np.float64)) ** 2))
        assert math.isclose(oracle.ed2(a, b), ref, rel_tol=1e-13)
        assert oracle.ed2(a, b) == oracle.ed2(b, a)


# ---------------------------------------------------------------- envelope / LB_Keogh
def test_envelope_examples_and_library():
    g = GOLD["envelope_spec"]
    U, L = oracle.envelope(g["q"], g["r"])
    assert U.tolist() == g["U"] and L.tolist() == g["L"]
    q = zwalks(1, 256, 9)[0]
    U0, L0 = oracle.envelope(q, 0)
    assert np.array_equal(U0, q) and np.array_equal(L0, q)
    for r in (1, 5, 25, 255, 256):
        U, L = oracle.envelope(q, r)
        assert np.array_equal(U, ndi.maximum_filter1d(q, 2 * r + 1, mode="nearest"))
        assert np.array_equal(L, ndi.minimum_filter1d(q, 2 * r + 1, mode="nearest"))
        assert np.all(L <= q) and np.all(q <= U)
    with pytest.raises(ValueError):
        oracle.envelope(q, 257)


def test_lb_keogh_hand_and_r0():
    g = GOLD["lb_keogh_hand"]
    U, L = oracle.envelope(g["q"], g["r"])
    assert oracle.lb_keogh2(U, L, g["c"]) == g["lbk2"]
    assert oracle.ed2(g["q"], g["c"]) == g["ed2"]
    assert oracle.dtw2(g["q"], g["c"], g["r"]) == g["dtw2"]
    X = zwalks(20, 256, 12)
    for a, b in zip(X[:-1], X[1:]):
        U, L = oracle.envelope(a, 0)
        assert oracle.lb_keogh2(U, L, b) == oracle.ed2(a, b)  # r = 0: LB_Keogh == ED^2
        U, L = oracle.envelope(a, 25)
        assert oracle.lb_keogh2(U, L, a) == 0.0  # a series lies inside its own envelope


# ------------------------------------------------------------------------------ DTW (O12)
def brute_dtw(q, c, r):
    """min over every warping path inside the band of the summed squared cost."""
    n = len(q)
    best = math.inf

    def walk(i, j, acc):
        nonlocal best
        acc += (float(q[i]) - float(c[j])) ** 2
        if acc >= best:
            return
        if i == n - 1 and j == n - 1:
            best = acc
            return
        for di, dj in ((1, 1), (1, 0), (0, 1)):
            a, b = i + di, j + dj
            if a < n and b < n and abs(a - b) <= r:
                walk(a, b, acc)

    walk(0, 0, 0.0)
    return best


def test_dtw_hand_values():
    g = GOLD["dtw_hand"]
    assert oracle.dtw2(g["q"], g["c"], 0) == g["r0"]
    assert oracle.dtw2(g["q"], g["c"], 1) == g["r1"]


def test_dtw_brute_force_tiny():
    rng = np.random.default_rng(21)
    for trial in range(60):
        n = int(rng.integers(1, 8))
        q = rng.standard_normal(n).astype(np.float32)
        c = rng.standard_normal(n).astype(np.float32)
        for r in range(0, n + 1):
            assert math.isclose(oracle.dtw2(q, c, r), brute_dtw(q, c, r), rel_tol=1e-12, abs_tol=1e-12)


def test_dtw_invariants():
    X = zwalks(30, 256, 13)
    for a, b in zip(X[:-1], X[1:]):
        e = oracle.ed2(a, b)
        assert oracle.dtw2(a, b, 0) == e  # r = 0 is the diagonal: bit-identical to ED^2
        prev = e
        for r in (1, 2, 5, 12, 25, 51, 128, 255):
            d = oracle.dtw2(a, b, r)
            assert d <= prev  # monotone non-increasing in the reach
            prev = d
        assert oracle.dtw2(a, b, 255) == oracle.dtw2(a, b, 256)
        assert math.isclose(oracle.dtw2(a, b, 25), oracle.dtw2(b, a, 25), rel_tol=1e-12)
        assert oracle.dtw2(a, a, 25) == 0.0


def test_lower_bound_chain_dtw():
    """LB_envPAA <= LB_Keogh <= DTW <= ED^2 (Alg. 10), r = 25, 2,500 pairs."""
    X = zwalks(50, 256, 14)
    Q = zwalks(50, 256, 15)
    _, S = oracle.isax_rows(X)
    for q in Q:
        U, L = oracle.envelope(q, 25)
        Up, Lp = oracle.paa64(U, 16), oracle.paa64(L, 16)
        for k in range(X.shape[0]):
            lbp = oracle.lb_env_paa2(Up, Lp, S[k], 256)
            lbk = oracle.lb_keogh2(U, L, X[k])
            d = oracle.dtw2(q, X[k], 25)
            assert lbp <= lbk <= d <= oracle.ed2(q, X[k])
    # r = 0: the envelope PAA bound equals the ED mindist
    q = Q[0]
    U, L = oracle.envelope(q, 0)
    Up, Lp = oracle.paa64(U, 16), oracle.paa64(L, 16)
    qp = oracle.paa64(q, 16)
    for k in range(X.shape[0]):
        assert oracle.lb_env_paa2(Up, Lp, S[k], 256) == oracle.mindist2(qp, S[k], 256)


def test_lb_keogh_reverse_lower_bounds_dtw():
    """LB_Keogh with the roles swapped -- the query's points against the CANDIDATE's envelope
    -- lower-bounds DTW too (the argument of P:1392-1405 is symmetric in the two series: every
    query point lies on the warping path, matched to a candidate point within the reach; the
    DTW refine's reverse filter): against brute force over every warping path on
    tiny inputs, and on 2,500 random-walk pairs at r = 25, where it is often the larger bound."""
    rng = np.random.default_rng(31)
    for trial in range(60):
        n = int(rng.integers(1, 8))
        q = rng.standard_normal(n).astype(np.float32)
        c = rng.standard_normal(n).astype(np.float32)
        for r in range(0, n + 1):
            Uc, Lc = oracle.envelope(c, r)
            assert oracle.lb_keogh2(Uc, Lc, q) <= brute_dtw(q, c, r) * (1 + 1e-12) + 1e-12
    X = zwalks(50, 256, 14)
    Q = zwalks(50, 256, 15)
    larger = 0
    for q in Q:
        U, L = oracle.envelope(q, 25)
        for k in range(X.shape[0]):
            Uc, Lc = oracle.envelope(X[k], 25)
            fwd = oracle.lb_keogh2(U, L, X[k])
            rev = oracle.lb_keogh2(Uc, Lc, q)
            assert rev <= oracle.dtw2(q, X[k], 25)
            larger += rev > fwd
    assert 0 < larger < 2500


def test_lb_env_paa_hand_value_reach1():
    """O11 at r > 0 on a worked example (Fig. fig:dtwsimd's ABOVE / BELOW / IN cases
    P:1471-1486), cardinality 4 (breakpoints -b, 0, b with b = Phi^-1(3/4), fp32):
      q = [0, 1, 0, 0, 2, 0, -1, 0], r = 1 -> U = [1,1,1,2,2,2,0,0], L = [0,0,0,0,0,-1,-1,-1]
      PAA (w = 4, m = 2): Ubar = [1, 1.5, 2, 0], Lbar = [0, 0, -0.5, -1]
      symbols [0, 3, 0, 3]: seg 0 BELOW (Lbar - hi(0) = 0 + b), seg 1 IN, seg 2 BELOW
      (-0.5 + b), seg 3 ABOVE (lo(3) - Ubar = b)
      LB = m ((b)^2 + (b - 0.5)^2 + (b)^2) with b = 0.6744897365570068 (fp32 of 0.67448975...)
         = 1.8806389552104292 (evaluated by hand to the last digit in fp64).
    The series c = [-1,-1, 1,1, -1,-1, 1,1] has exactly those symbols and LB_Keogh 5 (points
    0, 1, 4 below L by 1; points 6, 7 above U by 1), so the chain LB <= LB_Keogh <= DTW holds."""
    q = np.array([0, 1, 0, 0, 2, 0, -1, 0], np.float32)
    U, L = oracle.envelope(q, 1)
    assert U.tolist() == [1, 1, 1, 2, 2, 2, 0, 0] and L.tolist() == [0, 0, 0, 0, 0, -1, -1, -1]
    Up, Lp = oracle.paa64(U, 4), oracle.paa64(L, 4)
    assert Up.tolist() == [1.0, 1.5, 2.0, 0.0] and Lp.tolist() == [0.0, 0.0, -0.5, -1.0]
    c = np.array([-1, -1, 1, 1, -1, -1, 1, 1], np.float32)
    _, sym = oracle.isax(c, 4, 4)
    assert sym.tolist() == [0, 3, 0, 3]
    lb = oracle.lb_env_paa2(Up, Lp, sym, 8, card=4)
    assert lb == 1.8806389552104292
    assert oracle.lb_keogh2(U, L, c) == 5.0
    assert lb <= 5.0 <= oracle.dtw2(q, c, 1)
    # flipping any one case changes the value: all three cases are exercised
    assert oracle.lb_env_paa2(Up, Lp, np.array([3, 3, 0, 3], np.uint8), 8, card=4) < lb
    assert oracle.lb_env_paa2(Up, Lp, np.array([0, 3, 3, 3], np.uint8), 8, card=4) < lb
    assert oracle.lb_env_paa2(Up, Lp, np.array([0, 3, 0, 0], np.uint8), 8, card=4) < lb


def test_lb_rev_paa_hand_value_reach1():
    """O11b on a worked example (reading R19: LB_Keogh with the series' roles
    swapped, reduced by PAA as P:1411), cardinality 4 (breakpoints -b, 0, b,
    b = fp32(Phi^-1(3/4)) = 0.6744897365570068):
      candidate x = [0, 1, 0, 0, 2, 0, -1, 0], r = 1 -> U^x = [1,1,1,2,2,2,0,0],
      L^x = [0,0,0,0,0,-1,-1,-1]; w = 4 (m = 2): Ubar = [1, 1.5, 2, 0], Lbar = [0, 0, -0.5, -1]
      usym = [3, 3, 3, 2] (hi = +inf, +inf, +inf, b), lsym = [2, 2, 1, 0] (lo = 0, 0, -b, -inf)
      query q = [-1,-1, 1,1, -1,-1, 1,1], qbar = [-1, 1, -1, 1]:
      seg 0 below lo = 0 by 1; seg 1 inside; seg 2 below lo = -b by 1 - b; seg 3 above hi = b
      by 1 - b  ->  LB = m (1 + 0 + (1 - b)^2 + (1 - b)^2) = 2.4238277264269072 (fp64, summed in
      segment order).
    The reverse LB_Keogh of the pair is 5 (points 0, 1, 4 below L^x by 1; 6, 7 above U^x by
    1), so LB <= reverse LB_Keogh <= DTW."""
    x = np.array([0, 1, 0, 0, 2, 0, -1, 0], np.float32)
    q = np.array([-1, -1, 1, 1, -1, -1, 1, 1], np.float32)
    u, l = oracle.renv_sym(x, 1, 4, 4)
    assert u.tolist() == [3, 3, 3, 2] and l.tolist() == [2, 2, 1, 0]
    qp = oracle.paa64(q, 4)
    assert qp.tolist() == [-1.0, 1.0, -1.0, 1.0]
    lb = oracle.lb_rev_paa2(qp, u, l, 8, card=4)
    assert lb == 2.4238277264269072
    Ux, Lx = oracle.envelope(x, 1)
    assert oracle.lb_keogh2(Ux, Lx, q) == 5.0
    assert lb <= 5.0 <= oracle.dtw2(q, x, 1)
    # each case is live: moving one box so the query mean falls inside lowers the value
    assert oracle.lb_rev_paa2(qp, np.array([3, 3, 3, 3], np.uint8), l, 8, card=4) < lb
    assert oracle.lb_rev_paa2(qp, u, np.array([0, 2, 1, 0], np.uint8), 8, card=4) < lb
    assert oracle.lb_rev_paa2(qp, u, np.array([2, 2, 0, 0], np.uint8), 8, card=4) < lb


def test_lb_rev_paa_chain_and_r0_identity():
    """O11b lower-bounds the reverse LB_Keogh (hence DTW) on random walks at several reaches;
    at r = 0 (envelope = the series) it equals O6's mindist of the series' own symbols
    wherever O4's fp32-PAA symbols agree with O11b's fp64-mean symbols."""
    X = zwalks(60, 128, 41)
    Q = zwalks(6, 128, 42)
    tight = 0
    for r in (1, 5, 12):
        for q in Q:
            qp = oracle.paa64(q, 16)
            for x in X:
                u, l = oracle.renv_sym(x, r, 16)
                lb = oracle.lb_rev_paa2(qp, u, l, 128)
                Ux, Lx = oracle.envelope(x, r)
                rev = oracle.lb_keogh2(Ux, Lx, q)
                assert lb <= rev * (1 + 1e-12) + 1e-12
                assert rev <= oracle.dtw2(q, x, r) * (1 + 1e-12)
                tight += lb > 0.25 * rev
    assert tight > 0.1 * 3 * 6 * 60  # not a vacuous bound
    agree = 0
    for q in Q:
        qp = oracle.paa64(q, 16)
        for x in X:
            u, l = oracle.renv_sym(x, 0, 16)
            assert u.tolist() == l.tolist()
            _, sym = oracle.isax(x, 16)
            if sym.tolist() == u.tolist():
                agree += 1
                assert oracle.lb_rev_paa2(qp, u, l, 128) == oracle.mindist2(qp, sym, 128)
    assert agree >= 0.9 * len(Q) * len(X)


# ------------------------------------------------------------------------- 1-NN (O8/O13)
def test_nn_ed_vs_numpy_scan_and_threads():
    X = zwalks(3000, 256, 31)
    Q = zwalks(8, 256, 32)
    d2, ids = oracle.nn("ed", X, Q, threads=1, chunk=1 << 20)
    d2b, idsb = oracle.nn("ed", X, Q, threads=8, chunk=257)
    assert np.array_equal(ids, idsb) and np.array_equal(d2, d2b)
    D = ((X[None, :, :].astype(np.float64) - Q[:, None, :].astype(np.float64)) ** 2).sum(-1)
    assert np.array_equal(ids, D.argmin(1))
    assert np.allclose(d2, D.min(1), rtol=1e-13)


def test_nn_ties_lowest_id_and_exact_match():
    X = zwalks(500, 64, 33)
    X[400] = X[17]
    X[450] = X[17]
    d2, ids = oracle.nn("ed", X, X[[17, 400, 3]], threads=4, chunk=64)
    assert ids.tolist() == [17, 17, 3] and d2.tolist() == [0.0, 0.0, 0.0]
    d2, ids = oracle.nn("dtw", X, X[[450]], r=6, threads=4, chunk=64)
    assert ids.tolist() == [17] and d2.tolist() == [0.0]
    d2, ids = oracle.nn("ed", X, X[[17]], row_begin=1000, threads=2, chunk=100)
    assert ids.tolist() == [1017]


def test_nn_dtw_vs_brute_paths_tiny():
    rng = np.random.default_rng(41)
    X = rng.standard_normal((40, 6)).astype(np.float32)
    Q = rng.standard_normal((3, 6)).astype(np.float32)
    for r in (0, 1, 2, 5):
        d2, ids = oracle.nn("dtw", X, Q, r=r, threads=3, chunk=7)
        for qi, q in enumerate(Q):
            ref = [brute_dtw(q, x, r) for x in X]
            assert ids[qi] == int(np.argmin(ref))
            assert math.isclose(d2[qi], min(ref), rel_tol=1e-12, abs_tol=1e-12)


def test_knn_oracle_definition():
    """oracle.knn against an independent numpy fp64 brute force (k smallest of the sum of
    squares, ties to the lowest id), k = 1 against oracle.nn, and k > N padding."""
    rng = np.random.default_rng(11)
    X = rng.standard_normal((300, 24)).astype(np.float32)
    X[250] = X[17]
    Q = np.concatenate([X[[17]], rng.standard_normal((4, 24)).astype(np.float32)])
    d2, ids = oracle.knn("ed", X, Q, 9)
    for qi in range(Q.shape[0]):
        ref = ((X.astype(np.float64) - Q[qi].astype(np.float64)) ** 2).sum(axis=1)
        order = sorted(range(X.shape[0]), key=lambda i: (ref[i], i))[:9]
        assert list(ids[qi]) == order
        assert np.allclose(d2[qi], ref[order], rtol=1e-12, atol=0)
    assert list(ids[0, :2]) == [17, 250] and d2[0, 0] == 0.0 and d2[0, 1] == 0.0
    n1d, n1i = oracle.nn("ed", X, Q)
    k1d, k1i = oracle.knn("ed", X, Q, 1)
    assert np.array_equal(k1i[:, 0], n1i) and np.array_equal(k1d[:, 0], n1d)
    pd, pi = oracle.knn("ed", X[:3], Q[:1], 5)
    assert list(pi[0, 3:]) == [-1, -1] and np.all(np.isinf(pd[0, 3:]))
