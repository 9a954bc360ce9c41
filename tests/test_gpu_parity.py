"""Parity of the CUDA path (through the C-ABI) with the CPU oracle, element by element on
the same seeded inputs (device-generated rows copied back to the host for the oracle).

Bars:
  * symbols, PAA, breakpoints: bit-exact (integer / byte work and a fixed fp64 op order);
  * nearest-neighbour id: bit-exact, ties -> lowest id; d2 bit-exact (canonical fp64
    re-rank); dist within 1e-12 relative (it is sqrt(d2) on both sides);
  * fp32 per-row quantities (refine distances, LB_Keogh): 2^-16 relative of the oracle;
  * lower bounds: GPU LB <= true distance always (Property 1), and within
    the widened-box / round-down tolerance of the oracle's mindist (derived in the test).
"""
import math

import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def messi():
    from paper_2110_07519_b200 import messi as m
    return m


def gen_rows(N, n, seed=datagen.DATA_SEED, row_begin=0):
    x = torch.empty((N, n), dtype=torch.float32, device=DEV)
    if N:
        datagen.walks_cuda(x, row_begin, seed=seed)
    torch.cuda.synchronize()
    return x


@pytest.fixture(scope="module")
def c1():
    """Config 1: 100,000 x 256 random walks (seed 0), 10 queries (seed 1); 195.3 tiles."""
    X = gen_rows(100_000, 256)
    Q = gen_rows(10, 256, seed=datagen.QUERY_SEED)
    idx = messi().Index(X, keep_paa=True)
    yield X, Q, idx, X.cpu().numpy(), Q.cpu().numpy()
    idx.close()


# ------------------------------------------------------------------------ build (A1/A2)
def test_breakpoints_bit_exact():
    b = messi().messi_debug_breakpoints(0)
    assert np.array_equal(b, oracle.breakpoints(256)[1])


def test_summaries_bit_exact(c1):
    X, Q, idx, Xh, Qh = c1
    sym, paa = messi().messi_debug_summaries(idx.handle, X.shape[0], X.device, with_paa=True)
    P, S = oracle.isax_rows(Xh)
    assert np.array_equal(paa.cpu().numpy().view(np.uint32), P.view(np.uint32))
    assert np.array_equal(sym.cpu().numpy(), S)


def _interleave_key(S):
    key = np.zeros(S.shape[0], np.uint64)
    for bit in range(7, 3, -1):
        plane = np.zeros(S.shape[0], np.uint64)
        for s in range(16):
            plane |= ((S[:, s].astype(np.uint64) >> np.uint64(bit)) & np.uint64(1)) << np.uint64(s)
        key = (key << np.uint64(16)) | plane
    return key


def test_approximate_search_order_is_valid(c1):
    """The approximate-search order (reading R14, parity unpinned for the seed itself):
    keys sorted, perm a permutation, key(perm[i]) = bit-plane interleave of the symbols."""
    X, Q, idx, Xh, Qh = c1
    keys, perm = messi().messi_debug_order(idx.handle, X.shape[0], X.device)
    k = keys.cpu().numpy().view(np.uint64)
    p = perm.cpu().numpy().astype(np.int64)
    assert np.all(k[1:] >= k[:-1])
    assert np.array_equal(np.sort(p), np.arange(X.shape[0]))
    _, S = oracle.isax_rows(Xh)
    assert np.array_equal(k, _interleave_key(S)[p])


# ------------------------------------------------------------------ lower bounds (A3/A5)
# Every step-level check below reads the QUERY PATH'S OWN KERNELS (include/messi.h, inspection
# entry points): k_scan / fine_lb for the 8-bit bound, coarse_acc for the cardinality-16 one,
# k_filter_batch / box_lb for the ED tile boxes, k_tile_filter for the DTW ones, q8_bound_pass /
# ed2_group / ed2_exact_g for the ED refine, and the LB_Keogh filter + strip / band / warp
# refine kernels (frozen) for DTW.
U32 = 2.0 ** -24  # fp32 unit roundoff


def _lb_tol(d_seg, m):
    # GPU boxes are widened by one fp32 ulp (<= 4.8e-7 for |beta| < 4), table entries rounded
    # down to fp32 and summed rounding down: GPU <= oracle, and oracle - GPU <= m * sum_s
    # (2 d_s u + u^2) + 18 u * LB (16 roundings of the terms, 16 of the sum, the fp64 products)
    u = 4.8e-7
    return m * (2 * d_seg.sum(1) * u + 16 * u * u)


def _mindist_rows(qp, S, card=256):
    b32 = oracle.breakpoints(card)[1]
    return np.array([oracle.mindist2(qp, S[r], 256, card=card, beta32=b32) for r in range(S.shape[0])])


def test_lower_bounds_ed(c1):
    """The scan's 8-bit bound (k_scan: fine_lb over the fused ED kernel's own table) of EVERY C1
    row: GPU <= oracle mindist <= true ED^2 (Property 1), and oracle - GPU within
    the widened-box / round-down tolerance."""
    X, Q, idx, Xh, Qh = c1
    _, S = oracle.isax_rows(Xh)
    b32 = oracle.breakpoints()[1]
    lo = np.concatenate([[-np.inf], b32]).astype(np.float64)
    hi = np.concatenate([b32, [np.inf]]).astype(np.float64)
    for qi in range(2):
        lb = messi().messi_debug_lower_bounds(idx.handle, Q[qi].contiguous(), -1, X.shape[0]).cpu().numpy()
        assert not np.isnan(lb).any()  # every row came out of the scan kernel
        lb = lb.astype(np.float64)
        qp = oracle.paa64(Qh[qi])
        ref = _mindist_rows(qp, S)
        d_seg = np.maximum(0, np.maximum(lo[S] - qp, qp - hi[S]))
        tol = _lb_tol(d_seg, 16) + 18 * U32 * ref
        assert np.all(lb <= ref * (1 + 1e-12))
        assert np.all(ref - lb <= tol)
        assert np.all(ref <= oracle.ed2_rows(Xh, Qh[qi]))


@pytest.mark.parametrize("reach", [-1, 25])
def test_coarse_bounds(c1, reach):
    """The scan's coarse pass (cardinality 16 = the top 4 bits of every symbol):
    on every C1 row its bound never exceeds the 8-bit bound of the same row (the coarse box
    contains the fine one); ED: GPU <= the oracle's card-16 mindist <= true ED^2, within the
    widened-box / round-down tolerance."""
    X, Q, idx, Xh, Qh = c1
    N = X.shape[0]
    _, S = oracle.isax_rows(Xh)
    b16 = oracle.breakpoints(16)[1]
    for qi in range(2):
        q = Q[qi].contiguous()
        cb = messi().messi_debug_coarse_bounds(idx.handle, q, reach, N).cpu().numpy().astype(np.float64)
        fb = messi().messi_debug_lower_bounds(idx.handle, q, reach, N).cpu().numpy().astype(np.float64)
        assert not np.isnan(cb).any() and not np.isnan(fb).any()
        assert np.all(cb <= fb * (1 + 2.0 ** -20) + 1e-30)
        if reach < 0:
            qp = oracle.paa64(Qh[qi])
            ref = _mindist_rows(qp, S >> 4, card=16)
            lo = np.concatenate([[-np.inf], b16]).astype(np.float64)
            hi = np.concatenate([b16, [np.inf]]).astype(np.float64)
            d_seg = np.maximum(0, np.maximum(lo[S >> 4] - qp, qp - hi[S >> 4]))
            tol = _lb_tol(d_seg, 16) + 18 * U32 * ref
            assert np.all(cb <= ref * (1 + 1e-12))
            assert np.all(ref - cb <= tol)
            assert np.all(ref <= oracle.ed2_rows(Xh, Qh[qi]))
            # the coarse pass is a real filter: most rows fail it at the NN distance
            d2, _ = oracle.nn("ed", Xh[:20000], Qh[qi:qi + 1])
            assert np.mean(cb <= d2[0]) < 0.5


@pytest.mark.parametrize("reach", [-1, 25])
def test_tile_box_bounds(c1, reach):
    """The box of a tile (512 consecutive series in approximate-search order) bounds every
    member from below: tile LB <= each member's 8-bit bound <= its true distance (the node
    test of Alg. 7; Property 2).  ED: the batch filter kernel's
    fp32 zero-run bound (k_filter_batch), and every super-tile's bound <= its 16 tiles'; DTW:
    k_tile_filter."""
    X, Q, idx, Xh, Qh = c1
    N = X.shape[0]
    ntiles = (N + 511) // 512
    _, perm = messi().messi_debug_order(idx.handle, N, X.device)
    perm = perm.cpu().numpy().astype(np.int64)
    for qi in range(3):
        q = Q[qi].contiguous()
        tlb = messi().messi_debug_tile_bounds(idx.handle, q, reach, ntiles).cpu().numpy()
        assert not np.isnan(tlb).any()  # every tile listed by the filter kernel at threshold +inf
        flb = messi().messi_debug_lower_bounds(idx.handle, q, reach, N).cpu().numpy()
        member_min = np.full(ntiles, np.inf)
        np.minimum.at(member_min, np.arange(N) // 512, flb[perm])
        if reach < 0:
            assert np.all(tlb <= member_min * (1 + 16 * U32))  # fp32 sums rounded down, own orders
            ed = oracle.ed2_rows(Xh, Qh[qi])
            tmin = np.full(ntiles, np.inf)
            np.minimum.at(tmin, np.arange(N) // 512, ed[perm])
            assert np.all(tlb <= tmin)
            nsuper = (ntiles + 15) // 16
            slb = messi().messi_debug_super_bounds(idx.handle, q, nsuper).cpu().numpy()
            tpad = np.full(nsuper * 16, np.inf, np.float32)
            tpad[:ntiles] = tlb
            # the union box's exact bound is <= each tile's; both fp32 sums round down in their
            # own (lane-rotated) order, so compare within the 16 roundings of a sum
            assert np.all(slb <= tpad.reshape(nsuper, 16).min(axis=1) * (1 + 16 * U32))
            # the filter keeps a minority of tiles at the NN distance (pruning is real)
            d2, _ = oracle.nn("ed", Xh, Qh[qi:qi + 1])
            assert np.mean(tlb <= d2[0]) < 0.8
        else:
            assert np.all(tlb <= member_min * (1 + 1e-6) + 1e-6)  # fp64 bound rounded to nearest


def test_lower_bounds_dtw(c1):
    """The scan's envelope-PAA bound (k_scan over k_seed_dtw's table) of every C1 row:
    GPU <= the oracle's lb_env_paa2 (within rounding), and the chain LB <= LB_Keogh <= DTW."""
    X, Q, idx, Xh, Qh = c1
    _, S = oracle.isax_rows(Xh)
    r = 25
    for qi in range(2):
        lb = messi().messi_debug_lower_bounds(idx.handle, Q[qi].contiguous(), r, X.shape[0]).cpu().numpy()
        assert not np.isnan(lb).any()
        U, L = oracle.envelope(Qh[qi], r)
        Up, Lp = oracle.paa64(U), oracle.paa64(L)
        b32 = oracle.breakpoints(256)[1]
        ref = np.array([oracle.lb_env_paa2(Up, Lp, S[k], 256, beta32=b32) for k in range(S.shape[0])])
        assert np.all(lb <= ref * (1 + 1e-6) + 1e-9)
        assert np.all(lb >= ref * (1 - 1e-4) - 1e-3)
        lbk = np.array([oracle.lb_keogh2(U, L, Xh[k]) for k in range(0, S.shape[0], 50)])
        assert np.all(lb[::50] <= lbk)
        assert np.all(lbk <= oracle.dtw2_rows(Xh[::50], Qh[qi], r))


@pytest.mark.parametrize("r", [7, 25, 51])
def test_rev_paa_bounds_dtw(c1, r):
    """The DTW path's reverse envelope-PAA filter (k_renv + k_rev_paa_filter, the query path's
    own kernels, threshold +inf) on EVERY C1 row: GPU <= the oracle's lb_rev_paa2 (O11b) of the
    row's envelope symbols (safe: the kernel's symbols take rounded-up / -down means and its
    fp32 sums round down), GPU within 1e-4 of it on >= 99.9 % of the rows (tight), and the
    chain GPU <= reverse LB_Keogh <= DTW on a row sample."""
    X, Q, idx, Xh, Qh = c1
    Us, Ls = oracle.renv_sym_rows(Xh, r)
    for qi in range(2):
        lb = messi().messi_debug_rev_bounds(idx.handle, Q[qi].contiguous(), r, X.shape[0]).cpu().numpy()
        assert not np.isnan(lb).any()
        ref = oracle.lb_rev_paa2_rows(oracle.paa64(Qh[qi]), Us, Ls, Xh.shape[1])
        assert np.all(lb <= ref * (1 + 1e-9) + 1e-12)
        close = np.abs(lb - ref) <= 1e-4 * np.maximum(ref, 1.0)
        assert close.mean() >= 0.999, close.mean()
        assert (lb > 0).mean() > 0.5  # prunes something at all
        for k in range(0, Xh.shape[0], 997):
            Ux, Lx = oracle.envelope(Xh[k], r)
            rev = oracle.lb_keogh2(Ux, Lx, Qh[qi])
            assert lb[k] <= rev * (1 + 1e-9)
            assert rev <= oracle.dtw2(Qh[qi], Xh[k], r) * (1 + 1e-12)


# -------------------------------------------------------------- real distances (A7-A9)
def _quantise_like_rows(q):
    """The quantisation recipe of the rows, restated for one fp32 vector: s the
    smallest power of two with max|q| <= 127 s, c = rint(q / s)."""
    q = np.asarray(q, dtype=np.float32)
    mx = float(np.abs(q).max())
    if mx == 0.0:
        return 1.0, np.zeros(q.shape, np.int64)
    m, e = np.frexp(np.float32(mx))
    k = e - 7 if m * 128.0 <= 127.0 else e - 6
    s = float(np.ldexp(1.0, int(k)))
    return s, np.rint(q.astype(np.float64) / s).astype(np.int64)


def test_ed_refine_stages_every_row(c1):
    """The ED refine's own device code on EVERY C1 row (messi_debug_ed_refine):
      * q8i_bound_pass: dh2 is a lower bound of ||q^ - x^||^2 (query and row quantised with the
        same recipe; the sums are exact integers, so it is within 2^-40 of it), and its bound L
        never exceeds the true distance ||q - x|| (oracle ED; triangle inequality):
        the prune is safe; and L is tight (>= ||q^ - x^|| - e_x - ||q - q^|| up to the margins);
      * ed2_group (the exact pass): fp32 squared ED within (n/32 + 9) u relative of the
        oracle's (8 sequential fma per lane, a 5-level butterfly, the rounding of q - x);
      * ed2_exact_g (the re-rank): bit-identical to the oracle's fp64 ED^2."""
    X, Q, idx, Xh, Qh = c1
    N, n = X.shape
    q8, meta = messi().messi_debug_quantised(idx.handle, N, n, X.device)
    c = q8.cpu().numpy().view(np.int8).astype(np.float64)
    s = meta[:, 0].cpu().numpy().astype(np.float64)
    e = meta[:, 1].cpu().numpy().astype(np.float64)
    xq = s[:, None] * c
    ids = torch.arange(N, dtype=torch.int32, device=DEV)
    for qi in range(2):
        dh2, L, d32, d64 = messi().messi_debug_ed_refine(idx.handle, Q[qi].contiguous(), ids)
        dh2, L, d32, d64 = (t.cpu().numpy() for t in (dh2, L, d32, d64))
        sq, cq = _quantise_like_rows(Qh[qi])
        qhat = sq * cq.astype(np.float64)
        eq = np.sqrt(((Qh[qi].astype(np.float64) - qhat) ** 2).sum())
        ref_dh2 = ((xq - qhat) ** 2).sum(axis=1)
        assert np.all(dh2 <= ref_dh2 * (1 + 1e-15))
        assert np.all(dh2 >= ref_dh2 * (1 - 2.0 ** -40) - 1e-12)
        ed = oracle.ed2_rows(Xh, Qh[qi])
        assert np.all(L <= np.sqrt(ed))
        assert np.all(L >= np.sqrt(ref_dh2) * (1 - 2.0 ** -40) - e - eq * (1 + 2.0 ** -20) - 1e-9)
        assert np.all(np.abs(d32 - ed) <= (n // 32 + 9) * U32 * ed + 1e-30)
        assert np.array_equal(d64, ed)


REV_REACHES = (12, 25, 51)  # MESSI_REV_SPECS (refine.cuh) at n = 256


@pytest.mark.parametrize("reach,strip", [(0, None), (2, None), (5, None), (7, None), (12, None), (25, None),
                                         (51, None), (2, "0"), (5, "0")])
def test_dtw_stages_elementwise(c1, reach, strip, monkeypatch):
    """The DTW filter and refine KERNELS of the query path on 1,500 C1 rows (the ids handed
    to them as candidates, threshold +inf, refine frozen: no abandon):
      * LB_Keogh: at strip reaches (r >= 1 by default) the filter's LB_Keogh of the quantised row x^
        within fp32 summation error of its fp64 value, and (sqrt(LBK(x^)(1 - 2^-10)) - e)^2
        <= the oracle's raw LB_Keogh <= DTW; at other reaches the raw LB_Keogh within fp32
        error of the oracle's;
      * reverse LB_Keogh (r = 12, 25, 51: the query's points against the candidate's
        envelope): the filter's bound from the quantised row within rounding below its fp64
        value, <= the oracle's raw reverse LB_Keogh <= DTW (NaN, not computed, elsewhere);
      * refine (strip kernel r >= 1, register band r = 2, 5 under MESSI_DTW_STRIP=0, warp
        wavefront r = 0): fp32 DTW^2
        within (2n + 2) u relative of the oracle's fp64 DTW^2 (the error of a sum along one
        warping path of <= 2n - 1 cells)."""
    if strip is not None:  # "0": the register-band path (raw LB_Keogh filter, DtwThread<R>)
        monkeypatch.setenv("MESSI_DTW_STRIP", strip)
    X, Q, idx, Xh, Qh = c1
    N, n = X.shape
    rng = np.random.default_rng(100 + reach)
    ids_np = rng.choice(20_000, 1500, replace=False).astype(np.int32)
    ids = torch.from_numpy(ids_np).to(DEV)
    q = Q[2].contiguous()
    lbk, d32, quantised, lbr = messi().messi_debug_dtw_stages(idx.handle, q, reach, ids, rev=True)
    lbk, d32 = lbk.cpu().numpy().astype(np.float64), d32.cpu().numpy().astype(np.float64)
    lbr = lbr.cpu().numpy().astype(np.float64)
    assert not np.isnan(lbk).any() and not np.isnan(d32).any()
    assert quantised == (reach >= 1 and strip != "0")
    ref = oracle.dtw2_rows(Xh[ids_np], Qh[2], reach)
    assert np.all(np.abs(d32 - ref) <= (2 * n + 2) * U32 * ref + 1e-30)
    U, L = oracle.envelope(Qh[2], reach)
    raw = np.array([oracle.lb_keogh2(U, L, Xh[i]) for i in ids_np])
    assert np.all(raw <= ref * (1 + 1e-12))
    if quantised:
        q8, meta = messi().messi_debug_quantised(idx.handle, N, n, X.device)
        cq = q8[ids].cpu().numpy().view(np.int8).astype(np.float64)
        sc = meta[ids, 0].cpu().numpy().astype(np.float64)
        e = meta[ids, 1].cpu().numpy().astype(np.float64)
        xq = sc[:, None] * cq
        Ud, Ld = U.astype(np.float64), L.astype(np.float64)
        tq = (np.where(xq > Ud, xq - Ud, np.where(xq < Ld, xq - Ld, 0.0)) ** 2).sum(axis=1)
        assert np.all(np.abs(lbk - tq) <= (n + 4) * U32 * tq + 1e-30)
        bnd = np.maximum(0.0, np.sqrt(lbk * (1 - 2.0 ** -10)) - e) ** 2
        assert np.all(bnd <= raw * (1 + 1e-12))
        if reach in REV_REACHES and n == 256:
            # the filter's reverse bound (lbk_rev_q8): the query against the quantised row's
            # envelope widened by s/2, rounded down -- <= its fp64 value, >= that value less
            # the kernel's 2^-8 code-unit carry of q / s and fp32 rounding, <= the oracle's
            # raw reverse LB_Keogh <= DTW
            xq32 = xq.astype(np.float32)
            assert np.array_equal(xq32.astype(np.float64), xq)
            qd = Qh[2].astype(np.float64)
            T = np.empty(len(ids_np))
            T_lo = np.empty(len(ids_np))
            rawrev = np.empty(len(ids_np))
            for j, i in enumerate(ids_np):
                Uq, Lq = oracle.envelope(xq32[j], reach)
                m = np.maximum(np.maximum(qd - Uq, Lq - qd), sc[j] / 2) - sc[j] / 2
                T[j] = (m * m).sum()
                mlo = np.maximum(m - sc[j] * 2.0 ** -8, 0.0)  # q / s carried to 2^-8 (down)
                T_lo[j] = (mlo * mlo).sum()
                Ux, Lx = oracle.envelope(Xh[i], reach)
                rawrev[j] = oracle.lb_keogh2(Ux, Lx, Qh[2])
            assert not np.isnan(lbr).any()
            assert np.all(lbr <= T * (1 + 1e-12))
            assert np.all(lbr >= T_lo * (1 - (2 * n + 8) * U32))
            assert np.all(lbr <= rawrev * (1 + 1e-12))
            assert np.all(rawrev <= ref * (1 + 1e-12))
            assert (lbr > lbk).any()  # the reverse bound is the larger one for some rows
        else:
            assert np.isnan(lbr).all()
    else:
        assert np.isnan(lbr).all()
        assert np.all(np.abs(lbk - raw) <= (n // 32 + 8) * U32 * raw + 1e-30)


@pytest.mark.parametrize("count", [1, 2, 31, 32, 33, 63, 64, 65, 97, 127, 128, 129, 191, 193, 1000])
def test_dtw_refine_handout_counts(c1, count):
    """The strip refine's hand-out order (chunks of 64 entries, first half from the start of the
    list, second half from its end, holes past the middle) reaches EVERY list entry exactly
    once for list lengths around the chunk and half-chunk boundaries: the frozen refine over
    `count` candidates returns each one's fp32 DTW^2 (NaN where a candidate was never run)."""
    X, Q, idx, Xh, Qh = c1
    n = X.shape[1]
    reach = 25
    ids_np = np.random.default_rng(500 + count).choice(20_000, count, replace=False).astype(np.int32)
    ids = torch.from_numpy(ids_np).to(DEV)
    q = Q[1].contiguous()
    lbk, d32, quantised, _ = messi().messi_debug_dtw_stages(idx.handle, q, reach, ids, rev=True)
    d32 = d32.cpu().numpy().astype(np.float64)
    assert quantised and not np.isnan(d32).any()
    ref = oracle.dtw2_rows(Xh[ids_np], Qh[1], reach)
    assert np.all(np.abs(d32 - ref) <= (2 * n + 2) * U32 * ref + 1e-30)


def test_dtw_stages_long_series():
    """The strip refine at n = 2048 with r = 204 (10%) and r = 100 (64-thread CTAs, one query
    copy: the boundary rows fill shared memory), against the oracle's DTW on 160 rows each."""
    n = 2048
    X = gen_rows(3000, n, seed=5)
    Q = gen_rows(1, n, seed=6)
    Xh, Qh = X.cpu().numpy(), Q.cpu().numpy()
    idx = messi().Index(X)
    try:
        ids_np = np.random.default_rng(3).choice(3000, 160, replace=False).astype(np.int32)
        ids = torch.from_numpy(ids_np).to(DEV)
        for r in (204, 100):
            _, d32, quantised = messi().messi_debug_dtw_stages(idx.handle, Q[0].contiguous(), r, ids)
            d32 = d32.cpu().numpy().astype(np.float64)
            assert quantised
            ref = oracle.dtw2_rows(Xh[ids_np], Qh[0], r)
            assert np.all(np.abs(d32 - ref) <= (2 * n + 2) * U32 * ref + 1e-30)
    finally:
        idx.close()


@pytest.mark.parametrize("reach", [-1, 0, 3, 12, 25, 40])
def test_distances_elementwise(c1, reach):
    X, Q, idx, Xh, Qh = c1
    n = X.shape[1]
    ids = np.random.default_rng(7 + reach).choice(X.shape[0], 300, replace=False).astype(np.int32)
    d32, d64, lbk = messi().messi_debug_distances(idx.handle, Q[1].contiguous(), reach,
                                                  torch.from_numpy(ids).to(DEV))
    d32, d64 = d32.cpu().numpy().astype(np.float64), d64.cpu().numpy()
    if reach < 0:
        ref = np.array([oracle.ed2(Qh[1], Xh[i]) for i in ids])
    else:
        ref = np.array([oracle.dtw2(Qh[1], Xh[i], reach) for i in ids])
        assert not np.isnan(lbk.cpu().numpy()).any()
    assert np.array_equal(d64, ref)  # canonical fp64: bit-exact
    assert np.all(np.abs(d32 - ref) <= (2 * n + 2) * U32 * ref + 1e-30)


# ------------------------------------------------------- quantised-row bound
def test_quantised_rows_and_bound(c1):
    """The refine's quantised copy: c = rint(x / s) with s the smallest power of two such
    that max|x| <= 127 s; e >= ||x - s c|| (and tight); the bound ||q - s c|| - e never exceeds
    the true distance ||q - x|| (triangle inequality) -- checked in fp64 on every row of C1
    for every C1 query, and the kernel's own fp32 evaluation is covered by the 1-NN parity."""
    X, Q, idx, Xh, Qh = c1
    q8, meta = messi().messi_debug_quantised(idx.handle, X.shape[0], X.shape[1], X.device)
    c = q8.cpu().numpy().view(np.int8).astype(np.int64)
    s = meta[:, 0].cpu().numpy().astype(np.float64)
    e = meta[:, 1].cpu().numpy().astype(np.float64)
    x = Xh.astype(np.float64)
    assert np.all(np.abs(c) <= 127)
    m, ex = np.frexp(s)
    assert np.all(m == 0.5)  # powers of two
    mx = np.abs(x).max(axis=1)
    assert np.all(mx <= 127 * s) and np.all((mx > 127 * s / 2) | (mx == 0))
    assert np.array_equal(c, np.rint(x / s[:, None]).astype(np.int64))
    r = np.sqrt(((x - s[:, None] * c) ** 2).sum(axis=1))
    # e: round-up fp32 sum of the exact squares (n fmas + 5 butterfly adds) and a round-up
    # square root -- an upper bound, tight to (n + 8) u relative
    assert np.all(e >= r) and np.all(e <= r * (1 + (X.shape[1] + 8) * 2.0 ** -24) + 1e-30)
    deq = s[:, None] * c
    for qi in range(Q.shape[0]):
        q = Qh[qi].astype(np.float64)
        true = np.sqrt(((x - q) ** 2).sum(axis=1))
        lb = np.sqrt(((deq - q) ** 2).sum(axis=1)) - e
        assert np.all(lb <= true * (1 + 1e-12))


def test_quantised_lb_keogh_bound(c1):
    """The quantised LB_Keogh bound of the strip DTW path (k_lbk_filter_q8 and the strip
    refine's tail): for every row x of C1 and every suffix of its points,
    (sqrt(LBK_S(x^)) - e)^2 <= LBK_S(x) (the raw LB_Keogh of the suffix, oracle.lb_keogh2
    terms) <= DTW^2 when S is the whole row -- checked in fp64 with the GPU's own quantised
    rows, for two C1 queries and reaches 7 / 25."""
    X, Q, idx, Xh, Qh = c1
    rows = 3000
    q8, meta = messi().messi_debug_quantised(idx.handle, X.shape[0], X.shape[1], X.device)
    c = q8[:rows].cpu().numpy().view(np.int8).astype(np.float64)
    s = meta[:rows, 0].cpu().numpy().astype(np.float64)
    e = meta[:rows, 1].cpu().numpy().astype(np.float64)
    x = Xh[:rows].astype(np.float64)
    xq = s[:, None] * c
    for r in (7, 25):
        for qi in range(2):
            U, L = oracle.envelope(Qh[qi], r)
            U, L = np.asarray(U, dtype=np.float64), np.asarray(L, dtype=np.float64)
            term = lambda v: np.where(v > U, v - U, np.where(v < L, v - L, 0.0)) ** 2  # noqa: E731
            tx, tq = term(x), term(xq)
            for j in (0, 8, 64, 200):  # suffixes S = points j .. n-1
                raw = tx[:, j:].sum(axis=1)
                bnd = np.maximum(0.0, np.sqrt(tq[:, j:].sum(axis=1)) - e) ** 2
                assert np.all(bnd <= raw * (1 + 1e-12) + 1e-300)
            full = np.array([oracle.lb_keogh2(U, L, x[i]) for i in range(50)])
            assert np.allclose(full, tx[:50].sum(axis=1), rtol=1e-12, atol=0)
            d = oracle.dtw2_rows(Xh[:50], Qh[qi], r)
            assert np.all(tx[:50].sum(axis=1) <= np.asarray(d) * (1 + 1e-12))


# --------------------------------------------------------------------- 1-NN end to end
def check_nn(got, ref_d2, ref_id):
    dist, gid, d2 = got[:3]
    assert gid == ref_id, (gid, ref_id, d2, ref_d2)
    assert d2 == ref_d2
    assert math.isclose(dist, math.sqrt(ref_d2), rel_tol=1e-12, abs_tol=1e-300)


def test_nn_ed_config1(c1):
    X, Q, idx, Xh, Qh = c1
    d2, ids = oracle.nn("ed", Xh, Qh)
    for qi in range(Q.shape[0]):
        got = idx.query_ed(Q[qi], with_stats=True)
        check_nn(got, d2[qi], ids[qi])
        st = got[3]
        # series bounds are evaluated only inside the tiles the box filter keeps (Alg. 7)
        assert 1 <= st["tiles_scanned"] <= (X.shape[0] + 511) // 512
        assert st["lb_computed"] <= X.shape[0]
        assert st["seed_d2"] >= st["bsf_d2"] >= 0  # BSF only decreases (Obs. 1)
        assert st["near_best"] >= 1 and st["candidates"] >= st["refined"] >= st["exact"] >= 1


def test_nn_ed_host_query_and_batch(c1):
    X, Q, idx, Xh, Qh = c1
    d2, ids = oracle.nn("ed", Xh, Qh)
    m = messi()
    res, stats = m.result_buffer(Q.shape[0], DEV), m.stats_buffer(Q.shape[0], DEV)
    idx.query_batch(Q, None, res, stats)
    torch.cuda.synchronize()
    dist_b, id_b, d2_b = m.decode_results(res)
    assert np.array_equal(id_b.numpy(), ids) and np.array_equal(d2_b.numpy(), d2)
    for qi in range(3):  # host pointer path
        check_nn(idx.query_ed(Qh[qi]), d2[qi], ids[qi])


def test_nn_ed_batch_spans_launch_groups(c1):
    """More queries than one launch group of the batched ED path (kBatchMax = 128): 130
    queries (seed 1, rows 0..129 of the query stream) over the first 30,000 rows of C1, the
    last group holding 2; mixed with DTW calls on the same index before and after."""
    X, Q, idx, Xh, Qh = c1
    sub = 30_000
    X2 = X[:sub].contiguous()
    Q2 = gen_rows(130, 256, seed=datagen.QUERY_SEED)
    idx2 = messi().Index(X2)
    try:
        d2, ids = oracle.nn("ed", Xh[:sub], Q2.cpu().numpy())
        dref, iref = oracle.nn("dtw", Xh[:sub], Qh[:1], r=5)
        check_nn(idx2.query_dtw(Q[0], 5), dref[0], iref[0])
        m = messi()
        res, stats = m.result_buffer(130, DEV), m.stats_buffer(130, DEV)
        idx2.query_batch(Q2, None, res, stats)
        check_nn(idx2.query_dtw(Q[0], 5), dref[0], iref[0])
        torch.cuda.synchronize()
        _, id_b, d2_b = m.decode_results(res)
        assert np.array_equal(id_b.numpy(), ids) and np.array_equal(d2_b.numpy(), d2)
        for st in m.decode_stats(stats):
            assert st["near_best"] >= 1 and st["exact"] >= 1 and st["seed_d2"] >= st["bsf_d2"]
    finally:
        idx2.close()


@pytest.mark.parametrize("reach,strip", [(25, None), (7, None), (1, None), (3, None), (9, None), (51, None),
                                         (2, None), (5, None), (2, "0"), (5, "0"), (12, "0"), (25, "0")])
def test_nn_dtw(c1, reach, strip, monkeypatch):
    """Exact DTW 1-NN against the oracle.  Every reach >= 1 takes the strip kernel
    (k_refine_dtw_strip) by default; MESSI_DTW_STRIP=0 takes the register bands where they are
    instantiated (2, 5, 12, 25) with the raw LB_Keogh filter."""
    if strip is not None:
        monkeypatch.setenv("MESSI_DTW_STRIP", strip)
    X, Q, idx, Xh, Qh = c1
    sub = 20_000
    X2 = X[:sub].contiguous()
    idx2 = messi().Index(X2)
    try:
        d2, ids = oracle.nn("dtw", Xh[:sub], Qh[:3], r=reach)
        for qi in range(3):
            got = idx2.query_dtw(Q[qi], reach, with_stats=True)
            check_nn(got, d2[qi], ids[qi])
            st = got[3]
            assert st["candidates"] >= st["rev_paa_pass"] >= st["lbk_pass"] >= 1
            if reach in REV_REACHES and strip != "0":  # the reverse bound ran on the forward survivors
                assert st["rev_paa_pass"] >= st["exact"] >= st["lbk_pass"]
            else:
                assert st["exact"] == 0
        res = messi().result_buffer(3, DEV)
        idx2.query_batch(Q[:3].contiguous(), reach, res)
        torch.cuda.synchronize()
        _, id_b, d2_b = messi().decode_results(res)
        assert np.array_equal(id_b.numpy(), ids) and np.array_equal(d2_b.numpy(), d2)
    finally:
        idx2.close()


# ------------------------------------------------------------------------- edge cases
@pytest.mark.parametrize("N,n", [(1, 256), (7, 64), (513, 128), (2500, 16), (3000, 2048), (1025, 48)])
def test_nn_sizes_and_ragged(N, n):
    X = gen_rows(N, n, seed=5)
    Q = gen_rows(3, n, seed=6)
    Xh, Qh = X.cpu().numpy(), Q.cpu().numpy()
    idx = messi().Index(X)
    try:
        d2, ids = oracle.nn("ed", Xh, Qh)
        for qi in range(3):
            check_nn(idx.query_ed(Q[qi]), d2[qi], ids[qi])
        sub_rows = 400 if n <= 256 else 40
        for r in sorted({0, 2, min(5, n), n // 10, n}):  # n // 10: strip kernel (n = 2048: 64-thread CTAs)
            d2, ids = oracle.nn("dtw", Xh[:sub_rows], Qh[:1], r=r)
            sub = messi().Index(X[:sub_rows].contiguous())
            try:
                check_nn(sub.query_dtw(Q[0], r), d2[0], ids[0])
            finally:
                sub.close()
    finally:
        idx.close()


def test_duplicates_ties_lowest_id_and_zero_distance():
    N, n = 5000, 128
    X = gen_rows(N, n, seed=9)
    X[3000] = X[41]
    X[4999] = X[41]
    X[1234] = X[17]
    torch.cuda.synchronize()
    idx = messi().Index(X, row_begin=1000)
    try:
        for src, want in ((41, 41), (3000, 41), (4999, 41), (1234, 17)):
            dist, gid, d2 = idx.query_ed(X[src])
            assert (gid, d2, dist) == (1000 + want, 0.0, 0.0)
            dist, gid, d2 = idx.query_dtw(X[src], 12)
            assert (gid, d2) == (1000 + want, 0.0)
    finally:
        idx.close()


def test_all_rows_identical_and_constant_rows():
    N, n = 3000, 64
    base = gen_rows(1, n, seed=11)
    X = base.repeat(N, 1).contiguous()
    Q = gen_rows(2, n, seed=12)
    idx = messi().Index(X)
    try:
        d2, _ = oracle.nn("ed", X[:1].cpu().numpy(), Q.cpu().numpy())
        for qi in range(2):
            dist, gid, got = idx.query_ed(Q[qi])
            assert gid == 0 and got == d2[qi]
        dist, gid, got = idx.query_dtw(Q[0], 5)
        assert gid == 0
    finally:
        idx.close()
    Z = torch.zeros((700, n), dtype=torch.float32, device=DEV)  # constant (z-norm -> 0) rows
    Z[500] = gen_rows(1, n, seed=13)[0]
    idx = messi().Index(Z)
    try:
        q = gen_rows(1, n, seed=14)[0]
        d2, ids = oracle.nn("ed", Z.cpu().numpy(), q.cpu().numpy()[None])
        check_nn(idx.query_ed(q), d2[0], ids[0])
        dist, gid, got = idx.query_ed(torch.zeros(n, device=DEV))
        assert gid == 0 and got == 0.0
    finally:
        idx.close()


def test_near_tie_one_ulp():
    """Two rows differing in one ulp at one point: the fp32 refine cannot separate them,
    the exact fp64 re-rank must."""
    N, n = 4000, 256
    X = gen_rows(N, n, seed=15)
    q = gen_rows(1, n, seed=16)[0]
    d2, ids = oracle.nn("ed", X.cpu().numpy(), q.cpu().numpy()[None])
    nn = int(ids[0])
    twin = X[nn].clone()
    j = 100
    # move one point of the twin one ulp towards the query (strictly closer) and put the
    # twin at a HIGHER id than the original
    twin[j] = float(np.nextafter(np.float32(X[nn, j].item()), np.float32(q[j].item())))
    X[3999] = twin
    torch.cuda.synchronize()
    Xh = X.cpu().numpy()
    d2, ids = oracle.nn("ed", Xh, q.cpu().numpy()[None])
    idx = messi().Index(X)
    try:
        check_nn(idx.query_ed(q), d2[0], ids[0])
    finally:
        idx.close()


def test_noisy_queries_config5_shape():
    """Config 5's query workload at small scale: n = 128, sigma = 0.1."""
    N, n = 60_000, 128
    X = gen_rows(N, n)
    Q = torch.empty((20, n), dtype=torch.float32, device=DEV)
    datagen.noisy_queries_cuda(Q, N, sigma=0.1)
    torch.cuda.synchronize()
    d2, ids = oracle.nn("ed", X.cpu().numpy(), Q.cpu().numpy())
    idx = messi().Index(X)
    try:
        src = datagen.noisy_rows(20, N)
        hits = 0
        for qi in range(20):
            got = idx.query_ed(Q[qi])
            check_nn(got, d2[qi], ids[qi])
            hits += int(got[1] == src[qi])
        assert hits >= 15  # sigma = 0.1 noise: the source row is (almost always) the NN
    finally:
        idx.close()


def test_errors():
    m = messi()
    X = gen_rows(10, 64)
    with pytest.raises(m.MessiError) as e:
        m.messi_build(X[:0])
    assert e.value.status == m.MESSI_EEMPTY
    with pytest.raises(m.MessiError) as e:
        m.messi_build(gen_rows(10, 40))
    assert e.value.status == m.MESSI_EINVAL
    idx = m.Index(X)
    try:
        with pytest.raises(m.MessiError) as e:
            idx.query_dtw(X[0], 65)
        assert e.value.status == m.MESSI_EINVAL
        with pytest.raises(m.MessiError) as e:
            idx.query_dtw(X[0], -1)
        assert e.value.status == m.MESSI_EINVAL
        for bad_k in (0, 65):  # k-NN: 1 <= k <= 64
            with pytest.raises(m.MessiError) as e:
                idx.query_knn(X[0], bad_k)
            assert e.value.status == m.MESSI_EINVAL
        # the index stays usable after rejected calls
        _, gid, d2 = idx.query_ed(X[3])
        assert gid == 3 and d2 == 0.0
    finally:
        idx.close()
