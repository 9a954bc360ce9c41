"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (own
CUDA stream, batched sequential queries), on sampled outputs the oracle computes in full:
a few queries of each config answered by the CUDA path and by the oracle's brute force over
EVERY row (the rows are streamed device -> host in chunks; the oracle runs one serial call
per chunk on all host cores and merges (d2, id) lexicographically).  Bars: id and d2
bit-exact, dist within 1e-12.
"""
import math
import os

import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

DEV = "cuda:0"
CHUNK = 1 << 21


def messi():
    from paper_2110_07519_b200 import messi as m
    return m


def oracle_full(kind, X, Qh, reach=0):
    """Brute force over every row of the device tensor X, chunk by chunk."""
    d2 = np.full(Qh.shape[0], np.inf)
    ids = np.full(Qh.shape[0], -1, np.int64)
    for b in range(0, X.shape[0], CHUNK):
        part = X[b:b + CHUNK].cpu().numpy()
        pd, pi = oracle.nn(kind, part, Qh, r=reach, row_begin=b, chunk=max(1, part.shape[0] // 64))
        d2, ids = oracle.merge(d2, ids, pd, pi)
    return d2, ids


def run_batch(idx, Q, reach=None):
    m = messi()
    res = m.result_buffer(Q.shape[0], DEV)
    with torch.cuda.stream(idx.stream):
        idx.query_batch(Q, reach, res)
    torch.cuda.synchronize()
    return m.decode_results(res)


def check(got, d2, ids):
    dist, gid, gd2 = (t.numpy() for t in got)
    assert np.array_equal(gid, ids), (gid, ids)
    assert np.array_equal(gd2, d2)
    for a, b in zip(dist, d2):
        assert math.isclose(a, math.sqrt(b), rel_tol=1e-12)


def build(N, n, Q):
    X = torch.empty((N, n), dtype=torch.float32, device=DEV)
    datagen.walks_cuda(X, 0)
    torch.cuda.synchronize()
    idx = messi().Index(X, stream=torch.cuda.Stream(DEV))
    return X, idx


def test_config2_ed_10m():
    X, idx = build(10_000_000, 256, None)
    Q = torch.empty((100, 256), dtype=torch.float32, device=DEV)
    datagen.walks_cuda(Q, 0, seed=datagen.QUERY_SEED)
    try:
        got = run_batch(idx, Q)
        sample = [0, 17, 63, 99]
        d2, ids = oracle_full("ed", X, Q[sample].cpu().numpy())
        check(tuple(t[sample] for t in got), d2, ids)
    finally:
        idx.close()
        del X
        torch.cuda.empty_cache()


def oracle_full_knn(X, Qh, k):
    """k-NN brute force over every row of X, chunk by chunk (oracle.knn per chunk, then the
    k lexicographically smallest (d2, id) of the chunk lists)."""
    alld, alli = [], []
    for b in range(0, X.shape[0], CHUNK):
        part = X[b:b + CHUNK].cpu().numpy()
        d, i = oracle.knn("ed", part, Qh, k, row_begin=b)
        alld.append(d)
        alli.append(i)
    D, I = np.concatenate(alld, axis=1), np.concatenate(alli, axis=1)
    out_d, out_i = np.empty((Qh.shape[0], k)), np.empty((Qh.shape[0], k), np.int64)
    for qi in range(Qh.shape[0]):
        o = np.lexsort((I[qi], D[qi]))[:k]
        out_d[qi], out_i[qi] = D[qi, o], I[qi, o]
    return out_d, out_i


def test_config3_ed_100m():
    """The bench workload: 100M x 256 on one GPU, 100 queries batched; 3 sampled in full;
    and exact 10-NN of one query against the oracle's brute force."""
    X, idx = build(100_000_000, 256, None)
    Q = torch.empty((100, 256), dtype=torch.float32, device=DEV)
    datagen.walks_cuda(Q, 0, seed=datagen.QUERY_SEED)
    try:
        got = run_batch(idx, Q)
        sample = [0, 42, 99]
        d2, ids = oracle_full("ed", X, Q[sample].cpu().numpy())
        check(tuple(t[sample] for t in got), d2, ids)
        m = messi()
        res = m.result_buffer(Q.shape[0] * 10, DEV)
        with torch.cuda.stream(idx.stream):
            idx.query_batch_knn(Q, 10, res)
        torch.cuda.synchronize()
        _, kid, kd2 = m.decode_results(res)
        kd, ki = oracle_full_knn(X, Q[[7]].cpu().numpy(), 10)
        assert np.array_equal(kid.numpy().reshape(-1, 10)[7], ki[0])
        assert np.array_equal(kd2.numpy().reshape(-1, 10)[7], kd[0])
    finally:
        idx.close()
        del X
        torch.cuda.empty_cache()


def test_config4_dtw_10m():
    """Config 4 (10M x 256, reach 25) in the bench's launch configuration: 10 queries batched.
    Query 0 against the oracle's brute force over every row.  All 10 against an exact brute
    force over every row that COULD beat the GPU's answer: a row whose LB_Keogh exceeds the
    GPU's d2 has DTW > d2 (LB_Keogh <= DTW, pinned in test_oracle_pins), so the
    oracle's DTW over the rows with LB_Keogh <= d2 (selected here with fp64 torch and a 1e-9
    margin) must return exactly the GPU's (d2, id), ties to the lowest id."""
    X, idx = build(10_000_000, 256, None)
    nq = 10
    Q = torch.empty((nq, 256), dtype=torch.float32, device=DEV)
    datagen.walks_cuda(Q, 0, seed=datagen.QUERY_SEED)
    try:
        got = run_batch(idx, Q, reach=25)
        sample = [0]
        d2, ids = oracle_full("dtw", X, Q[sample].cpu().numpy(), reach=25)
        check(tuple(t[sample] for t in got), d2, ids)
        dist, gid, gd2 = (t.numpy() for t in got)
        Qh = Q.cpu().numpy()
        for qi in range(nq):
            U, L = oracle.envelope(Qh[qi], 25)
            Ud = torch.from_numpy(U.astype(np.float64)).to(DEV)
            Ld = torch.from_numpy(L.astype(np.float64)).to(DEV)
            sel = []
            for b in range(0, X.shape[0], CHUNK):
                c = X[b:b + CHUNK].double()
                lbk = ((c - Ud).clamp(min=0) ** 2 + (Ld - c).clamp(min=0) ** 2).sum(1)
                sel.append(torch.nonzero(lbk <= gd2[qi] * (1 + 1e-9)).flatten() + b)
                del c, lbk
            sel = torch.cat(sel)
            assert sel.numel() >= 1
            Xs = X[sel].cpu().numpy()
            sd, si = oracle.nn("dtw", Xs, Qh[qi:qi + 1], r=25)
            assert sd[0] == gd2[qi], (qi, sd[0], gd2[qi])
            assert int(sel[int(si[0])]) == gid[qi], (qi, int(sel[int(si[0])]), gid[qi])
    finally:
        idx.close()
        del X
        torch.cuda.empty_cache()


def test_config5_noisy_ed_100m_x128():
    """Config 5's shape on one GPU (all 100M x 128 rows, 51 GB): noisy dataset queries."""
    N, n = 100_000_000, 128
    X, idx = build(N, n, None)
    Q = torch.empty((50, n), dtype=torch.float32, device=DEV)
    datagen.noisy_queries_cuda(Q, N, sigma=0.1)
    torch.cuda.synchronize()
    try:
        got = run_batch(idx, Q)
        sample = [0, 25, 49]
        d2, ids = oracle_full("ed", X, Q[sample].cpu().numpy())
        check(tuple(t[sample] for t in got), d2, ids)
        src = datagen.noisy_rows(50, N)
        assert np.mean(got[1].numpy() == src) > 0.9  # the noisy source row is (almost always) the NN
    finally:
        idx.close()
        del X
        torch.cuda.empty_cache()
