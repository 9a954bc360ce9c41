"""Exact k-NN under DTW (the paper's k-NN for both measures, DTW
k-NN priced at P:2718-2719) through the C-ABI, against the oracle's k-NN by definition
(oracle.knn("dtw"): every row's fp64 banded DTW, the k smallest (d2, id)): ids and fp64 d2
bit-exact, ascending, ties to the lowest id.  Covers the three refine kernels (strip r >= 7,
register band r = 2 / 5, warp wavefront r = 0), batch and single calls, duplicates at the k-th
place, k > N, and k = 1 equal to the 1-NN path."""
import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _gen(N, n, seed, row_begin=0):
    x = torch.empty((N, n), dtype=torch.float32, device=DEV)
    datagen.walks_cuda(x, row_begin, seed=seed)
    torch.cuda.synchronize()
    return x


@pytest.fixture(scope="module")
def coll():
    from paper_2110_07519_b200 import messi as M
    X = _gen(12_000, 128, datagen.DATA_SEED)
    Q = _gen(6, 128, datagen.QUERY_SEED)
    idx = M.Index(X)
    yield X, Q, idx, X.cpu().numpy(), Q.cpu().numpy()
    idx.close()


@pytest.mark.parametrize("reach,k,strip", [(12, 5, None), (12, 64, None), (5, 10, None), (2, 3, None), (0, 7, None),
                                           (25, 2, None), (5, 10, "0"), (2, 3, "0")])
def test_dtw_knn_batch_exact(coll, reach, k, strip, monkeypatch):
    """strip "0": the register-band refine (MESSI_DTW_STRIP=0) instead of the default strip kernel."""
    from paper_2110_07519_b200 import messi as M
    if strip is not None:
        monkeypatch.setenv("MESSI_DTW_STRIP", strip)
    X, Q, idx, Xh, Qh = coll
    d2, ids = oracle.knn("dtw", Xh, Qh, k, r=reach)
    res, st = M.result_buffer(Q.shape[0] * k, DEV), M.stats_buffer(Q.shape[0], DEV)
    idx.query_batch_knn(Q, k, res, st, reach=reach)
    torch.cuda.synchronize()
    _, gid, gd2 = M.decode_results(res)
    assert np.array_equal(gid.numpy().reshape(-1, k), ids)
    assert np.array_equal(gd2.numpy().reshape(-1, k), d2)
    for s in M.decode_stats(st):
        assert s["near_best"] >= k and s["bsf_d2"] <= s["seed_d2"] * (1 + 1e-6)


def test_dtw_knn_single_k1_and_duplicates():
    from paper_2110_07519_b200 import messi as M
    X = _gen(5000, 64, 21)
    X[4000] = X[17]  # exact duplicates: tie on d2, the lower id first
    X[4001] = X[17]
    X[2500] = X[33]
    torch.cuda.synchronize()
    Xh = X.cpu().numpy()
    idx = M.Index(X, row_begin=100)
    try:
        for src in (17, 33):
            q = Xh[src] + np.float32(0.01)
            d2, ids = oracle.knn("dtw", Xh, q, 6, r=6, row_begin=100)
            dist, gid, gd2 = idx.query_dtw_knn(q, 6, 6)  # host query pointer
            assert list(gid) == list(ids[0]) and np.array_equal(gd2, d2[0])
            assert np.allclose(dist, np.sqrt(d2[0]), rtol=1e-12)
            n_dist, n_id, n_d2 = idx.query_dtw(q, 6)
            k_dist, k_id, k_d2 = idx.query_dtw_knn(q, 6, 1)
            assert k_id[0] == n_id and k_d2[0] == n_d2
    finally:
        idx.close()


def test_dtw_knn_more_than_rows():
    from paper_2110_07519_b200 import messi as M
    X = _gen(9, 32, 5)
    Q = _gen(2, 32, 6)
    Xh, Qh = X.cpu().numpy(), Q.cpu().numpy()
    idx = M.Index(X)
    try:
        d2, ids = oracle.knn("dtw", Xh, Qh, 12, r=3)
        for qi in range(2):
            dist, gid, gd2 = idx.query_dtw_knn(Q[qi], 3, 12)
            assert list(gid) == list(ids[qi])
            assert np.array_equal(gd2[:9], d2[qi][:9]) and np.all(np.isinf(gd2[9:])) and np.all(gid[9:] == -1)
    finally:
        idx.close()
