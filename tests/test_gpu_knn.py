"""Exact k-NN under ED (the paper's k-NN variant) through the
C-ABI, against the oracle's k-NN by definition (oracle.knn: every distance, k smallest
(d2, id)): ids and fp64 d2 bit-exact, ascending, ties to the lowest id; batch and single
calls; k = 1 equals the 1-NN path; shards with fewer than k rows; linked shards."""
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
    X = _gen(60_000, 256, datagen.DATA_SEED)
    Q = _gen(12, 256, datagen.QUERY_SEED)
    idx = M.Index(X)
    yield X, Q, idx, X.cpu().numpy(), Q.cpu().numpy()
    idx.close()


@pytest.mark.parametrize("k", [1, 2, 10, 64])
def test_knn_batch_exact(coll, k):
    from paper_2110_07519_b200 import messi as M
    X, Q, idx, Xh, Qh = coll
    d2, ids = oracle.knn("ed", Xh, Qh, k)
    res, st = M.result_buffer(Q.shape[0] * k, DEV), M.stats_buffer(Q.shape[0], DEV)
    idx.query_batch_knn(Q, k, res, st)
    torch.cuda.synchronize()
    _, gid, gd2 = M.decode_results(res)
    assert np.array_equal(gid.numpy().reshape(-1, k), ids)
    assert np.array_equal(gd2.numpy().reshape(-1, k), d2)
    for s in M.decode_stats(st):
        assert s["near_best"] >= k and s["bsf_d2"] <= s["seed_d2"]


def test_knn_single_and_k1_equals_nn(coll):
    X, Q, idx, Xh, Qh = coll
    d2, ids = oracle.knn("ed", Xh, Qh[:3], 5)
    for qi in range(3):
        dist, gid, gd2 = idx.query_knn(Qh[qi], 5)  # host query pointer
        assert list(gid) == list(ids[qi]) and np.array_equal(gd2, d2[qi])
        assert np.allclose(dist, np.sqrt(d2[qi]), rtol=1e-12)
        n_dist, n_id, n_d2 = idx.query_ed(Q[qi])
        k_dist, k_id, k_d2 = idx.query_knn(Q[qi], 1)
        assert k_id[0] == n_id and k_d2[0] == n_d2


@pytest.mark.parametrize("k", [8, 24])
def test_knn_duplicates_and_small_collection(k):
    """Exact duplicate rows (ties broken by id) and a collection smaller than k; k = 24 takes
    the warp-cooperative insert (k > 16), k = 8 the single-lane one."""
    from paper_2110_07519_b200 import messi as M
    X = _gen(3000, 64, datagen.DATA_SEED)
    X[2000:2005] = X[10]
    Q = X[[10, 11]].clone()
    torch.cuda.synchronize()
    idx = M.Index(X)
    try:
        d2, ids = oracle.knn("ed", X.cpu().numpy(), Q.cpu().numpy(), k)
        res = M.result_buffer(2 * k, DEV)
        idx.query_batch_knn(Q, k, res)
        torch.cuda.synchronize()
        _, gid, gd2 = M.decode_results(res)
        assert np.array_equal(gid.numpy().reshape(-1, k), ids) and np.array_equal(gd2.numpy().reshape(-1, k), d2)
        assert list(ids[0, :6]) == [10, 2000, 2001, 2002, 2003, 2004]
    finally:
        idx.close()
    Xs = X[:5].contiguous()
    idx2 = M.Index(Xs)
    try:
        dist, gid, gd2 = idx2.query_knn(Q[0], k)
        d2, ids = oracle.knn("ed", Xs.cpu().numpy(), Q[:1].cpu().numpy(), k)
        assert list(gid) == list(ids[0]) and list(gid[5:]) == [-1] * (k - 5) and np.all(np.isinf(gd2[5:]))
    finally:
        idx2.close()


@pytest.mark.parametrize("k", [9, 33])
def test_knn_linked_shards(k):
    """Shards sharing their k-th best (valid: one shard alone has k rows within it) still
    merge to the exact global k-NN."""
    from paper_2110_07519_b200 import messi as M
    from paper_2110_07519_b200.dist import shard_range
    X = _gen(45_000, 128, datagen.DATA_SEED)
    Q = _gen(6, 128, datagen.QUERY_SEED)
    idxs, parts = [], []
    streams = [torch.cuda.Stream() for _ in range(3)]
    for g in range(3):
        b, e = shard_range(X.shape[0], 3, g)
        parts.append(X[b:e].contiguous())
        idxs.append(M.Index(parts[-1], row_begin=b, stream=streams[g]))
    for g in range(3):
        M.messi_link_peers_local(idxs[g].handle, [idxs[h].handle for h in range(3) if h != g])
    try:
        res = [M.result_buffer(6 * k, DEV) for _ in range(3)]
        for g in range(3):
            idxs[g].query_batch_knn(Q, k, res[g])
        torch.cuda.synchronize()
        alld = np.concatenate([M.decode_results(r)[2].numpy().reshape(-1, k) for r in res], axis=1)
        alli = np.concatenate([M.decode_results(r)[1].numpy().reshape(-1, k) for r in res], axis=1)
        d2, ids = oracle.knn("ed", X.cpu().numpy(), Q.cpu().numpy(), k)
        for qi in range(6):
            cand = [(alld[qi, j], alli[qi, j]) for j in range(alld.shape[1]) if alli[qi, j] >= 0]
            cand.sort()
            assert [c[1] for c in cand[:k]] == list(ids[qi]) and [c[0] for c in cand[:k]] == list(d2[qi])
    finally:
        for i in idxs:
            i.close()
