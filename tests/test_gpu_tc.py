"""The tensor-core batched ED path (SURVEY 8(f) f4 (i)+(ii); tc.cuh) through the C-ABI:
exact 1-NN of many queries in one pass over the quantised rows, against the oracle's brute
force -- id and fp64 d2 bit-exact (ties to the lowest id); one and several passes (<= 256
queries each), n = 128 and 256, a collection that is not a multiple of the 128-row tile,
duplicates at zero distance, the exhaustive fallback when a query's candidate list overflows,
and the rejection of unsupported lengths."""
import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _gen(N, n, seed, row_begin=0):
    x = torch.empty((N, n), dtype=torch.float32, device=DEV)
    if N:
        datagen.walks_cuda(x, row_begin, seed=seed)
    torch.cuda.synchronize()
    return x


def _run_tc(idx, Q):
    from paper_2110_07519_b200 import messi as M
    res, st = M.result_buffer(Q.shape[0], DEV), M.stats_buffer(Q.shape[0], DEV)
    idx.query_batch_tc(Q, res, st)
    torch.cuda.synchronize()
    return M.decode_results(res), M.decode_stats(st)


@pytest.mark.parametrize("N,n,nq", [(100_000, 256, 10), (60_000, 128, 300), (1000, 256, 1), (70_001, 256, 257)])
def test_tc_matches_oracle(N, n, nq):
    from paper_2110_07519_b200 import messi as M
    X = _gen(N, n, datagen.DATA_SEED)
    Q = _gen(nq, n, datagen.QUERY_SEED)
    idx = M.Index(X)
    try:
        (dist, gid, d2), stats = _run_tc(idx, Q)
        ref_d2, ref_id = oracle.nn("ed", X.cpu().numpy(), Q.cpu().numpy())
        assert np.array_equal(gid.numpy(), ref_id)
        assert np.array_equal(d2.numpy(), ref_d2)
        assert np.allclose(dist.numpy(), np.sqrt(ref_d2), rtol=1e-12)
        for s in stats:
            assert s["lb_computed"] == N and s["near_best"] >= 1
            assert s["candidates"] >= s["exact"] >= 1  # survivors of the prescreen, then of the bound
            assert s["candidates"] < max(64, N // 100)  # the prescreen prunes
        # the same answers as the LUT batch path
        res = M.result_buffer(nq, DEV)
        idx.query_batch(Q, None, res)
        torch.cuda.synchronize()
        _, gid2, d22 = M.decode_results(res)
        assert np.array_equal(gid2.numpy(), gid.numpy()) and np.array_equal(d22.numpy(), d2.numpy())
    finally:
        idx.close()


def test_tc_duplicates_and_row_begin():
    from paper_2110_07519_b200 import messi as M
    X = _gen(9000, 128, 31)
    X[7000] = X[123]
    X[8999] = X[123]
    torch.cuda.synchronize()
    idx = M.Index(X, row_begin=5000)
    try:
        Q = torch.stack([X[7000], X[8999], X[5]]).contiguous()
        (dist, gid, d2), _ = _run_tc(idx, Q)
        assert list(gid.numpy()) == [5123, 5123, 5005] and list(d2.numpy()) == [0.0, 0.0, 0.0]
    finally:
        idx.close()


def test_tc_candidate_overflow_falls_back_exhaustively():
    """70,000 identical rows: every row is within the threshold, the candidate list of 65,536
    overflows and the query is answered by every row (the lowest id wins the tie)."""
    from paper_2110_07519_b200 import messi as M
    base = _gen(1, 256, 41)
    X = base.repeat(70_000, 1).contiguous()
    X[50_000] = _gen(1, 256, 42)[0]
    Q = _gen(2, 256, 43)
    idx = M.Index(X)
    try:
        (dist, gid, d2), st = _run_tc(idx, Q)
        ref_d2, ref_id = oracle.nn("ed", X.cpu().numpy(), Q.cpu().numpy())
        assert np.array_equal(gid.numpy(), ref_id) and np.array_equal(d2.numpy(), ref_d2)
    finally:
        idx.close()


def test_tc_rejects_other_lengths():
    from paper_2110_07519_b200 import messi as M
    X = _gen(500, 64, 7)
    idx = M.Index(X)
    try:
        with pytest.raises(M.MessiError) as e:
            idx.query_batch_tc(X[:2].contiguous())
        assert e.value.status == M.MESSI_EINVAL
    finally:
        idx.close()
