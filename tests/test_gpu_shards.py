"""Row-sharded collections whose shards share each query's best-so-far (include/messi.h,
messi_link_peers_*): the cross-shard lexicographic min of the local answers must equal the
oracle's brute force over the whole collection (exact id and d2), whether the shards are
linked or not -- linking only changes how much each shard prunes.

Emulated on one GPU (the box has one): two indexes of one process (messi_link_peers_local)
running concurrently on two streams, and two processes sharing the GPU through CUDA IPC
(messi_link_peers_ipc, the path bench.py takes on N GPUs) with a gloo process group.  The
kernels never wait on each other (they only raise each other's thresholds), so sharing one
GPU is safe."""
import os
import socket

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
    return x


def _run_shards(X, Q, link, nshards=2, rounds=2, reach=None, k=1):
    from paper_2110_07519_b200 import messi as M
    from paper_2110_07519_b200.dist import lexmin, shard_range
    N = X.shape[0]
    streams = [torch.cuda.Stream() for _ in range(nshards)]
    parts, idxs = [], []
    for g in range(nshards):
        b, e = shard_range(N, nshards, g)
        part = X[b:e].contiguous()
        parts.append(part)
        idxs.append(M.Index(part, row_begin=b, stream=streams[g]))
    if link:
        for g in range(nshards):
            M.messi_link_peers_local(idxs[g].handle, [idxs[h].handle for h in range(nshards) if h != g])
    out = []
    for _ in range(rounds):  # several launch epochs
        res = [M.result_buffer(Q.shape[0] * k, DEV) for _ in range(nshards)]
        sts = [M.stats_buffer(Q.shape[0], DEV) for _ in range(nshards)]
        for g in range(nshards):
            if k > 1:
                idxs[g].query_batch_knn(Q, k, res[g], sts[g], reach=reach)
            else:
                idxs[g].query_batch(Q, reach, res[g], sts[g])
        torch.cuda.synchronize()
        if k > 1:
            from paper_2110_07519_b200.dist import merge_knn  # noqa: F401 (host merge below)
            d2 = torch.cat([M.decode_results(r)[2].view(-1, k) for r in res], dim=1)
            gid = torch.cat([M.decode_results(r)[1].view(-1, k) for r in res], dim=1)
            order = [np.lexsort((g_.numpy(), np.where(g_.numpy() < 0, np.inf, d_.numpy())))[:k]
                     for d_, g_ in zip(d2, gid)]
            out.append((np.stack([d2[i].numpy()[o] for i, o in enumerate(order)]),
                        np.stack([gid[i].numpy()[o] for i, o in enumerate(order)]), None))
            continue
        d2 = torch.stack([M.decode_results(r)[2] for r in res])
        gid = torch.stack([M.decode_results(r)[1] for r in res])
        best, bid = lexmin(d2, gid)
        out.append((best.numpy(), bid.numpy(), [M.decode_stats(s) for s in sts]))
    for i in idxs:
        i.close()
    return out


@pytest.mark.parametrize("link", [False, True])
def test_linked_shards_exact(link):
    X = _gen(60_000, 256, datagen.DATA_SEED)
    Q = _gen(12, 256, datagen.QUERY_SEED)
    torch.cuda.synchronize()
    d2, ids = oracle.nn("ed", X.cpu().numpy(), Q.cpu().numpy())
    for best, bid, stats in _run_shards(X, Q, link, nshards=3):
        assert np.array_equal(bid, ids) and np.array_equal(best, d2)
        if link:
            # a linked shard may find nothing inside the shared threshold: (inf, -1)
            for shard in stats:
                for s in shard:
                    assert s["bsf_d2"] >= 0


@pytest.mark.parametrize("link", [False, True])
@pytest.mark.parametrize("reach", [25, 5])
def test_linked_shards_dtw_exact(link, reach):
    """DTW with linked shards (the shards share BSF0 and every later best of the
    same query through their DTW slots): the merged answers equal the oracle's, and linking
    only reduces the refine work of the shards."""
    X = _gen(30_000, 128, datagen.DATA_SEED)
    Q = _gen(6, 128, datagen.QUERY_SEED)
    torch.cuda.synchronize()
    d2, ids = oracle.nn("dtw", X.cpu().numpy(), Q.cpu().numpy(), r=reach)
    for best, bid, stats in _run_shards(X, Q, link, nshards=3, rounds=2, reach=reach):
        assert np.array_equal(bid, ids) and np.array_equal(best, d2)


def test_linked_shards_dtw_knn_exact():
    X = _gen(20_000, 128, datagen.DATA_SEED)
    Q = _gen(4, 128, datagen.QUERY_SEED)
    torch.cuda.synchronize()
    d2, ids = oracle.knn("dtw", X.cpu().numpy(), Q.cpu().numpy(), 5, r=12)
    for best, bid, _ in _run_shards(X, Q, True, nshards=2, rounds=1, reach=12, k=5):
        assert np.array_equal(bid, ids) and np.array_equal(best, d2)


def test_linked_shards_with_duplicates_across_shards():
    """Exact ties across shards (the same row in both halves): the lowest global id wins."""
    X = _gen(20_000, 128, datagen.DATA_SEED)
    X[15_000:15_010] = X[100:110]  # rows 15000.. duplicate rows 100.. (other shard)
    Q = X[100:106].clone()
    torch.cuda.synchronize()
    d2, ids = oracle.nn("ed", X.cpu().numpy(), Q.cpu().numpy())
    for best, bid, _ in _run_shards(X, Q, True, nshards=2, rounds=1):
        assert np.array_equal(bid, ids) and np.array_equal(best, d2)
        assert list(bid) == list(range(100, 106))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, out_path):
    import torch.distributed as dist
    from paper_2110_07519_b200 import messi as M
    from paper_2110_07519_b200.dist import link_shards, merge_results, shard_range
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    N, n = 40_000, 256
    b, e = shard_range(N, world, rank)
    part = torch.empty((e - b, n), dtype=torch.float32, device=DEV)
    datagen.walks_cuda(part, b, seed=datagen.DATA_SEED)
    Q = torch.empty((8, n), dtype=torch.float32, device=DEV)
    datagen.walks_cuda(Q, 0, seed=datagen.QUERY_SEED)
    torch.cuda.synchronize()
    idx = M.Index(part, row_begin=b)
    npeers = link_shards(idx)
    res = M.result_buffer(8, DEV)
    for _ in range(2):
        dist.barrier()
        idx.query_batch(Q, None, res, None)
        torch.cuda.synchronize()
        _, gid, d2 = M.decode_results_device(res)
        best, bid = merge_results(d2, gid)
    dist.barrier()
    idx.query_batch(Q[:3].contiguous(), 12, res, None)  # DTW, shared through the slots
    torch.cuda.synchronize()
    _, gid, d2 = M.decode_results_device(res)
    dbest, dbid = merge_results(d2[:3].contiguous(), gid[:3].contiguous())
    if rank == 0:
        np.savez(out_path, best=best.cpu().numpy(), bid=bid.cpu().numpy(), npeers=npeers,
                 dbest=dbest.cpu().numpy(), dbid=dbid.cpu().numpy())
    dist.barrier()
    idx.close()
    dist.destroy_process_group()


def test_ipc_linked_shards_two_processes(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "ipc.npz")
    mp.spawn(_ipc_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r = np.load(out)
    X = torch.empty((40_000, 256), dtype=torch.float32, device=DEV)
    datagen.walks_cuda(X, 0, seed=datagen.DATA_SEED)
    Q = _gen(8, 256, datagen.QUERY_SEED)
    torch.cuda.synchronize()
    d2, ids = oracle.nn("ed", X.cpu().numpy(), Q.cpu().numpy())
    assert int(r["npeers"]) == 1
    assert np.array_equal(r["bid"], ids) and np.array_equal(r["best"], d2)
    dd2, dids = oracle.nn("dtw", X.cpu().numpy(), Q[:3].cpu().numpy(), r=12)
    assert np.array_equal(r["dbid"], dids) and np.array_equal(r["dbest"], dd2)
