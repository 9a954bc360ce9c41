"""Multi-rank host logic on CPU (gloo, world_size 2): contiguous row sharding and the
exact cross-rank (d2, id) merge, checked against a single-process brute force."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2110_07519_b200.dist import lexmin, merge_results, shard_range


def test_shard_range_partitions():
    for N in (0, 1, 7, 100, 12_345):
        for G in (1, 2, 3, 8):
            parts = [shard_range(N, G, g) for g in range(G)]
            assert parts[0][0] == 0 and parts[-1][1] == N
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [e - b for b, e in parts]
            assert max(sizes) - min(sizes) <= 1


def test_lexmin_ties_go_to_lowest_id():
    d2 = torch.tensor([[1.0, 2.0, 5.0], [1.0, 3.0, float("inf")]], dtype=torch.float64)
    gid = torch.tensor([[7, 1, 4], [3, 0, -1]])
    best, bid = lexmin(d2, gid)
    assert best.tolist() == [1.0, 2.0, 5.0] and bid.tolist() == [3, 1, 4]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, X, Q, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = shard_range(X.shape[0], world, rank)
    # each rank answers over its own shard (global ids via row_begin) ...
    d2, ids = oracle.nn("ed", X[b:e], Q, row_begin=b, threads=1)
    # ... and the ranks merge with one all_gather
    gd2, gid = merge_results(torch.from_numpy(d2), torch.from_numpy(ids))
    if rank == 0:
        out.put((gd2.numpy(), gid.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_answers_equal_single_scan(world):
    rng = np.random.default_rng(0)
    X = rng.standard_normal((1001, 32)).astype(np.float32)
    X[900] = X[5]  # a cross-shard exact tie: the lower id (rank 0) must win
    Q = np.concatenate([X[[900]], rng.standard_normal((5, 32)).astype(np.float32)])
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, Q, out)) for r in range(world)]
    for p in procs:
        p.start()
    gd2, gid = out.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    d2, ids = oracle.nn("ed", X, Q)
    assert np.array_equal(gid, ids) and np.array_equal(gd2, d2)
    assert gid[0] == 5


def _knn_worker(rank, world, port, X, Q, k, out):
    from paper_2110_07519_b200.dist import merge_knn
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = shard_range(X.shape[0], world, rank)
    d2, ids = oracle.knn("ed", X[b:e], Q, k, row_begin=b)
    gd2, gid = merge_knn(torch.from_numpy(d2), torch.from_numpy(ids))
    if rank == 0:
        out.put((gd2.numpy(), gid.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("k", [1, 7])
def test_sharded_knn_merge_equals_single_scan(k):
    """k-NN across 2 ranks (gloo): the merge of the local k lists is the global k list,
    including cross-shard exact ties (lowest id first) and a shard with fewer than k rows."""
    rng = np.random.default_rng(1)
    X = rng.standard_normal((13, 16)).astype(np.float32)
    X[10] = X[2]  # cross-shard duplicate
    Q = np.concatenate([X[[10]], rng.standard_normal((3, 16)).astype(np.float32)])
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_knn_worker, args=(r, 2, port, X, Q, k, out)) for r in range(2)]
    for p in procs:
        p.start()
    gd2, gid = out.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    d2, ids = oracle.knn("ed", X, Q, k)
    assert np.array_equal(gid, ids) and np.array_equal(gd2, d2)
    assert gid[0, 0] == 2


def test_bench_rejects_gpus_world_size_mismatch():
    """bench.py --gpus N under a launcher whose WORLD_SIZE disagrees refuses to run (it would
    otherwise time a different number of GPUs than the command line names)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--no-cpu"], cwd=root, capture_output=True,
                         text=True, timeout=300, env=env)
    assert out.returncode != 0 and "WORLD_SIZE=1" in (out.stderr + out.stdout)
