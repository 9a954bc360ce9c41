"""bench.py's multi-rank path (torch.distributed.run, one process per rank, shards linked
over CUDA IPC, the exact merge) run end to end with 2 ranks sharing the one GPU of the box
(gloo process group: the driver's N-GPU runs use NCCL with one GPU per rank).  Checks that
rank 0 prints one well-formed JSON line for the 2-rank job."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_gloo():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--dist-backend", "gloo", "--rows", "4000000", "--queries", "32", "--steps", "3", "--warmup", "3",
           "--no-cpu", "--no-dtw", "--knn", "4"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["knn"]["value"] > 0
    assert d["config"]["parallelism"] == "row-shard x2"
    assert d["gpu_launches"] > 0 and d["e2e"]["value"] > 0


def test_bench_self_launch_two_ranks_matches_oracle(tmp_path):
    """`bench.py --gpus 2` WITHOUT a launcher (the driver's plain command): bench.py starts the
    two ranks itself (here sharing the box's one GPU over gloo; on an 8-GPU node one GPU per
    rank over NCCL), each rank builds its row shard, the shards are linked, and rank 0 dumps
    the merged (d2, gid) of the last timed step -- which must equal the oracle's brute force
    over the whole collection, bit for bit."""
    import numpy as np
    import torch

    import datagen
    import oracle
    dump = tmp_path / "merged.npz"
    rows, nq = 400_000, 16
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--dist-backend", "gloo", "--rows", str(rows),
           "--queries", str(nq), "--steps", "2", "--warmup", "3", "--repeats", "2", "--no-cpu", "--no-dtw",
           "--knn", "0", "--latency", "0", "--dump-results", str(dump)]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "row-shard x2" and d["repeats"]["n"] == 2
    got = np.load(dump)
    X = torch.empty((rows, 256), dtype=torch.float32, device="cuda")
    datagen.walks_cuda(X, 0, seed=datagen.DATA_SEED)
    Q = torch.empty((nq, 256), dtype=torch.float32, device="cuda")
    datagen.walks_cuda(Q, 0, seed=datagen.QUERY_SEED)
    d2, ids = oracle.nn("ed", X.cpu().numpy(), Q.cpu().numpy())
    assert np.array_equal(got["gid"], ids) and np.array_equal(got["d2"], d2)
