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
