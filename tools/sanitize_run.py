"""Small end-to-end run of every query path for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per gpurun call): C1-shaped data (20,000 x 256), ED 1-NN batch (two
launch groups), ED k-NN (lane and warp inserts), DTW 1-NN at reaches served by the strip,
band and warp kernels (four slots in flight), DTW k-NN, three linked shards of one process
(shared best-so-far over peer memory), and the inspection calls.  Exits non-zero on a wrong
answer count (answers are checked by the parity tests, not here)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2110_07519_b200 import messi as M  # noqa: E402

dev = torch.device("cuda:0")
N, n = 20_000, 256
X = torch.empty((N, n), dtype=torch.float32, device=dev)
datagen.walks_cuda(X, 0, seed=datagen.DATA_SEED)
Q = torch.empty((130, n), dtype=torch.float32, device=dev)
datagen.walks_cuda(Q, 0, seed=datagen.QUERY_SEED)
torch.cuda.synchronize()
idx = M.Index(X)
res = M.result_buffer(130 * 20, dev)
st = M.stats_buffer(130, dev)
idx.query_batch(Q, None, res, st)                       # ED, two launch groups (128 + 2)
idx.query_batch_knn(Q[:8].contiguous(), 5, res)          # ED k-NN, lane insert
idx.query_batch_knn(Q[:4].contiguous(), 20, res)         # ED k-NN, warp insert
for r in (25, 5, 0):                                      # strip, register band, warp refine
    idx.query_batch(Q[:6].contiguous(), r, res, st)
idx.query_batch_knn(Q[:4].contiguous(), 7, res, reach=12)  # DTW k-NN
if os.environ.get("SAN_TC", "1") == "1":
    idx.query_batch_tc(Q, res, st)                        # tensor-core batched path
torch.cuda.synchronize()
print("single:", idx.query_ed(Q[0])[1], idx.query_dtw(Q[1], 25)[1], idx.query_knn(Q[2], 3)[1][0])
# inspection calls (the same kernels with thresholds at +inf)
ids = torch.arange(0, N, 37, dtype=torch.int32, device=dev)
M.messi_debug_lower_bounds(idx.handle, Q[0].contiguous(), -1, N)
M.messi_debug_tile_bounds(idx.handle, Q[0].contiguous(), -1, (N + 511) // 512)
M.messi_debug_ed_refine(idx.handle, Q[0].contiguous(), ids)
M.messi_debug_dtw_stages(idx.handle, Q[0].contiguous(), 25, ids)
# three linked shards of one process
parts = [X[i * N // 3:(i + 1) * N // 3].contiguous() for i in range(3)]
shards = [M.Index(p, row_begin=i * N // 3) for i, p in enumerate(parts)]
for i, s in enumerate(shards):
    M.messi_link_peers_local(s.handle, [t.handle for j, t in enumerate(shards) if j != i])
outs = []
for s in shards:
    r = M.result_buffer(16, dev)
    s.query_batch(Q[:16].contiguous(), None, r)
    outs.append(r)
torch.cuda.synchronize()
for s in shards:
    s.close()
idx.close()
print("sanitize run ok")
