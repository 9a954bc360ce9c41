"""One TC pass on C2 (10M x 256) with 100 queries -- for ncu."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2110_07519_b200 import messi as M  # noqa: E402

N, n, nq = 10_000_000, 256, int(sys.argv[1]) if len(sys.argv) > 1 else 100
dev = torch.device("cuda:0")
X = torch.empty((N, n), dtype=torch.float32, device=dev)
datagen.walks_cuda(X, 0, seed=datagen.DATA_SEED)
Q = torch.empty((nq, n), dtype=torch.float32, device=dev)
datagen.walks_cuda(Q, 0, seed=datagen.QUERY_SEED)
idx = M.Index(X)
r = M.result_buffer(nq, dev)
for _ in range(3):
    idx.query_batch_tc(Q, r)
torch.cuda.synchronize()
print("ok", M.decode_results(r)[1][:4].tolist())
idx.close()
