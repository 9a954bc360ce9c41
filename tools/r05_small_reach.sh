# Round 2 (session 5): strip pipeline at every reach >= 1 by default: reach 2 / 5 timing both ways
# (10M x 256, 20 queries), then the DTW suites
python - <<'PY'
import os, sys, json, subprocess
code = r'''
import sys, torch
sys.path.insert(0, ".")
import datagen
from paper_2110_07519_b200 import messi as M
dev = torch.device("cuda:0")
X = torch.empty((10_000_000, 256), dtype=torch.float32, device=dev); datagen.walks_cuda(X, 0, seed=datagen.DATA_SEED)
Q = torch.empty((20, 256), dtype=torch.float32, device=dev); datagen.walks_cuda(Q, 0, seed=datagen.QUERY_SEED)
idx = M.Index(X); res = M.result_buffer(20, dev)
for reach in (2, 5):
    for _ in range(2): idx.query_batch(Q, reach, res)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3): idx.query_batch(Q, reach, res)
    b.record(); torch.cuda.synchronize()
    print("reach", reach, "q/s", round(60 / (a.elapsed_time(b) * 1e-3)))
'''
for env in ({}, {"MESSI_DTW_STRIP": "0"}, {}, {"MESSI_DTW_STRIP": "0"}):
    print(env, subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True).stdout.strip().replace("\n", "; "))
PY
timeout 1500 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_knn_dtw.py tests/test_gpu_shards.py "tests/test_gpu_fullsize.py::test_config4_dtw_10m" > gpurun_out/dtwtests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/dtwtests.log
