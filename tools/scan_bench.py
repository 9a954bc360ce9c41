"""Isolated coarse-scan throughput (tuning aid): python tools/scan_bench.py [rows] [reps]
Prints GB/s of algorithmic bytes (8 B/series + 8 B/survivor) and the fraction of the measured
HBM peak.  MESSI_LIB selects a library variant."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2110_07519_b200 import messi as M  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
X = torch.empty((rows, 256), dtype=torch.float32, device="cuda")
datagen.walks_cuda(X, 0)
Q = torch.empty((1, 256), dtype=torch.float32, device="cuda")
datagen.walks_cuda(Q, 0, seed=1)
torch.cuda.synchronize()
idx = M.Index(X)
M.messi_debug_scan_repeat(idx.handle, Q[0], 3)
ms, c, tiles = M.messi_debug_scan_repeat(idx.handle, Q[0], reps)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
gbs = (8192 * tiles + 8 * c) * reps / (ms / 1e3) / 1e9
print(json.dumps({"lib": os.environ.get("MESSI_LIB", "default"), "rows": rows, "us_per_scan": 1e3 * ms / reps,
                  "GBps": gbs, "frac": gbs / peak, "candidates": c, "tiles": tiles,
                  "tile_frac": tiles / ((rows + 511) // 512)}))
