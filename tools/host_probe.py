"""Host enqueue cost of the DTW batch path: time for messi_query_dtw_batch (100 queries) to
return (host) vs the device time of the same step (CUDA events), C4 shape."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen
from paper_2110_07519_b200 import messi as M

N = int(os.environ.get("PROBE_N", 10_000_000))
dev = torch.device("cuda:0")
X = datagen.walks_cuda(torch.empty((N, 256), dtype=torch.float32, device=dev), 0, seed=0)
Q = datagen.walks_cuda(torch.empty((100, 256), dtype=torch.float32, device=dev), 0, seed=1)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    idx = M.Index(X, stream=s)
    res, st = M.result_buffer(100, dev), M.stats_buffer(100, dev)
    for _ in range(3):
        idx.query_batch(Q, 25, res, st)
    torch.cuda.synchronize()
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        t0 = time.perf_counter()
        idx.query_batch(Q, 25, res, st)
        t1 = time.perf_counter()
        b.record(s)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print("enqueue %.2f ms  host total %.2f ms  device %.2f ms" % ((t1 - t0) * 1e3, (t2 - t0) * 1e3, a.elapsed_time(b)))
