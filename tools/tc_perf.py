"""Tensor-core batched path vs the LUT batch path: q/s on one collection for several query counts."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2110_07519_b200 import messi as M  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
noisy = len(sys.argv) > 3 and sys.argv[3] == "noisy"
dev = torch.device("cuda:0")
X = torch.empty((N, n), dtype=torch.float32, device=dev)
datagen.walks_cuda(X, 0, seed=datagen.DATA_SEED)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    idx = M.Index(X, stream=s)
    out = {"N": N, "n": n, "noisy": noisy}
    for nq in (100, 256, 1000):
        Q = torch.empty((nq, n), dtype=torch.float32, device=dev)
        if noisy:
            datagen.noisy_queries_cuda(Q, N, sigma=0.1)
        else:
            datagen.walks_cuda(Q, 0, seed=datagen.QUERY_SEED)
        torch.cuda.synchronize()
        r1, r2 = M.result_buffer(nq, dev), M.result_buffer(nq, dev)
        st = M.stats_buffer(nq, dev)
        for name, fn in (("lut", lambda: idx.query_batch(Q, None, r1)), ("tc", lambda: idx.query_batch_tc(Q, r2, st))):
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(5):
                fn()
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            out[f"{name}_{nq}"] = {"ms": ms, "qps": nq / ms * 1e3}
        M.messi_profile_enable(idx.handle, True)
        idx.query_batch_tc(Q, r2, st)
        kms = M.messi_profile_read(idx.handle, "scan")[0]
        M.messi_profile_enable(idx.handle, False)
        a, b = M.decode_results(r1), M.decode_results(r2)
        sts = M.decode_stats(st)
        out[f"tc_{nq}"].update({"kernel_ms": kms, "same_answers": bool(torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])),
                                "cand_mean": sum(x["candidates"] for x in sts) / nq,
                                "exact_mean": sum(x["exact"] for x in sts) / nq,
                                "rows8_gbs": N * n / (kms / 1e3) / 1e9,
                                "int8_tops": 2.0 * N * n * nq / (kms / 1e3) / 1e12})
    print(json.dumps(out))
    idx.close()
