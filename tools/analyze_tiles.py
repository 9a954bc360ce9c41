"""Design experiment (not a test): how many series a query must scan as a function of the
tile size of the box filter, and how many of them pass the 4-bit (cardinality-16) bound, at
the query's final BSF.  Uses the library's summaries, order and answers; bounds in fp64.

usage: python tools/analyze_tiles.py [--rows N] [--queries Q]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
from paper_2110_07519_b200 import messi as M  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=100_000_000)
    ap.add_argument("--queries", type=int, default=30)
    a = ap.parse_args()
    n = 256
    dev = torch.device("cuda:0")
    X = torch.empty((a.rows, n), dtype=torch.float32, device=dev)
    datagen.walks_cuda(X, 0, seed=datagen.DATA_SEED)
    Q = torch.empty((a.queries, n), dtype=torch.float32, device=dev)
    datagen.walks_cuda(Q, 0, seed=datagen.QUERY_SEED)
    torch.cuda.synchronize()
    idx = M.Index(X)
    res = M.result_buffer(a.queries, dev)
    idx.query_batch(Q, None, res, None)
    torch.cuda.synchronize()
    _, _, d2 = M.decode_results(res)
    sym, _ = M.messi_debug_summaries(idx.handle, a.rows, dev)
    _, perm = M.messi_debug_order(idx.handle, a.rows, dev)
    S = sym[perm.long()]  # sorted order
    del sym
    beta = torch.from_numpy(M.messi_debug_breakpoints(0).astype(np.float64)).to(dev)
    lo = torch.cat([torch.tensor([-np.inf], device=dev, dtype=torch.float64), beta])   # lo(v) = beta_v
    hi = torch.cat([beta, torch.tensor([np.inf], device=dev, dtype=torch.float64)])    # hi(v) = beta_{v+1}
    m = n // 16
    qbar = Q.double().view(a.queries, 16, m).mean(dim=2)
    out = {}
    sizes = [64, 128, 256, 512, 1024, 2048]
    for T in sizes:
        nt = a.rows // T
        Sb = S[:nt * T].view(nt, T, 16)
        bmin = Sb.min(dim=1).values.long()
        bmax = Sb.max(dim=1).values.long()
        kept = []
        for qi in range(a.queries):
            qb = qbar[qi]
            d = torch.clamp(torch.maximum(lo[bmin] - qb, qb - hi[bmax]), min=0)
            lb = m * (d * d).sum(dim=1)
            kept.append(int((lb <= float(d2[qi]) * (1 + 2 ** -12)).sum()) * T)
        out[T] = float(np.mean(kept))
        print(json.dumps({"tile": T, "series_in_kept_tiles_mean": out[T], "median": float(np.median(kept))}), flush=True)
    # 4-bit and 8-bit series bounds inside the kept 512-tiles, at the final BSF
    T = 512
    nt = a.rows // T
    Sb = S[:nt * T].view(nt, T, 16)
    bmin = Sb.min(dim=1).values.long()
    bmax = Sb.max(dim=1).values.long()
    c4, c8, ks = [], [], []
    for qi in range(a.queries):
        qb = qbar[qi]
        thr = float(d2[qi]) * (1 + 2 ** -12)
        d = torch.clamp(torch.maximum(lo[bmin] - qb, qb - hi[bmax]), min=0)
        keep = torch.nonzero(m * (d * d).sum(dim=1) <= thr).flatten()
        sub = Sb[keep].reshape(-1, 16).long()
        d8 = torch.clamp(torch.maximum(lo[sub] - qb, qb - hi[sub]), min=0)
        l8 = m * (d8 * d8).sum(dim=1)
        u = sub >> 4
        d4 = torch.clamp(torch.maximum(lo[16 * u] - qb, qb - hi[16 * u + 15]), min=0)
        l4 = m * (d4 * d4).sum(dim=1)
        ks.append(sub.shape[0])
        c8.append(int((l8 <= thr).sum()))
        c4.append(int((l4 <= thr).sum()))
    print(json.dumps({"kept_series": float(np.mean(ks)), "pass8": float(np.mean(c8)), "pass4": float(np.mean(c4)),
                      "pass4_over_pass8": float(np.sum(c4) / max(1, np.sum(c8)))}), flush=True)


if __name__ == "__main__":
    main()
