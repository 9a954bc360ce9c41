"""Workload sweeps, measured on one GPU: the DTW window (1/5/10/20% of n),
the series length at a fixed collection size, and the query noise of the tight-pruning
workload.  Each line: JSON with the config, queries/s (CUDA events around the batch call,
after warm-up) and the mean pruning counters.  Exactness of these paths is covered by the
parity tests (DTW reaches, lengths 16..2048, config-5 noise queries).

usage: python tools/sweep.py [--what dtw,length,noise] > profiles/r01_sweeps.jsonl
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
from paper_2110_07519_b200 import messi as M  # noqa: E402

DEV = torch.device("cuda:0")


def gen(N, n, seed):
    x = torch.empty((N, n), dtype=torch.float32, device=DEV)
    datagen.walks_cuda(x, 0, seed=seed)
    return x


def time_batch(idx, Q, reach, steps=2, warmup=1, knn=1):
    nq = Q.shape[0]
    res = M.result_buffer(nq * knn, DEV)
    stats = M.stats_buffer(nq, DEV)

    def step():
        if knn > 1:
            idx.query_batch_knn(Q, knn, res, stats)
        else:
            idx.query_batch(Q, reach, res, stats)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    st = M.decode_stats(stats)
    mean = {k: sum(s[k] for s in st) / len(st) for k in ("tiles_scanned", "coarse", "candidates", "lbk_pass",
                                                           "refined", "exact", "dtw_cells")}
    return nq / (ms / 1e3), ms, mean


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="dtw,length,noise,knn,dtw_length")
    a = ap.parse_args()
    what = a.what.split(",")
    if "dtw" in what:  # DTW window sweep, 10M x 256 (C4 collection), 20 queries
        X = gen(10_000_000, 256, datagen.DATA_SEED)
        Q = gen(20, 256, datagen.QUERY_SEED)
        torch.cuda.synchronize()
        idx = M.Index(X)
        for pct, r in ((1, 2), (5, 12), (10, 25), (20, 51)):
            qps, ms, mean = time_batch(idx, Q, r)
            print(json.dumps({"sweep": "dtw_window", "rows": 10_000_000, "n": 256, "window_pct": pct, "reach": r,
                              "queries": 20, "qps": qps, "ms_per_batch": ms, **mean}), flush=True)
        idx.close()
        del X, Q
        torch.cuda.empty_cache()
    if "dtw_length" in what:  # DTW at a 10% window, series length 128..2048 at 2.56 GB of rows, 10 queries
        for n in (128, 256, 512, 1024, 2048):
            N = 2_560_000_000 // (4 * n)
            X = gen(N, n, datagen.DATA_SEED)
            Q = gen(10, n, datagen.QUERY_SEED)
            torch.cuda.synchronize()
            idx = M.Index(X)
            r = n // 10
            qps, ms, mean = time_batch(idx, Q, r)
            print(json.dumps({"sweep": "dtw_length", "rows": N, "n": n, "reach": r, "queries": 10, "qps": qps,
                              "ms_per_batch": ms, **mean}), flush=True)
            idx.close()
            del X, Q
            torch.cuda.empty_cache()
    if "length" in what:  # ED, series length at 25.6 GB of rows, 100 queries
        for n in (128, 256, 512, 1024, 2048):
            N = 25_600_000_000 // (4 * n)
            X = gen(N, n, datagen.DATA_SEED)
            Q = gen(100, n, datagen.QUERY_SEED)
            torch.cuda.synchronize()
            idx = M.Index(X)
            qps, ms, mean = time_batch(idx, Q, None, steps=3)
            print(json.dumps({"sweep": "ed_length", "rows": N, "n": n, "gb": 4 * n * N / 1e9, "queries": 100,
                              "qps": qps, "ms_per_batch": ms, **mean}), flush=True)
            idx.close()
            del X, Q
            torch.cuda.empty_cache()
    if "noise" in what:  # ED, 100M x 128 (C5 collection), dataset rows + N(0, sigma^2) noise
        N = 100_000_000
        X = gen(N, 128, datagen.DATA_SEED)
        torch.cuda.synchronize()
        idx = M.Index(X)
        for sigma in (0.01, 0.05, 0.1):
            Q = torch.empty((100, 128), dtype=torch.float32, device=DEV)
            datagen.noisy_queries_cuda(Q, N, sigma=sigma)
            torch.cuda.synchronize()
            qps, ms, mean = time_batch(idx, Q, None, steps=3)
            print(json.dumps({"sweep": "ed_noise", "rows": N, "n": 128, "sigma": sigma, "queries": 100, "qps": qps,
                              "ms_per_batch": ms, **mean}), flush=True)
        idx.close()
        del X
        torch.cuda.empty_cache()
    if "knn" in what:  # exact k-NN on C2 (10M x 256)
        X = gen(10_000_000, 256, datagen.DATA_SEED)
        Q = gen(100, 256, datagen.QUERY_SEED)
        torch.cuda.synchronize()
        idx = M.Index(X)
        for k in (1, 5, 10, 50):
            qps, ms, mean = time_batch(idx, Q, None, steps=3, knn=k)
            print(json.dumps({"sweep": "ed_knn", "rows": 10_000_000, "n": 256, "k": k, "queries": 100, "qps": qps,
                              "ms_per_batch": ms, **mean}), flush=True)
        idx.close()


if __name__ == "__main__":
    main()
