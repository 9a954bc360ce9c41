"""Design experiment (not a test): DTW pruning at C4 -- how many rows pass the envelope-PAA
bound and the raw LB_Keogh at the seed BSF vs at the final answer, and how good the best of
the K smallest-LB_env candidates is as a seed.

usage: python tools/analyze_dtw.py [--rows N] [--queries Q] [--reach R]
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
    ap.add_argument("--rows", type=int, default=10_000_000)
    ap.add_argument("--queries", type=int, default=20)
    ap.add_argument("--reach", type=int, default=25)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    X = torch.empty((a.rows, 256), dtype=torch.float32, device=dev)
    datagen.walks_cuda(X, 0, seed=datagen.DATA_SEED)
    Q = torch.empty((a.queries, 256), dtype=torch.float32, device=dev)
    datagen.walks_cuda(Q, 0, seed=datagen.QUERY_SEED)
    torch.cuda.synchronize()
    idx = M.Index(X)
    res = M.result_buffer(a.queries, dev)
    stb = M.stats_buffer(a.queries, dev)
    idx.query_batch(Q, a.reach, res, stb)
    torch.cuda.synchronize()
    st = M.decode_stats(stb)
    _, ids, d2 = M.decode_results(res)
    eps = 1 + 2 ** -12
    rec = []
    for i in range(a.queries):
        q = Q[i].contiguous()
        lb = M.messi_debug_lower_bounds(idx.handle, q, a.reach, a.rows)
        s0, f = st[i]["seed_d2"], float(d2[i])
        cs = torch.nonzero(lb <= s0 * eps).flatten()
        cf = torch.nonzero(lb <= f * eps).flatten()
        # LB_Keogh of the seed candidates
        lbk = torch.empty(cs.numel(), dtype=torch.float32, device=dev)
        ci = cs.to(torch.int32).contiguous()
        M._check(M.lib().messi_debug_distances(idx.handle, M._ptr(q), a.reach, M._ptr(ci), ci.numel(), None, None,
                                               M._ptr(lbk)))
        order = torch.argsort(lb[cs])
        r = {"seed": s0, "final": f, "cand_seed": cs.numel(), "cand_final": cf.numel(),
             "lbk_seed": int((lbk <= s0 * eps).sum()), "lbk_final": int((lbk <= f * eps).sum())}
        for K in (256, 1024, 4096):
            top = cs[order[:K]].to(torch.int32)
            _, d64, _ = M.messi_debug_distances(idx.handle, q, a.reach, top)
            r[f"best_of_top{K}"] = float(d64.min())
        rec.append(r)
        print(json.dumps(r), flush=True)
    keys = [k for k in rec[0] if k not in ("seed", "final")]
    print(json.dumps({k: float(np.mean([x[k] for x in rec])) for k in keys}))
    print(json.dumps({"ratio_seed_final": float(np.mean([x["seed"] / x["final"] for x in rec])),
                      **{f"ratio_top{K}_final": float(np.mean([x[f"best_of_top{K}"] / x["final"] for x in rec]))
                         for K in (256, 1024, 4096)}}))


if __name__ == "__main__":
    main()
