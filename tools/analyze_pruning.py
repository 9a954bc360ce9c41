"""Pruning analysis at C3 (design experiment, not a test): per query, how many tiles / series
the box and iSAX bounds keep at the seed BSF vs at the final answer, and how many candidate
rows a quantised-row bound (int8 copy with per-row scale, error norm) would still send to the
exact fp32 refine.  Prints one JSON line per quantity summary.

usage: python tools/analyze_pruning.py [--rows N] [--queries Q]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
from paper_2110_07519_b200 import messi as M  # noqa: E402


def pct(x, ps=(50, 90, 99, 100)):
    t = torch.tensor(x, dtype=torch.float64)
    return {f"p{p}": float(torch.quantile(t, p / 100)) for p in ps} | {"mean": float(t.mean())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=100_000_000)
    ap.add_argument("--queries", type=int, default=100)
    ap.add_argument("--n", type=int, default=256)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    X = torch.empty((a.rows, a.n), dtype=torch.float32, device=dev)
    datagen.walks_cuda(X, 0, seed=datagen.DATA_SEED)
    Q = torch.empty((a.queries, a.n), dtype=torch.float32, device=dev)
    datagen.walks_cuda(Q, 0, seed=datagen.QUERY_SEED)
    torch.cuda.synchronize()
    idx = M.Index(X)
    res = M.result_buffer(a.queries, dev)
    stb = M.stats_buffer(a.queries, dev)
    idx.query_batch(Q, None, res, stb)
    torch.cuda.synchronize()
    st = M.decode_stats(stb)
    _, ids, d2 = M.decode_results(res)
    ntiles = (a.rows + 511) // 512
    eps = 1.0 + 2.0 ** -12
    # int8 copy: per-row scale s = max|x| / 127, q = round(x / s), err = ||x - s q||
    scale = torch.empty(a.rows, device=dev)
    for b in range(0, a.rows, 1 << 22):
        scale[b:b + (1 << 22)] = X[b:b + (1 << 22)].abs().amax(dim=1) / 127.0
    out = {k: [] for k in ("tiles_seed", "tiles_final", "cand_seed", "cand_final", "refined", "ratio",
                           "q8_pass_final", "q8_pass_seed", "ed_le_1p1", "tiles_final_half")}
    for i in range(a.queries):
        q = Q[i]
        tb = M.messi_debug_tile_bounds(idx.handle, q, -1, ntiles)
        lb = M.messi_debug_lower_bounds(idx.handle, q, -1, a.rows)
        s0, f = st[i]["seed_d2"], float(d2[i])
        out["tiles_seed"].append(int((tb <= s0 * eps).sum()))
        out["tiles_final"].append(int((tb <= f * eps).sum()))
        out["tiles_final_half"].append(int((tb <= 0.5 * (s0 + f) * eps).sum()))
        cs = torch.nonzero(lb <= s0 * eps).flatten()
        cf = torch.nonzero(lb <= f * eps).flatten()
        out["cand_seed"].append(cs.numel())
        out["cand_final"].append(cf.numel())
        out["refined"].append(st[i]["refined"])
        out["ratio"].append(s0 / f if f > 0 else 1.0)
        for name, c, thr in (("q8_pass_final", cf, f), ("q8_pass_seed", cs, s0)):
            rows = X[c]
            sc = scale[c]
            qi = torch.round(rows / sc[:, None]).clamp(-127, 127)
            deq = qi * sc[:, None]
            err = (rows.double() - deq.double()).norm(dim=1)
            dh = (deq.double() - q.double()[None]).norm(dim=1)
            lbq = (dh - err).clamp(min=0) ** 2
            out[name].append(int((lbq <= thr * eps).sum()))
            if name == "q8_pass_final":
                ed = ((rows.double() - q.double()[None]) ** 2).sum(1)
                out["ed_le_1p1"].append(int((ed <= 1.1 * f).sum()))
    for k, v in out.items():
        print(json.dumps({"quantity": k, **pct(v)}))
    print(json.dumps({"ntiles": ntiles, "rows": a.rows}))


if __name__ == "__main__":
    main()
