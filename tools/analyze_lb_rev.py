"""Design experiment (not a test, not the product): how much DTW refine work a second
lower bound would save at C4.  For each query, over the rows whose forward LB_Keogh (the
candidate's points against the query envelope, what the product filters on) is below the
final answer, it counts

  * how many the reverse LB_Keogh (the query's points against the CANDIDATE's envelope)
    rejects up front, and
  * the band rows the strip refine would compute (abandon tested every H rows at the final
    answer) with the current tail bound (forward LB_Keogh of the rows not done) and with the
    max of that and the reverse bound's suffix over the columns the rest of the path must
    still visit (i >= j0 + R),

the DTW rows simulated with plain torch ops on a sample of candidates.

usage: python tools/analyze_lb_rev.py [--rows N] [--queries Q] [--reach R] [--sample S]
"""
import argparse
import json
import os
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
from paper_2110_07519_b200 import messi as M  # noqa: E402


def envelope(x, r):
    """(U, L) of rows x [m, n]: max / min over |i - j| <= r."""
    up = F.max_pool1d(x.unsqueeze(1), 2 * r + 1, stride=1, padding=r).squeeze(1)
    lo = -F.max_pool1d(-x.unsqueeze(1), 2 * r + 1, stride=1, padding=r).squeeze(1)
    return up, lo


def block_envelope(x, r, B):
    """Superset envelope: for every point of block b (B points), the max / min over the
    blocks that any of its windows touches."""
    m, n = x.shape
    nb = n // B
    bm = x.view(m, nb, B).amax(2)
    bn = x.view(m, nb, B).amin(2)
    up = torch.empty_like(bm)
    lo = torch.empty_like(bn)
    for b in range(nb):
        a0 = max(0, (B * b - r) // B)
        a1 = min(nb - 1, (B * b + B - 1 + r) // B)
        up[:, b] = bm[:, a0:a1 + 1].amax(1)
        lo[:, b] = bn[:, a0:a1 + 1].amin(1)
    return up.repeat_interleave(B, 1), lo.repeat_interleave(B, 1)


def quant_halfstep(x):
    """s / 2 of k_quantise's scale (127 s >= max |x|, s a power of two)."""
    mx = x.abs().amax(1)
    k = torch.ceil(torch.log2(mx / 127.0))
    return 0.5 * torch.exp2(k)


def lbk_terms(x, up, lo):
    return torch.clamp(x - up, min=0) ** 2 + torch.clamp(lo - x, min=0) ** 2


def dtw_rowmins(c, q, r):
    """Row minima of the banded DTW matrix D(j, i), rows j = candidate points, [m, n]."""
    m, n = c.shape
    inf = float("inf")
    prev = torch.full((m, 2 * r + 3), inf, device=c.device)  # slot k+r+1 = column (j-1)+k, k in [-r, r]
    mins = torch.empty((m, n), device=c.device)
    cur = prev
    for j in range(n):
        cur = torch.full((m, 2 * r + 3), inf, device=c.device)
        for k in range(-r, r + 1):
            i = j + k
            if i < 0 or i >= n:
                continue
            d = (q[i] - c[:, j]) ** 2
            if j == 0 and i == 0:
                best = torch.zeros(m, device=c.device)
            else:
                best = torch.minimum(torch.minimum(prev[:, k + r + 1], prev[:, k + r + 2]), cur[:, k + r])
            cur[:, k + r + 1] = d + best
        mins[:, j] = cur.min(dim=1).values
        prev = cur
    fin = cur[:, r + 1]  # D(n-1, n-1)
    return mins, fin


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=10_000_000)
    ap.add_argument("--queries", type=int, default=8)
    ap.add_argument("--reach", type=int, default=25)
    ap.add_argument("--sample", type=int, default=20000)
    ap.add_argument("--H", type=int, default=8)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    n, R, H = 256, a.reach, a.H
    X = torch.empty((a.rows, n), dtype=torch.float32, device=dev)
    datagen.walks_cuda(X, 0, seed=datagen.DATA_SEED)
    Q = torch.empty((a.queries, n), dtype=torch.float32, device=dev)
    datagen.walks_cuda(Q, 0, seed=datagen.QUERY_SEED)
    torch.cuda.synchronize()
    idx = M.Index(X)
    res = M.result_buffer(a.queries, dev)
    stb = M.stats_buffer(a.queries, dev)
    idx.query_batch(Q, R, res, stb)
    torch.cuda.synchronize()
    _, ids, d2 = M.decode_results(res)
    st = M.decode_stats(stb)
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    out = []
    for qi in range(a.queries):
        q = Q[qi]
        bsf = float(d2[qi])
        seed = float(st[qi]["seed_d2"])
        qu, ql = envelope(q[None], R)
        fwd = torch.empty(a.rows, device=dev)
        for s in range(0, a.rows, 1 << 20):
            fwd[s:s + (1 << 20)] = lbk_terms(X[s:s + (1 << 20)], qu, ql).sum(1)
        cand = torch.nonzero(fwd <= max(bsf, seed)).flatten()
        C = X[cand]
        cu, cl = envelope(C, R)
        hs = quant_halfstep(C)[:, None]
        rev_terms = lbk_terms(q[None].expand_as(C), cu + hs, cl - hs)
        rev = rev_terms.sum(1)
        keep_rev = rev <= bsf
        blk = {}
        sp = fwd[cand] <= seed
        qa = q.abs()
        for name, msk in (("even", torch.arange(n, device=dev) % 2 == 0),
                          ("top50", qa >= qa.median()), ("top25", qa >= qa.quantile(0.75)),
                          ("half0", torch.arange(n, device=dev) < n // 2)):
            rs = (rev_terms * msk[None].float()).sum(1)
            blk[f"rej_seed_{name}"] = int((sp & (rs > seed)).sum())
        ratio = rev[sp] / seed
        blk["rev_over_thr_p10_p50"] = [float(ratio.quantile(0.1)), float(ratio.quantile(0.5))]
        fpass = fwd[cand] <= bsf
        seed_pass = fwd[cand] <= seed
        for B in (4, 8):
            bu, bl = block_envelope(C, R, B)
            rb = lbk_terms(q[None].expand_as(C), bu + hs, bl - hs).sum(1)
            blk[f"rev_reject_blk{B}"] = int((fpass & (rb > bsf)).sum())
            blk[f"rev_reject_blk{B}_seed"] = int((seed_pass & (rb > seed)).sum())
        # sampled abandon depths
        fidx = torch.nonzero(fwd[cand] <= bsf).flatten()
        pick = min(fidx.numel(), a.sample)
        sel = fidx[torch.randperm(fidx.numel(), generator=g, device=dev)[:pick]]
        Cs = C[sel]
        mins, fin = dtw_rowmins(Cs, q, R)
        ft = lbk_terms(Cs, qu, ql)
        fsuf = torch.flip(torch.cumsum(torch.flip(ft, [1]), 1), [1])  # fsuf[:, j] = sum_{t >= j}
        fsuf = torch.cat([fsuf, torch.zeros((pick, 1), device=dev)], 1)
        rsuf = torch.flip(torch.cumsum(torch.flip(rev_terms[sel], [1]), 1), [1])
        rsuf = torch.cat([rsuf, torch.zeros((pick, R + H + 2), device=dev)], 1)
        rows_a = torch.full((pick,), n, device=dev)
        rows_b = torch.full((pick,), n, device=dev)
        rows_b[~keep_rev[sel]] = 0
        done_a = torch.zeros(pick, dtype=torch.bool, device=dev)
        done_b = ~keep_rev[sel]
        for j0 in range(H, n + 1, H):
            rm = mins[:, j0 - 1]
            ba = rm + fsuf[:, j0] > bsf
            bb = rm + torch.maximum(fsuf[:, j0], rsuf[:, min(j0 + R, n)]) > bsf
            ab = ba & ~done_a
            rows_a[ab] = j0
            done_a |= ba
            bbn = bb & ~done_b
            rows_b[bbn] = j0
            done_b |= bb
        r = {"q": qi, "bsf": bsf, "seed": seed, "fwd_pass_seed": int(seed_pass.sum()),
             "rev_reject_seed": int((seed_pass & (rev > seed)).sum()), **blk,
             "fwd_pass": int(fpass.sum()), "rev_reject": int((fpass & ~keep_rev).sum()),
             "both_pass": int((fpass & keep_rev).sum()), "sample": pick,
             "rows_fwd_tail": float(rows_a.float().mean()), "rows_max_tail": float(rows_b.float().mean()),
             "rows_fwd_tail_filtered": float(torch.where(keep_rev[sel], rows_a, torch.zeros_like(rows_a)).float().mean()),
             "dtw_le_bsf": int((fin <= bsf * (1 + 2 ** -10)).sum())}
        out.append(r)
        print(json.dumps(r), flush=True)
    tot = {k: sum(r[k] for r in out) / len(out) for k in out[0] if k not in ("q", "bsf", "seed", "sample")}
    tot["work_ratio"] = sum(r["fwd_pass"] * r["rows_max_tail"] for r in out) / \
        sum(r["fwd_pass"] * r["rows_fwd_tail"] for r in out)
    tot["work_ratio_filter_only"] = sum(r["fwd_pass"] * r["rows_fwd_tail_filtered"] for r in out) / \
        sum(r["fwd_pass"] * r["rows_fwd_tail"] for r in out)
    print(json.dumps(tot))


if __name__ == "__main__":
    main()
