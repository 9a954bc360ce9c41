"""Row sharding and the cross-GPU exact merge (north_star: "each GPU returns a
local (dist, id) minimum, which NCCL all-reduces").

Rank g owns the contiguous global rows [shard_range(N, G, g)); its index is built with
row_begin = the first of them, so its local answer already carries the global id.  The
merge is the lexicographic min over ranks of (exact fp64 d2, global id) -- ties go to the
lowest id, as in the single-GPU answer -- done with ONE all_gather of 16 B per query per
rank (NCCL over NVLink on GPUs, gloo on CPU), batched over all queries of a step.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(N: int, world: int, rank: int):
    """[begin, end) of the rows rank `rank` owns out of N, contiguous, sizes differ by <= 1."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return (N * rank) // world, (N * (rank + 1)) // world


def lexmin(d2: torch.Tensor, gid: torch.Tensor):
    """Per column of [R, nq] candidates: the (d2, gid) lexicographic minimum (gid < 0 = none)."""
    d2 = torch.where(gid < 0, torch.full_like(d2, float("inf")), d2)
    best = d2.min(dim=0).values
    big = torch.iinfo(torch.int64).max
    cand = torch.where((d2 == best.unsqueeze(0)) & (gid >= 0), gid, torch.full_like(gid, big))
    bid = cand.min(dim=0).values
    bid = torch.where(bid == big, torch.full_like(bid, -1), bid)
    return best, bid


def merge_results(d2: torch.Tensor, gid: torch.Tensor, group=None):
    """Exact cross-rank merge of per-query local bests.  d2: float64 [nq], gid: int64 [nq] on
    the process group's device.  Returns (d2, gid) of the global answers on every rank."""
    world = dist.get_world_size(group)
    packed = torch.stack([d2.contiguous().view(torch.int64), gid.to(torch.int64)], dim=1).contiguous()
    home = packed.device
    if dist.get_backend(group) == "gloo" and packed.is_cuda:  # gloo exchanges host tensors
        packed = packed.cpu()
    parts = [torch.empty_like(packed) for _ in range(world)]
    dist.all_gather(parts, packed, group=group)
    allp = torch.stack(parts).to(home)  # [R, nq, 2]
    return lexmin(allp[:, :, 0].contiguous().view(torch.float64), allp[:, :, 1])


def link_shards(index, group=None):
    """Let the shards of this process group share each query's best-so-far during the
    batched ED kernels and the DTW path (include/messi.h, messi_link_peers_ipc): every rank
    publishes the CUDA IPC handles of its per-query state arrays, and opens those of all other
    ranks (their GPUs' memory, reached over NVLink).  Collective: every rank calls it, once per
    index; afterwards the ranks make the same query calls."""
    from . import messi as M
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    # sets 0, 1: the batched ED path's per-query states; 2: the DTW path's slot states
    mine = tuple(M.messi_batch_state_ipc(index.handle, s) for s in (0, 1, 2))
    allh = [None] * world
    dist.all_gather_object(allh, mine, group=group)
    peers = [allh[r] for r in range(world) if r != me]
    M.messi_link_peers_ipc(index.handle, peers)
    return len(peers)


def merge_knn(d2: torch.Tensor, gid: torch.Tensor, group=None):
    """Exact cross-rank k-NN merge: d2 float64 [nq, k], gid int64 [nq, k] (local answers, -1 =
    none) -> the k lexicographically smallest (d2, gid) of all ranks, per query."""
    world = dist.get_world_size(group)
    nq, k = d2.shape
    packed = torch.stack([d2.contiguous().view(torch.int64), gid.to(torch.int64)], dim=2).contiguous()
    home = packed.device
    if dist.get_backend(group) == "gloo" and packed.is_cuda:
        packed = packed.cpu()
    parts = [torch.empty_like(packed) for _ in range(world)]
    dist.all_gather(parts, packed, group=group)
    allp = torch.cat(parts, dim=1).to(home)  # [nq, R k, 2]
    ad = allp[:, :, 0].contiguous().view(torch.float64)
    ag = allp[:, :, 1]
    ad = torch.where(ag < 0, torch.full_like(ad, float("inf")), ad)
    big = torch.iinfo(torch.int64).max
    ag2 = torch.where(ag < 0, torch.full_like(ag, big), ag)
    # lexicographic: sort by id, then stable sort by distance
    o1 = torch.argsort(ag2, dim=1, stable=True)
    ad1, ag1 = torch.gather(ad, 1, o1), torch.gather(ag2, 1, o1)
    o2 = torch.argsort(ad1, dim=1, stable=True)
    bd, bi = torch.gather(ad1, 1, o2)[:, :k], torch.gather(ag1, 1, o2)[:, :k]
    bi = torch.where(bi == big, torch.full_like(bi, -1), bi)
    return bd, bi
