"""Multi-GPU sharding of the Falconn++ hot path.

One process per GPU, torch.distributed for the plumbing (NCCL on GPUs, gloo in
the CPU tests).  Shard g owns the contiguous global ids [g*n/G, (g+1)*n/G) and
builds its own index with ``id_offset`` so the ids it returns are global; every
GPU holds the same sign bitmasks (same seeds).  A query batch is replicated to
every rank, each rank answers from its shard, and the per-shard top-k lists are
merged after one all-gather with the reference's key order (score desc, id
asc), so ties still resolve to the lower global id.

Filter scope: ``per_shard`` applies the alpha/kappa filter inside each shard
(SURVEY 8(e) option A, the literal north-star reading); results then equal the
merge of per-shard oracles (tests/test_dist_gloo.py checks exactly that).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous id range of `rank` (sizes differ by at most one)."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return lo, hi


def merge_topk(scores: torch.Tensor, ids: torch.Tensor, k: int) -> tuple[torch.Tensor, torch.Tensor]:
    """Merge candidate lists [nq, m] into top-k by (score desc, id asc).

    Empty slots carry score -inf and id 0xFFFFFFFF (as int64) and sort last.
    """
    ids = ids.to(torch.int64)
    # stable two-pass sort: id asc, then score desc (stable keeps id order on ties)
    o1 = torch.argsort(ids, dim=1, stable=True)
    s1 = torch.gather(scores, 1, o1)
    i1 = torch.gather(ids, 1, o1)
    o2 = torch.argsort(s1, dim=1, descending=True, stable=True)
    s2 = torch.gather(s1, 1, o2)[:, :k]
    i2 = torch.gather(i1, 1, o2)[:, :k]
    return s2, i2


def allgather_merge(scores: torch.Tensor, ids: torch.Tensor, k: int, group=None):
    """All-gather per-rank [nq, k] lists and merge them (every rank gets the result)."""
    world = dist.get_world_size(group)
    if world == 1:
        return scores, ids.to(torch.int64)
    ids64 = ids.to(torch.int64)
    s_all = [torch.empty_like(scores) for _ in range(world)]
    i_all = [torch.empty_like(ids64) for _ in range(world)]
    dist.all_gather(s_all, scores.contiguous(), group=group)
    dist.all_gather(i_all, ids64.contiguous(), group=group)
    return merge_topk(torch.cat(s_all, dim=1), torch.cat(i_all, dim=1), k)
