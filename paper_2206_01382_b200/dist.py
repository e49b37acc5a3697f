"""Multi-GPU sharding of the Falconn++ hot path.

One process per GPU, torch.distributed for the plumbing (NCCL on GPUs, gloo in
the CPU tests).  Shard g owns the contiguous global ids [g*n/G, (g+1)*n/G) and
builds its own index with ``id_offset`` so the ids it returns are global; every
GPU holds the same sign bitmasks (same seeds).  A query batch is replicated to
every rank; stage A (hashing + probe selection) is split across the ranks and
the probe sets all-gathered (sharded_query), each rank answers from its shard,
and the per-shard top-k lists are merged after one all-gather with the
reference's key order (score desc, id asc) by the library's k-way merge kernel
(fpp_merge_topk), so ties still resolve to the lower global id.

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
    """Merge candidate lists [nq, m] into top-k by (score desc, id asc) -- the host
    (CPU-tensor) form used by the gloo tests with the oracle as the shard engine.
    CUDA tensors go through the device k-way merge kernel (merge_lists).

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


def merge_lists(s_all: torch.Tensor, i_all: torch.Tensor, k: int):
    """[G, nq, k] gathered shard lists -> merged [nq, k] (score desc, id asc).
    CUDA: the library's k-way merge kernel (fpp_merge_topk); CPU: merge_topk."""
    if s_all.is_cuda:
        import paper_2206_01382_b200 as fpp
        i32 = i_all if i_all.dtype == torch.int32 else i_all.to(torch.int32)
        ms, mi = fpp.merge_topk_device(s_all.contiguous(), i32.contiguous(), k,
                                       stream=torch.cuda.current_stream(s_all.device).cuda_stream)
        return ms, mi
    G, nq, kk = s_all.shape
    return merge_topk(s_all.permute(1, 0, 2).reshape(nq, G * kk),
                      i_all.to(torch.int64).permute(1, 0, 2).reshape(nq, G * kk), k)


def _backend(group=None) -> str:
    return dist.get_backend(group) if dist.is_initialized() else "none"


def all_gather_stacked(t: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather `t` from every rank into [G, *t.shape] (rank-major).  With NCCL the
    CUDA tensor is gathered in place over NVLink; with gloo (CPU tests, or several
    ranks sharing one GPU) it is staged through host memory."""
    world = dist.get_world_size(group)
    t = t.contiguous()
    if t.is_cuda and _backend(group) == "gloo":
        return all_gather_stacked(t.cpu(), group).to(t.device)
    out = torch.empty(world * t.numel(), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, t.reshape(-1), group=group)
    return out.view((world,) + tuple(t.shape))


def all_reduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    if t.is_cuda and _backend(group) == "gloo":
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        t.copy_(h)
        return t
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def allgather_merge(scores: torch.Tensor, ids: torch.Tensor, k: int, group=None):
    """All-gather per-rank [nq, k] lists and merge them (every rank gets the result)."""
    world = dist.get_world_size(group)
    if world == 1:
        return scores, ids.to(torch.int64)
    if scores.is_cuda:
        i32 = ids if ids.dtype in (torch.int32,) else ids.to(torch.int32)
        s_all = all_gather_stacked(scores, group)
        i_all = all_gather_stacked(i32, group)
        return merge_lists(s_all, i_all, k)
    ids64 = ids.to(torch.int64)
    s_all = [torch.empty_like(scores) for _ in range(world)]
    i_all = [torch.empty_like(ids64) for _ in range(world)]
    dist.all_gather(s_all, scores.contiguous(), group=group)
    dist.all_gather(i_all, ids64.contiguous(), group=group)
    return merge_topk(torch.cat(s_all, dim=1), torch.cat(i_all, dim=1), k)


def query_slice(nq: int, world: int, rank: int) -> tuple[int, int]:
    """Rank `rank`'s slice of a query batch for the stage-A split: equal slices of
    ceil(nq / world) rows (the last ones shorter or empty), so the gathered
    [world, per, P_eff] probe sets viewed as [world * per, P_eff] start with the
    batch's [nq, P_eff] in order."""
    per = -(-nq // world) if nq else 0
    return min(nq, rank * per), min(nq, (rank + 1) * per)


class GpuQueryEngine:
    """The rank's GPU index as a stage-A / stage-B engine (tensors on its device)."""

    def __init__(self, ix, stream=None):
        self.ix, self.stream = ix, stream

    def peff(self, qprobes: int) -> int:
        return self.ix.peff(qprobes)

    def probe_sets(self, Q, qprobes, out):
        self.ix.query_probe_sets_device(Q, qprobes, probes=out, stream=self.stream)

    def from_probe_sets(self, Q, probes, k, qprobes, ids, scores, stats=None):
        self.ix.query_from_probe_sets_device(Q, probes, ids, scores, k, qprobes, stats=stats,
                                             stream=self.stream)


def sharded_query_engine(engine, Q: torch.Tensor, ids: torch.Tensor, scores: torch.Tensor, k: int,
                         qprobes: int, group=None, stats=None):
    """Sharded batch query with stage A split across the ranks.

    Every rank holds the whole (replicated) batch Q and one shard.  Rank r computes the
    probe sets of its slice only (hashing and probe selection: the part of the query
    that does not depend on the shard); one all-gather gives every rank all probe sets
    (u32 bucket ids, P_eff per query); each rank resolves them in its own tables and
    runs stage B on the whole batch into ids/scores; the per-rank top-k lists are
    merged after an all-gather (score desc, id asc).  Returns the merged (scores, ids)
    on every rank.  Equals the replicated path (every rank running the whole query)
    because probe sets depend only on the queries and the hash functions, which all
    shards share.  `engine`: GpuQueryEngine, or the oracle engine of the CPU tests."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    nq = Q.shape[0]
    pe = engine.peff(qprobes)
    per = -(-nq // world) if nq else 0
    lo, hi = query_slice(nq, world, rank)
    mine = torch.zeros((per, pe), dtype=torch.int32, device=Q.device)
    if hi > lo:
        engine.probe_sets(Q[lo:hi], qprobes, mine[:hi - lo])
    if world > 1:
        allp = all_gather_stacked(mine, group).view(world * per, pe)[:nq]
    else:
        allp = mine[:nq]
    engine.from_probe_sets(Q, allp, k, qprobes, ids, scores, stats)
    return allgather_merge(scores, ids, k, group)


def sharded_query(ix, Qd, ids, scores, k: int, qprobes: int, group=None, stream=None, stats=None):
    """sharded_query_engine on the rank's GPU index (bench.py --gpus N)."""
    return sharded_query_engine(GpuQueryEngine(ix, stream), Qd, ids, scores, k, qprobes, group,
                                stats)


# ---------------------------------------------------------------------------
# Global-filter sharded build (SURVEY.md 8(e) option B): the union of the
# shard indexes equals the 1-GPU index exactly, for every G.
#   1. every rank hashes its shard and histograms (table, bucket) sizes;
#   2. all-reduce(sum) of the histograms -> the global bucket sizes B_g;
#   3. each rank writes min(keep(B_g), B_local) of its sorted bucket prefix
#      into globally agreed slots (sum_b keep(B_g), padded) -> all-gather;
#   4. per bucket the global cut = keep(B_g)-th smallest (score desc, id asc)
#      key of the gathered prefixes; each rank keeps its entries <= cut.
# The engine is the GPU library (GpuShardEngine) or, in the CPU tests, the
# oracle (tests/test_dist_gloo.py::OracleShardEngine).
# ---------------------------------------------------------------------------


class GpuShardEngine:
    """Phases of fpp_shard_* on the rank's GPU; tensors are CUDA torch tensors."""

    def __init__(self, X, id_offset: int, **params):
        import paper_2206_01382_b200 as fpp
        self.ix = fpp.Index.shard_begin(X, id_offset=id_offset, **params)
        self.device = X.device if getattr(X, "is_cuda", False) else torch.device("cuda", max(params.get("device", 0), 0))

    def hist(self) -> torch.Tensor:
        h = torch.empty(self.ix.shard_hist_len(), dtype=torch.int32, device=self.device)
        self.ix.shard_hist(h.data_ptr())
        return h

    def slots(self, ghist: torch.Tensor) -> int:
        return self.ix.shard_slots(ghist.data_ptr())

    def prefix(self, ghist: torch.Tensor, slots: int) -> torch.Tensor:
        p = torch.empty(max(slots, 1), dtype=torch.int64, device=self.device)
        self.ix.shard_prefix(ghist.data_ptr(), p.data_ptr())
        return p[:slots]

    def finish(self, ghist: torch.Tensor, all_prefix: torch.Tensor, world: int):
        self.ix.shard_finish(ghist.data_ptr(), all_prefix.data_ptr(), world)
        return self.ix


def build_global_filter(engine, group=None):
    """Run the exchange protocol over torch.distributed; returns engine.finish()."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    h = engine.hist()
    if world > 1:
        all_reduce_sum(h, group)
    slots = engine.slots(h)
    pre = engine.prefix(h, slots)
    if world > 1:
        allp = all_gather_stacked(pre, group).reshape(-1)
    else:
        allp = pre
    return engine.finish(h, allp, world)
