"""Multi-GPU host logic (paper_2206_01382_b200/dist.py) on CPU: world_size 2, gloo.

Each rank owns the contiguous id shard [g*n/G, (g+1)*n/G), builds its shard
index (here with the CPU oracle standing in for the per-GPU engine; the GPU
engine is bit-identical to it per tests/test_gpu_parity.py), answers the
replicated query batch, and the per-rank top-k lists are merged after an
all-gather with the (score desc, global id asc) order.  Checks:
  * the merge equals the single-process merge of the per-shard results;
  * with exhaustive probing of unfiltered shards the sharded answer equals the
    global brute force (ties resolved to the lower global id across shards).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_01382_b200 import dist as fdist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def make(n, d, nq):
    from oracle import oracle as orc
    X = orc.normalize(orc.synth(n, d, 6, 0.3, seed=2))
    Q = orc.normalize(orc.synth(nq, d, 6, 0.3, seed=2, stream=1))
    X[n - 1] = X[1]  # a duplicate across the shard boundary: tie -> lower global id
    return X, Q


def shard_answer(X, Q, lo, hi, cfg, k):
    from oracle import oracle as orc
    ox = orc.Index(X[lo:hi], **cfg["index"])
    ids, sc, _ = ox.query(Q, k, cfg["qprobes"])
    gids = np.where(ids == 0xFFFFFFFF, 0xFFFFFFFF, ids.astype(np.int64) + lo)
    return sc, gids


CFGS = {
    "filtered": {"index": dict(L=6, K=2, D=32, iprobes=3, alpha=0.2, kappa=5), "qprobes": 60},
    "exhaustive": {"index": dict(L=2, K=2, D=16, iprobes=1, alpha=1.0, kappa=0),
                   "qprobes": 2 * 4 * 16 * 16},
}


def worker(rank, world, port, out, name):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, d, nq, k = 1501, 32, 40, 10
    X, Q = make(n, d, nq)
    lo, hi = fdist.shard_range(n, world, rank)
    sc, gids = shard_answer(X, Q, lo, hi, CFGS[name], k)
    ms, mi = fdist.allgather_merge(torch.from_numpy(sc), torch.from_numpy(gids), k)
    if rank == 0:
        np.savez(out, scores=ms.numpy(), ids=mi.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["filtered", "exhaustive"])
def test_two_rank_merge(tmp_path, name):
    out = str(tmp_path / "res.npz")
    mp.spawn(worker, args=(2, free_port(), out, name), nprocs=2, join=True)
    got = np.load(out)
    n, d, nq, k = 1501, 32, 40, 10
    X, Q = make(n, d, nq)
    parts = [shard_answer(X, Q, *fdist.shard_range(n, 2, r), CFGS[name], k) for r in range(2)]
    es, ei = fdist.merge_topk(torch.from_numpy(np.concatenate([p[0] for p in parts], 1)),
                              torch.from_numpy(np.concatenate([p[1] for p in parts], 1)), k)
    assert np.array_equal(got["ids"], ei.numpy())
    assert np.array_equal(got["scores"], es.numpy())
    if name == "exhaustive":
        from oracle import oracle as orc
        bi, bs = orc.brute_force(X, Q, k)
        assert np.array_equal(got["ids"], bi.astype(np.int64))
        assert np.array_equal(got["scores"], bs)


class OracleQueryEngine:
    """CPU stand-in for dist.GpuQueryEngine (test infrastructure): probe sets from the
    oracle's query_debug, stage B as the oracle's search restricted to given probe
    sets (union of the buckets' kept entries, exact sequential fp64 inner products,
    top-k by score desc / id asc)."""

    def __init__(self, X, lo, cfg):
        from oracle import oracle as orc
        self.orc, self.X, self.lo = orc, X, lo
        self.ox = orc.Index(X, **cfg["index"])
        self.tabs = [self.ox.table(t) for t in range(cfg["index"]["L"])]

    def peff(self, qprobes):
        return int(self.ox.peff(qprobes))

    def probe_sets(self, Q, qprobes, out):
        for i, q in enumerate(Q.numpy()):
            p, _ = self.ox.query_debug(q, qprobes)
            assert len(p) == out.shape[1]
            out[i] = torch.from_numpy(p.astype(np.uint32).view(np.int32).copy())

    def from_probe_sets(self, Q, probes, k, qprobes, ids, scores, stats=None):
        L = self.orc.lib()
        NB = int(self.ox.NB)
        for i, q in enumerate(Q.numpy()):
            pb = probes[i].numpy().view(np.uint32).astype(np.int64)
            cand = set()
            for gb in pb.tolist():
                off, tid, _ = self.tabs[gb // NB]
                b = gb % NB
                cand.update(tid[off[b]:off[b + 1]].tolist())
            res = sorted(((-L.orc_inner_product(self.X[c], q, self.X.shape[1]), c) for c in cand))[:k]
            ids[i] = 0xFFFFFFFF
            scores[i] = -np.inf
            for j, (ns, c) in enumerate(res):
                ids[i, j] = c + self.lo
                scores[i, j] = -ns


def split_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, d, nq, k = 1501, 32, 37, 10
    X, Q = make(n, d, nq)
    lo, hi = fdist.shard_range(n, world, rank)
    cfg = CFGS["filtered"]
    eng = OracleQueryEngine(np.ascontiguousarray(X[lo:hi]), lo, cfg)
    ids = torch.empty((nq, k), dtype=torch.int64)
    sc = torch.empty((nq, k), dtype=torch.float64)
    ms, mi = fdist.sharded_query_engine(eng, torch.from_numpy(Q), ids, sc, k, cfg["qprobes"])
    if rank == 0:
        np.savez(out, scores=ms.numpy(), ids=mi.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_stage_a_split_equals_replicated(tmp_path, world):
    """dist.sharded_query_engine (stage A on each rank's slice of the batch, probe sets
    all-gathered, stage B per shard from the gathered probe sets, top-k merge) equals
    the replicated path (every rank answering the whole batch, merge) on the same
    shards; nq = 37 does not divide by the world size (a short / empty last slice)."""
    out = str(tmp_path / "split.npz")
    mp.spawn(split_worker, args=(world, free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    n, d, nq, k = 1501, 32, 37, 10
    X, Q = make(n, d, nq)
    parts = [shard_answer(X, Q, *fdist.shard_range(n, world, r), CFGS["filtered"], k)
             for r in range(world)]
    es, ei = fdist.merge_topk(torch.from_numpy(np.concatenate([p[0] for p in parts], 1)),
                              torch.from_numpy(np.concatenate([p[1] for p in parts], 1)), k)
    assert np.array_equal(got["ids"], ei.numpy())
    assert np.array_equal(got["scores"], es.numpy())


def test_query_slices_cover():
    for nq in (0, 1, 5, 37, 100):
        for w in (1, 2, 3, 8):
            rs = [fdist.query_slice(nq, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == nq
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))


def test_shard_ranges_cover():
    for n in (1, 7, 100, 1501):
        for w in (1, 2, 3, 8):
            rs = [fdist.shard_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_merge_topk_ties_and_empty():
    s = torch.tensor([[1.0, 0.5, -float("inf"), 1.0, 0.7, -float("inf")]], dtype=torch.float64)
    i = torch.tensor([[9, 3, 0xFFFFFFFF, 4, 8, 0xFFFFFFFF]], dtype=torch.int64)
    ms, mi = fdist.merge_topk(s, i, 4)
    assert mi.tolist() == [[4, 9, 8, 3]]
    assert ms.tolist() == [[1.0, 1.0, 0.7, 0.5]]


# --------------------------------------------- global-filter sharded build (8(e) B)
GF = dict(L=3, K=2, D=16, iProbes=3, alpha=0.2, kappa=4, seed=1)


def gf_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from shard_engine import OracleShardEngine
    n = 3001
    X, _ = make(n, 16, 1)
    lo, hi = fdist.shard_range(n, world, rank)
    kept = fdist.build_global_filter(OracleShardEngine(X[lo:hi], lo, **GF))
    allk = [None] * world
    dist.all_gather_object(allk, {k: v.tolist() for k, v in kept.items()})
    if rank == 0:
        import pickle
        with open(out, "wb") as f:
            pickle.dump(allk, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_global_filter_equals_single_index(tmp_path, world):
    import pickle
    out = str(tmp_path / "gf.pkl")
    mp.spawn(gf_worker, args=(world, free_port(), out), nprocs=world, join=True)
    allk = pickle.load(open(out, "rb"))
    from oracle import oracle as orc
    from shard_engine import ord_key
    n = 3001
    X, _ = make(n, 16, 1)
    ox = orc.Index(X, L=GF["L"], K=GF["K"], D=GF["D"], iprobes=GF["iProbes"], alpha=GF["alpha"],
                   kappa=GF["kappa"], seed=GF["seed"])
    union = {}
    for part in allk:
        for k, v in part.items():
            union.setdefault(k, []).extend(v)
    total = 0
    for t in range(GF["L"]):
        off, ids, sc = ox.table(t)
        for b in np.nonzero(np.diff(off))[0]:
            keys = (((~ord_key(sc[off[b]:off[b + 1]])) & np.uint64(0xFFFFFFFF)) << np.uint64(32)) \
                | ids[off[b]:off[b + 1]].astype(np.uint64)
            got = np.sort(np.array(union.pop((t, int(b)), []), dtype=np.uint64))
            assert np.array_equal(got, np.sort(keys)), (t, b)
            total += len(keys)
    assert not union  # no bucket kept by the shards that the single index drops
    assert total == sum(len(ox.table(t)[1]) for t in range(GF["L"]))
