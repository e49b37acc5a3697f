"""GPU parity: every intermediate of the CUDA path against the CPU oracle.

Bar (BASELINE.json north star): projections, hash codes,
index probes, kept-bucket CSR (ids + scores), ranked query lists, probe sets and
candidate sets are bit-exact; top-k ids identical (ties by lower id); scores are
asserted bit-exact too (the score kernel accumulates in the reference's
sequential fp64 order) -- the north-star tolerance would be 1e-5 relative.
All calls go through the C ABI (paper_2206_01382_b200 -> libfalconnpp_b200.so).
"""
import numpy as np
import pytest

from fpp_testutil import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

SCORE_RTOL = 1e-5  # north-star tolerance; the GPU path is in fact bit-exact


def data(fpp, n, d, clusters=0, sigma=0.0, seed=1, stream=0):
    return fpp.normalize(fpp.synth(n, d, clusters, sigma, seed=seed, stream=stream))


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


@pytest.mark.parametrize("d", [2, 5, 17, 32, 48, 64, 100, 128, 256, 300, 960])
def test_projection_bitexact(fpp, orc, d):
    X = data(fpp, 257, d)
    P = orc.lib().orc_pad_dimension(d)
    ix = fpp.Index.build(X, L=3, K=2, D=P, iProbes=1, alpha=1.0)
    for t in range(3):
        for f in range(2):
            seed = orc.lib().orc_derive_seed(1, t, f, 0)
            ref = orc.project_rows(X, P, seed)
            got = ix.project(X, t, f)
            assert np.array_equal(bits(got), bits(ref)), (d, t, f)
            assert np.array_equal(orc.cp_hash_rows(got), orc.cp_hash_rows(ref))


def test_projection_truncated_D(fpp, orc):
    X = data(fpp, 100, 200)  # d_pad 256, D = 64 < d_pad (rotation.cpp:51-53,96-98)
    ix = fpp.Index.build(X, L=2, K=2, D=64, iProbes=2, alpha=0.5)
    for t in range(2):
        for f in range(2):
            seed = orc.lib().orc_derive_seed(1, t, f, 0)
            assert np.array_equal(bits(ix.project(X, t, f)), bits(orc.project_rows(X, 64, seed)))


@pytest.mark.parametrize("K,D,ip,d", [(2, 128, 3, 128), (2, 512, 3, 300), (2, 1024, 3, 960),
                                      (2, 256, 5, 256), (1, 128, 3, 128), (2, 64, 1, 100),
                                      (2, 32, 16, 32), (1, 16, 9, 16), (2, 64, 7, 200)])
def test_index_probes_bitexact(fpp, orc, K, D, ip, d):
    X = data(fpp, 500, d, clusters=7, sigma=0.3)
    ix = fpp.Index.build(X, L=2, K=K, D=D, iProbes=ip, alpha=0.5)
    ox = orc.Index(X, L=2, K=K, D=D, iprobes=ip, alpha=0.5)
    for t in range(2):
        gb, gs = ix.index_probes(X, t)
        ob, os_ = ox.index_probes(X, t)
        assert np.array_equal(gb, ob), (K, D, ip, t)
        assert np.array_equal(bits(gs), bits(os_)), (K, D, ip, t)


CSR_CASES = [
    # name, n, d, clusters, sigma, L, K, D, ip, alpha, kappa
    ("c1_small", 20000, 128, 0, 0.0, 3, 2, 128, 3, 0.1, 20),
    ("clustered", 20000, 64, 20, 0.25, 3, 2, 64, 3, 0.05, 20),
    ("one_cluster_big_buckets", 30000, 64, 1, 0.05, 2, 2, 64, 3, 0.1, 20),
    ("alpha1_full_sort", 30000, 32, 1, 0.05, 2, 2, 32, 2, 1.0, 0),
    ("kappa0_stress", 20000, 128, 10, 0.3, 2, 2, 128, 3, 0.01, 0),
    ("K1", 10000, 64, 0, 0.0, 3, 1, 64, 3, 0.3, 5),
    ("d300", 8000, 300, 50, 0.3, 2, 2, 512, 3, 0.05, 20),
    # NB = 1024, B ~ 175 > 32 with keep = kappa = 20: every bucket on the warp top-k path
    ("topk_buckets", 60000, 32, 0, 0.0, 2, 2, 16, 3, 0.05, 20),
    # keep in (32, B): CTA path next to top-k buckets
    ("keep_gt_32", 60000, 32, 0, 0.0, 2, 2, 16, 3, 0.9, 20),
]


@pytest.mark.parametrize("case", CSR_CASES, ids=[c[0] for c in CSR_CASES])
def test_csr_bitexact(fpp, orc, case):
    _, n, d, C, sg, L, K, D, ip, al, ka = case
    X = data(fpp, n, d, C, sg)
    ix = fpp.Index.build(X, L=L, K=K, D=D, iProbes=ip, alpha=al, kappa=ka)
    ox = orc.Index(X, L=L, K=K, D=D, iprobes=ip, alpha=al, kappa=ka)
    tot = 0
    for t in range(L):
        go, gi, gs = ix.table(t)
        oo, oi, os_ = ox.table(t)
        assert np.array_equal(go, oo), t
        assert np.array_equal(gi, oi), t
        assert np.array_equal(gs, os_), t  # float == (canonical +-0)
        tot += len(oi)
    info = ix.info()
    assert info["kept_total"] == tot
    assert info["prefilter_total"] == n * L * ip


@pytest.mark.parametrize("qp", [50, 137, 1000, 5000, 40000])
def test_query_lists_bitexact(fpp, orc, qp):
    X = data(fpp, 3000, 100, 10, 0.3)
    Q = data(fpp, 9, 100, 10, 0.3, stream=1)
    L = 5
    ix = fpp.Index.build(X, L=L, K=2, D=128, iProbes=3, alpha=0.1)  # s > D for qp >= 5000
    ox = orc.Index(X, L=L, K=2, D=128, iprobes=3, alpha=0.1)
    s = ix.cap(qp)
    assert s == ox.cap(qp)
    gv, gc = ix.query_lists(Q, qp)
    for i in range(len(Q)):
        ov, oc = ox.query_lists(Q[i], s)
        assert np.array_equal(bits(gv[i]), bits(ov)), (qp, i)
        assert np.array_equal(gc[i], oc), (qp, i)


@pytest.mark.parametrize("K,D,d,qps", [
    (2, 512, 300, [1000, 5000, 10000, 20000]),  # d padded 300 -> 512
    (2, 512, 400, [2000, 4000]),
    (2, 1024, 960, [1000, 10000, 40000]),
    (2, 256, 200, [500, 3000, 9000]),
    (1, 512, 500, [100, 200, 700]),
])
def test_query_lists_preselect(fpp, orc, K, D, d, qps):
    # P >= 256 lists are built from a threshold-preselected subset (NS = P/4 or
    # P/2 keys sorted instead of P); s near and past the NS margins, K = 1
    X = data(fpp, 2000, d, 10, 0.3)
    Q = data(fpp, 12, d, 10, 0.3, stream=1)
    ix = fpp.Index.build(X, L=3, K=K, D=D, iProbes=2, alpha=0.1)
    ox = orc.Index(X, L=3, K=K, D=D, iprobes=2, alpha=0.1)
    for qp in qps:
        s = ix.cap(qp)
        gv, gc = ix.query_lists(Q, qp)
        for i in range(len(Q)):
            ov, oc = ox.query_lists(Q[i], s)
            assert np.array_equal(bits(gv[i]), bits(ov)), (qp, i)
            assert np.array_equal(gc[i], oc), (qp, i)


QUERY_CASES = [
    # name, n, d, clusters, sigma, L, K, D, ip, alpha, kappa, qprobes list
    ("c1_like", 20000, 128, 0, 0.0, 10, 2, 128, 3, 0.1, 20, [10, 100, 1000, 3000]),
    ("c2_like", 12000, 300, 100, 0.3, 8, 2, 512, 3, 0.05, 20, [8, 800, 2000, 20000]),
    ("c4_like_s_gt_D", 20000, 128, 100, 0.25, 6, 2, 128, 3, 0.01, 20, [5000, 100000]),
    ("K1", 5000, 64, 0, 0.0, 6, 1, 64, 2, 0.5, 10, [6, 60, 768]),
    ("wide_c3_like", 4000, 960, 20, 0.2, 4, 2, 1024, 3, 0.02, 20, [1000, 10000]),
    # d % 4 != 0: the scalar cp.async score path, narrow (32-float slices) and wide (96)
    ("odd_d_narrow", 6000, 17, 10, 0.3, 5, 2, 32, 3, 0.2, 10, [40, 400]),
    ("odd_d_wide", 6000, 250, 10, 0.3, 5, 2, 256, 3, 0.1, 10, [500, 3000]),
]


@pytest.mark.parametrize("case", QUERY_CASES, ids=[c[0] for c in QUERY_CASES])
def test_query_parity(fpp, orc, case):
    _, n, d, C, sg, L, K, D, ip, al, ka, qps = case
    X = data(fpp, n, d, C, sg)
    Q = data(fpp, 64, d, C, sg, stream=1)
    ix = fpp.Index.build(X, L=L, K=K, D=D, iProbes=ip, alpha=al, kappa=ka)
    ox = orc.Index(X, L=L, K=K, D=D, iprobes=ip, alpha=al, kappa=ka)
    k = 20
    for qp in qps:
        gi, gs, gst = ix.query(Q, k, qp, return_stats=True)
        oi, os_, ost = ox.query(Q, k, qp)
        assert np.array_equal(gst, ost), qp
        assert np.array_equal(gi, oi), qp
        ok = np.isfinite(os_)
        assert np.array_equal(np.isfinite(gs), ok)
        np.testing.assert_allclose(gs[ok], os_[ok], rtol=SCORE_RTOL, atol=0)
        assert np.array_equal(gs[ok], os_[ok]), "scores expected bit-exact"
        for qi in (0, 7, 31):
            gp, gc = ix.query_debug(Q[qi], qp)
            op, oc = ox.query_debug(Q[qi], qp)
            assert np.array_equal(gp, op), (qp, qi)
            assert np.array_equal(gc, oc), (qp, qi)


@pytest.mark.parametrize("beta", ["0.3", "1.0"])
def test_probe_threshold_fallback(fpp, orc, beta, monkeypatch):
    # FPP_PS_BETA=0.3: the optimistic first T_lo is too high for most queries, so
    # k_probe_select re-walks at the safe arm bound; 1.0 disables the first attempt
    monkeypatch.setenv("FPP_PS_BETA", beta)
    X = data(fpp, 12000, 300, 100, 0.3)
    Q = data(fpp, 48, 300, 100, 0.3, stream=1)
    ix = fpp.Index.build(X, L=8, K=2, D=512, iProbes=3, alpha=0.05)
    ox = orc.Index(X, L=8, K=2, D=512, iprobes=3, alpha=0.05)
    for qp in (800, 2000):
        gi, gs, gst = ix.query(Q, 20, qp, return_stats=True)
        oi, os_, ost = ox.query(Q, 20, qp)
        assert np.array_equal(gst, ost) and np.array_equal(gi, oi) and np.array_equal(gs, os_)
        gp, _ = ix.query_debug(Q[5], qp)
        op, _ = ox.query_debug(Q[5], qp)
        assert np.array_equal(gp, op)


def test_acceptance4_exhaustive_equals_bruteforce(fpp, orc):
    # alpha=1, iProbes=1, qProbes=L*4D^2 must equal brute force
    X = data(fpp, 2000, 32, seed=3)
    Q = data(fpp, 100, 32, seed=3, stream=1)
    L, D = 2, 32
    ix = fpp.Index.build(X, L=L, K=2, D=D, iProbes=1, alpha=1.0, kappa=0)
    gi, gs = ix.query(Q, 20, L * 4 * D * D)
    bi, bs = orc.brute_force(X, Q, 20)
    assert np.array_equal(gi, bi)
    assert np.array_equal(gs, bs)


def test_duplicates_tie_lower_id(fpp, orc):
    X = data(fpp, 1000, 64, seed=5)
    X[500:510] = X[3]  # exact duplicates: equal scores, lower id first
    Q = X[3:4].copy()
    # iProbes=1, alpha=1: keep = floor(B/1) = B, so every duplicate survives the filter
    ix = fpp.Index.build(X, L=4, K=2, D=64, iProbes=1, alpha=1.0, kappa=0)
    ox = orc.Index(X, L=4, K=2, D=64, iprobes=1, alpha=1.0, kappa=0)
    gi, gs = ix.query(Q, 20, 400)
    oi, os_, _ = ox.query(Q, 20, 400)
    assert np.array_equal(gi, oi)
    assert list(gi[0][:11]) == [3] + list(range(500, 510))


def test_fewer_candidates_than_k(fpp, orc):
    X = data(fpp, 5000, 64, seed=9)
    Q = data(fpp, 8, 64, seed=9, stream=1)
    ix = fpp.Index.build(X, L=1, K=2, D=64, iProbes=1, alpha=0.01, kappa=1)
    ox = orc.Index(X, L=1, K=2, D=64, iprobes=1, alpha=0.01, kappa=1)
    gi, gs, gst = ix.query(Q, 32, 1, return_stats=True)
    oi, os_, ost = ox.query(Q, 32, 1)
    assert np.array_equal(gi, oi) and np.array_equal(gst, ost)
    assert (gi == 0xFFFFFFFF).any() and np.isneginf(gs[gi == 0xFFFFFFFF]).all()


def test_empty_batch_and_errors(fpp):
    X = data(fpp, 100, 16)
    ix = fpp.Index.build(X, L=2, K=2, D=16, iProbes=1, alpha=1.0)
    ids, sc = ix.query(np.zeros((0, 16), np.float32), 5, 4)
    assert ids.shape == (0, 5)
    with pytest.raises(fpp.FppOutOfRange):
        ix.query(X[:2], 5, 1)  # qProbes < L
    with pytest.raises(fpp.FppOutOfRange):
        ix.query(X[:2], 101, 4)  # k > n
    with pytest.raises(fpp.FppDimensionError):
        ix.query(np.zeros((1, 15), np.float32), 5, 4)
    bad = X.copy()
    bad[7, 3] = np.nan
    with pytest.raises(fpp.FppNonFinite):
        fpp.Index.build(bad, L=2, K=2, D=16, iProbes=1, alpha=1.0)


@pytest.mark.parametrize("path", ["sliced", "grouped", "cluster", "global"])
def test_large_shard_collect_paths(fpp, orc, path, monkeypatch):
    # the large-shard visited sets (n > one SM's shared memory): sliced bitmap dedup
    # (id-slice counting sort + a shared-memory bitmap per slice), grouped dedup
    # (id-range counting sort + per-warp range bitmaps), the DSMEM-cluster bitmap and
    # the global-memory bitmap, forced at small n: the oracle's candidates/top-k/stats
    monkeypatch.setenv("FPP_FORCE_COLLECT", path)
    X = data(fpp, 20000, 64, 20, 0.3)
    Q = data(fpp, 40, 64, 20, 0.3, stream=1)
    ix = fpp.Index.build(X, L=6, K=2, D=64, iProbes=3, alpha=0.1)
    ox = orc.Index(X, L=6, K=2, D=64, iprobes=3, alpha=0.1)
    gi, gs, gst = ix.query(Q, 20, 600, return_stats=True)
    oi, os_, ost = ox.query(Q, 20, 600)
    assert np.array_equal(gst, ost) and np.array_equal(gi, oi) and np.array_equal(gs, os_)
    gp, gc = ix.query_debug(Q[3], 600)
    op, oc = ox.query_debug(Q[3], 600)
    assert np.array_equal(gc, oc)


def test_sliced_collect_natural_large_n(fpp, orc):
    # n = 2.2M points > the single-CTA bitmap limit (~1.8M) -> sliced dedup for real
    # (5 slices of 2^19 ids)
    X = data(fpp, 2_200_000, 16, 50, 0.2)
    Q = data(fpp, 16, 16, 50, 0.2, stream=1)
    ix = fpp.Index.build(X, L=2, K=2, D=16, iProbes=2, alpha=0.05, kappa=10)
    ox = orc.Index(X, L=2, K=2, D=16, iprobes=2, alpha=0.05, kappa=10)
    gi, gs, gst = ix.query(Q, 20, 100, return_stats=True)
    oi, os_, ost = ox.query(Q, 20, 100)
    assert np.array_equal(gst, ost) and np.array_equal(gi, oi) and np.array_equal(gs, os_)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_global_filter_equals_single_gpu_index(fpp, orc, world):
    # SURVEY 8(e) option B on one GPU: `world` shards built with fpp_shard_*, the
    # all-reduce / all-gather done in-process; the union of the shard indexes
    # must equal the 1-GPU index bucket for bucket, and the merged top-k must
    # equal the 1-GPU top-k bit for bit.
    import torch
    from paper_2206_01382_b200 import dist as fdist
    X = data(fpp, 30011, 64, 40, 0.3)
    Q = data(fpp, 48, 64, 40, 0.3, stream=1)
    prm = dict(L=3, K=2, D=64, iProbes=3, alpha=0.1, kappa=20)
    n = len(X)
    ranges = [fdist.shard_range(n, world, r) for r in range(world)]
    engines = [fdist.GpuShardEngine(X[lo:hi], lo, device=0, **prm) for lo, hi in ranges]
    gh = sum(e.hist() for e in engines)
    slots = [e.slots(gh) for e in engines]
    assert len(set(slots)) == 1
    allp = torch.cat([e.prefix(gh, slots[0]) for e in engines])
    shards = [e.finish(gh, allp, world) for e in engines]
    full = fpp.Index.build(X, **prm)
    for t in range(prm["L"]):
        fo, fi, fs = full.table(t)
        parts = [ix.table(t) for ix in shards]
        for b in np.nonzero(np.diff(fo))[0][:3000]:
            want = sorted(zip(fi[fo[b]:fo[b + 1]].tolist(), fs[fo[b]:fo[b + 1]].tolist()))
            got = []
            for (lo, _), (po, pi, ps) in zip(ranges, parts):
                got += [(int(i) + lo, s) for i, s in zip(pi[po[b]:po[b + 1]], ps[po[b]:po[b + 1]])]
            assert sorted(got) == want, (t, b)
        assert sum(len(p[1]) for p in parts) == len(fi)
    k, qp = 20, 400
    fi, fsc = full.query(Q, k, qp)
    outs = [ix.query(Q, k, qp) for ix in shards]
    ms, mi = fdist.merge_topk(torch.from_numpy(np.concatenate([o[1] for o in outs], 1)),
                              torch.from_numpy(np.concatenate([o[0].astype(np.int64) for o in outs], 1)), k)
    assert np.array_equal(mi.numpy(), fi.astype(np.int64))
    assert np.array_equal(ms.numpy(), fsc)


@pytest.mark.parametrize("n,d,k", [(5000, 300, 20), (3001, 17, 7), (2000, 960, 32), (40, 64, 32)])
def test_brute_force_exact(fpp, orc, n, d, k):
    # recall ground truth: inner_product scores bit for bit, ties to lower id
    X = data(fpp, n, d, 10, 0.3, seed=6)
    X[n // 2: n // 2 + 5] = X[3]  # exact duplicates: equal scores, lower id first
    Q = data(fpp, 37, d, 10, 0.3, seed=6, stream=1)
    Q[0] = X[3]
    ix = fpp.Index.build(X, L=2, K=2, D=orc.lib().orc_pad_dimension(d) if d >= 16 else 16,
                         iProbes=1, alpha=1.0)
    gi, gs = ix.brute_force(Q, k)
    bi, bs = orc.brute_force(X, Q, k)
    assert np.array_equal(gi, bi)
    assert np.array_equal(gs, bs)
    assert list(gi[0][:6]) == [3] + list(range(n // 2, n // 2 + 5))


@pytest.mark.parametrize("d,D", [(17, 32), (100, 128), (300, 512), (200, 64), (32, 16)])
def test_simhash_signatures_bitexact(fpp, orc, d, D):
    # SPEC.md "SimHash signatures": signs of the first 64 coordinates of the (t=0, f=0)
    # projection; bits >= D stay 0
    X = data(fpp, 700, d, 5, 0.3)
    ix = fpp.Index.build(X, L=2, K=2, D=D, iProbes=1, alpha=0.5)
    ox = orc.Index(X, L=2, K=2, D=D, iprobes=1, alpha=0.5)
    assert np.array_equal(ix.signatures(X), ox.simhash(X))
    if D < 64:
        assert int(np.bitwise_or.reduce(ix.signatures(X))) >> D == 0


@pytest.mark.parametrize("case", [("c2_like", 12000, 300, 100, 0.3, 8, 2, 512, 3, 0.05, 20),
                                  ("iid_d128", 20000, 128, 0, 0.0, 10, 2, 128, 3, 0.1, 20),
                                  ("K1", 5000, 64, 0, 0.0, 6, 1, 64, 2, 0.5, 10)],
                         ids=lambda c: c[0])
def test_rerank_parity(fpp, orc, case):
    # top-B by signature agreement (ties by lower id), then exact top-k
    _, n, d, C_, sg, L, K, D, ip, al, ka = case
    X = data(fpp, n, d, C_, sg)
    Q = data(fpp, 48, d, C_, sg, stream=1)
    ix = fpp.Index.build(X, L=L, K=K, D=D, iProbes=ip, alpha=al, kappa=ka)
    ox = orc.Index(X, L=L, K=K, D=D, iprobes=ip, alpha=al, kappa=ka)
    k = 20
    cap = L * (4 * D * D if K == 2 else 2 * D)
    for qp, B in ((800, 20), (800, 100), (2000, 500), (2000, 10 ** 6)):
        qp = min(qp, cap)
        gi, gs, gst = ix.query(Q, k, qp, return_stats=True, rerank=B)
        oi, os_, ost = ox.query(Q, k, qp, rerank=B)
        assert np.array_equal(gst, ost), (qp, B)
        assert np.array_equal(gi, oi), (qp, B)
        assert np.array_equal(gs, os_), (qp, B)
        assert (gst[:, 3] <= np.minimum(gst[:, 2], B)).all() and (gst[:, 3] > 0).all()
    # B >= U is the identity screen: equals the unscreened search
    qp = min(800, cap)
    gi0, gs0 = ix.query(Q, k, qp)
    gi1, gs1 = ix.query(Q, k, qp, rerank=10 ** 6)
    assert np.array_equal(gi0, gi1) and np.array_equal(gs0, gs1)
    with pytest.raises(fpp.FppOutOfRange):
        ix.query(Q, k, qp, rerank=k - 1)


def test_rerank_recall_bound(fpp, orc):
    # SPEC.md query invariants: recall with B > 0 <= recall with B = 0 at equal qProbes
    X = data(fpp, 20000, 128, 50, 0.3, seed=8)
    Q = data(fpp, 200, 128, 50, 0.3, seed=8, stream=1)
    ix = fpp.Index.build(X, L=10, K=2, D=128, iProbes=3, alpha=0.1)
    gt, _ = ix.brute_force(Q, 20)

    def recall(ids):
        return np.mean([len(set(a) & set(b)) / 20 for a, b in zip(ids, gt)])

    full = recall(ix.query(Q, 20, 1000)[0])
    for B in (20, 100, 400):
        assert recall(ix.query(Q, 20, 1000, rerank=B)[0]) <= full + 1e-12


@pytest.mark.parametrize("K,D,qps", [(2, 64, [8, 300, 3000]), (1, 128, [10, 200])])
def test_falconn_baseline_parity(fpp, orc, K, D, qps):
    # alpha = 1, iProbes = 1 forced; probes by ascending gap score
    X = data(fpp, 8000, 100 if D == 128 else 64, 20, 0.3)
    Q = data(fpp, 40, X.shape[1], 20, 0.3, stream=1)
    ix = fpp.Index.build(X, L=6, K=K, D=D, iProbes=3, alpha=0.1, mode="falconn_baseline")
    ox = orc.Index(X, L=6, K=K, D=D, iprobes=3, alpha=0.1, mode=1)
    inf = ix.info()
    assert (inf["alpha"], inf["iprobes"], inf["mode"]) == (1.0, 1, 1)
    for t in range(6):
        for u, v in zip(ix.table(t), ox.table(t)):
            assert np.array_equal(u, v)
    for qp in qps:
        gi, gs, gst = ix.query(Q, 10, qp, return_stats=True)
        oi, os_, ost = ox.query(Q, 10, qp)
        assert np.array_equal(gst, ost) and np.array_equal(gi, oi) and np.array_equal(gs, os_), qp
        for qi in (0, 11):
            gp, gc = ix.query_debug(Q[qi], qp)
            op, oc = ox.query_debug(Q[qi], qp)
            assert np.array_equal(gp, op) and np.array_equal(gc, oc), (qp, qi)
    # the first probe of every table is the true bucket in both modes
    iy = fpp.Index.build(X, L=6, K=K, D=D, iProbes=1, alpha=1.0)
    assert np.array_equal(ix.query_debug(Q[0], 6)[0], iy.query_debug(Q[0], 6)[0])


def test_centering_parity(fpp, orc, tmp_path):
    # SPEC.md:53-61 (dataset.cpp center()): index center(X); queries stay raw
    raw = fpp.synth(6000, 64, 10, 0.3, seed=12)
    X = fpp.normalize(raw) + np.float32(0.05)  # off-centre data
    Q = data(fpp, 30, 64, 10, 0.3, seed=12, stream=1)
    ix = fpp.Index.build(X, L=5, K=2, D=64, iProbes=3, alpha=0.1, centering=True)
    Xc, c = orc.center(X)
    ox = orc.Index(Xc, L=5, K=2, D=64, iprobes=3, alpha=0.1)
    assert np.array_equal(ix.center_vector(), c) and ix.info()["centering"] == 1
    for t in range(5):
        for u, v in zip(ix.table(t), ox.table(t)):
            assert np.array_equal(u, v)
    gi, gs, gst = ix.query(Q, 10, 400, return_stats=True)
    oi, os_, ost = ox.query(Q, 10, 400)
    assert np.array_equal(gi, oi) and np.array_equal(gs, os_) and np.array_equal(gst, ost)
    # FLPP keeps the center; load takes the raw rows again
    p = str(tmp_path / "c.flpp")
    ix.save(p)
    iy = fpp.Index.load(p, X)
    li, ls = iy.query(Q, 10, 400)
    assert np.array_equal(li, gi) and np.array_equal(ls, gs)
    assert np.array_equal(iy.center_vector(), c)


def test_large_batch_reordered_equals_oracle(fpp, orc):
    # batches with nq >= 256 and nq*d >= 512k run in stack-(0,0)-code order and are
    # scattered back: results (ids, scores, stats) must be the per-query oracle answers
    X = data(fpp, 6000, 480, 30, 0.3, seed=21)
    Q = data(fpp, 1100, 480, 30, 0.3, seed=21, stream=1)
    ix = fpp.Index.build(X, L=4, K=2, D=512, iProbes=3, alpha=0.1)
    ox = orc.Index(X, L=4, K=2, D=512, iprobes=3, alpha=0.1)
    for rr in (0, 50):
        gi, gs, gst = ix.query(Q, 10, 200, return_stats=True, rerank=rr)
        oi, os_, ost = ox.query(Q, 10, 200, rerank=rr)
        assert np.array_equal(gi, oi) and np.array_equal(gs, os_) and np.array_equal(gst, ost)


@pytest.mark.parametrize("geom", ["423", "432", "324", "423-tma"])
@pytest.mark.parametrize("d", [128, 300, 301, 960])
def test_score_early_termination_exact(fpp, orc, d, geom, monkeypatch, capfd):
    # k_score_pruned (Cauchy-Schwarz bound on the tail of each row against the running
    # k-th best) must return exactly the full gather's answers while reading less:
    # clustered data (many small clusters: most candidates are far), compared with
    # FPP_NO_PRUNE and the oracle, for two ring geometries (FPP_SC_PR)
    monkeypatch.setenv("FPP_SC_PR", geom.split("-")[0])
    if geom.endswith("-tma"):  # TMA bulk row copies + mbarrier ring (d % 4 == 0 only)
        monkeypatch.setenv("FPP_SC_TMA", "1")
    X = data(fpp, 20000, d, 200, 0.25, seed=31)
    Q = data(fpp, 300, d, 200, 0.25, seed=31, stream=1)
    ix = fpp.Index.build(X, L=16, K=2, D=128 if d <= 128 else 256, iProbes=3, alpha=0.2)
    ox = orc.Index(X, L=16, K=2, D=128 if d <= 128 else 256, iprobes=3, alpha=0.2)
    monkeypatch.setenv("FPP_DEBUG_PRUNE", "1")
    gi, gs, gst = ix.query(Q, 20, 20000, return_stats=True)
    err = capfd.readouterr().err
    monkeypatch.delenv("FPP_DEBUG_PRUNE")
    monkeypatch.setenv("FPP_NO_PRUNE", "1")
    fi, fs, fst = ix.query(Q, 20, 20000, return_stats=True)
    monkeypatch.delenv("FPP_NO_PRUNE")
    assert np.array_equal(gi, fi) and np.array_equal(gs, fs) and np.array_equal(gst, fst)
    oi, os_, ost = ox.query(Q, 20, 20000)
    assert np.array_equal(gi, oi) and np.array_equal(gst, ost)
    ok = np.isfinite(os_)
    assert np.array_equal(gs[ok], os_[ok])
    fr = [float(l.split("(")[1].split("%")[0]) for l in err.splitlines() if "[prune dbg]" in l]
    assert fr and max(fr) < 80.0, err  # the bound cut row reads


def test_score_early_termination_unstructured(fpp, orc, monkeypatch):
    # i.i.d. data: heads mostly survive, warps switch to full batches; still exact
    X = data(fpp, 30000, 200, 0, 0.0, seed=5)
    Q = data(fpp, 200, 200, 0, 0.0, seed=5, stream=1)
    ix = fpp.Index.build(X, L=8, K=2, D=256, iProbes=3, alpha=0.3)
    ox = orc.Index(X, L=8, K=2, D=256, iprobes=3, alpha=0.3)
    gi, gs, gst = ix.query(Q, 20, 3000, return_stats=True)
    oi, os_, ost = ox.query(Q, 20, 3000)
    assert np.array_equal(gi, oi) and np.array_equal(gst, ost)
    ok = np.isfinite(os_)
    assert np.array_equal(gs[ok], os_[ok])


@pytest.mark.parametrize("path", ["grouped", "sliced"])
@pytest.mark.parametrize("prune", ["0", "1"])
@pytest.mark.parametrize("n,qp", [(20000, 5000), (2000, 3000)])
def test_grouped_collect_every_id_once(fpp, orc, path, prune, n, qp, monkeypatch):
    # grouped / sliced dedup (the large-shard paths): every candidate id is scored once
    # (SPEC.md:352 -- stats.exact = unique candidates), so ids, scores and all four
    # stats columns equal the oracle's, with and without early termination; n = 2000
    # packs many entries into few groups (heavy repeats)
    monkeypatch.setenv("FPP_FORCE_COLLECT", path)
    monkeypatch.setenv("FPP_PRUNE" if prune == "1" else "FPP_NO_PRUNE", "1")
    X = data(fpp, n, 128, 200, 0.25, seed=41)
    Q = data(fpp, 300, 128, 200, 0.25, seed=41, stream=1)
    ix = fpp.Index.build(X, L=12, K=2, D=128, iProbes=3, alpha=0.2)
    ox = orc.Index(X, L=12, K=2, D=128, iprobes=3, alpha=0.2)
    oi, os_, ost = ox.query(Q, 20, qp)
    gi, gs = ix.query(Q, 20, qp)
    assert np.array_equal(gi, oi)
    ok = np.isfinite(os_)
    assert np.array_equal(gs[ok], os_[ok])
    si, ss, sst = ix.query(Q, 20, qp, return_stats=True)
    assert np.array_equal(si, oi) and np.array_equal(sst, ost)
    assert (sst[:, 3] == sst[:, 2]).all() and (ost[:, 1] >= ost[:, 2]).all()
    for qi in (0, 99):
        _, gc = ix.query_debug(Q[qi], qp)
        _, oc = ox.query_debug(Q[qi], qp)
        assert np.array_equal(gc, oc)


def test_query_out_buffers(fpp, orc):
    # query(..., out=(ids, scores)) writes into caller-owned arrays (bench.py's e2e leg
    # passes page-locked ones): same answers as the allocating call; bad shapes rejected
    X = data(fpp, 5000, 64, 20, 0.3, seed=7)
    Q = data(fpp, 50, 64, 20, 0.3, seed=7, stream=1)
    ix = fpp.Index.build(X, L=6, K=2, D=64, iProbes=3, alpha=0.2)
    gi, gs = ix.query(Q, 10, 300)
    oi = np.zeros((50, 10), np.uint32)
    os_ = np.zeros((50, 10), np.float64)
    ri, rs = ix.query(Q, 10, 300, out=(oi, os_))
    assert ri is oi and rs is os_
    assert np.array_equal(oi, gi) and np.array_equal(os_, gs)
    with pytest.raises(ValueError):
        ix.query(Q, 10, 300, out=(np.zeros((50, 9), np.uint32), os_))


@pytest.mark.parametrize("d,D,ip", [(64, 64, 5), (128, 128, 3), (256, 256, 5)])
def test_index_probes_equal_magnitudes(fpp, orc, d, D, ip):
    # rows with six non-zeros: a projection takes at most 32 distinct |p| values, each at
    # several coordinates, so the top-r selection meets exact |p| ties among its kept keys
    # (the high-word group minimum must fall back to the low words: j ascending)
    rng = np.random.default_rng(7)
    X = np.zeros((300, d), np.float32)
    for i in range(300):
        X[i, rng.choice(d, 6, replace=False)] = rng.standard_normal(6).astype(np.float32)
    X = fpp.normalize(X)
    ix = fpp.Index.build(X, L=3, K=2, D=D, iProbes=ip, alpha=0.5)
    ox = orc.Index(X, L=3, K=2, D=D, iprobes=ip, alpha=0.5)
    for t in range(3):
        gb, gs = ix.index_probes(X, t)
        ob, os_ = ox.index_probes(X, t)
        assert np.array_equal(gb, ob), (d, t)
        assert np.array_equal(bits(gs), bits(os_)), (d, t)


def test_top_r_insertion_keeps_tie_order(fpp, orc):
    # regression (found by profiles/soak_parity.py): the lane-local top-R insertion of the
    # shuffle-FHT path (d_pad < 64, and the tie fallback above) must shift the displaced
    # entries unconditionally -- with a strict compare a displaced entry slipped behind a
    # successor of equal |p| (here j = 2 and j = 22 of row 18, table 2), swapping two index
    # probes and so the kept set of four buckets
    X = data(fpp, 10205, 17, clusters=5, sigma=0.3, seed=850085278)
    prm = dict(L=3, K=1, D=32, alpha=1.0, kappa=5, seed=850085278)
    ix = fpp.Index.build(X, iProbes=8, **prm)
    ox = orc.Index(X, iprobes=8, **prm)
    for t in range(3):
        gb, gs = ix.index_probes(X, t)
        ob, os_ = ox.index_probes(X, t)
        assert np.array_equal(gb, ob), t
        assert np.array_equal(bits(gs), bits(os_)), t
        go, gi, gsc = ix.table(t)
        oo, oi, osc = ox.table(t)
        assert np.array_equal(go, oo) and np.array_equal(gi, oi) and np.array_equal(bits(gsc), bits(osc))


def test_random_configurations_equal_oracle(fpp, orc):
    # a short, seeded run of profiles/soak_parity.py's generator: random (n, d, K, D, iProbes,
    # L, alpha, kappa, clusters, k, qProbes, stats on/off); ids, scores, stats = the oracle's
    rng = np.random.default_rng(20260121)
    for _ in range(60):
        d = int(rng.choice([8, 17, 32, 48, 64, 100, 128, 200, 256, 300, 320, 512, 960]))
        n = int(rng.integers(500, 6000))
        K = int(rng.choice([1, 2, 2, 2]))
        P = int(orc.lib().orc_pad_dimension(d))
        D = int(rng.choice([P, P, max(P // 2, 2)]))
        ip = int(rng.integers(1, min(D, 8) + 1))
        L = int(rng.integers(1, 6))
        prm = dict(L=L, K=K, D=D, alpha=float(rng.choice([1.0, 0.5, 0.1, 0.02])),
                   kappa=int(rng.choice([0, 5, 20])), seed=int(rng.integers(1, 1 << 30)))
        clusters = int(rng.choice([0, 5, 40]))
        X = data(fpp, n, d, clusters, 0.3, seed=prm["seed"])
        Q = data(fpp, int(rng.integers(1, 70)), d, clusters, 0.3, seed=prm["seed"], stream=1)
        ix = fpp.Index.build(X, iProbes=ip, **prm)
        ox = orc.Index(X, iprobes=ip, **prm)
        NB = (2 * D) ** K
        for _ in range(2):
            k = min(int(rng.choice([1, 7, 20, 32, 33, 50, 100])), n)
            qp = int(rng.integers(L, min(L * NB, 20000) + 1))
            gi, gs, gst = ix.query(Q, k, qp, return_stats=True)
            oi, os_, ost = ox.query(Q, k, qp)
            case = dict(n=n, d=d, ip=ip, k=k, qp=qp, clusters=clusters, **prm)
            assert np.array_equal(gi, oi), case
            assert np.array_equal(gs, os_), case
            assert np.array_equal(gst, ost), case
            gi2, gs2 = ix.query(Q, k, qp)  # the stats-off (timed) path
            assert np.array_equal(gi2, oi) and np.array_equal(gs2, os_), case
        ix.close()
