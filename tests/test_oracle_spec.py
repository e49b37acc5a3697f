"""SPEC.md worked examples and acceptance properties, against the CPU oracle.

The reference ships no tests; these are the SPEC's own
[TRIVIAL]/[DERIVED] examples (line numbers cited per test) plus acceptance
criteria #4, #5 and #10 at desk scale.
"""
import numpy as np
import pytest


def f32(*v):
    return np.array(v, dtype=np.float32)


def test_fht_examples(orc):
    a = f32(1, 0)
    orc.lib().orc_fht(a, 2)
    assert list(a) == [1, 1]
    b = f32(1, 1)
    orc.lib().orc_fht(b, 2)
    assert list(b) == [2, 0]
    v = np.random.default_rng(1).standard_normal(256).astype(np.float32)
    w = v.copy()
    orc.lib().orc_fht(w, 256)
    orc.lib().orc_fht(w, 256)
    np.testing.assert_allclose(w, 256 * v, rtol=1e-5, atol=1e-4)


def test_project_examples(orc):
    seed = orc.lib().orc_derive_seed(1, 0, 0, 0)
    assert not orc.project(np.zeros(64, np.float32), 64, seed).any()
    x = np.random.default_rng(2).standard_normal(64).astype(np.float32)
    assert np.array_equal(orc.project(2 * x, 64, seed), 2 * orc.project(x, 64, seed))


def test_cross_polytope_hash_examples(orc):
    assert orc.lib().orc_cp_hash(f32(0.6, -0.8), 2) == 3
    assert orc.lib().orc_cp_hash(f32(0.9, 0.1), 2) == 0
    assert orc.lib().orc_cp_hash(f32(0.5, 0.5), 2) == 0
    assert orc.lib().orc_cp_hash(f32(-0.0, 0.0), 2) == 0  # -0.0 counts as >= 0


def index_probes(orc, p1, p2, ip, D=2):
    b = np.empty(ip, np.uint32)
    s = np.empty(ip, np.float32)
    orc.lib().orc_index_probes(np.concatenate([f32(*p1), f32(*p2)]), 2, D, ip, b, s)
    return list(b), list(s)


def test_bucket_id_examples(orc):  # SPEC.md:181-183 via the iProbes=1 probe
    assert index_probes(orc, (0.9, 0.1), (0.9, 0.1), 1)[0] == [0]          # (0,0) -> 0
    assert index_probes(orc, (0.1, -0.9), (0.1, -0.9), 1)[0] == [15]       # (3,3) -> 15
    assert index_probes(orc, (0.1, 0.9), (-0.9, 0.1), 1)[0] == [1 * 4 + 2]  # (1,2) -> 6


def test_index_probe_sequence_examples(orc):
    b, s = index_probes(orc, (0.9, 0.2), (0.8, 0.3), 4)
    # pairs (0,0):1.7 (0,1):1.2 (1,0):1.0 (1,1):0.5 -> buckets h1*2D+h2
    assert b == [0, 1, 4, 5]
    np.testing.assert_allclose(s, [1.7, 1.2, 1.0, 0.5], rtol=1e-6)
    assert all(s[i] >= s[i + 1] for i in range(3))
    b1, _ = index_probes(orc, (0.9, 0.2), (0.8, 0.3), 1)
    assert b1 == [0]


def test_query_probe_sequence_examples(orc):
    vals = np.array([[[0.9, 0.2], [0.8, 0.3]]], np.float32)   # L=1, K=2, s=2
    codes = np.array([[[0, 1], [0, 1]]], np.uint32)
    assert list(orc.probe_set_lists(vals, codes, 2, 1)) == [0]          # qProbes = L
    assert list(orc.probe_set_lists(vals, codes, 2, 2)) == [0, 1]       # + (0,1):1.2
    assert list(orc.probe_set_lists(vals, codes, 2, 3)) == [0, 1, 4]    # + (1,0):1.0
    assert list(orc.probe_set_lists(vals, codes, 2, 4)) == [0, 1, 4, 5]
    # prefix monotone
    prev = set()
    for p in range(1, 5):
        cur = set(orc.probe_set_lists(vals, codes, 2, p).tolist())
        assert prev <= cur
        prev = cur


def test_filter_bucket_examples(orc):
    assert orc.keep_count(100, 0.1, 3, 20) == 20
    assert orc.keep_count(5, 1.0, 1, 0) == 5
    assert orc.keep_count(10, 0.5, 1, 0) == 5
    assert orc.keep_count(3, 0.01, 1, 20) == 3
    assert orc.keep_count(100000, 0.05, 3, 20) == 1666  # floor(double(alpha)*B/iP)


def test_inner_product_examples(orc):
    ip = orc.lib().orc_inner_product
    assert ip(f32(1, 0), f32(0, 1), 2) == 0.0
    assert abs(ip(f32(0.6, 0.8), f32(0.6, 0.8), 2) - 1.0) < 1e-6
    assert abs(ip(f32(0.6, 0.8), f32(0.8, 0.6), 2) - 0.96) < 1e-6


def test_normalize_examples(orc):
    np.testing.assert_allclose(orc.normalize(np.array([[3, 4]], np.float32)), [[0.6, 0.8]],
                               rtol=1e-7)
    assert list(orc.normalize(np.array([[0, 1]], np.float32))[0]) == [0, 1]
    with pytest.raises(ValueError):
        orc.normalize(np.array([[0, 0]], np.float32))


def data(orc, n, d, clusters=0, sigma=0.0, seed=1, stream=0):
    return orc.normalize(orc.synth(n, d, clusters, sigma, seed=seed, stream=stream))


def test_build_alpha1_is_plain_falconn(orc):
    X = data(orc, 3000, 32)
    ox = orc.Index(X, L=3, K=2, D=32, iprobes=1, alpha=1.0, kappa=0)
    for t in range(3):
        off, ids, sc = ox.table(t)
        assert len(ids) == 3000 and sorted(ids) == list(range(3000))
        for b in np.nonzero(np.diff(off))[0][:200]:  # sorted by (score desc, id asc)
            seg_s, seg_i = sc[off[b]:off[b + 1]], ids[off[b]:off[b + 1]]
            order = sorted(range(len(seg_s)), key=lambda j: (-seg_s[j], seg_i[j]))
            assert order == list(range(len(seg_s)))


def test_acceptance4_exhaustive_equals_bruteforce(orc):
    X = data(orc, 2000, 32, seed=3)
    Q = data(orc, 100, 32, seed=3, stream=1)
    L, D = 2, 32
    ox = orc.Index(X, L=L, K=2, D=D, iprobes=1, alpha=1.0, kappa=0)
    ids, sc, st = ox.query(Q, 20, L * 4 * D * D)
    bi, bs = orc.brute_force(X, Q, 20)
    assert np.array_equal(ids, bi)
    assert np.array_equal(sc, bs)
    assert (st[:, 2] == 2000).all()  # every point is a candidate


def test_acceptance5_monotone_and_filter_subset(orc):
    X = data(orc, 4000, 64, 8, 0.3)
    Q = data(orc, 10, 64, 8, 0.3, stream=1)
    full = orc.Index(X, L=4, K=2, D=64, iprobes=3, alpha=1.0, kappa=20)
    for alpha in (0.1, 0.5):
        ox = orc.Index(X, L=4, K=2, D=64, iprobes=3, alpha=alpha, kappa=20)
        for t in range(4):
            fo, fi, _ = full.table(t)
            go, gi, _ = ox.table(t)
            for b in np.nonzero(np.diff(go))[0]:
                assert set(gi[go[b]:go[b + 1]]) <= set(fi[fo[b]:fo[b + 1]])
    L = 4
    for q in Q[:4]:
        prev_p, prev_c = set(), set()
        for qp in (L, 2 * L, 4 * L, 8 * L, 64 * L, 512 * L):
            p, c = full.query_debug(q, qp)
            assert prev_p <= set(p.tolist()) and prev_c <= set(c.tolist())
            prev_p, prev_c = set(p.tolist()), set(c.tolist())


def test_acceptance10_thread_independence(orc):
    X = data(orc, 5000, 64, 10, 0.3)
    Q = data(orc, 40, 64, 10, 0.3, stream=1)
    res = []
    for th in (1, 4, 8):
        ox = orc.Index(X, L=4, K=2, D=64, iprobes=3, alpha=0.1, threads=th)
        tables = [ox.table(t) for t in range(4)]
        res.append((tables, ox.query(Q, 20, 200, threads=th)))
    for tables, q in res[1:]:
        for (a, b) in zip(tables, res[0][0]):
            assert all(np.array_equal(x, y) for x, y in zip(a, b))
        assert all(np.array_equal(x, y) for x, y in zip(q, res[0][1]))


def test_self_query_returns_self(orc):
    X = data(orc, 5000, 64, seed=4)
    ox = orc.Index(X, L=20, K=2, D=64, iprobes=3, alpha=0.1)
    ids, sc, _ = ox.query(X[:50], 1, 20)
    assert (ids[:, 0] == np.arange(50)).mean() >= 0.99
    assert np.allclose(sc[ids[:, 0] == np.arange(50), 0], 1.0, atol=1e-6)


def test_topk_fewer_candidates_than_k(orc):
    X = data(orc, 3000, 32, seed=6)
    ox = orc.Index(X, L=1, K=2, D=32, iprobes=1, alpha=0.01, kappa=1)
    ids, sc, st = ox.query(X[:5], 20, 1)
    for i in range(5):
        u = int(st[i, 2])
        assert u < 20
        assert (ids[i, u:] == 0xFFFFFFFF).all() and np.isneginf(sc[i, u:]).all()
        assert all(sc[i, j] >= sc[i, j + 1] for j in range(u - 1))


def test_brute_force_examples(orc):
    E = np.eye(3, dtype=np.float32)
    ids, sc = orc.brute_force(E, E[:1], 1)
    assert ids[0, 0] == 0 and sc[0, 0] == 1.0
    ids, _ = orc.brute_force(E, E[:1], 3)
    assert list(ids[0]) == [0, 1, 2]  # ties (0, 0) broken by lower id
