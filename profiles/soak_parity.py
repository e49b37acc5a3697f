"""Randomised GPU-vs-oracle soak (not a pytest module): random small configurations for
a bounded time; ids, scores and stats must equal the oracle's.
usage: python profiles/soak_parity.py [seconds] [seed]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2206_01382_b200 as fpp
from oracle import oracle as orc

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 12345)
t0, cases = time.time(), 0
while time.time() - t0 < budget:
    d = int(rng.choice([8, 17, 32, 48, 64, 100, 128, 200, 256, 300, 320, 512, 960]))
    n = int(rng.integers(500, 12000))
    K = int(rng.choice([1, 2, 2, 2]))
    P = 1 << max(int(d - 1).bit_length(), 0)
    D = int(rng.choice([P, P, max(P // 2, 2)]))
    ip = int(rng.integers(1, min(D, 8) + 1))
    L = int(rng.integers(1, 7))
    alpha = float(rng.choice([1.0, 0.5, 0.1, 0.02]))
    kappa = int(rng.choice([0, 5, 20]))
    clusters = int(rng.choice([0, 5, 40]))
    seed = int(rng.integers(1, 1 << 30))
    if rng.random() < 0.1:
        n = int(rng.integers(20000, 60000))  # (a few larger shards)
    if os.environ.get("SOAK_BIG"):  # the walking screen at scale: admission hash / bitmap / log paths
        d = int(rng.choice([64, 128, 128, 256]))
        n = int(rng.integers(200_000, 1_500_000))
        K, P = 2, d
        D = d
        ip, L = 3, int(rng.integers(4, 10))
        alpha, kappa = float(rng.choice([0.01, 0.05, 0.3])), 20
        clusters = int(rng.choice([100, 2000]))
    X = fpp.normalize(fpp.synth(n, d, clusters, 0.3, seed=seed))
    if rng.random() < 0.15 and not os.environ.get("SOAK_BIG"):
        # sparse rows (1-6 non-zeros): projections with many equal |p| -- tie order everywhere
        m = int(rng.choice([1, 2, 3, 6]))
        X = np.zeros((n, d), np.float32)
        for i in range(n):
            X[i, rng.choice(d, min(m, d), replace=False)] = rng.standard_normal(min(m, d)).astype(np.float32)
        X[np.abs(X).sum(axis=1) == 0, 0] = 1.0
        X = fpp.normalize(X)
    if rng.random() < 0.3:  # exact duplicates: equal scores, ties to the lower id
        src = rng.integers(0, n, size=max(1, n // 50))
        X[rng.integers(0, n, size=len(src))] = X[src]
    nq = int(rng.integers(1, 90)) if rng.random() < 0.85 else int(rng.integers(600, 2500))
    if os.environ.get("SOAK_BIG"):
        nq = 150
    Q = fpp.normalize(fpp.synth(nq, d, clusters, 0.3, seed=seed, stream=1))
    if rng.random() < 0.3:
        Q[: min(nq, 5)] = X[: min(nq, 5)]  # queries that are data points
    prm = dict(L=L, K=K, D=D, alpha=alpha, kappa=kappa, seed=seed)
    # variants: falconn_baseline mode, centering, a 2..3-shard MultiIndex on one device
    variant = str(rng.choice(["plain", "plain", "baseline", "centering", "multi"]))
    if variant == "baseline":
        ix = fpp.Index.build(X, iProbes=ip, mode="falconn_baseline", **prm)
        ox = orc.Index(X, iprobes=ip, mode=1, **prm)
    elif variant == "centering":
        X = X + np.float32(0.03)
        ix = fpp.Index.build(X, iProbes=ip, centering=True, **prm)
        ox = orc.Index(orc.center(X)[0], iprobes=ip, **prm)
    elif variant == "multi":
        G = int(rng.integers(2, 4))
        ix = fpp.MultiIndex.build(X, num_gpus=G, devices=[0] * G, iProbes=ip, **prm)
        ox = orc.Index(X, iprobes=ip, **prm)
    else:
        ix = fpp.Index.build(X, iProbes=ip, **prm)
        ox = orc.Index(X, iprobes=ip, **prm)
    NB = (2 * D) ** K
    for _ in range(3):
        k = int(rng.choice([1, 7, 20, 32, 33, 50, 100]))
        k = min(k, n)
        qp = int(rng.integers(L, min(L * NB, 30000) + 1))
        stats = bool(rng.integers(0, 2))
        rr = int(rng.choice([0, 0, k, 3 * k, 50 * k])) if variant in ("plain", "baseline") else 0
        kw = dict(rerank=rr) if rr else {}
        # scheduling / path switches (none may change a result)
        for var in ("FPP_FORCE_COLLECT", "FPP_PRUNE", "FPP_NO_PRUNE", "FPP_NO_REORDER", "FPP_SERIAL"):
            os.environ.pop(var, None)
        env = {}
        if rng.random() < 0.3:
            env["FPP_FORCE_COLLECT"] = str(rng.choice(["grouped", "sliced", "cluster", "global"]))
        if rng.random() < 0.3:
            env[str(rng.choice(["FPP_PRUNE", "FPP_NO_PRUNE"]))] = "1"
        if rng.random() < 0.2:
            env["FPP_NO_REORDER"] = "1"
        if rng.random() < 0.2:
            env["FPP_SERIAL"] = "1"
        os.environ.update(env)
        if os.environ.get("SOAK_LOG"):
            print("Q", dict(variant=variant, n=n, d=d, ip=ip, k=k, qp=qp, stats=stats, rerank=rr,
                            clusters=clusters, nq=len(Q), **prm), file=sys.stderr, flush=True)
        try:
            if stats:
                gi, gs, gst = ix.query(Q, k, qp, return_stats=True, **kw)
            else:
                gi, gs = ix.query(Q, k, qp, **kw)
        except Exception as ex:
            print("EXCEPTION", ex, env, dict(variant=variant, n=n, d=d, ip=ip, k=k, qp=qp, stats=stats, rerank=rr,
                                        clusters=clusters, nq=len(Q), **prm), flush=True)
            sys.exit(2)
        oi, os_, ost = ox.query(Q, k, qp, **kw)
        ncol = 3 if variant == "multi" else ost.shape[1]  # (the multi index reports no exact count)
        ok = np.array_equal(gi, oi) and np.array_equal(gs, os_) and \
            (not stats or np.array_equal(gst[:, :ncol], ost[:, :ncol]))
        if not ok:
            print("MISMATCH", env, dict(variant=variant, n=n, d=d, ip=ip, k=k, qp=qp, stats=stats, rerank=rr,
                                   clusters=clusters, nq=len(Q), **prm), flush=True)
            sys.exit(1)
    ix.close()
    cases += 1
print(f"soak ok: {cases} random configurations x 3 queries batches in {time.time() - t0:.0f} s")
