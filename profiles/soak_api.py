"""Randomised soak of the other entry points against the oracle (companion of
soak_parity.py): CSR tables, brute force (any k), FLPP save -> load round trips, the
device API on user streams, and the split path (probe sets computed by one index, stage B
from them) on random configurations.  usage: python profiles/soak_api.py [seconds] [seed]"""
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2206_01382_b200 as fpp
from oracle import oracle as orc

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
t0, cases = time.time(), 0
tmp = tempfile.mkdtemp()


def fail(what, cfg):
    print("MISMATCH", what, cfg, flush=True)
    sys.exit(1)


while time.time() - t0 < budget:
    d = int(rng.choice([5, 16, 33, 64, 100, 128, 256, 300, 960]))
    n = int(rng.integers(300, 9000))
    K = int(rng.choice([1, 2, 2]))
    P = int(orc.lib().orc_pad_dimension(d))
    D = int(rng.choice([P, max(P // 2, 2)]))
    ip = int(rng.integers(1, min(D, 16) + 1))
    L = int(rng.integers(1, 5))
    prm = dict(L=L, K=K, D=D, alpha=float(rng.choice([1.0, 0.3, 0.05])), kappa=int(rng.choice([0, 3, 20])),
               seed=int(rng.integers(1, 1 << 30)))
    clusters = int(rng.choice([0, 8]))
    X = fpp.normalize(fpp.synth(n, d, clusters, 0.3, seed=prm["seed"]))
    nq = int(rng.integers(1, 60))
    Q = fpp.normalize(fpp.synth(nq, d, clusters, 0.3, seed=prm["seed"], stream=1))
    cfg = dict(n=n, d=d, ip=ip, clusters=clusters, nq=nq, **prm)
    ix = fpp.Index.build(X, iProbes=ip, **prm)
    ox = orc.Index(X, iprobes=ip, **prm)
    for t in range(L):  # CSR: offsets, ids, scores
        for u, v in zip(ix.table(t), ox.table(t)):
            if not np.array_equal(np.asarray(u).view(np.uint32), np.asarray(v).view(np.uint32)):
                fail(("table", t), cfg)
    k = min(int(rng.choice([1, 10, 32, 40, 97])), n)
    bi, bs = ix.brute_force(Q, k)
    ri, rs = orc.brute_force(X, Q, k)
    if not (np.array_equal(bi, ri) and np.array_equal(bs, rs)):
        fail(("brute", k), cfg)
    NB = (2 * D) ** K
    qp = int(rng.integers(L, min(L * NB, 8000) + 1))
    oi, os_, ost = ox.query(Q, k, qp)
    # FLPP round trip
    path = os.path.join(tmp, "i.flpp")
    ix.save(path)
    iy = fpp.Index.load(path, X)
    li, ls, lst = iy.query(Q, k, qp, return_stats=True)
    if not (np.array_equal(li, oi) and np.array_equal(ls, os_) and np.array_equal(lst, ost)):
        fail(("flpp", k, qp), cfg)
    # device API on a user stream + the split path through the loaded index
    Qd = torch.from_numpy(Q).cuda()
    st = torch.cuda.Stream()
    ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    sc = torch.empty((nq, k), dtype=torch.float64, device="cuda")
    with torch.cuda.stream(st):
        ix.query_device(Qd, ids, sc, k, qp, stream=st.cuda_stream)
        probes = ix.query_probe_sets_device(Qd, qp, stream=st.cuda_stream)
        ids2 = torch.empty_like(ids)
        sc2 = torch.empty_like(sc)
        iy.query_from_probe_sets_device(Qd, probes, ids2, sc2, k, qp, stream=st.cuda_stream)
    st.synchronize()
    for a, b, what in ((ids, sc, "device"), (ids2, sc2, "split")):
        if not (np.array_equal(a.cpu().numpy().view(np.uint32), oi) and np.array_equal(b.cpu().numpy(), os_)):
            fail((what, k, qp), cfg)
    ix.close()
    iy.close()
    cases += 1
print(f"api soak ok: {cases} random configurations in {time.time() - t0:.0f} s")
