"""Feasibility study (GPU box): how many C4 bucket entries could a per-bucket (or
per-block) cap bound skip?  For a block of entries B with center c and radius
rho = max ||x - c|| (x in B):  x.q = c.q + (x - c).q <= c.q + rho ||q||.  A block
whose bound is below the query's final k-th best cannot contribute.  Prints the
fraction of walked entries in skippable blocks for whole buckets and for CSR-order
blocks of 8/16 entries.  Not product code: an analysis probe."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2206_01382_b200 as fpp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
NQS = 1000
cfg = dict(d=128, clusters=10_000, sigma=0.25, L=50, K=2, D=128, iprobes=3, alpha=0.01)
t0 = time.time()
X = fpp.normalize(fpp.synth(n, 128, cfg["clusters"], cfg["sigma"], seed=1, stream=0))
Q = fpp.normalize(fpp.synth(NQS, 128, cfg["clusters"], cfg["sigma"], seed=1, stream=1))
print(f"data {time.time() - t0:.1f}s", flush=True)
dev = torch.device("cuda", 0)
Xd = torch.from_numpy(X).to(dev)
Qd = torch.from_numpy(Q).to(dev)
ix = fpp.Index.build(Xd, L=50, K=2, D=128, iProbes=3, alpha=0.01)
NB = ix.info()["num_buckets"]
ids = torch.empty((NQS, 20), dtype=torch.int32, device=dev)
sc = torch.empty((NQS, 20), dtype=torch.float64, device=dev)
ix.query_device(Qd, ids, sc, 20, 5000)
thr = sc[:, -1].float()  # final k-th best
probes = ix.query_probe_sets_device(Qd, 5000).long()  # [nq, P] global bucket ids t*NB+b
torch.cuda.synchronize()
print("thr quantiles", torch.quantile(thr, torch.tensor([0.05, 0.5, 0.95], device=dev)).tolist())
qn = Qd.norm(dim=1)

for BS in (0, 8, 16, 32):
    # per table: blocks = whole buckets (BS = 0) or CSR-order runs of BS entries
    tot_e = 0
    skip_e = 0
    skip_e_half = 0
    for t in range(50):
        off, tid, _ = ix.table(t)
        off = torch.from_numpy(off.astype(np.int64)).to(dev)
        tid = torch.from_numpy(tid.astype(np.int64)).to(dev)
        lens = off[1:] - off[:-1]
        bidx = torch.repeat_interleave(torch.arange(NB, device=dev), lens)  # bucket of entry
        pos_in = torch.arange(len(tid), device=dev) - off[bidx]
        blk = pos_in // BS if BS else torch.zeros_like(pos_in)
        nblk_b = (lens + BS - 1) // BS if BS else (lens > 0).long()
        blk_base = torch.cumsum(nblk_b, 0) - nblk_b
        gb = blk_base[bidx] + blk  # global block id
        NBL = int(nblk_b.sum())
        xe = Xd[tid]
        cnt = torch.zeros(NBL, device=dev).index_add_(0, gb, torch.ones(len(tid), device=dev))
        cen = torch.zeros((NBL, 128), device=dev).index_add_(0, gb, xe) / cnt[:, None].clamp(min=1)
        r = (xe - cen[gb]).norm(dim=1)
        rho = torch.zeros(NBL, device=dev).scatter_reduce_(0, gb, r, "amax")
        # this table's probes of each query
        m = (probes // NB) == t
        for q0 in range(0, NQS, 100):
            pr = probes[q0:q0 + 100]
            mm = m[q0:q0 + 100]
            qi, pj = mm.nonzero(as_tuple=True)
            b = pr[qi, pj] % NB
            nb_ = nblk_b[b]
            # expand to blocks
            rep = torch.repeat_interleave(torch.arange(len(b), device=dev), nb_)
            within = torch.arange(len(rep), device=dev) - (torch.cumsum(nb_, 0) - nb_)[rep]
            g = blk_base[b][rep] + within
            qq = qi[rep] + q0
            bound = (cen[g] * Qd[qq]).sum(1) + rho[g] * qn[qq]
            c = cnt[g]
            tot_e += int(c.sum())
            skip_e += int(c[bound < thr[qq]].sum())
            skip_e_half += int(c[bound < thr[qq] - 0.05].sum())
    print(f"block {BS or 'bucket'}: entries {tot_e / NQS:.0f}/query, skippable at final thr "
          f"{skip_e / tot_e:.3f}, at thr-0.05 {skip_e_half / tot_e:.3f}", flush=True)
