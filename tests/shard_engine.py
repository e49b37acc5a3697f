"""CPU engine of the global-filter sharded build protocol (paper_2206_01382_b200.dist).

Test infrastructure: the per-point index probes come from the oracle
(orc_index_probes_rows, bit-identical to the GPU's k_hash_build); the
protocol arithmetic (keep counts, prefixes, cuts) restates the device
kernels of fpp_build.cu with numpy.
"""
import numpy as np
import torch


def ord_key(s):
    u = (np.asarray(s, np.float32) + np.float32(0)).view(np.uint32).astype(np.uint64)
    return np.where(u & 0x80000000, (~u) & 0xFFFFFFFF, u | 0x80000000)


def keep_count(B, alpha, ip, kappa):
    f = np.floor(np.float64(np.float32(alpha)) * B.astype(np.float64) / ip).astype(np.int64)
    return np.minimum(B, np.maximum(kappa, f))


class OracleShardEngine:
    def __init__(self, X, id_offset, L, K, D, iProbes, alpha, kappa=20, seed=1):
        from oracle import oracle as orc
        self.L, self.ip, self.alpha, self.kappa = L, iProbes, alpha, kappa
        self.lo = id_offset
        ox = orc.Index(X, L=L, K=K, D=D, iprobes=iProbes, alpha=1.0, kappa=0, seed=seed)
        self.NB = int(ox.NB)
        n = X.shape[0]
        self.seg = {}  # (t, b) -> sorted keys (score desc, global id asc)
        self.h = np.zeros(L * self.NB, np.int64)
        for t in range(L):
            b, s = ox.index_probes(X, t)
            ids = np.repeat(np.arange(n, dtype=np.uint64) + np.uint64(id_offset), iProbes)
            keys = (((~ord_key(s.reshape(-1))) & np.uint64(0xFFFFFFFF)) << np.uint64(32)) | ids
            bb = b.reshape(-1).astype(np.int64)
            order = np.lexsort((keys, bb))
            bb, keys = bb[order], keys[order]
            ub, start = np.unique(bb, return_index=True)
            ends = list(start[1:]) + [len(bb)]
            for u, a, e in zip(ub, start, ends):
                self.seg[(t, int(u))] = keys[a:e]
                self.h[t * self.NB + int(u)] = e - a

    def hist(self):
        return torch.from_numpy(self.h.astype(np.int32).copy())

    def slots(self, gh):
        self.kg = keep_count(gh.numpy().astype(np.int64), self.alpha, self.ip, self.kappa)
        self.off = np.concatenate([[0], np.cumsum(self.kg)])
        return int(self.off[-1])

    def prefix(self, gh, slots):
        pre = np.full(slots, np.uint64(0xFFFFFFFFFFFFFFFF), np.uint64)
        for (t, b), keys in self.seg.items():
            x = t * self.NB + b
            k = int(self.kg[x])
            m = min(k, len(keys))
            pre[self.off[x]:self.off[x] + m] = keys[:m]
        return torch.from_numpy(pre.view(np.int64))

    def finish(self, gh, allp, world):
        G = gh.numpy().astype(np.int64)
        allp = allp.numpy().view(np.uint64).reshape(world, -1)
        kept = {}
        for (t, b), keys in self.seg.items():
            x = t * self.NB + b
            k = int(self.kg[x])
            if k == 0:
                continue
            if k >= G[x]:
                cut = np.uint64(0xFFFFFFFFFFFFFFFF)
            else:
                merged = np.sort(allp[:, self.off[x]:self.off[x] + k].reshape(-1))
                cut = merged[k - 1]
            sel = keys[keys <= cut]
            if len(sel):
                kept[(t, b)] = sel
        return kept
