"""One C5-shaped build at a reduced n (ncu target for k_hash_build): n points of d = 256
i.i.d. Gaussian rows, L = 64, K = 2, D = 256, iProbes = 5, alpha = 0.005.
usage: python profiles/build_probe.py [n] [L]"""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_01382_b200 as fpp

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
L = int(sys.argv[2]) if len(sys.argv) > 2 else 64
g = torch.Generator(device="cuda").manual_seed(1)
X = torch.randn(n, 256, device="cuda", generator=g)
X /= X.norm(dim=1, keepdim=True)
for _ in range(2):
    ix = fpp.Index.build(X, L=L, K=2, D=256, iProbes=5, alpha=0.005, kappa=20, seed=1)
    t = ix.timings()
    print({k: round(v, 2) for k, v in t.items() if k in ("hash_ms", "sort_ms")}, n / (t["hash_ms"] + t["sort_ms"]) * 1e-3, "M pts/s")
    ix.close()
