"""Regenerate tests/golden/fingerprints.json from the UNMODIFIED reference.

Uses oracle/_ref/libfpp_ref.so (reference rotation.cpp + dataset.cpp +
common.hpp compiled by oracle/Makefile; needs /root/reference, i.e. this
container).  Recipe = SURVEY.md section 8(c):
  x[i] = float(int32(mix64(i) >> 40) - 2^23) * 2^-23, i < n*d;  Dataset(x, d);
  normalize once;  SpinnerStack(d, pad(d), derive_seed(1, t, f));
  proj = chained fnv1a64(row bytes, h) from h = 0;
  hash = chained fnv1a64(&u32 cross_polytope_hash(row), 4, h) from h = 0
         (argmax |p|, lowest index on ties; i if p >= 0 else D + i);
  norm = fnv1a64(normalized bytes) with the default basis.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle  # noqa: E402

N = 20000
DIMS = (128, 256, 300, 960)


def mix64(z):
    z = z + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def raw_rows(n, d):
    i = np.arange(n * d, dtype=np.uint64)
    with np.errstate(over="ignore"):
        v = (mix64(i) >> np.uint64(40)).astype(np.int64) - (1 << 23)
    return (v.astype(np.float32) * np.float32(1.0 / (1 << 23))).reshape(n, d)


def cp_hash(P):
    a = np.abs(P)
    i = np.argmax(a, axis=1)  # first max = lowest index on ties
    v = P[np.arange(len(P)), i]
    D = P.shape[1]
    return np.where(v >= 0, i, D + i).astype(np.uint32)


def chained(rows_bytes_iter):
    h = 0
    for b in rows_bytes_iter:
        h = oracle.fnv1a64(b, h)
    return h


def main():
    R = oracle.ref()
    if R is None:
        raise SystemExit("oracle/_ref/libfpp_ref.so missing: run `make -C oracle` with /root/reference")
    out = {"n": N, "recipe": "SURVEY.md 8(c)", "dims": {}}
    for d in DIMS:
        X = raw_rows(N, d).copy()
        assert R.ref_normalize(X.reshape(-1), N, d) == -1
        P = 1
        while P < d:
            P <<= 1
        entry = {"norm": format(oracle.fnv1a64(X), "016x"), "stacks": {}}
        for t in (0, 1):
            for f in (0, 1):
                seed = R.ref_derive_seed(1, t, f, 0)
                Y = np.empty((N, P), np.float32)
                assert R.ref_project(d, P, seed, X.reshape(-1), N, Y.reshape(-1)) == 0
                proj = chained(Y[r] for r in range(N))
                hs = cp_hash(Y)
                hh = chained(hs[r:r + 1] for r in range(N))
                entry["stacks"][f"{t},{f}"] = {"proj": format(proj, "016x"), "hash": format(hh, "016x")}
        out["dims"][str(d)] = entry
    with open(os.path.join(HERE, "fingerprints.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out)[:300])


if __name__ == "__main__":
    main()
