"""Pin the CPU oracle (oracle/fpp_oracle.c) to the reference.

1. Golden fingerprints (tests/golden/fingerprints.json, generated from the
   unmodified reference build by tests/golden/make_fingerprints.py; identical
   to SURVEY.md section 8(c)): normalized bytes, projections and hash codes of
   20,000 rows at d = 128 / 256 / 300 / 960, four stacks each.
2. Direct comparison with oracle/_ref (the reference's own rotation.cpp /
   dataset.cpp / common.hpp) on random inputs when that build is present.
"""
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "fingerprints.json")))


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


@pytest.mark.parametrize("d", [128, 256, 300, 960])
def test_fingerprints(orc, d):
    g = GOLD["dims"][str(d)]
    n = GOLD["n"]
    X = orc.normalize(raw_rows(n, d))  # dataset.cpp:24-38, exactly once
    assert format(orc.fnv1a64(X), "016x") == g["norm"]
    P = orc.lib().orc_pad_dimension(d)
    for key, want in g["stacks"].items():
        t, f = (int(v) for v in key.split(","))
        Y = orc.project_rows(X, P, orc.lib().orc_derive_seed(1, t, f, 0))
        # chained fnv over rows == fnv over the concatenation (streaming hash)
        assert format(orc.fnv1a64(Y, 0), "016x") == want["proj"], (d, key)
        assert format(orc.fnv1a64(orc.cp_hash_rows(Y), 0), "016x") == want["hash"], (d, key)


def ref_or_skip(orc):
    R = orc.ref()
    if R is None:
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return R


def test_common_vs_reference(orc):
    R = ref_or_skip(orc)
    rng = np.random.default_rng(5)
    for z in rng.integers(0, 2**63, 200, dtype=np.uint64).tolist() + [0, 1, 2**64 - 1]:
        assert orc.lib().orc_mix64(z) == R.ref_mix64(z)
        assert orc.lib().orc_derive_seed(z, 3, 7, 11) == R.ref_derive_seed(z, 3, 7, 11)
    b = rng.integers(0, 255, 1000, dtype=np.uint8)
    assert orc.lib().orc_fnv1a64(b.ctypes.data, 1000, 0xCBF29CE484222325) == \
        R.ref_fnv1a64(b.ctypes.data, 1000, 0xCBF29CE484222325)


@pytest.mark.parametrize("n", [1, 2, 8, 64, 1024])
def test_fht_vs_reference(orc, n):
    R = ref_or_skip(orc)
    v = np.random.default_rng(n).standard_normal(n).astype(np.float32)
    a, b = v.copy(), v.copy()
    orc.lib().orc_fht(a, n)
    assert R.ref_fht(b, n) == 0
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_fht_rejects_non_power_of_two(orc):
    R = ref_or_skip(orc)
    assert R.ref_fht(np.zeros(6, np.float32), 6) == -1  # rotation.cpp:18-20


@pytest.mark.parametrize("d,D", [(2, 2), (5, 8), (17, 32), (100, 128), (128, 128), (200, 64),
                                 (300, 512), (960, 1024), (64, 256)])
def test_project_vs_reference(orc, d, D):
    R = ref_or_skip(orc)
    X = np.random.default_rng(d).standard_normal((50, d)).astype(np.float32)
    seed = orc.lib().orc_derive_seed(1, 4, 1, 0)
    want = np.empty((50, D), np.float32)
    assert R.ref_project(d, D, seed, X.reshape(-1), 50, want.reshape(-1)) == 0
    got = orc.project_rows(X, D, seed)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_normalize_and_inner_product_vs_reference(orc):
    R = ref_or_skip(orc)
    X = np.random.default_rng(9).standard_normal((500, 37)).astype(np.float32)
    a = orc.normalize(X)
    b = X.copy()
    assert R.ref_normalize(b.reshape(-1), 500, 37) == -1
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    for i in range(20):
        assert orc.lib().orc_inner_product(a[i], a[i + 1], 37) == \
            R.ref_inner_product(a[i], a[i + 1], 37)


def test_center_vs_reference(orc):
    # dataset.cpp:40-57 center(): double mean, float center, fp32 subtraction
    R = ref_or_skip(orc)
    import ctypes as C
    X = np.random.default_rng(5).standard_normal((3001, 41)).astype(np.float32) + 0.3
    a, ca = orc.center(X)
    b = X.copy()
    cb = np.empty(41, np.float32)
    R.ref_center.restype = C.c_int64
    R.ref_center.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p]
    assert R.ref_center(b.ctypes.data, 3001, 41, cb.ctypes.data) == -1
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert np.array_equal(ca.view(np.uint32), cb.view(np.uint32))


def test_normalize_is_not_idempotent(orc):
    # dataset.hpp:50-52 claims idempotence; bit-wise it is not,
    # which is why inputs are normalized exactly once on the host.
    X = orc.normalize(raw_rows(20000, 128))
    Y = orc.normalize(X)
    changed = int((X != Y).any(axis=1).sum())
    assert changed > 0
