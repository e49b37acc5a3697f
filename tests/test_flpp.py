"""FLPP index persistence (SPEC.md:270-278 save/load; format :283-287).

GPU: load(save(ix)) answers queries bit-identically; the same (dataset, config)
saves byte-identical files; an index written from the CPU restatement's CSR
loads and answers exactly like the restatement; every SPEC error class
(magic, version, truncation, checksum) plus dataset-reference mismatches.
CPU: the numpy format tool round-trips and detects corruption.
"""
import os

import numpy as np
import pytest

from fpp_testutil import gpu_available

CFG = dict(L=4, K=2, D=64, iProbes=3, alpha=0.1, kappa=10)


def data(fpp, n, d, seed=1, stream=0):
    return fpp.normalize(fpp.synth(n, d, 8, 0.3, seed=seed, stream=stream))


def test_flpp_tool_roundtrip_and_corruption(tmp_path):
    from paper_2206_01382_b200 import flpp
    rng = np.random.default_rng(0)
    K, D, L = 2, 4, 2
    NB = 4 * D * D
    tables = []
    for _ in range(L):
        sizes = rng.integers(0, 3, NB)
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint32)
        ids = rng.integers(0, 100, off[-1]).astype(np.uint32)
        sc = rng.random(off[-1]).astype(np.float32)
        tables.append((off, ids, sc))
    p = str(tmp_path / "a.flpp")
    flpp.write(p, L=L, K=K, D=D, alpha=0.5, iprobes=2, kappa=3, seed=7, n=100, d=5, tables=tables,
               content_hash_value=123)
    r = flpp.read(p)
    assert (r["L"], r["K"], r["D"], r["seed"], r["n"], r["d"], r["content_hash"]) == \
        (L, K, D, 7, 100, 5, 123)
    for (o, i, s), (o2, i2, s2) in zip(tables, r["tables"]):
        assert np.array_equal(o, o2) and np.array_equal(i, i2) and np.array_equal(s, s2)
    raw = bytearray(open(p, "rb").read())
    raw[-12] ^= 1  # a body byte
    open(p, "wb").write(raw)
    with pytest.raises(ValueError, match="checksum"):
        flpp.read(p)


@pytest.mark.gpu
def test_flpp_gpu_roundtrip_bit_identical(fpp, tmp_path):
    if not gpu_available():
        pytest.skip("needs a CUDA device")
    X = data(fpp, 3000, 64)
    Q = data(fpp, 40, 64, stream=1)
    ix = fpp.Index.build(X, **CFG)
    a, b = str(tmp_path / "a.flpp"), str(tmp_path / "b.flpp")
    ix.save(a)
    fpp.Index.build(X, **CFG).save(b)
    assert open(a, "rb").read() == open(b, "rb").read()  # determinism: byte-identical
    iy = fpp.Index.load(a, X)
    for qp in (4, 200, 2000):
        gi, gs, gst = ix.query(Q, 10, qp, return_stats=True)
        li, ls, lst = iy.query(Q, 10, qp, return_stats=True)
        assert np.array_equal(gi, li) and np.array_equal(gs, ls) and np.array_equal(gst, lst)
    for t in range(CFG["L"]):
        for u, v in zip(ix.table(t), iy.table(t)):
            assert np.array_equal(u, v)
    assert ix.info()["kept_total"] == iy.info()["kept_total"]



@pytest.mark.gpu
def test_flpp_cross_implementation(fpp, orc, tmp_path):
    if not gpu_available():
        pytest.skip("needs a CUDA device")
    from paper_2206_01382_b200 import flpp
    X = data(fpp, 3000, 64, seed=4)
    Q = data(fpp, 40, 64, seed=4, stream=1)
    ox = orc.Index(X, L=CFG["L"], K=2, D=64, iprobes=3, alpha=0.1, kappa=10)
    # CPU restatement's CSR -> FLPP -> fpp_load: answers like the restatement
    p = str(tmp_path / "orc.flpp")
    flpp.write(p, L=CFG["L"], K=2, D=64, alpha=0.1, iprobes=3, kappa=10, seed=1, n=3000, d=64,
               tables=[ox.table(t) for t in range(CFG["L"])],
               content_hash_value=flpp.content_hash(X))
    iy = fpp.Index.load(p, X)
    gi, gs, gst = iy.query(Q, 10, 300, return_stats=True)
    oi, os_, ost = ox.query(Q, 10, 300)
    assert np.array_equal(gi, oi) and np.array_equal(gs, os_) and np.array_equal(gst, ost)
    # GPU build -> fpp_save -> numpy reader: the restatement's CSR
    g = str(tmp_path / "gpu.flpp")
    fpp.Index.build(X, **CFG).save(g)
    r = flpp.read(g)
    for t in range(CFG["L"]):
        for u, v in zip(r["tables"][t], ox.table(t)):
            assert np.array_equal(u, v)


@pytest.mark.gpu
def test_flpp_errors(fpp, tmp_path):
    if not gpu_available():
        pytest.skip("needs a CUDA device")
    X = data(fpp, 1000, 32)
    ix = fpp.Index.build(X, L=2, K=2, D=32, iProbes=2, alpha=0.2)
    p = str(tmp_path / "x.flpp")
    ix.save(p)
    good = open(p, "rb").read()

    def load_bytes(raw, XX=X):
        q = str(tmp_path / "y.flpp")
        open(q, "wb").write(raw)
        return fpp.Index.load(q, XX)

    with pytest.raises(fpp.FppFormatError, match="magic"):
        load_bytes(b"FLPQ" + good[4:])
    bad_version = bytearray(good)
    bad_version[4] += 1  # version + 1
    with pytest.raises(fpp.FppUnsupported, match="version 2"):
        load_bytes(bytes(bad_version))
    with pytest.raises(fpp.FppFormatError, match="truncated"):
        load_bytes(good[:len(good) // 2])
    flipped = bytearray(good)
    flipped[-1] ^= 0x40  # the footer no longer matches the body
    with pytest.raises(fpp.FppFormatError, match="checksum"):
        load_bytes(bytes(flipped))
    X2 = X.copy()
    X2[0, 0] = np.nextafter(X2[0, 0], 2.0)
    with pytest.raises(fpp.FppFormatError, match="content hash"):
        load_bytes(good, X2)
    with pytest.raises(fpp.FppDimensionError):
        load_bytes(good, X[:999])
    with pytest.raises(fpp.FppIOError):
        fpp.Index.load(str(tmp_path / "missing.flpp"), X)
    assert load_bytes(good).info()["kept_total"] == ix.info()["kept_total"]
