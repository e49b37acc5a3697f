"""FLPP index files in numpy (no device): read / write the format that
fpp_save / fpp_load use (include/falconnpp.h).

A table is given as CSR over its 4D^2 (K=2) or 2D (K=1) buckets: offsets
[NB+1] u32, ids [kept] u32, scores [kept] f32, each bucket in (score desc, id
asc) order.  Used to inspect GPU-written indexes and to hand an index built
elsewhere (e.g. by the CPU restatement in the tests) to fpp_load.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"FLPP"
VERSION = 1
FNV_BASIS, FNV_PRIME = 0xCBF29CE484222325, 0x100000001B3


def fnv1a64(data: bytes, h: int = FNV_BASIS) -> int:
    """common.hpp:50-57 (byte-serial; meant for test-sized files)."""
    a = np.frombuffer(data, dtype=np.uint8)
    hv = np.uint64(h)
    prime = np.uint64(FNV_PRIME)
    with np.errstate(over="ignore"):
        for b in a.tolist():
            hv = (hv ^ np.uint64(b)) * prime
    return int(hv)


def content_hash(X) -> int:
    return fnv1a64(np.ascontiguousarray(X, dtype=np.float32).tobytes())


def _nb(K: int, D: int) -> int:
    return 4 * D * D if K == 2 else 2 * D


def write(path, *, L, K, D, alpha, iprobes, kappa, seed, n, d, tables, content_hash_value,
          id_offset=0, version=VERSION):
    """tables: list of (offsets, ids, scores) per table."""
    head = MAGIC + struct.pack("<IIIIfIIIIIQQI", version, L, K, D, alpha, iprobes, kappa, 0, 0,
                               id_offset, seed, n, d)
    head += struct.pack("<I", 0) + struct.pack("<Q", content_hash_value)
    body = bytearray()
    for off, ids, sc in tables:
        off = np.asarray(off, dtype=np.uint32)
        nz = np.nonzero(np.diff(off))[0]
        body += struct.pack("<I", len(nz))
        for b in nz:
            o0, o1 = int(off[b]), int(off[b + 1])
            body += struct.pack("<II", int(b), o1 - o0)
            rec = np.empty((o1 - o0, 2), dtype=np.uint32)
            rec[:, 0] = np.asarray(ids[o0:o1], dtype=np.uint32)
            rec[:, 1] = np.asarray(sc[o0:o1], dtype=np.float32).view(np.uint32)
            body += rec.tobytes()
    with open(path, "wb") as f:
        f.write(head)
        f.write(body)
        f.write(struct.pack("<Q", fnv1a64(bytes(body))))


def read(path) -> dict:
    """Parse and verify (magic, version, checksum); returns header fields + tables."""
    raw = open(path, "rb").read()
    if raw[:4] != MAGIC:
        raise ValueError("bad magic")
    hdr = struct.unpack_from("<IIIIfIIIIIQQI", raw, 4)
    version, L, K, D, alpha, iprobes, kappa, centering, mode, id_offset, seed, n, d = hdr
    if version != VERSION:
        raise ValueError(f"unsupported FLPP version {version}")
    pos = 4 + struct.calcsize("<IIIIfIIIIIQQI")
    if centering:
        pos += 4 * d
    (plen,) = struct.unpack_from("<I", raw, pos)
    pos += 4 + plen
    (chash,) = struct.unpack_from("<Q", raw, pos)
    pos += 8
    body0 = pos
    NB = _nb(K, D)
    tables = []
    for _ in range(L):
        (nz,) = struct.unpack_from("<I", raw, pos)
        pos += 4
        off = np.zeros(NB + 1, dtype=np.uint32)
        ids, sc, cur, last = [], [], 0, 0
        for _ in range(nz):
            b, cnt = struct.unpack_from("<II", raw, pos)
            pos += 8
            rec = np.frombuffer(raw, dtype=np.uint32, count=2 * cnt, offset=pos).reshape(cnt, 2)
            pos += 8 * cnt
            off[last + 1:b + 1] = cur
            cur += cnt
            off[b + 1] = cur
            last = b + 1
            ids.append(rec[:, 0].copy())
            sc.append(rec[:, 1].copy().view(np.float32))
        off[last:] = cur
        tables.append((off, np.concatenate(ids) if ids else np.zeros(0, np.uint32),
                       np.concatenate(sc) if sc else np.zeros(0, np.float32)))
    (footer,) = struct.unpack_from("<Q", raw, pos)
    if footer != fnv1a64(raw[body0:pos]):
        raise ValueError("body checksum mismatch")
    return dict(version=version, L=L, K=K, D=D, alpha=alpha, iprobes=iprobes, kappa=kappa,
                id_offset=id_offset, seed=seed, n=n, d=d, content_hash=chash, tables=tables)
