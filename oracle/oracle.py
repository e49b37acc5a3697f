"""ctypes binding of the CPU oracle (oracle/liboracle.so) and of the unmodified
reference build (oracle/_ref/libfpp_ref.so).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libfpp_ref.so")

u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class Params(C.Structure):
    _fields_ = [("L", C.c_uint32), ("K", C.c_uint32), ("D", C.c_uint32),
                ("iprobes", C.c_uint32), ("kappa", C.c_uint32),
                ("alpha", C.c_float), ("seed", C.c_uint64), ("mode", C.c_uint32)]


class Stats(C.Structure):
    _fields_ = [("probes", C.c_uint64), ("entries", C.c_uint64),
                ("candidates", C.c_uint64), ("exact", C.c_uint64)]


NATIVE = False  # the loaded library was built with -march=native on this host


def _native_path() -> str:
    """oracle/_native/<host cpu>/liboracle.so: -march=native binaries are per host CPU."""
    import hashlib
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln for ln in f if ln.startswith("model name")), "")
    except OSError:
        pass
    tag = hashlib.sha1(model.encode()).hexdigest()[:12]
    return os.path.join(HERE, "_native", tag, "liboracle.so")


def use_native() -> bool:
    """Switch later lib() users to an -march=native build for this host (the
    reference's own flag, proj/CMakeLists.txt:20-22; -ffp-contract=off keeps every
    fp op as the portable build's).  Objects built before keep their library.  Used
    by bench.py's timing legs only; returns False if it cannot be built here."""
    global _lib, NATIVE
    if NATIVE:
        return True
    so = _native_path()
    src = os.path.join(HERE, "fpp_oracle.c")
    try:
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            os.makedirs(os.path.dirname(so), exist_ok=True)
            subprocess.run(["make", "-s", "-C", HERE, "native", f"NATIVE_SO={so}"], check=True,
                           capture_output=True, timeout=300)
        _lib = _load(so)
        NATIVE = True
    except Exception:
        NATIVE = False
    return NATIVE


def build_oracle(with_ref: bool = True) -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    targets = ["all"] if with_ref and os.path.isdir("/root/reference/proj") else [LIB]
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build_oracle(with_ref=False)
        _lib = _load(LIB)
    return _lib


def _load(path):
        L = C.CDLL(path)
        L.orc_mix64.restype = C.c_uint64
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_derive_seed.argtypes = [C.c_uint64] * 4
        L.orc_fnv1a64.restype = C.c_uint64
        L.orc_fnv1a64.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64]
        L.orc_pad_dimension.restype = C.c_uint32
        L.orc_pad_dimension.argtypes = [C.c_uint32]
        L.orc_fht.argtypes = [f32p, C.c_uint32]
        L.orc_signs.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, f32p]
        L.orc_project.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, f32p, f32p]
        L.orc_project_rows.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, f32p, C.c_uint64,
                                       f32p, C.c_int]
        L.orc_cp_hash_rows.argtypes = [f32p, C.c_uint64, C.c_uint32, u32p]
        L.orc_index_probes_rows.argtypes = [C.c_void_p, f32p, C.c_uint64, C.c_uint32, u32p,
                                            f32p]
        L.orc_index_from_csr.restype = C.c_void_p
        L.orc_index_from_csr.argtypes = [f32p, C.c_uint64, C.c_uint32, C.POINTER(Params), u32p,
                                         u32p, f32p, u64p]
        L.orc_synth.argtypes = [f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_float, C.c_uint64,
                                C.c_uint32, C.c_int]
        L.orc_synth_rows.argtypes = [f32p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32,
                                     C.c_float, C.c_uint64, C.c_uint32, C.c_int]
        L.orc_index_probes_rows_mt.argtypes = [C.c_void_p, f32p, C.c_uint64, C.c_uint32, u32p,
                                               f32p, C.c_int]
        L.orc_csr_from_entries.restype = C.c_uint64
        L.orc_csr_from_entries.argtypes = [u32p, f32p, C.c_uint64, C.c_uint32, C.c_uint32,
                                           C.c_float, C.c_uint32, C.c_uint32, C.c_int, u32p, u32p,
                                           f32p]
        L.orc_keep_count.restype = C.c_uint32
        L.orc_keep_count.argtypes = [C.c_uint32, C.c_float, C.c_uint32, C.c_uint32]
        L.orc_probe_set_lists.restype = C.c_uint64
        L.orc_probe_set_lists.argtypes = [f32p, u32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.c_uint32, C.c_uint64, u64p]
        L.orc_normalize.restype = C.c_int64
        L.orc_normalize.argtypes = [f32p, C.c_uint64, C.c_uint32]
        L.orc_center.restype = None
        L.orc_center.argtypes = [f32p, C.c_uint64, C.c_uint32, f32p]
        L.orc_inner_product.restype = C.c_double
        L.orc_inner_product.argtypes = [f32p, f32p, C.c_uint32]
        L.orc_cp_hash.restype = C.c_uint32
        L.orc_cp_hash.argtypes = [f32p, C.c_uint32]
        L.orc_rank.argtypes = [f32p, C.c_uint32, C.c_uint32, f32p, u32p]
        L.orc_index_probes.argtypes = [f32p, C.c_uint32, C.c_uint32, C.c_uint32, u32p, f32p]
        L.orc_build.restype = C.c_void_p
        L.orc_build.argtypes = [f32p, C.c_uint64, C.c_uint32, C.POINTER(Params), C.c_int,
                                C.c_uint32, C.c_uint32]
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_num_buckets.restype = C.c_uint64
        L.orc_num_buckets.argtypes = [C.c_void_p]
        L.orc_table_size.restype = C.c_uint64
        L.orc_table_size.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_table.argtypes = [C.c_void_p, C.c_uint32, u32p, u32p, f32p]
        L.orc_query_cap.restype = C.c_uint32
        L.orc_query_cap.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_query_probes.restype = C.c_uint64
        L.orc_query_probes.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_query.restype = C.c_int
        L.orc_query.argtypes = [C.c_void_p, f32p, C.c_uint64, C.c_uint32, C.c_uint32, u32p,
                                f64p, C.c_void_p, C.c_int]
        L.orc_query_rerank.restype = C.c_int
        L.orc_query_rerank.argtypes = [C.c_void_p, f32p, C.c_uint64, C.c_uint32, C.c_uint32,
                                       C.c_uint32, u32p, f64p, C.c_void_p, C.c_int]
        L.orc_simhash_rows.restype = None
        L.orc_simhash_rows.argtypes = [C.c_void_p, f32p, C.c_uint64, u64p, C.c_int]
        L.orc_query_debug.restype = C.c_int
        L.orc_query_debug.argtypes = [C.c_void_p, f32p, C.c_uint32, u64p,
                                      C.POINTER(C.c_uint64), u32p, C.POINTER(C.c_uint64)]
        L.orc_query_lists.argtypes = [C.c_void_p, f32p, C.c_uint32, f32p, u32p]
        L.orc_brute_force.argtypes = [f32p, C.c_uint64, C.c_uint32, f32p, C.c_uint64,
                                      C.c_uint32, u32p, f64p, C.c_int]
        return L


def ref():
    """The unmodified reference (rotation.cpp + dataset.cpp), or None."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_LIB):
            return None
        R = C.CDLL(REF_LIB)
        R.ref_mix64.restype = C.c_uint64
        R.ref_mix64.argtypes = [C.c_uint64]
        R.ref_derive_seed.restype = C.c_uint64
        R.ref_derive_seed.argtypes = [C.c_uint64] * 4
        R.ref_fnv1a64.restype = C.c_uint64
        R.ref_fnv1a64.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        R.ref_fht.restype = C.c_int
        R.ref_fht.argtypes = [f32p, C.c_uint64]
        R.ref_project.restype = C.c_int
        R.ref_project.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, f32p, C.c_uint64, f32p]
        R.ref_normalize.restype = C.c_int64
        R.ref_normalize.argtypes = [f32p, C.c_uint64, C.c_uint32]
        R.ref_inner_product.restype = C.c_double
        R.ref_inner_product.argtypes = [f32p, f32p, C.c_uint32]
        _ref = R
    return _ref


# ------------------------------------------------------------------ helpers

def fnv1a64(arr: np.ndarray, h: int = 0xCBF29CE484222325) -> int:
    a = np.ascontiguousarray(arr)
    return lib().orc_fnv1a64(a.ctypes.data, a.nbytes, h)


def project(x: np.ndarray, D: int, seed: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(D, np.float32)
    lib().orc_project(x.shape[-1], D, seed, x, out)
    return out


def project_rows(X: np.ndarray, D: int, seed: int, threads: int = 0) -> np.ndarray:
    X = np.ascontiguousarray(X, dtype=np.float32)
    out = np.empty((X.shape[0], D), np.float32)
    lib().orc_project_rows(X.shape[1], D, seed, X.reshape(-1), X.shape[0], out.reshape(-1),
                           threads or os.cpu_count())
    return out


def cp_hash_rows(Pm: np.ndarray) -> np.ndarray:
    Pm = np.ascontiguousarray(Pm, dtype=np.float32)
    out = np.empty(Pm.shape[0], np.uint32)
    lib().orc_cp_hash_rows(Pm.reshape(-1), Pm.shape[0], Pm.shape[1], out)
    return out


def synth(n: int, d: int, clusters: int = 0, sigma: float = 0.0, seed: int = 1,
          stream: int = 0, threads: int = 0, row0: int = 0) -> np.ndarray:
    X = np.empty((n, d), np.float32)
    lib().orc_synth_rows(X.reshape(-1), row0, n, d, clusters, sigma, seed, stream,
                         threads or os.cpu_count())
    return X


def center(X: np.ndarray):
    """dataset.cpp:40-57 restated: returns (centered copy, center)."""
    X = np.array(X, dtype=np.float32, order="C", copy=True)
    c = np.empty(X.shape[1], np.float32)
    lib().orc_center(X.reshape(-1), X.shape[0], X.shape[1], c)
    return X, c


def normalize(X: np.ndarray) -> np.ndarray:
    X = np.array(X, dtype=np.float32, order="C", copy=True)
    r = lib().orc_normalize(X.reshape(-1), X.shape[0], X.shape[1])
    if r >= 0:
        raise ValueError(f"normalize: zero-norm row {r}")
    return X


class Index:
    """Oracle index over a borrowed dataset X (kept alive here)."""

    def __init__(self, X: np.ndarray, L: int, K: int, D: int, iprobes: int, alpha: float,
                 kappa: int = 20, seed: int = 1, threads: int = 0,
                 t_begin: int = 0, t_end: int = 0, csr=None, mode: int = 0):
        self.X = np.ascontiguousarray(X, dtype=np.float32)
        self.n, self.d = self.X.shape
        self._L = lib()  # the library this index lives in (use_native() may switch later)
        self.prm = Params(L, K, D, iprobes, kappa, alpha, seed, mode)
        self.L, self.K, self.D = L, K, D
        self.t_begin, self.t_end = t_begin, (t_end or L)
        if csr is not None:  # (offsets [L][NB+1], ids, scores, table_base [L+1])
            off, ids, sc, tb = (np.ascontiguousarray(a) for a in csr)
            self.h = self._L.orc_index_from_csr(self.X.reshape(-1), self.n, self.d,
                                              C.byref(self.prm), off.reshape(-1), ids, sc, tb)
        else:
            self.h = self._L.orc_build(self.X.reshape(-1), self.n, self.d, C.byref(self.prm),
                                     threads, t_begin, t_end)
        if not self.h:
            raise ValueError("oracle build: invalid configuration")
        self.NB = self._L.orc_num_buckets(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self._L.orc_free(self.h)
            self.h = None

    def table(self, t: int):
        tot = self._L.orc_table_size(self.h, t)
        off = np.empty(self.NB + 1, np.uint32)
        ids = np.empty(max(tot, 1), np.uint32)
        sc = np.empty(max(tot, 1), np.float32)
        self._L.orc_table(self.h, t, off, ids, sc)
        return off, ids[:tot], sc[:tot]

    def index_probes_mt(self, X: np.ndarray, t: int, threads: int = 0):
        """index_probes over rows X with OpenMP (streamed table checks)."""
        X = np.ascontiguousarray(X, dtype=np.float32)
        ip = self.prm.iprobes
        b = np.empty(X.shape[0] * ip, np.uint32)
        s = np.empty(X.shape[0] * ip, np.float32)
        self._L.orc_index_probes_rows_mt(self.h, X.reshape(-1), X.shape[0], t, b, s,
                                       threads or os.cpu_count())
        return b, s

    def index_probes(self, X: np.ndarray, t: int):
        X = np.ascontiguousarray(X, dtype=np.float32)
        ip = self.prm.iprobes
        b = np.empty(X.shape[0] * ip, np.uint32)
        s = np.empty(X.shape[0] * ip, np.float32)
        self._L.orc_index_probes_rows(self.h, X.reshape(-1), X.shape[0], t, b, s)
        return b.reshape(-1, ip), s.reshape(-1, ip)

    def cap(self, qprobes: int) -> int:
        return self._L.orc_query_cap(self.h, qprobes)

    def peff(self, qprobes: int) -> int:
        return self._L.orc_query_probes(self.h, qprobes)

    def query(self, Q: np.ndarray, k: int, qprobes: int, threads: int = 0, rerank: int = 0):
        """search; rerank = SimHash budget B (0 = off, :330-338).
        stats columns: probes, entries, candidates, exact inner products."""
        Q = np.ascontiguousarray(Q, dtype=np.float32)
        nq = Q.shape[0]
        ids = np.empty(nq * k, np.uint32)
        sc = np.empty(nq * k, np.float64)
        st = (Stats * max(nq, 1))()
        r = self._L.orc_query_rerank(self.h, Q.reshape(-1), nq, k, qprobes, rerank, ids, sc,
                                   C.cast(st, C.c_void_p), threads)
        if r != 0:
            raise ValueError("oracle query: invalid arguments")
        stats = np.array([(s.probes, s.entries, s.candidates, s.exact) for s in st[:nq]],
                         dtype=np.uint64)
        return ids.reshape(nq, k), sc.reshape(nq, k), stats.reshape(nq, 4)

    def simhash(self, X: np.ndarray, threads: int = 0) -> np.ndarray:
        X = np.ascontiguousarray(X, dtype=np.float32)
        out = np.empty(X.shape[0], np.uint64)
        self._L.orc_simhash_rows(self.h, X.reshape(-1), X.shape[0], out, threads)
        return out

    def query_debug(self, q: np.ndarray, qprobes: int):
        q = np.ascontiguousarray(q, dtype=np.float32)
        pe = self.peff(qprobes)
        probes = np.empty(pe + self.L, np.uint64)
        cands = np.empty(self.n, np.uint32)
        np_ = C.c_uint64()
        nc = C.c_uint64()
        self._L.orc_query_debug(self.h, q, qprobes, probes, C.byref(np_), cands, C.byref(nc))
        return probes[:np_.value].copy(), cands[:nc.value].copy()

    def query_lists(self, q: np.ndarray, s: int):
        q = np.ascontiguousarray(q, dtype=np.float32)
        vals = np.empty(self.L * self.K * s, np.float32)
        codes = np.empty(self.L * self.K * s, np.uint32)
        self._L.orc_query_lists(self.h, q, s, vals, codes)
        return vals.reshape(self.L, self.K, s), codes.reshape(self.L, self.K, s)


def csr_from_entries(eb: np.ndarray, es: np.ndarray, n: int, iprobes: int, NB: int,
                     alpha: float, kappa: int, id0: int = 0, threads: int = 0):
    """Alg. 1 lines 5-6 for one table from its pre-filter entries (bucket, score) of
    points id0 .. id0+n-1 ([n][iprobes] flat): returns the CSR (offsets, ids, scores)."""
    eb = np.ascontiguousarray(eb, dtype=np.uint32).reshape(-1)
    es = np.ascontiguousarray(es, dtype=np.float32).reshape(-1)
    off = np.empty(NB + 1, np.uint32)
    ids = np.empty(max(1, n * iprobes), np.uint32)
    sc = np.empty(max(1, n * iprobes), np.float32)
    tot = lib().orc_csr_from_entries(eb, es, n, iprobes, NB, alpha, kappa, id0,
                                     threads or os.cpu_count(), off, ids, sc)
    return off, ids[:tot].copy(), sc[:tot].copy()


def keep_count(B: int, alpha: float, iprobes: int, kappa: int) -> int:
    return lib().orc_keep_count(B, alpha, iprobes, kappa)


def probe_set_lists(vals: np.ndarray, codes: np.ndarray, D: int, peff: int) -> np.ndarray:
    """vals/codes [L][K][s] -> probe ids t*NB + bucket (sorted)."""
    vals = np.ascontiguousarray(vals, dtype=np.float32)
    codes = np.ascontiguousarray(codes, dtype=np.uint32)
    L, K, s = vals.shape
    out = np.empty(peff + L, np.uint64)
    n = lib().orc_probe_set_lists(vals.reshape(-1), codes.reshape(-1), L, K, D, s, peff, out)
    return np.sort(out[:n])


def brute_force(X: np.ndarray, Q: np.ndarray, k: int, threads: int = 0):
    X = np.ascontiguousarray(X, dtype=np.float32)
    Q = np.ascontiguousarray(Q, dtype=np.float32)
    nq = Q.shape[0]
    ids = np.empty(nq * k, np.uint32)
    sc = np.empty(nq * k, np.float64)
    lib().orc_brute_force(X.reshape(-1), X.shape[0], X.shape[1], Q.reshape(-1), nq, k, ids,
                          sc, threads or os.cpu_count())
    return ids.reshape(nq, k), sc.reshape(nq, k)
