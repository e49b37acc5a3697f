"""paper_2206_01382_b200 -- B200-native Falconn++ hot path (index build + batched query).

Python mirror of the reference's index/query API (SPEC.md:245-253 build,
SPEC.md:321-329 search; north star ``build(X, L, K, D, iProbes, alpha)`` /
``query(Q, k, qProbes)``) over the C ABI in include/falconnpp.h.  All compute
runs in libfalconnpp_b200.so (hand-written sm_100a CUDA); there is no CPU
fallback -- without the library this package fails to import, and without a
GPU every compute call raises ``FppCudaError``.

Errors mirror the reference's ``std::invalid_argument`` (dataset.cpp:10-18,
rotation.cpp:18-20,42-49): configuration / range / dimension errors raise
``ValueError`` subclasses carrying the library's message.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _build

__all__ = ["Index", "normalize", "synth", "merge_topk_device", "device_count", "FppError", "FppInvalidArgument",
           "FppEmptyDataset", "FppDimensionError", "FppOutOfRange", "FppNonFinite",
           "FppZeroNorm", "FppCudaError", "FppOutOfMemory", "FppUnsupported", "FppFormatError",
           "FppIOError", "content_hash", "center", "MODES", "lib",
           "LIB_PATH", "Params", "QueryStats", "Timings"]

# FPP_LIB_PATH: a variant build (python -m paper_2206_01382_b200._build <name> -D...) for
# tuning experiments; the default is the in-tree library
LIB_PATH = os.environ.get("FPP_LIB_PATH") or _build.LIB

FPP_OK = 0
MODES = {"falconnpp": 0, "falconn_baseline": 1}
ABI_VERSION = 6  # include/falconnpp.h FPP_ABI_VERSION this binding was written against
ERRORS = {1: "INVALID_ARGUMENT", 2: "EMPTY_DATASET", 3: "DIMENSION", 4: "OUT_OF_RANGE",
          5: "NON_FINITE", 6: "ZERO_NORM", 7: "CUDA", 8: "OUT_OF_MEMORY", 9: "UNSUPPORTED",
          10: "FORMAT", 11: "IO"}


class FppError(Exception):
    code = -1


class FppInvalidArgument(FppError, ValueError):
    code = 1


class FppEmptyDataset(FppError, ValueError):
    code = 2


class FppDimensionError(FppError, ValueError):
    code = 3


class FppOutOfRange(FppError, ValueError):
    code = 4


class FppNonFinite(FppError, ValueError):
    code = 5


class FppZeroNorm(FppError, ValueError):
    code = 6


class FppCudaError(FppError, RuntimeError):
    code = 7


class FppOutOfMemory(FppError, MemoryError):
    code = 8


class FppUnsupported(FppError, NotImplementedError):
    code = 9


class FppFormatError(FppError, ValueError):
    """Index file: bad magic, truncated, checksum or dataset-hash mismatch."""
    code = 10


class FppIOError(FppError, OSError):
    code = 11


_EXC = {c.code: c for c in (FppInvalidArgument, FppEmptyDataset, FppDimensionError, FppOutOfRange,
                            FppNonFinite, FppZeroNorm, FppCudaError, FppOutOfMemory,
                            FppUnsupported, FppFormatError, FppIOError)}


class Params(C.Structure):
    _fields_ = [("L", C.c_uint32), ("K", C.c_uint32), ("D", C.c_uint32),
                ("iprobes", C.c_uint32), ("kappa", C.c_uint32), ("alpha", C.c_float),
                ("seed", C.c_uint64), ("device", C.c_int32), ("id_offset", C.c_uint32),
                ("scratch_bytes", C.c_uint64), ("centering", C.c_uint32), ("mode", C.c_uint32)]


class QueryStats(C.Structure):
    _fields_ = [("probes", C.c_uint64), ("entries", C.c_uint64), ("candidates", C.c_uint64),
                ("exact", C.c_uint64)]


class Timings(C.Structure):
    _fields_ = [("hash_ms", C.c_double), ("sort_ms", C.c_double), ("qhash_ms", C.c_double),
                ("probe_ms", C.c_double), ("collect_ms", C.c_double), ("score_ms", C.c_double),
                ("launches", C.c_uint64), ("score_rows", C.c_uint64), ("entries", C.c_uint64),
                ("probes", C.c_uint64), ("score_bytes", C.c_uint64),
                ("score_launches", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class IndexInfo(C.Structure):
    _fields_ = [("n", C.c_uint64), ("d", C.c_uint32), ("d_pad", C.c_uint32), ("L", C.c_uint32),
                ("K", C.c_uint32), ("D", C.c_uint32), ("iprobes", C.c_uint32),
                ("kappa", C.c_uint32), ("alpha", C.c_float), ("seed", C.c_uint64),
                ("num_buckets", C.c_uint64), ("kept_total", C.c_uint64),
                ("prefilter_total", C.c_uint64), ("device_bytes", C.c_uint64),
                ("max_bucket", C.c_uint32), ("id_offset", C.c_uint32),
                ("centering", C.c_uint32), ("mode", C.c_uint32), ("device", C.c_int32)]


vp = C.c_void_p
u32, u64, f32, i32 = C.c_uint32, C.c_uint64, C.c_float, C.c_int

# (name, restype, argtypes) -- every symbol declared in include/falconnpp.h
SIGNATURES = [
    ("fpp_abi_version", C.c_int, []),
    ("fpp_last_error", C.c_char_p, []),
    ("fpp_default_params", None, [C.POINTER(Params)]),
    ("fpp_device_count", C.c_int, []),
    ("fpp_build", C.c_int, [vp, u64, u32, C.POINTER(Params), C.POINTER(vp)]),
    ("fpp_build_device", C.c_int, [vp, u64, u32, C.POINTER(Params), C.POINTER(vp)]),
    ("fpp_free", None, [vp]),
    ("fpp_query", C.c_int, [vp, vp, u64, u32, u32, vp, vp, vp]),
    ("fpp_query_device", C.c_int, [vp, vp, u64, u32, u32, vp, vp, vp, vp]),
    ("fpp_query_probe_sets_device", C.c_int, [vp, vp, u64, u32, vp, vp]),
    ("fpp_query_from_probe_sets_device", C.c_int, [vp, vp, u64, vp, u32, u32, vp, vp, vp, vp]),
    ("fpp_query_rerank", C.c_int, [vp, vp, u64, u32, u32, u32, vp, vp, vp]),
    ("fpp_query_rerank_device", C.c_int, [vp, vp, u64, u32, u32, u32, vp, vp, vp, vp]),
    ("fpp_signatures", C.c_int, [vp, vp, u64, vp]),
    ("fpp_index_info_get", C.c_int, [vp, C.POINTER(IndexInfo)]),
    ("fpp_table_size", u64, [vp, u32]),
    ("fpp_table_csr", C.c_int, [vp, u32, vp, vp, vp]),
    ("fpp_project", C.c_int, [vp, vp, u64, u32, u32, vp]),
    ("fpp_index_probes", C.c_int, [vp, vp, u64, u32, vp, vp]),
    ("fpp_query_cap", u32, [vp, u32]),
    ("fpp_query_probes", u64, [vp, u32]),
    ("fpp_query_lists", C.c_int, [vp, vp, u64, u32, vp, vp]),
    ("fpp_query_debug", C.c_int, [vp, vp, u32, vp, C.POINTER(u64), vp, C.POINTER(u64)]),
    ("fpp_timings_get", C.c_int, [vp, C.POINTER(Timings)]),
    ("fpp_timings_reset", C.c_int, [vp]),
    ("fpp_shard_begin", C.c_int, [vp, u64, u32, C.POINTER(Params), C.POINTER(vp)]),
    ("fpp_shard_begin_device", C.c_int, [vp, u64, u32, C.POINTER(Params), C.POINTER(vp)]),
    ("fpp_shard_hist_len", u64, [vp]),
    ("fpp_shard_hist", C.c_int, [vp, vp]),
    ("fpp_shard_slots", C.c_int, [vp, vp, C.POINTER(u64)]),
    ("fpp_shard_prefix", C.c_int, [vp, vp, vp]),
    ("fpp_shard_finish", C.c_int, [vp, vp, vp, u32]),
    ("fpp_brute_force", C.c_int, [vp, vp, u64, u32, vp, vp]),
    ("fpp_brute_force_device", C.c_int, [vp, vp, u64, u32, vp, vp, vp]),
    ("fpp_save", C.c_int, [vp, C.c_char_p]),
    ("fpp_load", C.c_int, [C.c_char_p, vp, u64, u32, i32, C.POINTER(vp)]),
    ("fpp_load_device", C.c_int, [C.c_char_p, vp, u64, u32, i32, C.POINTER(vp)]),
    ("fpp_content_hash", u64, [vp, u64, u32]),
    ("fpp_center", C.c_int, [vp, u64, u32, vp]),
    ("fpp_index_center", C.c_int, [vp, vp]),
    ("fpp_normalize", C.c_int, [vp, u64, u32]),
    ("fpp_synth", C.c_int, [vp, u64, u32, u32, f32, u64, u32, i32]),
    ("fpp_synth_rows", C.c_int, [vp, u64, u64, u32, u32, f32, u64, u32, i32]),
    ("fpp_merge_topk", C.c_int, [vp, vp, u32, u64, u32, vp, vp, i32, vp]),
    ("fpp_multi_build", C.c_int, [vp, u64, u32, C.POINTER(Params), u32, vp, C.POINTER(vp)]),
    ("fpp_multi_query", C.c_int, [vp, vp, u64, u32, u32, vp, vp, vp]),
    ("fpp_multi_shards", u32, [vp]),
    ("fpp_multi_shard", vp, [vp, u32]),
    ("fpp_multi_free", None, [vp]),
]

_lib = None


def lib():
    """Load libfalconnpp_b200.so (building it with nvcc if absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            _build.build()
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.fpp_abi_version() != ABI_VERSION:
            raise ImportError(f"{LIB_PATH}: ABI {L.fpp_abi_version()} != binding ABI {ABI_VERSION}"
                              " (rebuild with paper_2206_01382_b200._build.build(force=True))")
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != FPP_OK:
        msg = lib().fpp_last_error().decode(errors="replace")
        raise _EXC.get(rc, FppError)(f"[{ERRORS.get(rc, rc)}] {msg}")


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def _f32(X) -> np.ndarray:
    X = np.ascontiguousarray(X, dtype=np.float32)
    if X.ndim == 1:
        X = X.reshape(1, -1)
    return X


def device_count() -> int:
    return lib().fpp_device_count()


def normalize(X: np.ndarray) -> np.ndarray:
    """normalize(Dataset) (dataset.cpp:24-38); returns a normalized copy."""
    X = np.array(_f32(X), copy=True)
    _check(lib().fpp_normalize(_ptr(X), X.shape[0], X.shape[1]))
    return X


def synth(n: int, d: int, clusters: int = 0, sigma: float = 0.0, seed: int = 1, stream: int = 0,
          threads: int = 0, row0: int = 0) -> np.ndarray:
    """Pinned synthetic data; rows [row0, row0+n) of the dataset
    (a shard when row0 > 0).  Rows are NOT normalized."""
    X = np.empty((n, d), np.float32)
    _check(lib().fpp_synth_rows(_ptr(X), row0, n, d, clusters, sigma, seed, stream, threads))
    return X


def merge_topk_device(scores, ids, k: int, out_scores=None, out_ids=None, stream=None):
    """k-way merge of all-gathered shard top-k lists on the device (fpp_merge_topk).

    scores float64 / ids int32|uint32 CUDA tensors [lists, nq, k] (each list sorted by
    score desc, id asc; empty slots id 0xFFFFFFFF and -inf) -> [nq, k] merged lists in
    the same order."""
    _require_tensor(scores, "scores", ("torch.float64",), scores.device, ndim=3)
    _require_tensor(ids, "ids", ("torch.int32", "torch.uint32"), scores.device, ndim=3)
    G, nq, kk = scores.shape
    if tuple(ids.shape) != (G, nq, kk) or kk != k:
        raise FppInvalidArgument("merge_topk: scores/ids must both be [lists, nq, k]")
    import torch
    if out_scores is None:
        out_scores = torch.empty((nq, k), dtype=torch.float64, device=scores.device)
    if out_ids is None:
        out_ids = torch.empty((nq, k), dtype=ids.dtype, device=scores.device)
    _require_tensor(out_scores, "out_scores", ("torch.float64",), scores.device, shape=(nq, k))
    _require_tensor(out_ids, "out_ids", ("torch.int32", "torch.uint32"), scores.device,
                    shape=(nq, k))
    _check(lib().fpp_merge_topk(C.c_void_p(scores.data_ptr()), C.c_void_p(ids.data_ptr()), G, nq,
                                k, C.c_void_p(out_scores.data_ptr()),
                                C.c_void_p(out_ids.data_ptr()), scores.device.index or 0,
                                C.c_void_p(stream) if stream else None))
    return out_scores, out_ids


def _require_tensor(t, name, dtypes, device, shape=None, ndim=None):
    """Device-API argument check (the ABI takes raw pointers): a contiguous CUDA tensor
    of one of `dtypes` on `device` with the given shape -- else FppInvalidArgument."""
    if not _is_torch_cuda(t):
        raise FppInvalidArgument(f"{name}: must be a CUDA torch tensor")
    if str(t.dtype) not in dtypes:
        raise FppInvalidArgument(f"{name}: dtype {t.dtype}, expected {' or '.join(dtypes)}")
    if not t.is_contiguous():
        raise FppInvalidArgument(f"{name}: must be contiguous")
    if device is not None and t.device != device:
        raise FppInvalidArgument(f"{name}: on {t.device}, expected {device}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise FppInvalidArgument(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if ndim is not None and t.dim() != ndim:
        raise FppInvalidArgument(f"{name}: must be {ndim}-D")


class Index:
    """A built Falconn++ index resident on one GPU (SPEC.md:237-242 FalconnPPIndex)."""

    def __init__(self, handle, params: Params, n: int, d: int, X_ref=None):
        self._h = handle
        self.params = params
        self.n, self.d = n, d
        self._X_ref = X_ref

    # --------------------------------------------------------------- build
    @classmethod
    def build(cls, X, L: int, K: int, D: int, iProbes: int, alpha: float, kappa: int = 20,
              seed: int = 1, device: int = -1, id_offset: int = 0, scratch_bytes: int = 0,
              centering: bool = False, mode: str = "falconnpp"):
        """Index::build(X, L, K, D, iProbes, alpha) -- SPEC.md:245-253.

        X is host (numpy) n x d fp32, already normalized, or a CUDA torch tensor.
        centering: index center(X) (queries stay raw, scores x'.q).
        mode: "falconnpp" or "falconn_baseline" (alpha = 1, iProbes = 1, probes by
        ascending gap score).
        """
        p = Params(L, K, D, iProbes, kappa, alpha, seed, device, id_offset, scratch_bytes,
                   int(bool(centering)), MODES[mode] if isinstance(mode, str) else int(mode))
        h = C.c_void_p()
        if _is_torch_cuda(X):
            X = X.contiguous()
            if X.dtype.__str__() != "torch.float32":
                raise FppInvalidArgument("build: X must be float32")
            n, d = X.shape
            if device < 0:
                p.device = X.device.index or 0
            _check(lib().fpp_build_device(C.c_void_p(X.data_ptr()), n, d, C.byref(p), C.byref(h)))
        else:
            X = _f32(X)
            n, d = X.shape
            _check(lib().fpp_build(_ptr(X), n, d, C.byref(p), C.byref(h)))
        return cls(h, p, n, d)

    @classmethod
    def shard_begin(cls, X, L: int, K: int, D: int, iProbes: int, alpha: float, kappa: int = 20,
                    seed: int = 1, device: int = -1, id_offset: int = 0):
        """Phase 1 of the global-filter sharded build (see paper_2206_01382_b200.dist)."""
        p = Params(L, K, D, iProbes, kappa, alpha, seed, device, id_offset, 0, 0, 0)
        h = C.c_void_p()
        if _is_torch_cuda(X):
            X = X.contiguous()
            n, d = X.shape
            if device < 0:
                p.device = X.device.index or 0
            _check(lib().fpp_shard_begin_device(C.c_void_p(X.data_ptr()), n, d, C.byref(p),
                                                C.byref(h)))
        else:
            X = _f32(X)
            n, d = X.shape
            _check(lib().fpp_shard_begin(_ptr(X), n, d, C.byref(p), C.byref(h)))
        return cls(h, p, n, d)

    def brute_force(self, Q, k: int):
        """Exact top-k over the index's dataset (recall ground truth):
        inner_product scores bit for bit, ties to the lower id."""
        Q = _f32(Q)
        nq = Q.shape[0]
        if Q.shape[1] != self.d:
            raise FppDimensionError("brute_force_topk: dimension mismatch")
        ids = np.empty((nq, k), np.uint32)
        sc = np.empty((nq, k), np.float64)
        _check(lib().fpp_brute_force(self._h, _ptr(Q), nq, k, _ptr(ids), _ptr(sc)))
        return ids, sc

    def brute_force_device(self, Q, ids, scores, k: int, stream=None):
        """Device-resident exact top-k on torch CUDA tensors (checked like query_device)."""
        dev = self.device_obj()
        _require_tensor(Q, "Q", ("torch.float32",), dev, ndim=2)
        if Q.shape[1] != self.d:
            raise FppDimensionError("brute_force_topk: dimension mismatch")
        _require_tensor(ids, "ids", ("torch.int32", "torch.uint32"), dev, shape=(Q.shape[0], k))
        _require_tensor(scores, "scores", ("torch.float64",), dev, shape=(Q.shape[0], k))
        _check(lib().fpp_brute_force_device(self._h, C.c_void_p(Q.data_ptr()), Q.shape[0], k,
                                            C.c_void_p(ids.data_ptr()),
                                            C.c_void_p(scores.data_ptr()),
                                            C.c_void_p(stream) if stream else None))

    # --------------------------------------------------------- persistence
    def save(self, path) -> None:
        """save(index, path) -- SPEC.md:270-278; FLPP format (include/falconnpp.h)."""
        _check(lib().fpp_save(self._h, os.fsencode(path)))

    @classmethod
    def load(cls, path, X, device: int = -1):
        """load(path) -- the dataset is stored by reference: pass the same X (host
        numpy or CUDA tensor); its content hash must match the file's."""
        h = C.c_void_p()
        if _is_torch_cuda(X):
            X = X.contiguous()
            n, d = X.shape
            dev = (X.device.index or 0) if device < 0 else device
            _check(lib().fpp_load_device(os.fsencode(path), C.c_void_p(X.data_ptr()), n, d, dev,
                                         C.byref(h)))
        else:
            X = _f32(X)
            n, d = X.shape
            _check(lib().fpp_load(os.fsencode(path), _ptr(X), n, d, max(device, 0), C.byref(h)))
        inf = IndexInfo()
        _check(lib().fpp_index_info_get(h, C.byref(inf)))
        p = Params(inf.L, inf.K, inf.D, inf.iprobes, inf.kappa, inf.alpha, inf.seed,
                   max(device, 0), inf.id_offset, 0, inf.centering, inf.mode)
        return cls(h, p, n, d)

    def shard_hist_len(self) -> int:
        return lib().fpp_shard_hist_len(self._h)

    def shard_hist(self, out_dev_ptr: int) -> None:
        _check(lib().fpp_shard_hist(self._h, C.c_void_p(out_dev_ptr)))

    def shard_slots(self, global_hist_ptr: int) -> int:
        v = u64()
        _check(lib().fpp_shard_slots(self._h, C.c_void_p(global_hist_ptr), C.byref(v)))
        return v.value

    def shard_prefix(self, global_hist_ptr: int, prefix_ptr: int) -> None:
        _check(lib().fpp_shard_prefix(self._h, C.c_void_p(global_hist_ptr), C.c_void_p(prefix_ptr)))

    def shard_finish(self, global_hist_ptr: int, all_prefix_ptr: int, world: int) -> None:
        _check(lib().fpp_shard_finish(self._h, C.c_void_p(global_hist_ptr),
                                      C.c_void_p(all_prefix_ptr), world))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None and getattr(self, "_borrowed", None) is None:
            _lib.fpp_free(h)
        self._h = None

    def close(self):
        self.__del__()

    # --------------------------------------------------------------- query
    def query(self, Q, k: int, qProbes: int, return_stats: bool = False, rerank: int = 0,
              out=None):
        """Index::query(Q, k, qProbes) -- SPEC.md:321-329, batch over rows of Q.

        rerank = SimHash budget B (0 = off, else B >= k).
        Returns ids [nq,k] uint32 (0xFFFFFFFF past min(k,U)), scores [nq,k] fp64
        (-inf past min(k,U)) and optionally stats [nq,4] (probes, entries,
        candidates collected, exact inner products).  out = (ids, scores): caller-owned
        C-contiguous result arrays (e.g. page-locked, so the device writes them directly).
        """
        Q = _f32(Q)
        if Q.shape[1] != self.d:
            raise FppDimensionError(f"search: query dim {Q.shape[1]} != index dim {self.d}")
        nq = Q.shape[0]
        if out is not None:
            ids, sc = out
            if (ids.shape != (nq, k) or ids.dtype != np.uint32 or not ids.flags.c_contiguous
                    or sc.shape != (nq, k) or sc.dtype != np.float64
                    or not sc.flags.c_contiguous):
                raise ValueError("query: out must be (uint32 [nq,k], float64 [nq,k]) "
                                 "C-contiguous arrays")
        else:
            ids = np.empty((nq, k), np.uint32)
            sc = np.empty((nq, k), np.float64)
        st = (QueryStats * max(nq, 1))() if return_stats else None
        stp = C.cast(st, C.c_void_p) if st is not None else None
        if rerank:
            _check(lib().fpp_query_rerank(self._h, _ptr(Q), nq, k, qProbes, rerank, _ptr(ids),
                                          _ptr(sc), stp))
        else:
            _check(lib().fpp_query(self._h, _ptr(Q), nq, k, qProbes, _ptr(ids), _ptr(sc), stp))
        if return_stats:
            stats = np.array([(s.probes, s.entries, s.candidates, s.exact) for s in st[:nq]],
                             dtype=np.uint64).reshape(nq, 4)
            return ids, sc, stats
        return ids, sc

    def query_device(self, Q, ids, scores, k: int, qProbes: int, stats=None, stream=None,
                     rerank: int = 0):
        """Device-resident batch query on torch CUDA tensors (no host copies):
        Q float32 [nq, d], ids int32/uint32 [nq, k], scores float64 [nq, k], stats (if
        given) int64 [nq, 4], all contiguous on the index's device (checked: the ABI
        takes raw pointers)."""
        dev = self.device_obj()
        _require_tensor(Q, "Q", ("torch.float32",), dev, ndim=2)
        if Q.shape[1] != self.d:
            raise FppDimensionError(f"search: query dim {Q.shape[1]} != index dim {self.d}")
        nq = Q.shape[0]
        _require_tensor(ids, "ids", ("torch.int32", "torch.uint32"), dev, shape=(nq, k))
        _require_tensor(scores, "scores", ("torch.float64",), dev, shape=(nq, k))
        if stats is not None:
            _require_tensor(stats, "stats", ("torch.int64",), dev, shape=(nq, 4))
        args = (C.c_void_p(ids.data_ptr()), C.c_void_p(scores.data_ptr()),
                C.c_void_p(stats.data_ptr()) if stats is not None else None,
                C.c_void_p(stream) if stream else None)
        if rerank:
            _check(lib().fpp_query_rerank_device(self._h, C.c_void_p(Q.data_ptr()), nq,
                                                 k, qProbes, rerank, *args))
        else:
            _check(lib().fpp_query_device(self._h, C.c_void_p(Q.data_ptr()), nq, k,
                                          qProbes, *args))

    def query_probe_sets_device(self, Q, qProbes: int, probes=None, stream=None):
        """Stage A alone (multi-GPU split): the probe sets of the
        queries Q (float32 [nq, d] on the index device) as global bucket ids, int32
        (uint32 bits) [nq, P_eff] -- resolvable by any shard with the same parameters
        and seed (query_from_probe_sets_device)."""
        import torch
        dev = self.device_obj()
        _require_tensor(Q, "Q", ("torch.float32",), dev, ndim=2)
        if Q.shape[1] != self.d:
            raise FppDimensionError(f"search: query dim {Q.shape[1]} != index dim {self.d}")
        nq, pe = Q.shape[0], self.peff(qProbes)
        if probes is None:
            probes = torch.empty((nq, pe), dtype=torch.int32, device=dev)
        _require_tensor(probes, "probes", ("torch.int32", "torch.uint32"), dev, shape=(nq, pe))
        _check(lib().fpp_query_probe_sets_device(self._h, C.c_void_p(Q.data_ptr()), nq, qProbes,
                                                 C.c_void_p(probes.data_ptr()),
                                                 C.c_void_p(stream) if stream else None))
        return probes

    def query_from_probe_sets_device(self, Q, probes, ids, scores, k: int, qProbes: int,
                                     stats=None, stream=None):
        """Stage B from probe sets (query_probe_sets_device of any shard) resolved in
        this index's tables; the same answers as query_device on Q."""
        dev = self.device_obj()
        _require_tensor(Q, "Q", ("torch.float32",), dev, ndim=2)
        if Q.shape[1] != self.d:
            raise FppDimensionError(f"search: query dim {Q.shape[1]} != index dim {self.d}")
        nq = Q.shape[0]
        _require_tensor(probes, "probes", ("torch.int32", "torch.uint32"), dev,
                        shape=(nq, self.peff(qProbes)))
        _require_tensor(ids, "ids", ("torch.int32", "torch.uint32"), dev, shape=(nq, k))
        _require_tensor(scores, "scores", ("torch.float64",), dev, shape=(nq, k))
        if stats is not None:
            _require_tensor(stats, "stats", ("torch.int64",), dev, shape=(nq, 4))
        _check(lib().fpp_query_from_probe_sets_device(
            self._h, C.c_void_p(Q.data_ptr()), nq, C.c_void_p(probes.data_ptr()), k, qProbes,
            C.c_void_p(ids.data_ptr()), C.c_void_p(scores.data_ptr()),
            C.c_void_p(stats.data_ptr()) if stats is not None else None,
            C.c_void_p(stream) if stream else None))

    def device_obj(self):
        import torch
        if getattr(self, "_dev", None) is None:
            self._dev = torch.device("cuda", self.info()["device"])
        return self._dev

    def center_vector(self) -> np.ndarray:
        c = np.empty(self.d, np.float32)
        _check(lib().fpp_index_center(self._h, _ptr(c)))
        return c

    def signatures(self, X) -> np.ndarray:
        """64-bit SimHash signatures of rows X (as stored for the index's points)."""
        X = _f32(X)
        out = np.empty(X.shape[0], np.uint64)
        _check(lib().fpp_signatures(self._h, _ptr(X), X.shape[0], _ptr(out)))
        return out

    # ------------------------------------------------------- introspection
    def info(self) -> dict:
        inf = IndexInfo()
        _check(lib().fpp_index_info_get(self._h, C.byref(inf)))
        return {k: getattr(inf, k) for k, _ in inf._fields_}

    def table(self, t: int):
        NB = self.info()["num_buckets"]
        tot = lib().fpp_table_size(self._h, t)
        off = np.empty(NB + 1, np.uint32)
        ids = np.empty(max(tot, 1), np.uint32)
        sc = np.empty(max(tot, 1), np.float32)
        _check(lib().fpp_table_csr(self._h, t, _ptr(off), _ptr(ids), _ptr(sc)))
        return off, ids[:tot], sc[:tot]

    def project(self, X, t: int, f: int) -> np.ndarray:
        X = _f32(X)
        out = np.empty((X.shape[0], self.params.D), np.float32)
        _check(lib().fpp_project(self._h, _ptr(X), X.shape[0], t, f, _ptr(out)))
        return out

    def index_probes(self, X, t: int):
        X = _f32(X)
        ip = self.params.iprobes
        b = np.empty((X.shape[0], ip), np.uint32)
        s = np.empty((X.shape[0], ip), np.float32)
        _check(lib().fpp_index_probes(self._h, _ptr(X), X.shape[0], t, _ptr(b), _ptr(s)))
        return b, s

    def cap(self, qProbes: int) -> int:
        return lib().fpp_query_cap(self._h, qProbes)

    def peff(self, qProbes: int) -> int:
        return lib().fpp_query_probes(self._h, qProbes)

    def query_lists(self, Q, qProbes: int):
        Q = _f32(Q)
        s = self.cap(qProbes)
        L, K = self.params.L, self.params.K
        v = np.empty((Q.shape[0], L, K, s), np.float32)
        c = np.empty((Q.shape[0], L, K, s), np.uint32)
        _check(lib().fpp_query_lists(self._h, _ptr(Q), Q.shape[0], qProbes, _ptr(v), _ptr(c)))
        return v, c

    def query_debug(self, q, qProbes: int):
        q = _f32(q)
        pe = self.peff(qProbes)
        probes = np.empty(pe, np.uint64)
        cands = np.empty(self.n, np.uint32)
        npr, nc = u64(), u64()
        _check(lib().fpp_query_debug(self._h, _ptr(q), qProbes, _ptr(probes), C.byref(npr),
                                     _ptr(cands), C.byref(nc)))
        return probes[:npr.value].copy(), cands[:nc.value].copy()

    def timings(self) -> dict:
        t = Timings()
        _check(lib().fpp_timings_get(self._h, C.byref(t)))
        return t.as_dict()

    def reset_timings(self) -> None:
        _check(lib().fpp_timings_reset(self._h))


class MultiIndex:
    """build(X, config) / query(Q, k, qProbes) over num_gpus devices in one process
    (fpp_multi_*, include/falconnpp.h): contiguous id shards built by the global-filter
    protocol, so every answer equals the 1-GPU index's for every num_gpus.
    devices: one CUDA ordinal per shard (default 0..num_gpus-1; ordinals may repeat)."""

    def __init__(self, handle, params: Params, n: int, d: int):
        self._h = handle
        self.params = params
        self.n, self.d = n, d

    @classmethod
    def build(cls, X, L: int, K: int, D: int, iProbes: int, alpha: float, kappa: int = 20,
              seed: int = 1, num_gpus: int = 1, devices=None, mode: str = "falconnpp"):
        p = Params(L, K, D, iProbes, kappa, alpha, seed, -1, 0, 0, 0,
                   MODES[mode] if isinstance(mode, str) else int(mode))
        X = _f32(X)
        n, d = X.shape
        dv = None
        if devices is not None:
            if len(devices) != num_gpus:
                raise FppInvalidArgument("build: len(devices) != num_gpus")
            dv = (C.c_int32 * num_gpus)(*[int(x) for x in devices])
        h = C.c_void_p()
        _check(lib().fpp_multi_build(_ptr(X), n, d, C.byref(p), num_gpus,
                                     C.cast(dv, C.c_void_p) if dv is not None else None,
                                     C.byref(h)))
        return cls(h, p, n, d)

    @property
    def num_shards(self) -> int:
        return lib().fpp_multi_shards(self._h)

    def shard(self, g: int) -> "Index":
        """Shard g as a borrowed Index (introspection; owned by this MultiIndex)."""
        h = lib().fpp_multi_shard(self._h, g)
        if not h:
            raise FppOutOfRange(f"shard {g} of {self.num_shards}")
        ix = Index(None, self.params, 0, self.d)
        ix._h = C.c_void_p(h)
        ix._borrowed = self  # keeps the owner alive; Index.__del__ must not free it
        inf = ix.info()
        ix.n = inf["n"]
        return ix

    def query(self, Q, k: int, qProbes: int, return_stats: bool = False):
        Q = _f32(Q)
        if Q.shape[1] != self.d:
            raise FppDimensionError(f"search: query dim {Q.shape[1]} != index dim {self.d}")
        nq = Q.shape[0]
        ids = np.empty((nq, k), np.uint32)
        sc = np.empty((nq, k), np.float64)
        st = (QueryStats * max(nq, 1))() if return_stats else None
        stp = C.cast(st, C.c_void_p) if st is not None else None
        _check(lib().fpp_multi_query(self._h, _ptr(Q), nq, k, qProbes, _ptr(ids), _ptr(sc), stp))
        if return_stats:
            stats = np.array([(s.probes, s.entries, s.candidates, s.exact) for s in st[:nq]],
                             dtype=np.uint64).reshape(nq, 4)
            return ids, sc, stats
        return ids, sc

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.fpp_multi_free(h)
            self._h = None

    def close(self):
        self.__del__()


def center(X):
    """center(Dataset) (dataset.cpp:40-57): returns (X - mean, mean) in fp32; the mean is
    the reference's sequential double sum per coordinate, rows are not renormalized."""
    X = np.array(X, dtype=np.float32, order="C", copy=True)
    c = np.empty(X.shape[1], np.float32)
    _check(lib().fpp_center(_ptr(X), X.shape[0], X.shape[1], _ptr(c)))
    return X, c


def content_hash(X) -> int:
    """fnv1a64 of the fp32 bytes (common.hpp:50-57): the FLPP dataset reference."""
    X = _f32(X)
    return int(lib().fpp_content_hash(_ptr(X), X.shape[0], X.shape[1]))


def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)
