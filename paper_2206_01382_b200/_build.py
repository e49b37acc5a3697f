"""Compile the CUDA library libfalconnpp_b200.so in-tree (sm_100a only).

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, one object per .cu,
linked into paper_2206_01382_b200/lib/libfalconnpp_b200.so.  Rebuilds only when a
source or header is newer than the library.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libfalconnpp_b200.so")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-ccbin", "/usr/bin/g++", "-Xcompiler",
         "-fPIC,-fopenmp,-O3", "-Xptxas", "-v", "-I" + INCLUDE]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(INCLUDE, "falconnpp.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def build(force: bool = False, verbose: bool = False, variant: str = "",
          extra: tuple = ()) -> str:
    """variant: build lib/var_<variant>.so with the extra nvcc flags instead (tuning
    experiments; loaded with FPP_LIB_PATH)."""
    lib = os.path.join(LIBDIR, f"var_{variant}.so") if variant else LIB
    if not variant and not force and not needs_build():
        return LIB
    objdir = os.path.join(LIBDIR, "obj" + (f"_{variant}" if variant else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        # FPP_NVCC_EXTRA: extra flags for experiments (e.g. -DFPP_CO_CL_THREADS=512)
        cmd = [NVCC] + ARCH + FLAGS + os.environ.get("FPP_NVCC_EXTRA", "").split() + \
            list(extra) + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        log = os.path.join(objdir, os.path.basename(src) + ".ptxas.txt")
        with open(log, "w") as f:
            f.write(r.stderr)
        if verbose:
            print(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = lib + ".tmp"
    cmd = [NVCC] + ARCH + ["-shared", "-ccbin", "/usr/bin/g++", "-o", tmp] + objs + \
        ["-Xcompiler", "-fopenmp", "-lgomp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import sys
    if len(sys.argv) > 1:  # python -m paper_2206_01382_b200._build <variant> -DFLAG=..
        print(build(variant=sys.argv[1], extra=tuple(sys.argv[2:])))
    else:
        print(build(force=True, verbose=False))
