#!/usr/bin/env python
"""bench.py -- Falconn++ hot path on B200: batched query throughput (+ build points/s).

Default (N=1): BASELINE.json configs[3] ("c4", the config the metric is quoted on at
1/2/4/8 B200): n=10M d=128 10,000-cluster mixture (sigma 0.25) normalized, L=50 K=2
D=128 iProbes=3 alpha=0.01 kappa=20, 100,000 queries, qProbes=5,000, k=20.  A step
= one batched query of all nq queries through the hot path (hash -> probe select ->
bucket walk/dedup -> row gather + fp64 dot + top-k).  The same run adds a C5 build
block (configs[4]: n=50M d=256 L=64 iProbes=5 alpha=0.005, points/s and the FP32-add
roofline) unless --no-c5.

  python bench.py [--gpus N --steps K --warmup W --config c4 --qprobes 5000]
  python bench.py --impl reference ...   # the CPU oracle port on the host cores

Parity is checked in every N=1 run (outside the timed region): the oracle rebuilds
tables {0, L/2, L-1} from the same X and compares their CSR bytes with the GPU's,
then answers a query sample (ids, scores, stats) over the GPU CSR; C5 streams X back
and rebuilds table 0.  The line carries "parity" and the exit code is 1 on any
mismatch.

Multi-GPU: `--gpus N` without WORLD_SIZE re-launches itself under torchrun (one
rank per GPU, NCCL; FPP_DIST_BACKEND=gloo or fewer visible GPUs than ranks: gloo,
ranks sharing GPUs round-robin -- a correctness mode, not a scaling number).  Rank
g indexes ids [g*n/G,(g+1)*n/G) with the global filter (all-reduce of bucket
histograms + all-gather of bucket prefixes: the shards hold exactly the 1-GPU
index), queries are replicated, per-rank top-k lists are all-gathered and merged
by the library's merge kernel; value = nq*K / (max over ranks of the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: n, d, clusters, sigma, L, K, D, iprobes, alpha, nq, qprobes(headline), sweep
    "c1": dict(n=100_000, d=128, clusters=0, sigma=0.0, L=50, K=2, D=128, iprobes=3, alpha=0.1,
               nq=1000, qprobes=1000, sweep=[50, 200, 1000]),
    "c2": dict(n=1_200_000, d=300, clusters=1000, sigma=0.3, L=100, K=2, D=512, iprobes=3,
               alpha=0.05, nq=10_000, qprobes=10_000, sweep=[1000, 2000, 5000, 10_000, 20_000],
               rerank=[200, 1000, 4000]),
    "c3": dict(n=1_000_000, d=960, clusters=500, sigma=0.2, L=100, K=2, D=1024, iprobes=3,
               alpha=0.02, nq=1000, qprobes=10_000, sweep=[10_000]),
    "c4": dict(n=10_000_000, d=128, clusters=10_000, sigma=0.25, L=50, K=2, D=128, iprobes=3,
               alpha=0.01, nq=100_000, qprobes=5000, sweep=[1000, 5000]),
    # index-build throughput config (BASELINE.json configs[4]); build-only
    "c5": dict(n=50_000_000, d=256, clusters=0, sigma=0.0, L=64, K=2, D=256, iprobes=5,
               alpha=0.005, nq=0, qprobes=0, sweep=[]),
}
K_TOP = 20
KAPPA = 20
SEED = 1
SM_COUNT, FP32_LANES = 148, 128  # B200: FP32 adds per SM per clock (scalar FADD)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_info():
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count()}


def config_dict(name, cfg, qprobes, world):
    """The workload description shared by both arms (same keys, same values)."""
    d = {"workload": name, "n": cfg["n"], "d": cfg["d"], "clusters": cfg["clusters"],
         "sigma": cfg["sigma"], "L": cfg["L"], "K": cfg["K"], "D": cfg["D"],
         "iProbes": cfg["iprobes"], "alpha": cfg["alpha"], "kappa": KAPPA, "k": K_TOP,
         "seed": SEED, "parallelism": f"shard{world}" if world > 1 else "single"}
    if cfg["nq"]:
        xb = cfg["n"] * cfg["d"] * 4
        d.update(qProbes=qprobes, nq=cfg["nq"],
                 l2=("inputs larger than L2 (X %.2f GB gathered at random); no flush" % (xb / 1e9))
                 if xb > 126e6 else
                 ("X (%.0f MB) fits the 126 MB L2: a correctness config, not flushed" % (xb / 1e6)))
    return d


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_data(cfg, lo, hi, gen):
    """Rows [lo,hi) of the pinned synthetic dataset + all queries, normalized once."""
    X = gen.normalize(gen.synth(hi - lo, cfg["d"], cfg["clusters"], cfg["sigma"], seed=SEED,
                                stream=0, row0=lo))
    Q = gen.normalize(gen.synth(cfg["nq"], cfg["d"], cfg["clusters"], cfg["sigma"], seed=SEED,
                                stream=1)) if cfg["nq"] else None
    return np.ascontiguousarray(X), Q


def oracle_lib(native: bool = True):
    """The oracle (test infrastructure: parity checker + CPU arm).  On the GPU box it is
    rebuilt once with -march=native (the reference's flag, proj/CMakeLists.txt:20-22)
    when gcc is there; the prebuilt x86-64-v3 library otherwise."""
    from oracle import oracle as orc
    if native and not os.environ.get("FPP_ORACLE_PREBUILT"):
        orc.use_native()
    else:
        orc.lib()
    return orc


# --------------------------------------------------------------------- traffic
def dram_traffic(config, qprobes):
    """ncu DRAM bytes per launch of the dominant kernel for this exact command
    (profiles/dram_traffic.json, written by profiles/traffic.py from an ncu --set full
    capture), or None."""
    p = os.path.join(ROOT, "profiles", "dram_traffic.json")
    try:
        with open(p) as f:
            j = json.load(f)
        e = j.get(config)
        if e and e.get("qprobes") == qprobes:
            return e
    except Exception:
        pass
    return None


# ---------------------------------------------------------------------- parity
def parity_tables(cfg, X, ix, orc, threads, tables):
    """Oracle rebuild of `tables` from the same X; CSR bytes compared with the GPU's."""
    res = {"tables": [], "csr_equal": True, "entries_checked": 0}
    for t in tables:
        t0 = time.perf_counter()
        ob = orc.Index(X, L=cfg["L"], K=cfg["K"], D=cfg["D"], iprobes=cfg["iprobes"],
                       alpha=cfg["alpha"], kappa=KAPPA, seed=SEED, threads=threads,
                       t_begin=t, t_end=t + 1)
        oo, oi, os_ = ob.table(t)
        del ob
        go, gi, gs = ix.table(t)
        eq = (np.array_equal(go, oo) and np.array_equal(gi, oi)
              and np.array_equal(gs.view(np.uint32), os_.view(np.uint32)))
        res["tables"].append(int(t))
        res["entries_checked"] += int(len(oi))
        res["csr_equal"] = bool(res["csr_equal"] and eq)
        log(f"[parity] table {t}: {len(oi)} kept entries, equal={eq} "
            f"({time.perf_counter() - t0:.1f}s)")
    return res


def import_gpu_csr(cfg, X, ix, orc):
    """The GPU CSR (tables sampled above verified bit-exact) wrapped for the CPU oracle."""
    offs, ids, scs, tb = [], [], [], [0]
    for t in range(cfg["L"]):
        o, i, s = ix.table(t)
        offs.append(o)
        ids.append(i)
        scs.append(s)
        tb.append(tb[-1] + len(i))
    csr = (np.stack(offs), np.concatenate(ids), np.concatenate(scs), np.array(tb, np.uint64))
    return orc.Index(X, L=cfg["L"], K=cfg["K"], D=cfg["D"], iprobes=cfg["iprobes"],
                     alpha=cfg["alpha"], kappa=KAPPA, seed=SEED, csr=csr)


def parity_queries(ox, Q, sample, gids, gsc, gst, qprobes, threads):
    """Oracle answers for the query sample vs the GPU's (ids, scores, stats)."""
    oi, os_, ost = ox.query(Q[sample], K_TOP, qprobes, threads=threads)
    ok = np.isfinite(os_)
    rel = 0.0
    if ok.any():
        rel = float(np.max(np.abs(gsc[sample][ok] - os_[ok]) / np.maximum(np.abs(os_[ok]), 1e-300)))
    return {"queries": int(len(sample)), "ids_equal": bool(np.array_equal(gids[sample], oi)),
            "scores_max_rel_err": rel, "scores_bit_equal": bool(np.array_equal(gsc[sample], os_)),
            "stats_equal": bool(gst is None or np.array_equal(gst[sample], ost)),
            "tolerance": "ids identical, scores within 1e-5 relative (north star)"}


def parity_ok(p):
    if not p:
        return True
    ok = True
    if "csr_equal" in p:
        ok &= p["csr_equal"]
    q = p.get("query_sample")
    if q:
        ok &= q["ids_equal"] and q["stats_equal"] and q["scores_max_rel_err"] <= 1e-5
    if "e2e_equals_device" in p:
        ok &= p["e2e_equals_device"]
    if "merged_equals_single" in p:
        ok &= p["merged_equals_single"]
    return bool(ok)


# ---------------------------------------------------------------- reference arm
def run_reference(args, cfg, qprobes):
    """--impl reference: the CPU oracle port (the reference ships no hashing/index/query
    code) on the host cores, same config/metric/unit."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    orc = oracle_lib()
    threads = os.cpu_count() or 1
    n = cfg["n"]
    t0 = time.perf_counter()
    X, Q = make_data(cfg, 0, n, orc)
    log(f"[reference] data {time.perf_counter() - t0:.1f}s; oracle build of {cfg['L']} tables "
        f"on {threads} threads ...")
    t0 = time.perf_counter()
    ox = orc.Index(X, L=cfg["L"], K=cfg["K"], D=cfg["D"], iprobes=cfg["iprobes"],
                   alpha=cfg["alpha"], kappa=KAPPA, seed=SEED, threads=threads)
    tbuild = time.perf_counter() - t0
    log(f"[reference] build {tbuild:.1f}s")
    m = min(len(Q), threads)
    t0 = time.perf_counter()
    ox.query(Q[:m], K_TOP, qprobes, threads=threads)
    dt = max(time.perf_counter() - t0, 1e-6)
    ns = int(min(len(Q), max(m, m * args.ref_step_s / dt)))  # ~ref_step_s of CPU per step
    for w in range(args.warmup):
        ox.query(Q[:m], K_TOP, qprobes, threads=threads)
    times = []
    for s in range(args.steps):
        a = (s * ns) % max(1, len(Q) - ns + 1)
        t0 = time.perf_counter()
        ox.query(Q[a:a + ns], K_TOP, qprobes, threads=threads)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    qps = ns * args.steps / tot
    line = {
        "metric": "queries/s (k=20)", "value": qps, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "none (1 process)",
        "vs_baseline": None, "dtype": "f32 (FHT, pair scores) / f64 (inner products)",
        "data": "synthetic (pinned seeded generator, DESIGN.md section 6)", "impl": "reference",
        "config": config_dict(args.config, cfg, qprobes, 1),
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "port",
                         "cpu": cpu_info(),
                         "sample": f"{ns} of {cfg['nq']} queries per step (a sliding window), "
                                   f"full {cfg['L']}-table oracle index built on the CPU "
                                   f"in {tbuild:.0f}s; oracle -march="
                                   f"{'native' if orc.NATIVE else 'x86-64-v3'}"},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "build": {"points_per_s": n / tbuild, "wall_s": tbuild,
                  "note": "full oracle index build (all tables), all host threads"},
    }
    print(json.dumps(line), flush=True)
    return 0


def build_cpu_sample(cfg, npts, threads, orc):
    """Oracle build of one table over a same-distribution sample, as points/s for all L."""
    Xs = orc.normalize(orc.synth(npts, cfg["d"], cfg["clusters"], cfg["sigma"], seed=SEED))
    t0 = time.perf_counter()
    ob = orc.Index(Xs, L=cfg["L"], K=cfg["K"], D=cfg["D"], iprobes=cfg["iprobes"],
                   alpha=cfg["alpha"], kappa=KAPPA, seed=SEED, threads=threads, t_begin=0, t_end=1)
    dt = time.perf_counter() - t0
    del ob
    return npts / (dt * cfg["L"])


def run_reference_build(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    orc = oracle_lib()
    threads = os.cpu_count() or 1
    npts = 1_000_000
    vals = [build_cpu_sample(cfg, npts, threads, orc) for _ in range(max(1, args.steps))]
    v = float(np.median(vals))
    print(json.dumps({
        "metric": "index-build points/s", "value": v, "unit": "points/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "impl": "reference",
        "data": "synthetic i.i.d. N(0,1) normalized", "config": config_dict(args.config, cfg, 0, 1),
        "cpu_baseline": {"value": v, "unit": "points/s", "cores": threads, "kind": "port",
                         "cpu": cpu_info(),
                         "sample": f"{npts} points x 1 of {cfg['L']} tables per step, "
                                   f"extrapolated linearly in L (tables are independent)"},
        "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)
    return 0


# ------------------------------------------------------------------ dist setup
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(args):
    """--gpus N without a launcher: re-run this script under torchrun, one rank per GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the driver counts ranks from NCCL's log
    log("[bench] launching:", " ".join(cmd))
    return subprocess.call(cmd, env=env)


class Dist:
    def __init__(self):
        import torch
        import torch.distributed as dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        ndev = max(1, torch.cuda.device_count())
        self.dev = self.local % ndev
        torch.cuda.set_device(self.dev)
        self.backend = None
        if self.world > 1:
            be = os.environ.get("FPP_DIST_BACKEND", "nccl")
            if be == "nccl" and self.world > ndev:
                log(f"[bench] {self.world} ranks on {ndev} GPU(s): gloo (ranks share GPUs; "
                    f"correctness mode, not a scaling measurement)")
                be = "gloo"
            self.backend = be
            if be == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.dev))
            else:
                dist.init_process_group("gloo")
        self.dist = dist
        self.torch = torch

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, vals):
        t = self.torch.tensor(vals, dtype=self.torch.float64)
        if self.world > 1:
            if self.backend == "nccl":
                t = t.cuda()
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return [float(x) for x in t.cpu().tolist()]

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# ----------------------------------------------------------------- build block
def build_block(cfg, name, steps, warmup, dd, check_tables, threads):
    """Build throughput (K1 + K2) on device-generated data, FP32-add and HBM fractions,
    and the streamed oracle check of `check_tables` (X copied back chunk by chunk)."""
    import torch

    import paper_2206_01382_b200 as fpp
    from paper_2206_01382_b200 import dist as fdist
    world, rank, local = dd.world, dd.rank, dd.dev
    n, d = cfg["n"], cfg["d"]
    lo, hi = fdist.shard_range(n, world, rank)
    # i.i.d. N(0,1) rows generated on the device (torch Philox, seed 1 + shard offset),
    # normalized on the device (double norm): same distribution as the host generator;
    # the parity check copies the very bytes back to the host
    gen = torch.Generator(device="cuda")
    gen.manual_seed(SEED * 1_000_003 + lo)
    X = torch.empty((hi - lo, d), dtype=torch.float32, device="cuda")
    for a in range(0, hi - lo, 1 << 22):
        b = min(hi - lo, a + (1 << 22))
        blk = torch.randn((b - a, d), generator=gen, device="cuda", dtype=torch.float32)
        X[a:b] = blk / blk.double().norm(dim=1, keepdim=True).float()
    torch.cuda.synchronize()
    prm = dict(L=cfg["L"], K=cfg["K"], D=cfg["D"], iProbes=cfg["iprobes"], alpha=cfg["alpha"],
               kappa=KAPPA, seed=SEED, device=local)

    def one_build():
        if world > 1:  # global filter over the process group
            return fdist.build_global_filter(fdist.GpuShardEngine(X, lo, **prm))
        return fpp.Index.build(X, id_offset=lo, **prm)

    for _ in range(warmup):
        ix = one_build()
        info = ix.info()
        del ix
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dd.barrier()
    torch.cuda.synchronize()
    dev_ms = []
    ix = None
    with ClockSampler(local) as clk:
        ev0.record()
        for s in range(steps):
            if ix is not None:
                del ix
            ix = one_build()
            t = ix.timings()
            dev_ms.append((t["hash_ms"], t["sort_ms"]))
        ev1.record()
        torch.cuda.synchronize()
    dd.barrier()
    t_ms = dd.max([ev0.elapsed_time(ev1)])[0]
    info = ix.info()
    pps = n * steps / (t_ms / 1e3)
    hash_ms = float(np.mean([a for a, _ in dev_ms]))
    sort_ms = float(np.mean([b for _, b in dev_ms]))
    clocks = clk.summary()
    mhz = clocks["sm_mhz"] or 1965.0
    adds = (hi - lo) * cfg["L"] * cfg["K"] * 3 * cfg["D"] * int(np.log2(cfg["D"]))
    fp32_peak = SM_COUNT * FP32_LANES * mhz * 1e6
    # shared-memory crossbar (128 B/clk/SM): the five layout transposes of a projection
    # write and read the padded vector once each
    P = 1 << max(int(d - 1).bit_length(), 0)
    smem_tr_bytes = (hi - lo) * cfg["L"] * cfg["K"] * 5 * 2 * P * 4
    smem_peak = SM_COUNT * 128 * mhz * 1e6
    bytes_build = (4 * (hi - lo) * d + 24 * (hi - lo) * cfg["L"] * cfg["iprobes"]
                   + 8 * info["kept_total"] + 4 * cfg["L"] * (info["num_buckets"] + 1))
    hbm, peak_kind = peaks()
    step_s = t_ms / steps / 1e3
    out = {
        "workload": name, "points_per_s": pps, "ms_per_build": t_ms / steps, "steps": steps,
        "warmup": warmup, "n": n, "n_gpus": world,
        "data": "synthetic i.i.d. N(0,1) rows normalized, generated on the device (torch Philox)",
        "roofline": {
            "kernel": "k_hash_build", "bound": "fp32 (FHT butterflies)",
            "fht_adds_per_build": adds, "fht_adds_per_s": adds / (hash_ms / 1e3),
            "fp32_add_peak_per_s": fp32_peak,
            "fp32_peak_basis": f"{SM_COUNT} SMs x {FP32_LANES} FADD/clk x {mhz:.0f} MHz "
                               f"(median SM clock under load)",
            "fp32_frac_hash_kernel": adds / (hash_ms / 1e3) / fp32_peak,
            "fp32_frac_build": adds / step_s / fp32_peak,
            "smem_transpose_bytes_per_build": smem_tr_bytes,
            "smem_peak_bytes_per_s": smem_peak,
            "smem_frac_hash_kernel_transposes": smem_tr_bytes / (hash_ms / 1e3) / smem_peak,
            "smem_note": "k_hash_build is bound by shared-memory wavefronts, not FP32 issue: ncu "
                         "l1tex__data_pipe_lsu_wavefronts 83.6% of peak (transposes ~60% of them, the "
                         "top-r selection and spills the rest), issue-active 73%, FMA pipe 42% "
                         "(profiles/r02_c5_hash_build.json)",
            "hbm_algorithmic_bytes": bytes_build, "hbm_achieved_gbs": bytes_build / step_s / 1e9,
            "hbm_peak": hbm, "peak_kind": peak_kind, "hbm_frac": bytes_build / step_s / 1e9 / hbm,
            "hash_ms": hash_ms, "sort_ms": sort_ms},
        "kept_total": info["kept_total"], "prefilter_total": info["prefilter_total"],
        "clocks": clocks,
    }
    if check_tables and world == 1 and rank == 0:
        out["parity"] = build_parity_streamed(cfg, X, ix, check_tables, threads)
    del ix, X
    torch.cuda.empty_cache()
    return out


def build_parity_streamed(cfg, Xd, ix, tables, threads):
    """Oracle CSR of `tables` from the GPU's own X bytes, streamed to the host in chunks
    (the C5 dataset is 51 GB): per chunk the oracle's index probes, then the oracle's
    bucket sort + alpha/kappa filter (orc_csr_from_entries), compared with the GPU CSR."""
    orc = oracle_lib(native=False)
    n, ip = Xd.shape[0], cfg["iprobes"]
    t0 = time.perf_counter()
    ox = orc.Index(np.zeros((1, cfg["d"]), np.float32), L=cfg["L"], K=cfg["K"], D=cfg["D"],
                   iprobes=ip, alpha=cfg["alpha"], kappa=KAPPA, seed=SEED, threads=1,
                   t_begin=0, t_end=1)  # signs only (a 1-point shell)
    eb = {t: np.empty(n * ip, np.uint32) for t in tables}
    es = {t: np.empty(n * ip, np.float32) for t in tables}
    step = 1 << 21
    for a in range(0, n, step):
        b = min(n, a + step)
        xh = Xd[a:b].cpu().numpy()
        for t in tables:
            bb, ss = ox.index_probes_mt(xh, t, threads)
            eb[t][a * ip:b * ip] = bb
            es[t][a * ip:b * ip] = ss
    res = {"tables": list(tables), "csr_equal": True, "entries_checked": 0,
           "method": "oracle index probes over the GPU's X bytes (streamed D2H) + oracle "
                     "bucket sort and alpha/kappa filter"}
    NB = int(ox.NB)
    for t in tables:
        oo, oi, os_ = orc.csr_from_entries(eb[t], es[t], n, ip, NB, cfg["alpha"], KAPPA,
                                           threads=threads)
        go, gi, gs = ix.table(t)
        eq = (np.array_equal(go, oo) and np.array_equal(gi, oi)
              and np.array_equal(gs.view(np.uint32), os_.view(np.uint32)))
        res["csr_equal"] = bool(res["csr_equal"] and eq)
        res["entries_checked"] += int(len(oi))
        log(f"[parity c5] table {t}: {len(oi)} kept entries, equal={eq}")
    res["seconds"] = time.perf_counter() - t0
    return res


def run_build(args, cfg):
    """Build-only throughput (config c5): points/s of the full index build (K1 + K2)."""
    dd = Dist()
    threads = os.cpu_count() or 1
    L = cfg["L"]
    blk = build_block(cfg, args.config, args.steps, args.warmup, dd,
                      [0, L - 1] if not args.no_parity else [], threads)
    cpu = None
    if dd.world == 1 and dd.rank == 0 and not args.no_cpu_baseline:
        orc = oracle_lib()
        cpu = {"value": build_cpu_sample(cfg, 1_000_000, threads, orc), "unit": "points/s",
               "cores": threads, "kind": "port", "cpu": cpu_info(),
               "sample": f"oracle build of 1 of {L} tables over 1M points of the same "
                         f"distribution, extrapolated linearly in L"}
    rc = 0
    if dd.rank == 0:
        par = blk.pop("parity", None)
        rc = 0 if parity_ok(par) else 1
        print(json.dumps({
            "metric": "index-build points/s", "value": blk["points_per_s"], "unit": "points/s",
            "n_gpus": dd.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": blk["ms_per_build"], "higher_is_better": True,
            "scaling": "strong" if dd.world > 1 else "none (1 GPU)", "vs_baseline": None,
            "dtype": "f32", "data": blk["data"],
            "config": config_dict(args.config, cfg, 0, dd.world),
            "roofline": blk["roofline"], "build": {"kept_total": blk["kept_total"],
                                                   "prefilter_total": blk["prefilter_total"]},
            "e2e": {"value": blk["points_per_s"], "unit": "points/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0,
                    "note": "inputs device-resident (device-generated); build via fpp_build_device"},
            "gpu_launches": None, "cpu_baseline": cpu, "clocks": blk["clocks"], "parity": par,
        }), flush=True)
    dd.close()
    return rc


# ----------------------------------------------------------------- query bench
def run_query_bench(args, cfg, qprobes):
    dd = Dist()
    torch = dd.torch
    import paper_2206_01382_b200 as fpp
    from paper_2206_01382_b200 import dist as fdist

    world, rank, local = dd.world, dd.rank, dd.dev
    threads = os.cpu_count() or 1
    n, d, nq = cfg["n"], cfg["d"], cfg["nq"]
    lo, hi = fdist.shard_range(n, world, rank)
    t0 = time.perf_counter()
    X, Q = make_data(cfg, lo, hi, fpp)
    log(f"[rank {rank}] data {time.perf_counter() - t0:.1f}s shard [{lo},{hi})")

    # ---------------------------------------------------------------- build
    Xd = torch.from_numpy(X).cuda()
    dd.barrier()
    torch.cuda.synchronize()
    tb0 = time.perf_counter()
    prm = dict(L=cfg["L"], K=cfg["K"], D=cfg["D"], iProbes=cfg["iprobes"], alpha=cfg["alpha"],
               kappa=KAPPA, seed=SEED, device=local)
    if world > 1:  # global filter: the shards together hold exactly the 1-GPU index
        ix = fdist.build_global_filter(fdist.GpuShardEngine(Xd, lo, **prm))
    else:
        ix = fpp.Index.build(Xd, id_offset=lo, **prm)
    torch.cuda.synchronize()
    tbuild = time.perf_counter() - tb0
    tim = ix.timings()
    build_dev_ms = tim["hash_ms"] + tim["sort_ms"]
    tbuild_max, tbuild_dev_max = dd.max([tbuild, build_dev_ms / 1e3])
    info = ix.info()
    log(f"[rank {rank}] build {tbuild:.3f}s (device {build_dev_ms:.1f} ms: hash "
        f"{tim['hash_ms']:.1f} sort {tim['sort_ms']:.1f}) kept {info['kept_total']}")
    del Xd

    # ---------------------------------------------------------------- query
    Qd = torch.from_numpy(Q).cuda()
    ids_d = torch.empty((nq, K_TOP), dtype=torch.int32, device="cuda")
    sc_d = torch.empty((nq, K_TOP), dtype=torch.float64, device="cuda")
    st_d = torch.empty((nq, 4), dtype=torch.int64, device="cuda")
    # the queries and every timing event run on one explicit stream: the legacy
    # default stream (handle 0) would mean "library stream" to the C ABI, and
    # events on the legacy stream do not order with the library's non-blocking streams
    torch.cuda.synchronize()
    qstream = torch.cuda.Stream()
    torch.cuda.set_stream(qstream)
    stream = qstream.cuda_stream
    merged = {}

    def step(qp, stats=None):
        if world > 1 and not args.replicate_stage_a:
            # stage A split across the ranks, probe sets all-gathered
            merged["s"], merged["i"] = fdist.sharded_query(ix, Qd, ids_d, sc_d, K_TOP, qp,
                                                           stream=stream, stats=stats)
            return
        ix.query_device(Qd, ids_d, sc_d, K_TOP, qp, stats=stats, stream=stream)
        if world > 1:
            merged["s"], merged["i"] = fdist.allgather_merge(sc_d, ids_d, K_TOP)

    step(qprobes, st_d)
    torch.cuda.synchronize()
    st_local = st_d.cpu().numpy().astype(np.uint64)
    P_sum, E_sum, U_sum, _ = (int(x) for x in st_local.sum(axis=0))
    for _ in range(args.warmup - 1):
        step(qprobes)
    ix.reset_timings()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dd.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record()
        for _ in range(args.steps):
            step(qprobes)
        ev1.record()
        torch.cuda.synchronize()
    dd.barrier()
    t_ms = dd.max([ev0.elapsed_time(ev1)])[0]
    tim = ix.timings()
    qps = nq * args.steps / (t_ms / 1e3)
    if world > 1:
        g_ids = merged["i"].cpu().numpy().astype(np.int64).astype(np.uint32)
        g_sc = merged["s"].cpu().numpy()
    else:
        g_ids = ids_d.cpu().numpy().view(np.uint32).copy()
        g_sc = sc_d.cpu().numpy().copy()

    # roofline of the dominant kernel (the score gather).  frac: ncu DRAM bytes per
    # launch of this exact command (profiles/dram_traffic.json) / the launch's duration
    # measured here with CUDA events / the measured HBM peak (north star: "from ncu
    # DRAM GB/s counters").  requested_frac: the row bytes the kernel asked the memory
    # system for (fpp_timings.score_bytes, L2 hits included) over the same time.
    # algorithmic_*: SURVEY 8(d)'s full-row bytes 4*d*U (+ lists, query, output); with
    # exact early termination the kernel reads only row prefixes of most candidates.
    hbm, peak_kind = peaks()
    row_bytes_step = tim["score_bytes"] / args.steps if tim.get("score_bytes") else 4 * d * U_sum
    score_bytes_step = row_bytes_step + 4 * U_sum + 4 * d * nq + 12 * K_TOP * nq
    score_bytes_full = 4 * d * U_sum + 4 * U_sum + 4 * d * nq + 12 * K_TOP * nq
    path_bytes_full = 8 * P_sum + 4 * E_sum + 4 * d * U_sum + 4 * d * nq + 12 * K_TOP * nq
    score_ms = tim["score_ms"] / args.steps
    score_launches = max(1.0, tim["score_launches"] / args.steps)
    launch_s = score_ms / score_launches / 1e3
    tr = dram_traffic(args.config, qprobes) if world == 1 else None
    pruned = row_bytes_step < 4 * d * U_sum
    kname = ("k_score_screen" if 64 <= d <= 256 and d % 4 == 0 else "k_score_pruned") \
        if pruned else "k_score"
    roof = {"kernel": tr["kernel"].split("(")[0].replace("void ", "") if tr else kname,
            "bound": "hbm", "unit": "GB/s",
            "peak": hbm, "peak_kind": peak_kind,
            "kernel_ms_per_launch": launch_s * 1e3, "launches_per_step": score_launches,
            "kernel_ms_per_step": score_ms, "share_of_step": score_ms / (t_ms / args.steps),
            "requested_bytes_per_launch": score_bytes_step / score_launches,
            "requested_gbs": score_bytes_step / score_launches / launch_s / 1e9,
            "requested_frac": score_bytes_step / score_launches / launch_s / 1e9 / hbm,
            "row_bytes_read_fraction": row_bytes_step / max(1, 4 * d * U_sum),
            "algorithmic_bytes_per_launch": score_bytes_full / score_launches,
            "algorithmic_gbs": score_bytes_full / score_launches / launch_s / 1e9}
    if tr:
        # the captured launch's DRAM bytes per query, times this run's queries per launch
        # (chunks differ in size), over this run's CUDA-event launch time
        per_q = tr["dram_bytes_per_launch"] / tr.get("queries_per_launch", 8192)
        bytes_launch = per_q * nq / score_launches
        roof.update(achieved=bytes_launch / launch_s / 1e9,
                    traffic=bytes_launch, traffic_per_query=per_q,
                    frac=bytes_launch / launch_s / 1e9 / hbm,
                    frac_basis="ncu dram__bytes_read.sum + dram__bytes_write.sum per query of the "
                               f"captured launch ({tr.get('source', 'profiles/dram_traffic.json')}) "
                               "x queries per launch / CUDA-event launch time (this run) / measured "
                               "HBM peak")
    else:
        roof.update(achieved=roof["requested_gbs"], traffic=None, frac=roof["requested_frac"],
                    frac_basis="requested row bytes (no ncu DRAM capture for this config/qProbes "
                               "in profiles/dram_traffic.json); L2 hits included")

    # --------------------------------------------------------- e2e (host API)
    Qh = torch.empty((nq, d), dtype=torch.float32).pin_memory().numpy()
    Qh[:] = Q
    # page-locked result buffers too: the device writes ids/scores straight into them
    ids_h = torch.empty((nq, K_TOP), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
    sc_h = torch.empty((nq, K_TOP), dtype=torch.float64).pin_memory().numpy()
    e_ids = e_sc = None

    def e2e_step():
        ix.query(Qh, K_TOP, qprobes, out=(ids_h, sc_h))
        if world > 1:
            s_t = torch.from_numpy(sc_h).cuda()
            i_t = torch.from_numpy(ids_h.view(np.int32)).cuda()
            ms, mi = fdist.allgather_merge(s_t, i_t, K_TOP)
            return ms.cpu().numpy(), mi.cpu().numpy().astype(np.int64).astype(np.uint32)
        return sc_h, ids_h

    e2e_step()
    dd.barrier()
    te0 = time.perf_counter()
    for _ in range(args.steps):
        e_sc, e_ids = e2e_step()
    te = time.perf_counter() - te0
    e2e_qps = nq * args.steps / dd.max([te])[0]
    parity = {"e2e_equals_device": bool(np.array_equal(e_ids, g_ids)
                                        and np.array_equal(e_sc, g_sc))}

    # ---------------------------------------------- qProbes sweep (+ recall)
    sweep = []
    gt_info = None
    if not args.no_sweep and world == 1:
        gt = None
        if not args.no_recall:
            # exact ground truth on the GPU (fpp_brute_force: inner_product bit for bit,
            # ties to the lower id -- SPEC.md:490-503), timed separately from the sweep
            nr = min(nq, 1000)
            gt_ids = torch.empty((nr, K_TOP), dtype=torch.int32, device="cuda")
            gt_sc = torch.empty((nr, K_TOP), dtype=torch.float64, device="cuda")
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record()
            ix.brute_force_device(Qd[:nr].contiguous(), gt_ids, gt_sc, K_TOP, stream=stream)
            g1.record()
            torch.cuda.synchronize()
            gt = gt_ids.cpu().numpy().view(np.uint32)
            gt_info = {"queries": nr, "ms": g0.elapsed_time(g1),
                       "method": "exact fp64 brute force on the GPU (fpp_brute_force)"}
        for qp in cfg["sweep"]:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            step(qp)
            torch.cuda.synchronize()
            e0.record()
            step(qp)
            e1.record()
            torch.cuda.synchronize()
            row = {"qprobes": qp, "queries_per_s": nq / (e0.elapsed_time(e1) / 1e3)}
            if gt is not None:
                got = ids_d[:len(gt)].cpu().numpy().view(np.uint32)
                rec = np.mean([len(set(got[i]) & set(gt[i])) / K_TOP for i in range(len(gt))])
                row["recall_at_20"] = float(rec)
            sweep.append(row)
        # SimHash rerank at the headline qProbes: exact distances
        # per query drop from U_q to B
        for B in cfg.get("rerank", []):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ix.query_device(Qd, ids_d, sc_d, K_TOP, qprobes, stream=stream, rerank=B)
            torch.cuda.synchronize()
            e0.record()
            ix.query_device(Qd, ids_d, sc_d, K_TOP, qprobes, stream=stream, rerank=B)
            e1.record()
            torch.cuda.synchronize()
            row = {"qprobes": qprobes, "rerank_B": B,
                   "queries_per_s": nq / (e0.elapsed_time(e1) / 1e3)}
            if gt is not None:
                got = ids_d[:len(gt)].cpu().numpy().view(np.uint32)
                row["recall_at_20"] = float(np.mean([len(set(got[i]) & set(gt[i])) / K_TOP
                                                     for i in range(len(gt))]))
            sweep.append(row)

    # ------------------------------------------------ parity + CPU baseline
    cpu = None
    if world == 1 and rank == 0:
        orc = oracle_lib(native=False)  # the checker: the prebuilt (portable) oracle
        if not args.no_parity:
            L = cfg["L"]
            parity.update(parity_tables(cfg, X, ix, orc, threads, sorted({0, L // 2, L - 1})))
            ox = import_gpu_csr(cfg, X, ix, orc)
            m = min(nq, args.parity_queries)
            sample = np.unique(np.linspace(0, nq - 1, m).astype(np.int64))
            t0 = time.perf_counter()
            parity["query_sample"] = parity_queries(ox, Q, sample, g_ids, g_sc,
                                                    st_local.astype(np.uint64), qprobes, threads)
            parity["query_sample"]["seconds"] = time.perf_counter() - t0
            parity["note"] = ("oracle tables rebuilt from X and compared byte for byte; the query "
                              "sample runs the oracle's search over the GPU CSR")
            del ox
        if not args.no_cpu_baseline:
            try:
                orc = oracle_lib(native=True)  # timing: -march=native on this host if possible
                ox = import_gpu_csr(cfg, X, ix, orc)
                m = min(len(Q), threads)
                t0 = time.perf_counter()
                ox.query(Q[:m], K_TOP, qprobes, threads=threads)
                dt = max(time.perf_counter() - t0, 1e-6)
                ns = int(min(len(Q), max(m, m * 12.0 / dt)))
                t0 = time.perf_counter()
                ox.query(Q[:ns], K_TOP, qprobes, threads=threads)
                tq = time.perf_counter() - t0
                del ox
                cpu = {"value": ns / tq, "unit": "queries/s", "cores": threads, "kind": "port",
                       "cpu": cpu_info(),
                       "sample": f"{ns} of {nq} queries at qProbes={qprobes} over the full "
                                 f"{cfg['L']}-table index (GPU CSR, sampled tables verified "
                                 f"bit-exact above); {threads} OpenMP threads; oracle -march="
                                 f"{'native' if orc.NATIVE else 'x86-64-v3'}",
                       "build_points_per_s": build_cpu_sample(cfg, min(n, 1_000_000), threads, orc),
                       "build_sample": f"1 of {cfg['L']} tables over min(n, 1M) points of the "
                                       f"same distribution, extrapolated linearly in L"}
            except Exception as e:  # reported, not fatal
                cpu = {"value": None, "error": repr(e)}
    elif world > 1 and not args.no_parity and n <= 2_000_000:
        # merged shard answers vs a single-rank index over the full X (rank 0)
        if rank == 0:
            Xf, _ = make_data(dict(cfg, nq=0), 0, n, fpp)
            full = fpp.Index.build(Xf, **dict(prm, device=local))
            fi, fs = full.query(Q, K_TOP, qprobes)
            parity["merged_equals_single"] = bool(np.array_equal(fi, g_ids)
                                                  and np.array_equal(fs, g_sc))
            del full, Xf
        dd.barrier()

    # ------------------------------------------------------ C5 build block
    c5 = None
    if not args.no_c5 and args.config == "c4" and world == 1:
        del ix
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        c5 = build_block(CONFIGS["c5"], "c5", 2, 1, dd, [] if args.no_parity else [0], threads)

    rc = 0
    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": "queries/s (k=20)", "value": qps, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
            "higher_is_better": True,
            "scaling": "strong (n fixed, sharded n/G)" if world > 1 else "none (1 GPU)",
            "vs_baseline": None, "dtype": "f32 (FHT, pair scores) / f64 (inner products)",
            "data": "synthetic (pinned seeded generator, DESIGN.md section 6; stands in for the "
                    "paper's corpora)",
            "config": config_dict(args.config, cfg, qprobes, world),
            "roofline": roof,
            "path": {"algorithmic_bytes_per_step_full_rows": path_bytes_full,
                     "mean_probes": P_sum / nq, "mean_entries": E_sum / nq,
                     "mean_candidates": U_sum / nq,
                     "phase_ms_per_step": {k: tim[k] / args.steps for k in
                                           ("qhash_ms", "probe_ms", "collect_ms", "score_ms")},
                     "note": "phase times overlap (two-stream pipeline)"},
            "build": {"points_per_s": n / tbuild_max, "device_points_per_s": n / tbuild_dev_max,
                      "wall_s": tbuild_max, "device_s": tbuild_dev_max,
                      "kept_total": info["kept_total"],
                      "prefilter_total": info["prefilter_total"]},
            "e2e": {"value": e2e_qps, "unit": "queries/s",
                    "h2d_bytes_per_step": nq * d * 4,
                    "d2h_bytes_per_step": nq * K_TOP * (4 + 8)},
            "gpu_launches": int(tim["launches"]),
            "cpu_baseline": cpu,
            "parity": parity,
            "sweep": sweep,
            "ground_truth": gt_info,
            "build_c5": c5,
            "clocks": clocks,
            "dist_backend": dd.backend,
        }
        ok = parity_ok(parity) and parity_ok((c5 or {}).get("parity"))
        line["parity_ok"] = ok
        print(json.dumps(line), flush=True)
        rc = 0 if ok else 1
    dd.close()
    return rc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=0,
                    help="timed steps (default: 5; the short c1-c3 steps default to enough "
                         "steps for about a second, so the clock sampler sees the timed region)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--qprobes", type=int, default=0)
    ap.add_argument("--replicate-stage-a", action="store_true",
                    help="N>1: every rank hashes and probe-selects the whole batch (the "
                         "round-1 path) instead of its slice + an all-gather of probe sets")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-recall", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 build block (c4 runs)")
    ap.add_argument("--parity-queries", type=int, default=400)
    ap.add_argument("--ref-step-s", type=float, default=3.0,
                    help="reference arm: seconds of CPU work per timed step")
    ap.add_argument("--mode", default="", choices=["", "query", "build"],
                    help="query (default for c1-c4) or build-only throughput (default for c5)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.steps <= 0:
        args.steps = ({"c1": 1000, "c2": 60, "c3": 400}.get(args.config, 5)
                      if args.impl == "ours" else 5)
    cfg = CONFIGS[args.config]
    qprobes = args.qprobes or cfg["qprobes"]
    mode = args.mode or ("build" if args.config == "c5" else "query")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if args.impl == "reference":  # rank 0 alone runs; no launcher needed
            os.environ.update(WORLD_SIZE=str(args.gpus), RANK="0")
        else:
            return spawn_ranks(args)
    if args.impl == "reference":
        if mode == "build":
            return run_reference_build(args, cfg)
        return run_reference(args, cfg, qprobes)
    if mode == "build":
        return run_build(args, cfg)
    return run_query_bench(args, cfg, qprobes)


if __name__ == "__main__":
    sys.exit(main())
