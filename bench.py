#!/usr/bin/env python
"""bench.py -- Falconn++ hot path on B200: batched query throughput (+ build points/s).

Default (N=1): BASELINE.json configs[1] ("c2"): n=1.2M d=300 1000-cluster mixture
(sigma 0.3) normalized, L=100 K=2 D=512 iProbes=3 alpha=0.05 kappa=20, 10,000
queries, k=20, headline qProbes=10,000 (the 1k-20k sweep is reported beside it).
A step = one batched query of all nq queries through the hot path (hash ->
probe select -> bucket walk/dedup -> row gather + fp64 dot + top-k).

  python bench.py [--gpus N --steps K --warmup W --config c2 --qprobes 10000]
  python bench.py --impl reference ...   # CPU oracle port on the host cores

Multi-GPU (torchrun, one rank per GPU): rank g indexes ids [g*n/G,(g+1)*n/G)
with the global filter (NCCL all-reduce of bucket histograms + all-gather of
bucket prefixes: the shards hold exactly the 1-GPU index), queries are
replicated, per-rank top-k lists are merged after an NCCL all-gather;
value = nq*K / (max over ranks of the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
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
               alpha=0.01, nq=100_000, qprobes=5000, sweep=[5000]),
    # index-build throughput config (BASELINE.json configs[4]); build-only
    "c5": dict(n=50_000_000, d=256, clusters=0, sigma=0.0, L=64, K=2, D=256, iprobes=5,
               alpha=0.005, nq=0, qprobes=0, sweep=[]),
}
K_TOP = 20
KAPPA = 20
SEED = 1


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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
    X = gen.synth(hi, cfg["d"], cfg["clusters"], cfg["sigma"], seed=SEED, stream=0)[lo:hi]
    X = gen.normalize(X)
    Q = gen.normalize(gen.synth(cfg["nq"], cfg["d"], cfg["clusters"], cfg["sigma"], seed=SEED,
                                stream=1))
    return np.ascontiguousarray(X), Q


def cpu_baseline(cfg, X, Q, ix, qprobes, budget_s=20.0):
    """Oracle port on this host: query sample over the GPU-built (bit-exact) CSR, and one
    table of the build extrapolated linearly in L."""
    from oracle import oracle as orc
    threads = os.cpu_count() or 1
    L = cfg["L"]
    info = ix.info()
    offs, ids, scs, tb = [], [], [], [0]
    for t in range(L):
        o, i, s = ix.table(t)
        offs.append(o)
        ids.append(i)
        scs.append(s)
        tb.append(tb[-1] + len(i))
    csr = (np.stack(offs), np.concatenate(ids), np.concatenate(scs), np.array(tb, np.uint64))
    ox = orc.Index(X, L=L, K=cfg["K"], D=cfg["D"], iprobes=cfg["iprobes"], alpha=cfg["alpha"],
                   kappa=KAPPA, seed=SEED, csr=csr)
    del csr, offs, ids, scs
    # calibrate then run a bounded sample of queries with all host threads
    m = min(len(Q), threads)
    t0 = time.perf_counter()
    ox.query(Q[:m], K_TOP, qprobes, threads=threads)
    dt = max(time.perf_counter() - t0, 1e-6)
    ns = int(min(len(Q), max(m, m * budget_s * 0.6 / dt)))
    t0 = time.perf_counter()
    ox.query(Q[:ns], K_TOP, qprobes, threads=threads)
    tq = time.perf_counter() - t0
    qps = ns / tq
    # build: one table, all threads, extrapolated to L tables
    t0 = time.perf_counter()
    ob = orc.Index(X, L=L, K=cfg["K"], D=cfg["D"], iprobes=cfg["iprobes"], alpha=cfg["alpha"],
                   kappa=KAPPA, seed=SEED, threads=threads, t_begin=0, t_end=1)
    tb1 = time.perf_counter() - t0
    del ob
    build_pps = len(X) / (tb1 * L)
    return {"value": qps, "unit": "queries/s", "cores": threads, "kind": "port",
            "sample": f"{ns} of {len(Q)} queries at qProbes={qprobes} over the full "
                      f"{L}-table index (CSR imported from the GPU build, bit-exact); "
                      f"{threads} OpenMP threads",
            "build_points_per_s": build_pps,
            "build_sample": f"1 of {L} tables on all {len(X)} points, extrapolated linearly in L",
            "kept_total": info["kept_total"]}


def run_reference(args, cfg, qprobes):
    """--impl reference: the CPU oracle port (the reference ships no hashing/index/query
    code) on the host cores, same config/metric/unit."""
    from oracle import oracle as orc
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n = cfg["n"]
    X, Q = make_data(cfg, 0, n, orc)
    log(f"[reference] oracle build of {cfg['L']} tables on {threads} threads ...")
    t0 = time.perf_counter()
    ox = orc.Index(X, L=cfg["L"], K=cfg["K"], D=cfg["D"], iprobes=cfg["iprobes"],
                   alpha=cfg["alpha"], kappa=KAPPA, seed=SEED, threads=threads)
    tbuild = time.perf_counter() - t0
    log(f"[reference] build {tbuild:.1f}s")
    m = min(len(Q), threads)
    t0 = time.perf_counter()
    ox.query(Q[:m], K_TOP, qprobes, threads=threads)
    dt = max(time.perf_counter() - t0, 1e-6)
    ns = int(min(len(Q), max(m, m * 8.0 / dt)))  # ~8 s per step
    for w in range(args.warmup):
        ox.query(Q[:m], K_TOP, qprobes, threads=threads)
    times = []
    for s in range(args.steps):
        t0 = time.perf_counter()
        ox.query(Q[:ns], K_TOP, qprobes, threads=threads)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    qps = ns * args.steps / tot
    line = {
        "metric": "queries/s (k=20)", "value": qps, "unit": "queries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32/f64",
        "data": "synthetic (pinned seeded generator, DESIGN.md section 6)", "impl": "reference",
        "config": {"workload": args.config, "n": n, "d": cfg["d"], "L": cfg["L"], "K": cfg["K"],
                   "D": cfg["D"], "iProbes": cfg["iprobes"], "alpha": cfg["alpha"],
                   "kappa": KAPPA, "qProbes": qprobes, "k": K_TOP, "nq_per_step": ns},
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "port",
                         "sample": f"{ns} of {cfg['nq']} queries per step, full {cfg['L']}-table "
                                   f"oracle index built on CPU"},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "build_points_per_s": n / tbuild,
    }
    print(json.dumps(line), flush=True)


def build_cpu_sample(cfg, npts, threads):
    """Oracle build of one table over a same-distribution sample, as points/s for all L."""
    from oracle import oracle as orc
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
        return
    threads = os.cpu_count() or 1
    npts = 200_000
    vals = [build_cpu_sample(cfg, npts, threads) for _ in range(max(1, args.steps))]
    v = float(np.median(vals))
    print(json.dumps({
        "metric": "index-build points/s", "value": v, "unit": "points/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "impl": "reference",
        "data": "synthetic i.i.d. N(0,1) normalized", "config": {"workload": args.config, **cfg},
        "cpu_baseline": {"value": v, "unit": "points/s", "cores": threads, "kind": "port",
                         "sample": f"{npts} points x 1 of {cfg['L']} tables per step, "
                                   f"extrapolated linearly in L"},
        "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_build(args, cfg):
    """Build-only throughput (config c5): points/s of the full index build (K1 + K2)."""
    import torch
    import torch.distributed as dist

    import paper_2206_01382_b200 as fpp
    from paper_2206_01382_b200 import dist as fdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, d = cfg["n"], cfg["d"]
    lo, hi = fdist.shard_range(n, world, rank)
    # i.i.d. N(0,1) rows generated on the device (torch Philox, seed 1 + shard offset),
    # normalized on the device: same distribution as the host generator, not the same bytes
    gen = torch.Generator(device="cuda")
    gen.manual_seed(SEED * 1_000_003 + lo)
    X = torch.empty((hi - lo, d), dtype=torch.float32, device="cuda")
    for a in range(0, hi - lo, 1 << 22):
        b = min(hi - lo, a + (1 << 22))
        blk = torch.randn((b - a, d), generator=gen, device="cuda", dtype=torch.float32)
        X[a:b] = blk / blk.double().norm(dim=1, keepdim=True).float()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    def one_build():
        prm = dict(L=cfg["L"], K=cfg["K"], D=cfg["D"], iProbes=cfg["iprobes"], alpha=cfg["alpha"],
                   kappa=KAPPA, seed=SEED, device=local)
        if world > 1:  # global filter over NCCL
            return fdist.build_global_filter(fdist.GpuShardEngine(X, lo, **prm))
        return fpp.Index.build(X, id_offset=lo, **prm)

    for _ in range(args.warmup):
        ix = one_build()
        info = ix.info()
        del ix
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    dev_ms = []
    with ClockSampler(local) as clk:
        ev0.record()
        for _ in range(args.steps):
            ix = one_build()
            t = ix.timings()
            dev_ms.append((t["hash_ms"], t["sort_ms"]))
            del ix
        ev1.record()
        torch.cuda.synchronize()
    barrier()
    t_ms = ev0.elapsed_time(ev1)
    tt = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    pps = n * args.steps / (t_ms / 1e3)
    hash_ms = float(np.mean([a for a, _ in dev_ms]))
    sort_ms = float(np.mean([b for _, b in dev_ms]))
    flops = (hi - lo) * cfg["L"] * cfg["K"] * 3 * cfg["D"] * int(np.log2(cfg["D"]))
    bytes_build = (4 * (hi - lo) * d + 24 * (hi - lo) * cfg["L"] * cfg["iprobes"]
                   + 8 * info["kept_total"])
    hbm, peak_kind = peaks()
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        cpu = {"value": build_cpu_sample(cfg, 200_000, threads), "unit": "points/s",
               "cores": threads, "kind": "port",
               "sample": f"oracle build of 1 of {cfg['L']} tables over 200000 points of the same "
                         f"distribution, extrapolated linearly in L"}
    if rank == 0:
        print(json.dumps({
            "metric": "index-build points/s", "value": pps, "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic i.i.d. N(0,1) rows normalized, generated on device (torch Philox)",
            "config": {"workload": args.config, "n": n, "d": d, "L": cfg["L"], "K": cfg["K"],
                       "D": cfg["D"], "iProbes": cfg["iprobes"], "alpha": cfg["alpha"],
                       "kappa": KAPPA, "parallelism": f"shard{world}" if world > 1 else "single"},
            "roofline": {"kernel": "k_hash_build", "bound": "fp32 (FHT butterflies)",
                         "fht_adds_per_s": flops / (hash_ms / 1e3),
                         "hbm_achieved_gbs": bytes_build / ((hash_ms + sort_ms) / 1e3) / 1e9,
                         "hbm_peak": hbm, "peak_kind": peak_kind,
                         "hbm_frac": bytes_build / ((hash_ms + sort_ms) / 1e3) / 1e9 / hbm,
                         "hash_ms": hash_ms, "sort_ms": sort_ms},
            "build": {"kept_total": info["kept_total"], "prefilter_total": info["prefilter_total"]},
            "e2e": {"value": pps, "unit": "points/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0,
                    "note": "inputs device-resident (device-generated); build via fpp_build_device"},
            "gpu_launches": None, "cpu_baseline": cpu, "clocks": clk.summary(),
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--qprobes", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-recall", action="store_true")
    ap.add_argument("--mode", default="", choices=["", "query", "build"],
                    help="query (default for c1-c4) or build-only throughput (default for c5)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    qprobes = args.qprobes or cfg["qprobes"]
    mode = args.mode or ("build" if args.config == "c5" else "query")
    if args.impl == "reference":
        if mode == "build":
            return run_reference_build(args, cfg)
        return run_reference(args, cfg, qprobes)
    if mode == "build":
        return run_build(args, cfg)

    import torch
    import torch.distributed as dist

    import paper_2206_01382_b200 as fpp
    from paper_2206_01382_b200 import dist as fdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, d, nq = cfg["n"], cfg["d"], cfg["nq"]
    lo, hi = fdist.shard_range(n, world, rank)
    t0 = time.perf_counter()
    X, Q = make_data(cfg, lo, hi, fpp)
    log(f"[rank {rank}] data {time.perf_counter() - t0:.1f}s shard [{lo},{hi})")

    def barrier():
        if world > 1:
            dist.barrier()

    # ---------------------------------------------------------------- build
    Xd = torch.from_numpy(X).cuda()
    barrier()
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
    tb_t = torch.tensor([tbuild, build_dev_ms / 1e3], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tb_t, op=dist.ReduceOp.MAX)
    tbuild_max, tbuild_dev_max = tb_t.tolist()
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

    def step(qp, stats=None):
        ix.query_device(Qd, ids_d, sc_d, K_TOP, qp, stats=stats, stream=stream)
        if world > 1:
            fdist.allgather_merge(sc_d, ids_d.view(torch.int32).to(torch.int64) & 0xFFFFFFFF,
                                  K_TOP)

    step(qprobes, st_d)
    torch.cuda.synchronize()
    st = st_d.cpu().numpy().astype(np.uint64)
    P_sum, E_sum, U_sum, _ = (int(x) for x in st.sum(axis=0))
    for _ in range(args.warmup - 1):
        step(qprobes)
    ix.reset_timings()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record()
        for _ in range(args.steps):
            step(qprobes)
        ev1.record()
        torch.cuda.synchronize()
    barrier()
    t_ms = ev0.elapsed_time(ev1)
    tt = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    tim = ix.timings()
    qps = nq * args.steps / (t_ms / 1e3)

    # roofline of the dominant kernel (the score gather): bytes it moves per launch /
    # launch time.  Row bytes are the library's exact count of candidate-row bytes read
    # (fpp_timings.score_bytes): with exact early termination (k_score_pruned) a
    # candidate that cannot reach the top-k is read only up to the slice whose bound
    # rules it out, so this is below SURVEY 8(d)'s full-row formula 4*d*U, which is
    # reported beside it ("*_full_rows").
    hbm, peak_kind = peaks()
    row_bytes_step = tim["score_bytes"] / args.steps if tim.get("score_bytes") else 4 * d * U_sum
    score_bytes_step = row_bytes_step + 4 * U_sum + 4 * d * nq + 12 * K_TOP * nq
    score_bytes_full = 4 * d * U_sum + 4 * U_sum + 4 * d * nq + 12 * K_TOP * nq
    path_bytes_step = 8 * P_sum + 4 * E_sum + row_bytes_step + 4 * d * nq + 12 * K_TOP * nq
    path_bytes_full = 8 * P_sum + 4 * E_sum + 4 * d * U_sum + 4 * d * nq + 12 * K_TOP * nq
    score_ms = tim["score_ms"] / args.steps
    achieved = score_bytes_step / (score_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "score_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                tj = json.load(f)
            if tj.get("config") == args.config and tj.get("qprobes") == qprobes:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    launches_per_step = tim["launches"] / args.steps
    # 5 kernels per query chunk (lists, probe select, scan, collect, score) plus 5 for
    # the batch reorder (nq >= 256 and nq*d >= 512k, fpp_query.cu run_query)
    reorder = nq >= 256 and nq * d >= 512 * 1024
    score_launches_per_step = max(1.0, (launches_per_step - (5 if reorder else 0)) / 5.0)

    # --------------------------------------------------------- e2e (host API)
    import torch as _t
    Qh = _t.empty((nq, d), dtype=_t.float32).pin_memory().numpy()
    Qh[:] = Q
    # page-locked result buffers too: the device writes ids/scores straight into them
    ids_h = _t.empty((nq, K_TOP), dtype=_t.int32).pin_memory().numpy().view(np.uint32)
    sc_h = _t.empty((nq, K_TOP), dtype=_t.float64).pin_memory().numpy()
    ix.query(Qh, K_TOP, qprobes, out=(ids_h, sc_h))
    barrier()
    te0 = time.perf_counter()
    for _ in range(args.steps):
        ix.query(Qh, K_TOP, qprobes, out=(ids_h, sc_h))
        if world > 1:
            s_t = torch.from_numpy(sc_h).cuda()
            i_t = torch.from_numpy(ids_h.astype(np.int64)).cuda()
            ms, mi = fdist.allgather_merge(s_t, i_t, K_TOP)
            mi.cpu()
    te = time.perf_counter() - te0
    tet = torch.tensor([te], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tet, op=dist.ReduceOp.MAX)
    e2e_qps = nq * args.steps / float(tet.item())

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
            ix.reset_timings()
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

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(cfg, X, Q, ix, qprobes)
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "error": repr(e)}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": "queries/s (k=20)", "value": qps, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f32 (FHT, pair scores) / f64 (inner products)",
            "data": "synthetic (pinned seeded generator, DESIGN.md section 6; stands in for the "
                    "paper's corpora)",
            "config": {"workload": args.config, "n": n, "d": d, "clusters": cfg["clusters"],
                       "sigma": cfg["sigma"], "L": cfg["L"], "K": cfg["K"], "D": cfg["D"],
                       "iProbes": cfg["iprobes"], "alpha": cfg["alpha"], "kappa": KAPPA,
                       "qProbes": qprobes, "k": K_TOP, "nq": nq,
                       "parallelism": f"shard{world}" if world > 1 else "single",
                       "l2": "inputs larger than L2 (X %.2f GB gathered at random)" % (
                           n * d * 4 / 1e9)},
            "roofline": {"kernel": "k_score_pruned" if row_bytes_step < 4 * d * U_sum else "k_score",
                         "bound": "hbm", "achieved": achieved,
                         "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "algorithmic_bytes_per_launch": score_bytes_step / score_launches_per_step,
                         "algorithmic_bytes_per_step": score_bytes_step,
                         "row_bytes_read_fraction": row_bytes_step / max(1, 4 * d * U_sum),
                         "algorithmic_bytes_per_step_full_rows": score_bytes_full,
                         "launches_per_step": launches_per_step,
                         "kernel_ms_per_step": score_ms,
                         "share_of_step": score_ms / (t_ms / args.steps)},
            "path": {"algorithmic_bytes_per_step": path_bytes_step,
                     "algorithmic_bytes_per_step_full_rows": path_bytes_full,
                     "achieved_gbs": path_bytes_step / (t_ms / args.steps / 1e3) / 1e9,
                     "frac_of_hbm": path_bytes_step / (t_ms / args.steps / 1e3) / 1e9 / hbm,
                     "mean_probes": P_sum / nq, "mean_entries": E_sum / nq,
                     "mean_candidates": U_sum / nq,
                     "phase_ms_per_step": {k: tim[k] / args.steps for k in
                                           ("qhash_ms", "probe_ms", "collect_ms", "score_ms")}},
            "build": {"points_per_s": n / tbuild_max, "device_points_per_s": n / tbuild_dev_max,
                      "wall_s": tbuild_max, "device_s": tbuild_dev_max,
                      "kept_total": info["kept_total"],
                      "prefilter_total": info["prefilter_total"]},
            "e2e": {"value": e2e_qps, "unit": "queries/s",
                    "h2d_bytes_per_step": nq * d * 4,
                    "d2h_bytes_per_step": nq * K_TOP * (4 + 8)},
            "gpu_launches": int(tim["launches"]),
            "cpu_baseline": cpu,
            "sweep": sweep,
            "ground_truth": gt_info,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
