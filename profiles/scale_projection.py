"""Per-rank work of the G-GPU C4 query on ONE GPU (no multi-GPU box here): rank 0's kernels
at shard size n/G, timed alone with CUDA events -- the data behind DESIGN.md section 9's
scaling projection.  For G in (1, 2, 4, 8): all G global-filter shards are built on device
0 (the all-reduce / all-gather done in process, as tests/test_gpu_scale.py does), then rank
0's part of dist.sharded_query is timed: stage A on its nq/G slice
(fpp_query_probe_sets_device), stage B on all nq queries against its shard
(fpp_query_from_probe_sets_device), the k-way merge of G lists.  The collectives are NOT
run; their bytes are printed so a link bandwidth can be applied.
usage: python profiles/scale_projection.py [c4] > gpurun_out/scale_projection.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2206_01382_b200 as fpp
from paper_2206_01382_b200 import dist as fdist

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = bench.CONFIGS[name]
qp, k = cfg["qprobes"], 20
X, Q = bench.make_data(cfg, 0, cfg["n"], fpp)
n, nq = len(X), len(Q)
prm = dict(L=cfg["L"], K=cfg["K"], D=cfg["D"], iProbes=cfg["iprobes"], alpha=cfg["alpha"],
           kappa=bench.KAPPA, seed=bench.SEED)
Qd = torch.from_numpy(Q).cuda()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
rows = []
for G in (1, 2, 4, 8):
    ranges = [fdist.shard_range(n, G, r) for r in range(G)]
    engines = [fdist.GpuShardEngine(X[lo:hi], lo, device=0, **prm) for lo, hi in ranges]
    gh = sum(e.hist() for e in engines)
    slots = engines[0].slots(gh)
    for e in engines[1:]:
        e.slots(gh)
    allp = torch.cat([e.prefix(gh, slots) for e in engines])
    shards = [e.finish(gh, allp, G) for e in engines]
    ix = shards[0]
    for s in shards[1:]:
        s.close()
    del engines, shards, allp
    torch.cuda.empty_cache()
    probes = ix.query_probe_sets_device(Qd, qp)  # every query's probe set (the all-gather's result)
    pe = probes.shape[1]
    lo, hi = fdist.query_slice(nq, G, 0)
    Qs = Qd[lo:hi].contiguous()
    ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    sc = torch.empty((nq, k), dtype=torch.float64, device="cuda")
    lists_s = torch.empty((G, nq, k), dtype=torch.float64, device="cuda").fill_(-1.0)
    lists_i = torch.full((G, nq, k), -1, dtype=torch.int32, device="cuda")
    best = None
    ts = torch.cuda.Stream()  # (a non-default stream: handle 0 would select the library's own)
    for rep in range(4):  # first pass warms up
        torch.cuda.synchronize()
        with torch.cuda.stream(ts):
            st = ts.cuda_stream  # the calls are ordered on this stream
            ev[0].record()
            ix.query_probe_sets_device(Qs, qp, stream=st)
            ev[1].record()
            ix.query_from_probe_sets_device(Qd, probes, ids, sc, k, qp, stream=st)
            ev[2].record()
            fdist.merge_lists(lists_s, lists_i, k)
            ev[3].record()
        torch.cuda.synchronize()
        t = [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
        if rep and (best is None or sum(t) < sum(best)):
            best = t
    a, b, m = best
    row = {"G": G, "shard_points": ranges[0][1] - ranges[0][0], "kept_entries": ix.info()["kept_total"],
           "stage_a_ms": a, "stage_b_ms": b, "merge_ms": m, "rank_ms": a + b + m,
           "allgather_probe_bytes_per_rank": int((hi - lo) * pe * 4) if G > 1 else 0,
           "allgather_topk_bytes_per_rank": int(nq * k * 12) if G > 1 else 0}
    rows.append(row)
    print(json.dumps(row), flush=True)
    ix.close()
    del probes
    torch.cuda.empty_cache()
t1 = rows[0]["rank_ms"]
for r in rows:
    # all-gather time at an assumed 300 GB/s per-GPU effective NVLink rate (G - 1 peers' data arrive)
    comm = (r["G"] - 1) * (r["allgather_probe_bytes_per_rank"] + r["allgather_topk_bytes_per_rank"]) / 300e9 * 1e3
    r["comm_ms_at_300GBs"] = comm
    r["projected_speedup_compute_only"] = t1 / r["rank_ms"]
    r["projected_speedup_with_comm"] = t1 / (r["rank_ms"] + comm)
    r["projected_queries_per_s"] = nq / ((r["rank_ms"] + comm) / 1e3)
print(json.dumps({"workload": name, "nq": nq, "qprobes": qp, "rows": rows,
                  "note": "rank 0's kernels timed alone on one B200 at shard size n/G; collectives not run "
                          "(bytes listed; 300 GB/s assumed for the projection)"}))
