"""Summarize ncu outputs into profiles/ (launch-list shares + per-kernel metrics).

usage: python profiles/summarize.py <launches.csv> <report.ncu-rep> <out-prefix>
"""
import collections
import csv
import json
import subprocess
import sys

launches, rep, out = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(open(launches)) if len(r) > 5]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void ", "").split("<")[0].strip().replace("fpp::", "")
    v = float(r[vi].replace(",", ""))
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v for _, v in agg.values())
QUERY = ("k_query_lists", "k_probe_select", "k_scan_eq", "k_collect", "k_collect_cluster", "k_score",
         "k_score_pruned", "k_score_screen", "k_order_keys", "k_order_sort", "k_gather_rows",
         "k_scatter_results", "k_merge_topk")
qtot = sum(v for k, (_, v) in agg.items() if k in QUERY) or 1
lines = ["| kernel | launches | total ms | share of all | share of query |", "|---|---|---|---|---|"]
for k, (c, v) in agg.items():
    qs = f"{100 * v / qtot:.1f}%" if k in QUERY else "-"
    lines.append(f"| {k} | {c} | {v / 1e6:.2f} | {100 * v / tot:.1f}% | {qs} |")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rr = list(csv.reader(raw.splitlines()))
H, U = rr[0], rr[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct"]
kern = []
for r in rr[2:]:
    d = {"kernel": r[H.index("Kernel Name")][:60]}
    for w in want:
        if w in H:
            d[w] = f"{r[H.index(w)]} {U[H.index(w)]}".strip()
    st = []
    for i, c in enumerate(H):
        if c.startswith("smsp__pcsamp_warps_issue_stalled") and not c.endswith("not_issued"):
            try:
                st.append((c.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i])))
            except ValueError:
                pass
    st.sort(key=lambda x: -x[1])
    tot_s = sum(v for _, v in st) or 1
    d["top_stalls"] = [f"{a} {100 * b / tot_s:.0f}%" for a, b in st[:4]]
    kern.append(d)
with open(out + "_launches.md", "w") as f:
    f.write("Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; "
            "cold-cache, serialised: compare shares)\n\n" + "\n".join(lines) + "\n")
with open(out + "_kernels.json", "w") as f:
    json.dump(kern, f, indent=1)
print("\n".join(lines))
for d in kern:
    print(json.dumps(d))
