"""Aggregate an ncu `--page source --print-source sass` CSV by opcode:
instructions executed and warp-stall samples (usage: sass_hist.py file.csv [topN])."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
ins = defaultdict(float)
smp = defaultdict(float)
for r in rows[2:]:
    if len(r) < len(h) or r[ix["Source"]] == "Source":
        continue
    op = r[ix["Source"]].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1] if len(op) > 1 else o
    o = o.split(".")[0]
    ins[o] += float(r[ix["Instructions Executed"]] or 0)
    smp[o] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
ti, ts = sum(ins.values()), sum(smp.values())
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print(f"total instructions {ti:.3e}, stall samples {ts:.0f}")
for o in sorted(ins, key=lambda k: -ins[k])[:top]:
    print(f"{o:10s} inst {ins[o] / ti * 100:5.1f}%  samples {smp[o] / ts * 100:5.1f}%")
