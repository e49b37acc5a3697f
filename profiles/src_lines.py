"""Per-CUDA-source-line stall samples and instructions from an ncu `--page source --csv
--print-source cuda,sass` export (usage: src_lines.py file.csv [topN])."""
import csv
import os
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
smp, ins, text = defaultdict(float), defaultdict(float), {}
f, h, cur = "?", None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        h = r
        ismp = h.index("Warp Stall Sampling (All Samples)")
        iins = h.index("Instructions Executed")
        continue
    if h is None or len(r) < len(h):
        continue
    if r[0]:
        try:
            cur = (f, int(r[0]))
        except ValueError:
            continue
        text[cur] = r[1]
    try:
        smp[cur] += float(r[ismp] or 0)
        ins[cur] += float(r[iins] or 0)
    except ValueError:
        pass
ts, ti = sum(smp.values()) or 1, sum(ins.values()) or 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"stall samples {ts:.0f}, instructions {ti:.3e}")
for k in sorted(smp, key=lambda k: -smp[k])[:top]:
    print(f"{k[0][:12]}:{k[1]:<5d} smp {100 * smp[k] / ts:5.1f}%  ins {100 * ins[k] / ti:5.1f}%  "
          f"{text.get(k, '')[:80].strip()}")
