"""Global-memory instructions of one kernel from an ncu `--page source --csv --print-source
sass` export: L2 theoretical sectors (and excess over ideal), executions, stall samples.
usage: mem_instr.py file.csv [topN]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
out = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    try:
        sec = float(r[ix["L2 Theoretical Sectors Global"]] or 0)
        exc = float(r[ix["L2 Theoretical Sectors Global Excessive"]] or 0)
        ex = float(r[ix["Instructions Executed"]] or 0)
        smp = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    if sec > 0:
        out.append((sec, exc, ex, smp, r[0][-5:], r[1].strip()[:70]))
tot = sum(o[0] for o in out)
print(f"L2 theoretical sectors (global) {tot:.3e}")
for o in sorted(out, key=lambda o: -o[0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{100 * o[0] / tot:5.1f}%  sectors {o[0]:.2e} excess {o[1]:.2e} exec {o[2]:.2e} smp {o[3]:7.0f} {o[4]} {o[5]}")
