"""Write the DRAM traffic of the dominant query kernel into profiles/dram_traffic.json.

usage: python profiles/traffic.py <report.ncu-rep> <config> <qprobes> <kernel-substring> <source-note>
                                  [queries-per-launch (default 8192)]

Reads one `ncu --set full` capture (dram__bytes_read.sum + dram__bytes_write.sum and
gpu__time_duration.sum of the first launch whose name contains <kernel-substring>) and
records it per (config, qProbes); bench.py divides those bytes by its own CUDA-event
launch time for roofline.frac (north star: "ncu DRAM GB/s counters").
"""
import csv
import json
import os
import subprocess
import sys

rep, config, qprobes, kname, note = sys.argv[1:6]
qpl = int(sys.argv[6]) if len(sys.argv) > 6 else 8192
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rr = list(csv.reader(raw.splitlines()))
H, U = rr[0], rr[1]


def val(r, m):
    v = float(r[H.index(m)].replace(",", ""))
    u = U[H.index(m)]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
    return v * scale.get(u, 1.0)


row = next(r for r in rr[2:] if kname in r[H.index("Kernel Name")])
ent = {"qprobes": int(qprobes), "kernel": row[H.index("Kernel Name")][:80],
       "dram_bytes_per_launch": val(row, "dram__bytes_read.sum") + val(row, "dram__bytes_write.sum"),
       "dram_read_bytes": val(row, "dram__bytes_read.sum"),
       "dram_write_bytes": val(row, "dram__bytes_write.sum"),
       "gpu_time_ms": val(row, "gpu__time_duration.sum"),
       "grid": row[H.index("launch__grid_size")],
       "queries_per_launch": qpl,
       "source": note}
ent["ncu_gbs"] = ent["dram_bytes_per_launch"] / ent["gpu_time_ms"] / 1e6
p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dram_traffic.json")
j = json.load(open(p)) if os.path.exists(p) else {}
j[config] = ent
json.dump(j, open(p, "w"), indent=1)
print(json.dumps(ent, indent=1))
