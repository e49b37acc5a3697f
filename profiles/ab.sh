#!/bin/bash
# A/B bench lines for one config under different env settings (one GPU).
# usage: profiles/ab.sh <config> <tag> "<ENV=.. ENV2=..>" ["<ENV...>" ...]
cfg=$1; tag=$2; shift 2
mkdir -p gpurun_out/$tag
i=0
for e in "$@"; do
  env $e python -X faulthandler bench.py --config $cfg --no-c5 --no-cpu-baseline --no-sweep \
      --no-parity > gpurun_out/$tag/ab$i.json 2> gpurun_out/$tag/ab$i.err
  rc=$?
  [ $rc != 0 ] && echo "$e: rc=$rc" && tail -25 gpurun_out/$tag/ab$i.err
  python - gpurun_out/$tag/ab$i.json "$e" <<'PY'
import json, sys
try:
    j = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    ph = j["path"]["phase_ms_per_step"]
    print(f"{sys.argv[2]:40s} {j['value']:10.0f} q/s  {j['ms_per_step']:7.2f} ms  " +
          " ".join(f"{k[:-3]}={v:.1f}" for k, v in ph.items()) +
          f"  readfrac={j['roofline']['row_bytes_read_fraction']:.3f}")
except Exception as ex:
    print(sys.argv[2], "FAILED", ex)
PY
  i=$((i+1))
done
