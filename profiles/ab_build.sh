#!/bin/bash
# A/B of the C5 build throughput under env settings (one GPU): profiles/ab_build.sh <tag> "<ENV>"...
tag=$1; shift
mkdir -p gpurun_out/$tag
i=0
for e in "$@"; do
  env $e python -X faulthandler bench.py --config c5 --steps 2 --warmup 1 --no-parity --no-cpu-baseline \
      > gpurun_out/$tag/b$i.json 2> gpurun_out/$tag/b$i.err || { echo "$e: rc=$?"; tail -20 gpurun_out/$tag/b$i.err; }
  python - gpurun_out/$tag/b$i.json "$e" <<'PY'
import json, sys
try:
    j = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = j["roofline"]
    print(f"{sys.argv[2]:44s} {j['value'] / 1e6:7.2f} M pts/s  hash {r['hash_ms']:7.1f} ms  sort {r['sort_ms']:6.1f} ms  fp32 {r['fp32_frac_hash_kernel']:.3f}")
except Exception as ex:
    print(sys.argv[2], "FAILED", ex)
PY
  i=$((i+1))
done
