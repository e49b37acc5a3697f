#!/bin/bash
# one --set full capture of the score kernel of a query config (ONE GPU, after the same
# bench command exited 0 without ncu).  usage: profiles/ncu_score.sh <config> <tag> [skip] [env...]
set -u
cfg=$1; tag=$2; skip=${3:-3}; shift 3 || true
out=gpurun_out/$tag
mkdir -p $out
env "$@" ncu --set full --import-source on --clock-control none -k regex:'k_score' \
    --launch-skip $skip --launch-count 1 -o $out/score \
    python bench.py --config $cfg --steps 1 --warmup 3 --no-c5 --no-cpu-baseline --no-sweep --no-parity \
    > $out/score.log 2>&1
echo "score rc=$?"
