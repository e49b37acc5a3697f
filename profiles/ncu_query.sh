#!/bin/bash
# ncu recipe for one query config (run under gpurun on ONE GPU, after the same bench
# command exited 0 without ncu).  usage: profiles/ncu_query.sh <config> <tag> [skip]
#   1. launch list (gpu__time_duration.sum, --clock-control none): shares per kernel
#   2. --set full captures of the query kernels (first launch after `skip` of each)
set -u
cfg=$1; tag=$2; skip=${3:-8}
out=gpurun_out/$tag
mkdir -p $out
B="python bench.py --config $cfg --steps 1 --warmup 3 --no-c5 --no-cpu-baseline --no-sweep --no-parity"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
    $B > $out/launches.log 2>&1
echo "launches rc=$?"
ncu --set full --import-source on --clock-control none \
    -k regex:'k_score_screen|k_score_pruned|k_score\b|k_collect|k_probe_select|k_query_lists' \
    --launch-skip $skip --launch-count 4 -o $out/full $B > $out/full.log 2>&1
echo "full rc=$?"
