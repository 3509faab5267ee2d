#!/bin/bash
# one ncu --set full capture (with source) of a bench_kernel case (development tool; run under gpurun):
#   bash tools/ncu_one.sh <tag> <kernel regex> <bench_kernel args...>
cd "$(dirname "$0")/.." || exit 1
tag=$1; rx=$2; shift 2
mkdir -p gpurun_out
timeout 300 python tools/bench_kernel.py "$@" --reps 10 > gpurun_out/plain_$tag.log 2>&1 || { echo plain failed; tail -5 gpurun_out/plain_$tag.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s 6 -c 2 -o gpurun_out/prof_$tag -f python tools/bench_kernel.py "$@" --reps 10 > gpurun_out/ncu_$tag.log 2>&1; echo ncu=$?
