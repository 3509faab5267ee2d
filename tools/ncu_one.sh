#!/bin/bash
# ncu --set full of kernel A/B for one bench_kernel invocation: ncu_one.sh <tag> <bench_kernel args...>
cd "$(dirname "$0")/.." || exit 1
TAG=$1; shift
CMD="python tools/bench_kernel.py $* --reps 6 --copies 1"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo plain failed; tail gpurun_out/plain_$TAG.log; exit 1; }
tail -1 gpurun_out/plain_$TAG.log
ncu --set full --clock-control none --import-source on -k regex:"k_assemble|k_node_finish" -s 4 -c 2 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
