#!/bin/bash
# round evidence, call 2 of 2: one ncu --set full capture of the bench step's kernels
#   bash tools/evidence_full.sh <tag>
cd "$(dirname "$0")/.." || exit 1
TAG=${1:-x}
CMD="python bench.py --steps 20 --warmup 3 --no-extras --no-cpu"
timeout 300 $CMD > gpurun_out/plain_full_$TAG.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_assemble|k_node_finish" -s 12 -c 4 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu=$?
