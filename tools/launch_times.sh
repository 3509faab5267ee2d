#!/bin/bash
# per-launch device times of the bench step kernels (cold, serialized; compare shares)
cd "$(dirname "$0")/.." || exit 1
CMD="python bench.py --steps 20 --warmup 3 --no-extras --no-cpu"
timeout 300 $CMD > gpurun_out/plain_lt.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_lt.log 2>&1; echo ncu_lt=$?
