#!/bin/bash
# round evidence, call 1 of 2 (on the GPU box): GPU tests, the default bench line (with the
# oracle cpu_baseline), the reference arm, and the ncu launch list of the bench command.
#   bash tools/evidence.sh <tag>
cd "$(dirname "$0")/.." || exit 1
TAG=${1:-x}
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest_exit=$?; tail -2 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench=$?; tail -2 gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo ref=$?
CMD="python bench.py --steps 20 --warmup 3 --no-extras --no-cpu"
timeout 300 $CMD > gpurun_out/plain_lt_$TAG.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_lt_$TAG.log 2>&1; echo ncu_lt=$?
