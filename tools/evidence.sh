#!/bin/bash
# round evidence in one call: GPU tests, smoke, default bench line, reference arm, ncu launch list
# of the bench command and one ncu --set full capture of the bench step's kernels (each ncu run
# only after the same command exited 0 without ncu)
#   bash tools/evidence.sh <tag>
cd "$(dirname "$0")/.." || exit 1
TAG=${1:-x}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest_exit=$?; tail -3 gpurun_out/pytest_gpu_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke=$?
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench=$?; tail -2 gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo ref=$?
CMD="python bench.py --steps 20 --warmup 3 --no-extras --no-cpu"
timeout 300 $CMD > gpurun_out/plain_lt_$TAG.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_lt_$TAG.log 2>&1; echo ncu_lt=$?
timeout 300 $CMD > gpurun_out/plain_full_$TAG.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_assemble|k_node_finish" -s 12 -c 4 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu_full=$?
