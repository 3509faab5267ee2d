#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
python - << 'PY'
import glob, os, sys
lib = "paper_2601_03086_b200/libpfem.so"
t = os.path.getmtime(lib)
stale = [f for f in glob.glob("paper_2601_03086_b200/csrc/*") if os.path.getmtime(f) > t]
if stale: sys.exit(f"STALE libpfem.so: {stale}")
PY
[ $? -ne 0 ] && exit 1
# one GPU iteration: quick GPU tests, bench (json), short bench + ncu full capture of k_assemble
# usage (on the GPU box via gpurun): bash tools/gpu_iter.sh <tag> [pytest -k expr]
TAG=${1:-x}
K=${2:-"not cg_config4_scaled"}
timeout 900 python -m pytest tests -q -m gpu -x --timeout 600 -k "$K" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; tail -2 gpurun_out/bench.err
CMD="python bench.py --steps 20 --warmup 3 --no-extras --no-cpu"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_assemble|k_node_finish" -s 12 -c 4 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
