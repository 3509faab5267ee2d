#!/bin/bash
# focused timings of the 4 headline kernels + ncu full of config 4 K.v (tag = $1)
cd "$(dirname "$0")/.." || exit 1
python - << 'PY' || exit 1
import glob, os, sys
t = os.path.getmtime("paper_2601_03086_b200/libpfem.so")
stale = [f for f in glob.glob("paper_2601_03086_b200/csrc/*") if os.path.getmtime(f) > t]
sys.exit(f"STALE libpfem.so: {stale}" if stale else 0)
PY
TAG=${1:-x}
for a in "--config 3 --op er" "--config 3 --op kv" "--config 4 --op kv" "--config 5 --op er"; do
  timeout 300 python tools/bench_kernel.py $a --reps 40 2>&1 | tail -1
done | tee gpurun_out/kernels_$TAG.jsonl
if [ -n "$2" ]; then
  CMD="python tools/bench_kernel.py $2 --reps 6 --copies 1"
  timeout 300 $CMD > gpurun_out/plain_k.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_assemble|k_node_finish" -s 4 -c 2 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_k.log 2>&1; echo ncu=$?
fi
