#!/bin/bash
# kernel-A-alone times (PFEM_DEBUG=32; needs a PFEM_DBG=1 build: python tools/ab_build.py dbg PFEM_DBG=1,
# then PFEM_LIB=libpfem_dbg.so) for configs 4 K.v and 5 E+R, plus ncu full captures of both
cd "$(dirname "$0")/.." || exit 1
TAG=${1:-x}
for a in "--config 4 --op kv" "--config 5 --op er"; do
  for d in 0 32; do
    PFEM_DEBUG=$d timeout 300 python tools/bench_kernel.py $a --reps 40 2>&1 | tail -1 | \
      python -c "import sys,json; l=sys.stdin.read(); d=json.loads(l) if l.startswith('{') else None; print('dbg=$d', d['config'], d['op'], round(d['median_us'],1)) if d else print(l[-200:])"
  done
done | tee gpurun_out/prof45_$TAG.txt
for a in "--config 4 --op kv" "--config 5 --op er"; do
  c=$(echo $a | cut -d' ' -f2)
  CMD="python tools/bench_kernel.py $a --reps 6 --copies 1"
  timeout 300 $CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_assemble|k_node_finish" -s 4 -c 2 -o gpurun_out/prof_${TAG}_c$c $CMD > gpurun_out/ncu_${TAG}_c$c.log 2>&1; echo ncu_c$c=$?
done
