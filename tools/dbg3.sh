#!/bin/bash
# config-3 E+R (and K.v) kernel time under PFEM_DEBUG ablation switches; the kernel-side switches
# need a build with them compiled in: python tools/ab_build.py dbg PFEM_DBG=1, then PFEM_LIB=libpfem_dbg.so
cd "$(dirname "$0")/.." || exit 1
for d in 0 32 33 34 40 35 43 59; do
  for op in er kv; do
    PFEM_DEBUG=$d timeout 300 python tools/bench_kernel.py --config 3 --op $op --reps 40 2>&1 | tail -1 | \
      python -c "import sys,json; l=sys.stdin.read(); d=json.loads(l) if l.startswith('{') else None; print('dbg=$d', '$op', round(d['median_us'],1)) if d else print(l[-200:])"
  done
done | tee gpurun_out/dbg3_${1:-x}.txt
