#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
for pf in 0 148 296 592 1184; do
  for a in "--config 4 --op kv" "--config 5 --op er"; do
    PFEM_PF=$pf timeout 300 python tools/bench_kernel.py $a --reps 40 2>&1 | tail -1 | \
      python -c "import sys,json; l=sys.stdin.read(); d=json.loads(l) if l.startswith('{') else None; print('pf=$pf', '$a', round(d['median_us'],1)) if d else print(l[-200:])"
  done
done | tee gpurun_out/pf_sweep2.txt
