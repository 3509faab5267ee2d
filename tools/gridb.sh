#!/bin/bash
# kernel-B grid cap sweep (PFEM_GRIDB) on config 3 E+R / K.v and config 4 K.v
cd "$(dirname "$0")/.." || exit 1
for g in 1184 592 296 148; do
  for a in "--config 3 --op er" "--config 4 --op kv"; do
    PFEM_GRIDB=$g timeout 300 python tools/bench_kernel.py $a --reps 40 2>&1 | tail -1 | \
      python -c "import sys,json; l=sys.stdin.read(); d=json.loads(l) if l.startswith('{') else None; print('gridb=$g', d['config'], d['op'], round(d['median_us'],1)) if d else print(l[-200:])"
  done
done | tee gpurun_out/gridb_${1:-x}.txt
for a in "--config 3 --op er" "--config 4 --op kv"; do
  PFEM_DEBUG=128 timeout 300 python tools/bench_kernel.py $a --reps 40 2>&1 | tail -1 | \
    python -c "import sys,json; l=sys.stdin.read(); d=json.loads(l); print('nopdl', d['config'], d['op'], round(d['median_us'],1))"
done | tee -a gpurun_out/gridb_${1:-x}.txt
