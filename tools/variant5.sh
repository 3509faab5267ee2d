#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
for v in 0 1; do
  for a in "--config 5 --op er" "--config 4 --op kv" "--config 5 --op er --order input"; do
    PFEM_VARIANT=$v timeout 300 python tools/bench_kernel.py $a --reps 40 2>&1 | tail -1 | \
      python -c "import sys,json; l=sys.stdin.read(); d=json.loads(l) if l.startswith('{') else None; print('variant=$v', '$a', round(d['median_us'],1), d['n_occ']) if d else print(l[-300:])"
  done
done | tee gpurun_out/variant5.txt
