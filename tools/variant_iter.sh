#!/bin/bash
# kernel A variants side by side: "ENV ..." settings x the 4 headline kernels (+ direct-variant parity)
cd "$(dirname "$0")/.." || exit 1
TAG=${1:-v}; shift
SETS=${@:-"PFEM_VARIANT=0 PFEM_VARIANT=1"}
for V in $SETS; do
  for a in "--config 3 --op er" "--config 3 --op kv" "--config 4 --op kv" "--config 5 --op er"; do
    env ${V//,/ } timeout 300 python tools/bench_kernel.py $a --reps 40 2>&1 | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$V', d['config'], d['op'], round(d['median_us'],1), round(d['frac'],3))"
  done
done | tee gpurun_out/variants_$TAG.txt
PFEM_VARIANT=1 timeout 900 python -m pytest tests -m gpu -x -q -k "not cg_config4" 2>&1 | tail -2
