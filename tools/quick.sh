#!/bin/bash
# quick GPU iteration: the 4 headline kernel timings + GPU parity (without the long CG test)
cd "$(dirname "$0")/.." || exit 1
TAG=${1:-q}
for a in "--config 3 --op er" "--config 3 --op kv" "--config 4 --op kv" "--config 5 --op er"; do
  timeout 300 python tools/bench_kernel.py $a --reps 40 2>&1 | tail -1 | \
    python -c "import sys,json; l=sys.stdin.read(); d=json.loads(l) if l.startswith('{') else None; print(d['config'], d['op'], round(d['median_us'],1), round(d['frac'],3)) if d else print(l)"
done | tee gpurun_out/quick_$TAG.txt
timeout 900 python -m pytest tests -q -m gpu -x -k "not cg_config4" 2>&1 | tail -3
