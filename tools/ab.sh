#!/bin/bash
# same-box A/B: .ab/head (HEAD tree) vs the working tree's libpfem.so and libpfem_<tag>.so builds
#   bash tools/ab.sh <out-tag> [lib tags ...]
cd "$(dirname "$0")/.." || exit 1
OUT=${1:-ab}; shift
run4() {  # $1 label, rest: env
  local label=$1; shift
  for a in "--config 3 --op er" "--config 3 --op kv" "--config 4 --op kv" "--config 5 --op er"; do
    env "$@" timeout 300 python tools/bench_kernel.py $a --reps 40 2>&1 | tail -1 | \
      python -c "import sys,json; l=sys.stdin.read(); d=json.loads(l) if l.startswith('{') else None; print('$label', d['config'], d['op'], round(d['median_us'],1), round(d['frac'],3)) if d else print('$label', l[-300:])"
  done
}
{
[ -d .ab/head ] && (cd .ab/head && run4 head X=1)
run4 cur X=1
for t in "$@"; do run4 $t PFEM_LIB=libpfem_$t.so; done
} | tee gpurun_out/ab_$OUT.txt
