#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
for lib in libpfem.so libpfem_eb512.so; do
  for be in 256 512; do
    for op in er kv; do
      PFEM_LIB=$lib timeout 300 python tools/bench_kernel.py --config 3 --op $op --reps 40 --block-elems $be 2>&1 | tail -1 | \
        python -c "import sys,json; l=sys.stdin.read(); d=json.loads(l) if l.startswith('{') else None; print('$lib', $be, '$op', round(d['median_us'],1), d['n_occ']) if d else print(l[-300:])"
    done
  done
done | tee gpurun_out/eb512.txt
