#!/bin/bash
# Same-box A/B timing of in-tree library builds (development tool; run under gpurun):
#   bash tools/ab_kernels.sh OUT "libpfem.so libpfem_old.so" ["--config 3 --op er" ...]
# Each (case, build) pair is timed by tools/bench_kernel.py (median of 60 calls, rotating
# copies), alternating builds twice so drift shows; one line per run in OUT.
cd "$(dirname "$0")/.." || exit 1
out=$1; libs=$2; shift 2
cases=("$@")
[ ${#cases[@]} -eq 0 ] && cases=("--config 3 --op er" "--config 3 --op kv" "--config 4 --op kv" "--config 5 --op er" "--config 2 --op er")
for rep in 1 2; do
  for c in "${cases[@]}"; do
    for lib in $libs; do
      r=$(timeout 180 python tools/bench_kernel.py $c --lib $lib --reps 60 2>&1 | tail -1 |
          python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['median_us'],1), round(d['frac'],3))" 2>&1)
      echo "$lib | $c | $r" >> "$out"
    done
  done
done
