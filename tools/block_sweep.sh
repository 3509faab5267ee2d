#!/bin/bash
# kernel timings vs plan block size (direct form for blocks above the staged capacity)
cd "$(dirname "$0")/.." || exit 1
TAG=${1:-x}
{
for be in 256 384 512 768; do timeout 300 python tools/bench_kernel.py --config 4 --op kv --reps 40 --block-elems $be | tail -1; done
for be in 512 768 1024 1360; do timeout 300 python tools/bench_kernel.py --config 5 --op er --reps 40 --block-elems $be | tail -1; done
for be in 256 512; do PFEM_VARIANT=1 timeout 300 python tools/bench_kernel.py --config 3 --op er --reps 40 --block-elems $be | tail -1; done
} 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['config'], d['op'], d['n_blocks'], d['n_occ'], round(d['median_us'], 1), round(d['frac'], 3))
" | tee gpurun_out/block_sweep_$TAG.txt
