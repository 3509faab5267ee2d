cd /root/repo
for o in input locality; do for dbg in 0 32; do
  PFEM_DEBUG=$dbg python tools/bench_kernel.py --config 5 --op er --reps 40 --order $o | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$o dbg$dbg', round(d['median_us'],1), d['n_occ'])"
done; done
