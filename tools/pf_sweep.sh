cd /root/repo
for pf in 0 300 700 1400 2800; do
  for c in "--config 5 --op er" "--config 4 --op kv"; do
  PFEM_PF=$pf python tools/bench_kernel.py $c --reps 40 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pf$pf', d['config'], round(d['median_us'],1))"
  done
done
