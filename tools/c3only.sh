cd /root/repo
for V in "$@"; do
  for a in "--config 3 --op er" "--config 3 --op kv"; do
    env ${V//,/ } timeout 300 python tools/bench_kernel.py $a --reps 40 2>&1 | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$V', d['config'], d['op'], round(d['median_us'],1), round(d['frac'],3))"
  done
done
