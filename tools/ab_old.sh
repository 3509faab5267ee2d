# same-box comparison of an older tree (.ab/old, its own binding and library) with HEAD
cd /root/repo
for t in . .ab/old .ab/c8b8d76; do
  for a in "--config 4 --op kv" "--config 5 --op er" "--config 3 --op er"; do
    (cd $t && python tools/bench_kernel.py $a --reps 40 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$t', d['config'], d['op'], round(d['median_us'],1))")
  done
done
