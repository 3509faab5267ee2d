import json, sys
j = json.load(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/bench.json'))
r = j['roofline']
print('value %.3e  ms/step %.4f  ER %.1f us frac %.3f  TG %.1f us frac %.3f  launches %s clocks %s' % (
    j['value'], j['ms_per_step'], r['avg_launch_us'], r['frac'], r['tangent']['avg_launch_us'], r['tangent']['frac'],
    j.get('gpu_launches'), j.get('clocks')))
for k, v in j.get('extras', {}).items():
    print(k, {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v.items()} if isinstance(v, dict) else v)
