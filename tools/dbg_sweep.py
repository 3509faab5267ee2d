"""Time config-3 fused E+R under PFEM_DEBUG switches (each in a fresh process)."""
import json, os, subprocess, sys
res = {}
for d in [0, 1, 2, 4, 8, 1 | 2, 1 | 2 | 4 | 8, 1 | 2 | 4 | 8 | 16, 2 | 4 | 8]:
    env = dict(os.environ, PFEM_DEBUG=str(d))
    out = subprocess.run([sys.executable, "bench.py", "--steps", "300", "--warmup", "10", "--no-extras", "--no-cpu"],
                         env=env, capture_output=True, text=True)
    try:
        j = json.loads(out.stdout.strip().splitlines()[-1])
        res[d] = (round(j["roofline"]["avg_launch_us"], 1), round(j["roofline"]["tangent"]["avg_launch_us"], 1))
    except Exception as e:
        res[d] = str(out.stderr[-300:])
    print(d, res[d], flush=True)
