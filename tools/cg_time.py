"""Config-4 CG timing (development tool): ms per iteration vs the K.v time, zero start."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_03086_b200 as pf  # noqa: E402
from pfem_gen import config4  # noqa: E402

p = config4()
dev = "cuda"
m = pf.Mesh(torch.as_tensor(p.coords, device=dev), torch.as_tensor(p.conn, device=dev), dtype=torch.float64)
if len(sys.argv) > 1 and sys.argv[1] == "otf":
    m.geometry = "on_the_fly"
mat = pf.Material("linear", "young_poisson", torch.as_tensor(p.p0, device=dev), torch.as_tensor(p.p1, device=dev))
mask = torch.as_tensor(p.mask, device=dev)
f = torch.as_tensor(p.f_ext, device=dev)
x0 = torch.zeros_like(f)
pf.cg(m, mat, f, x0, mask=mask, tol=1e-8, max_iter=100)
for pre in ("none", "jacobi"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, rep = pf.cg(m, mat, f, x0, mask=mask, tol=1e-8, max_iter=20000, precond=pre)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{pre}: iterations {rep['iterations']} time {dt:.3f} s  ms/it {dt / rep['iterations'] * 1e3:.4f} "
          f"true {rep['true_rel_res_final']:.2e}")
v = torch.randn((1,) + f.shape, dtype=torch.float64, device=dev)
kv = torch.empty_like(v)
for _ in range(5):
    pf.tangent_apply(m, mat, v, mask=mask, out=kv)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    pf.tangent_apply(m, mat, v, mask=mask, out=kv)
b.record()
torch.cuda.synchronize()
print(f"Kv {a.elapsed_time(b) / 50 * 1e3:.1f} us")
