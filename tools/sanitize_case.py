"""Small workload that exercises every kernel family once, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck, one tool per gpurun call):

    compute-sanitizer --tool racecheck python tools/sanitize_case.py

Staged (several samples) and direct (one sample) element kernels with kernel B, COLOUR mode,
masked tangent, CG (pipelined CSR iteration and COLOUR), Jacobi PCG, Newton, the pretraining
loss, heat conduction, on-the-fly geometry and the Q4 / Q8 path, on meshes small enough that
the sanitizer's slowdown stays in minutes."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2601_03086_b200 as pf  # noqa: E402
from pfem_gen import beam_q4, config1, cook_q8, fourier_field, kuhn_cube, plate_with_holes, small_cube_problem  # noqa: E402


def main():
    dev = "cuda"
    rng = np.random.default_rng(0)
    # 2-D plate, NH fp32, 5 samples (staged form, ragged sample chunk) and 1 sample (direct form)
    c, t, _ = plate_with_holes(24, np.random.default_rng(1))
    for dt in (torch.float32, torch.float64):
        m = pf.Mesh(torch.as_tensor(c, device=dev), torch.as_tensor(t, device=dev), dtype=dt, block_elems=97)
        mat = pf.Material("neohookean", "lame", torch.as_tensor(rng.uniform(0.3, 1, len(t)), dtype=dt, device=dev),
                          torch.as_tensor(rng.uniform(0.3, 1, len(t)), dtype=dt, device=dev))
        for S in (5, 1):
            u = torch.as_tensor(np.stack([0.05 * fourier_field(c, rng) for _ in range(S)]), dtype=dt, device=dev)
            f = torch.as_tensor(0.01 * rng.standard_normal(c.shape), dtype=dt, device=dev)
            for mode in ("csr", "colour"):
                pf.energy(m, mat, u, f_ext=f, elem_energy=True, residual=True, mode=mode)
                mask = torch.as_tensor((rng.random(c.size) < 0.2).astype(np.uint8), device=dev)
                pf.tangent_apply(m, mat, u, u=u, mask=mask, mode=mode)
                pf.pretrain_loss(m, mat, u, f_ext=f, mode=mode)
            m.geometry = "on_the_fly"
            pf.energy(m, mat, u, elem_energy=True, residual=True)
            m.geometry = "stored"
        W, tot, r = pf.heat(m, torch.as_tensor(np.exp(rng.standard_normal(len(t))), dtype=dt, device=dev),
                            torch.as_tensor(rng.standard_normal((3, len(c))), dtype=dt, device=dev))
    # 3-D cube, NH fp32 (staged T4) and the fused CG / PCG on the config-4 recipe
    c3, t3 = kuhn_cube(9, brick=4)
    m3 = pf.Mesh(torch.as_tensor(c3, device=dev), torch.as_tensor(t3, device=dev), dtype=torch.float32)
    mat3 = pf.Material("neohookean", "lame", torch.tensor([0.4], device=dev), torch.tensor([0.6], device=dev))
    u3 = torch.as_tensor(np.stack([0.1 * fourier_field(c3, rng) for _ in range(4)]), dtype=torch.float32, device=dev)
    pf.energy(m3, mat3, u3, elem_energy=True, residual=True)
    pf.tangent_apply(m3, mat3, u3, u=u3)
    p = small_cube_problem(n_nodes=8, brick=4)
    m4 = pf.Mesh(torch.as_tensor(p.coords, device=dev), torch.as_tensor(p.conn, device=dev), dtype=torch.float64)
    mat4 = pf.Material("linear", "young_poisson", torch.as_tensor(p.p0, device=dev), torch.as_tensor(p.p1, device=dev))
    f4 = torch.as_tensor(p.f_ext, device=dev)
    mk4 = torch.as_tensor(p.mask, device=dev)
    for mode in ("csr", "colour"):
        pf.cg(m4, mat4, f4, torch.zeros_like(f4), mask=mk4, tol=1e-8, mode=mode)
        pf.cg(m4, mat4, f4, torch.zeros_like(f4), mask=mk4, tol=1e-8, mode=mode, precond="jacobi")
    p1 = config1()
    m1 = pf.Mesh(torch.as_tensor(p1.coords, device=dev), torch.as_tensor(p1.conn, device=dev))
    mat1 = pf.Material("linear", "young_poisson", torch.as_tensor(p1.p0, device=dev), torch.as_tensor(p1.p1, device=dev))
    f1 = torch.as_tensor(p1.f_ext, device=dev)
    pf.newton(m1, mat1, torch.zeros_like(f1), f_ext=f1, mask=torch.as_tensor(p1.mask, device=dev), tol=1e-12, cg_tol=1e-12)
    # quadrilaterals
    for mk in (beam_q4, cook_q8):
        pq = mk(n_cells=6)
        mq = pf.Mesh(torch.as_tensor(pq.coords, device=dev), torch.as_tensor(pq.conn, device=dev), elem_type=pq.elem)
        matq = pf.Material(pq.model, pq.param_kind, torch.as_tensor(pq.p0, device=dev), torch.as_tensor(pq.p1, device=dev))
        fq = torch.as_tensor(pq.f_ext, device=dev)
        pf.newton(mq, matq, torch.zeros_like(fq), f_ext=fq, mask=torch.as_tensor(pq.mask, device=dev),
                  tol=1e-10 * float(np.linalg.norm(pq.f_ext)), cg_tol=1e-10)
    torch.cuda.synchronize()
    print("sanitize case done")


if __name__ == "__main__":
    main()
