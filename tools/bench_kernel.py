"""Focused kernel timing for one config / op (development tool; bench.py is the contract).

    python tools/bench_kernel.py --config 4 --op kv --reps 50
    python tools/bench_kernel.py --config 5 --op er --reps 50
    python tools/bench_kernel.py --config 3 --op er --reps 50 [--mode colour] [--block-elems N]

Rotates over 3 copies (inputs > L2) and prints one JSON line with the median and mean per-call
time (CUDA events) and the algorithmic-bytes bandwidth."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2601_03086_b200 as pf  # noqa: E402
from bench import bytes_energy_residual, bytes_tangent, load_peaks  # noqa: E402
from pfem_gen import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--op", default="er", choices=["er", "kv", "e", "r"])
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--copies", type=int, default=3)
    ap.add_argument("--mode", default="csr")
    ap.add_argument("--block-elems", type=int, default=0)
    ap.add_argument("--dtype", default=None)
    ap.add_argument("--order", default="auto", choices=["auto", "input", "locality"])
    ap.add_argument("--otf", action="store_true", help="geometry formed on the fly from coords")
    ap.add_argument("--lib", default=None, help="an alternative in-tree build (libpfem_<tag>.so)")
    ap.add_argument("--brick", type=int, default=0, help="configs 3 / 4: generator brick size (0 = default)")
    a = ap.parse_args()
    if a.lib:
        from paper_2601_03086_b200 import _lib
        _lib.load(os.path.join(ROOT, "paper_2601_03086_b200", a.lib))
    if a.brick and a.config in (3, 4):
        prob = CONFIGS[a.config](brick=a.brick)
    else:
        prob = CONFIGS[a.config]() if a.config != 2 else CONFIGS[2](dtype=a.dtype or "f32")
    dt = torch.float32 if (a.dtype or prob.dtype) == "f32" else torch.float64
    s = 4 if dt == torch.float32 else 8
    dev = "cuda"
    pe, pn = prob.parts()
    sets = []
    t0 = time.perf_counter()
    for c in range(a.copies):
        m = pf.Mesh(torch.as_tensor(prob.coords, device=dev), torch.as_tensor(prob.conn, device=dev), dtype=dt,
                    part_elem=pe if prob.n_parts > 1 else None, part_node=pn if prob.n_parts > 1 else None,
                    block_elems=a.block_elems, elem_order=a.order, geometry="on_the_fly" if a.otf else "stored")
        mat = pf.Material(prob.model, prob.param_kind, torch.as_tensor(np.asarray(prob.p0), dtype=dt, device=dev),
                          torch.as_tensor(np.asarray(prob.p1), dtype=dt, device=dev))
        u = torch.as_tensor(prob.u, dtype=dt, device=dev)
        v = torch.randn_like(u)
        mask = torch.as_tensor(prob.mask, device=dev) if prob.mask is not None else None
        S = u.shape[0]
        outs = (torch.empty((S, prob.n_parts), dtype=dt, device=dev), torch.empty((S, prob.n_elems), dtype=dt, device=dev),
                torch.empty_like(u))
        sets.append(dict(m=m, mat=mat, u=u, v=v, mask=mask, outs=outs, kv=torch.empty_like(u)))
    torch.cuda.synchronize()
    prep = (time.perf_counter() - t0) / a.copies

    def call(st):
        if a.op == "er":
            pf.energy(st["m"], st["mat"], st["u"], elem_energy=True, residual=True, out=st["outs"], mode=a.mode)
        elif a.op == "e":
            pf.energy(st["m"], st["mat"], st["u"], out=(st["outs"][0], None, None), mode=a.mode)
        elif a.op == "r":
            pf.residual(st["m"], st["mat"], st["u"], out=st["outs"][2], mode=a.mode)
        else:
            pf.tangent_apply(st["m"], st["mat"], st["v"], u=st["u"] if prob.model == "neohookean" else None,
                             mask=st["mask"], out=st["kv"], mode=a.mode)

    for i in range(6):
        call(sets[i % len(sets)])
    torch.cuda.synchronize()
    ts = []
    for i in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call(sets[i % len(sets)])
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    us = np.array([x.elapsed_time(y) * 1e3 for x, y in ts])
    E, N, d, S = prob.n_elems, prob.n_nodes, prob.dim, prob.u.shape[0]
    mat_pe = int(len(np.asarray(prob.p0)) > 1) + int(len(np.asarray(prob.p1)) > 1)
    if a.op == "er":
        B = bytes_energy_residual(E, N, d, S, s, True, mat_pe, prob.n_parts)
    elif a.op == "kv":
        B = bytes_tangent(E, N, d, S, s, prob.model == "neohookean", mat_pe, prob.mask is not None)
    else:
        B = bytes_energy_residual(E, N, d, S, s, False, mat_pe, prob.n_parts)
    peak, _ = load_peaks()
    med = float(np.median(us))
    print(json.dumps({"config": a.config, "op": a.op, "mode": a.mode, "E": E, "S": S, "median_us": med,
                      "mean_us": float(us.mean()), "GBps": B / (med * 1e-6) / 1e9, "frac": B / (med * 1e-6) / 1e9 / peak,
                      "bytes": B, "prepare_s": prep, "n_blocks": sets[0]["m"].n_blocks, "n_occ": sets[0]["m"].n_occ}))


if __name__ == "__main__":
    main()
