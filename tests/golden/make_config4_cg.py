"""Oracle-only golden for the full-size config-4 CG (reading R18;
PAPER.md App. B, warm start P:395-417).

    python tests/golden/make_config4_cg.py [--threads N]

Calls only ``oracle/`` and the seeded generators in ``pfem_gen/`` (no CUDA path).  Writes

- ``config4_ustar_f32.npz``: u*, the oracle CG solution at tol 1e-12 from zero, rounded to
  float32 (the warm start is built from this stored array by both sides:
  x0 = u* + 0.01 rms(u*) xi on free DOFs, xi seeded 4004, ``pfem_gen.configs.warm_start``);
- ``config4_cg.json``: for x0 = 0 and x0 = warm, the oracle iteration counts to 1e-8 under the
  dot-product orders 0 (ascending), 1 (descending) and 2 (pairwise) — the oracle's own
  spread — the first 50 entries of the order-0 residual history, rel_res0 and the true
  relative residual at exit, and the wall time per solve on this host (context only).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from pfem_gen.configs import config4, warm_start  # noqa: E402

TOL = 1e-8
ORDERS = (0, 1, 2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--n-nodes", type=int, default=80)
    ap.add_argument("--out", default=HERE)
    a = ap.parse_args()
    oracle.set_threads(a.threads)
    p = config4(n_nodes=a.n_nodes)
    om = oracle.prepare_problem(p)
    shape = p.coords.shape
    f, mask = p.f_ext, p.mask
    suffix = "" if a.n_nodes == 80 else f"_n{a.n_nodes}"
    res = {"config": "config4", "n_nodes_axis": a.n_nodes, "n_nodes": int(p.n_nodes), "n_elems": int(p.n_elems),
           "tol": TOL, "dot_orders": list(ORDERS), "threads": a.threads or os.cpu_count()}
    t0 = time.time()
    ustar, rep = om.cg(f, mask, np.zeros(shape), tol=1e-12, max_iter=50000, history=False)
    res["ustar"] = {"tol": 1e-12, "iterations": rep["iterations"], "status": rep["status"],
                    "true_rel_res_final": rep["true_rel_res_final"], "seconds": time.time() - t0}
    print("u*", res["ustar"], flush=True)
    us32 = ustar.astype(np.float32)
    np.savez_compressed(os.path.join(a.out, f"config4_ustar_f32{suffix}.npz"), ustar=us32)
    x_warm = warm_start(us32.astype(np.float64), mask, seed=4004)
    for name, x0 in (("zero", np.zeros(shape)), ("warm", x_warm)):
        runs = {}
        for o in ORDERS:
            t0 = time.time()
            _, rep = om.cg(f, mask, x0, tol=TOL, max_iter=50000, history=True, dot_order=o)
            runs[str(o)] = {"iterations": rep["iterations"], "status": rep["status"],
                            "rel_res0": rep["rel_res0"], "rel_res_final": rep["rel_res_final"],
                            "true_rel_res_final": rep["true_rel_res_final"], "seconds": time.time() - t0}
            if o == 0:
                runs[str(o)]["history50"] = [float(h) for h in rep["history"][:50]]
                h = rep["history"]
                runs[str(o)]["first_below"] = {str(t): int(np.argmax(h < t)) if np.any(h < t) else None
                                               for t in (1e-3, 1e-6)}
            print(name, o, {k: v for k, v in runs[str(o)].items() if k != "history50"}, flush=True)
        its = [r["iterations"] for r in runs.values()]
        res[name] = {"runs": runs, "spread": [min(its), max(its)]}
    with open(os.path.join(a.out, f"config4_cg{suffix}.json"), "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
