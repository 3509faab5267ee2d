"""Shared test helpers: build the GPU mesh / material from a pfem_gen.Problem and the
oracle mesh from the SAME (dtype-rounded) inputs (reading R14: fp32 runs round the
fp64 inputs to fp32 and the fp64 oracle consumes the rounded values)."""
from __future__ import annotations

import numpy as np
import torch

DT = {"f32": torch.float32, "f64": torch.float64}
NP = {"f32": np.float32, "f64": np.float64}
TOL = {"f32": 2e-5, "f64": 1e-12}     # north star (BASELINE.json): rel-L2 bars


def rounded(a, dtype):
    return np.asarray(a, dtype=np.float64).astype(NP[dtype]).astype(np.float64)


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def max_rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))


def gpu_problem(prob, dtype=None, block_elems=0, dev="cuda", elem_order="auto"):
    """(Mesh, Material, u tensor) for the CUDA path."""
    import paper_2601_03086_b200 as pf
    dtype = dtype or prob.dtype
    td = DT[dtype]
    pe, pn = prob.parts()
    mesh = pf.Mesh(torch.as_tensor(prob.coords, device=dev), torch.as_tensor(prob.conn, device=dev), dtype=td,
                   part_elem=pe if prob.n_parts > 1 else None, part_node=pn if prob.n_parts > 1 else None,
                   block_elems=block_elems, elem_order=elem_order)
    mat = pf.Material(prob.model, prob.param_kind, torch.as_tensor(np.asarray(prob.p0), dtype=td, device=dev),
                      torch.as_tensor(np.asarray(prob.p1), dtype=td, device=dev))
    u = torch.as_tensor(prob.u, dtype=td, device=dev)
    return mesh, mat, u


def oracle_problem(orc, prob, dtype=None):
    """Oracle mesh whose material parameters are the dtype-rounded inputs."""
    dtype = dtype or prob.dtype
    pe, pn = prob.parts()
    return orc.prepare(prob.coords, prob.conn, prob.model, prob.param_kind, rounded(prob.p0, dtype),
                       rounded(prob.p1, dtype), pe, pn)


PER_ENTRY = 100.0   # reading R31: per-entry bar = PER_ENTRY * rel-L2 bar, scale-relative


def assert_field(a, b, dtype, what=""):
    """Parity of one output array (reading R13 / R31): the whole-array rel-L2 bar of the north
    star, and next to it a per-entry bar |a_i - b_i| <= 100 tol (|b_i| + rms(b)), so that a
    single wrong element or node cannot hide inside a small global norm."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    tol = TOL[dtype]
    e = rel_l2(a, b)
    assert e < tol, (what, "rel-L2", e)
    rms = float(np.sqrt(np.mean(b * b))) if b.size else 0.0
    worst = float(np.max(np.abs(a - b) / (np.abs(b) + rms + 1e-300))) if b.size else 0.0
    assert worst < PER_ENTRY * tol, (what, "per-entry", worst)
    return e, worst


def assert_totals(t, ref, scale, dtype, what="totals"):
    """Per-(sample, part) totals (reading R32): |t - ref| <= tol * scale entry by entry, where
    scale = |W| + |f.u| is the sum of the magnitudes of the two terms of Pi = W - f.u (no
    f_ext: scale = |W|), so the cancellation in W - f.u is not charged to the kernel."""
    t = np.asarray(t, np.float64)
    ref = np.asarray(ref, np.float64)
    scale = np.asarray(scale, np.float64)
    err = np.abs(t - ref) / np.maximum(scale, 1e-300)
    assert float(np.max(err)) < TOL[dtype], (what, float(np.max(err)))
