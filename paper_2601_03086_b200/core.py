"""Thin torch-facing wrappers of the C-ABI (same names as include/pfem.h without the
``pfem_`` prefix).  torch supplies device memory and the current stream; every
computation runs in libpfem's CUDA kernels.  Nothing here computes the method.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib as L

_DT = {torch.float32: L.F32, torch.float64: L.F64}
_TD = {L.F32: torch.float32, L.F64: torch.float64}
MODES = {"csr": L.ASSEMBLE_CSR, "colour": L.ASSEMBLE_COLOUR, "color": L.ASSEMBLE_COLOUR}
MODELS = {"linear": L.LINEAR, "neohookean": L.NEOHOOKEAN}
KINDS = {"lame": L.LAME, "young_poisson": L.YOUNG_POISSON,
         "young_poisson_plane_stress": L.YOUNG_POISSON_PLANE_STRESS}


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("libpfem takes CUDA tensors only (no CPU fallback)")


GEOMETRY = {"stored": 0, "on_the_fly": 1}
ELEM_TYPES = {"simplex": 0, "q4": 1, "q8": 2}


class Mesh:
    """A prepared mesh (pfem_mesh_prepare): geometry, CSR, colouring and assembly plan."""

    def __init__(self, coords: torch.Tensor, conn: torch.Tensor, dtype=torch.float64, part_elem=None,
                 part_node=None, block_elems: int = 0, max_colours: int = 128, stream=None,
                 elem_order: str = "auto", geometry: str = "stored", elem_type: str = "simplex"):
        lib = L.load()
        _require_cuda(coords, conn)
        dev = coords.device
        self.coords = coords.to(torch.float64).contiguous()
        self.conn = conn.to(torch.int32).contiguous()
        N, d = self.coords.shape
        E = self.conn.shape[0]
        nv = {"simplex": d + 1, "q4": 4, "q8": 8}[elem_type]
        if self.conn.shape[1] != nv:
            raise ValueError(f"conn must be [E, {nv}] for {elem_type} elements")
        if elem_type != "simplex" and d != 2:
            raise ValueError("Q4 / Q8 elements are 2-D")
        self.elem_type = elem_type
        self.dim, self.n_nodes, self.n_elems = d, N, E
        self.dtype = dtype
        K = 1
        self.part_elem = self.part_node = None
        if part_elem is not None:
            self.part_elem = torch.as_tensor(part_elem, dtype=torch.int32, device=dev).contiguous()
            self.part_node = torch.as_tensor(part_node, dtype=torch.int32, device=dev).contiguous()
            K = self.part_elem.numel() - 1
        self.n_parts = K
        self.grad = torch.empty((d * d, E), dtype=dtype, device=dev)
        self.vol = torch.empty(E, dtype=dtype, device=dev)
        self.csr_ptr = torch.empty(N + 1, dtype=torch.int32, device=dev)
        self.csr_ent = torch.empty(E * nv, dtype=torch.int32, device=dev)
        self.colour = torch.empty(E, dtype=torch.int32, device=dev)
        self.colour_elems = torch.empty(E, dtype=torch.int32, device=dev)
        self.colour_ptr = torch.empty(max_colours + 1, dtype=torch.int32, device=dev)
        m = L.pfem_mesh()
        m.dim, m.n_nodes, m.n_elems, m.n_parts = d, N, E, K
        m.dtype = _DT[dtype]
        m.block_elems = block_elems
        m.elem_order = {"input": 0, "locality": 1, "auto": 2}[elem_order]
        m.geometry = GEOMETRY[geometry]
        m.elem_type = ELEM_TYPES[elem_type]
        m.coords, m.conn = self.coords.data_ptr(), self.conn.data_ptr()
        m.part_elem = self.part_elem.data_ptr() if self.part_elem is not None else None
        m.part_node = self.part_node.data_ptr() if self.part_node is not None else None
        m.grad, m.vol = self.grad.data_ptr(), self.vol.data_ptr()
        m.csr_ptr, m.csr_ent = self.csr_ptr.data_ptr(), self.csr_ent.data_ptr()
        m.colour, m.colour_elems, m.colour_ptr = (self.colour.data_ptr(), self.colour_elems.data_ptr(),
                                                 self.colour_ptr.data_ptr())
        m.max_colours = max_colours
        self._m = m
        L.check(lib.pfem_mesh_prepare(C.byref(m), _stream(stream)))
        self._ws = {}

    # ------------------------------------------------------------------ info
    @property
    def geometry(self) -> str:
        """"stored" (prepared grad / vol) or "on_the_fly" (formed from coords in the element pass)."""
        return {v: k for k, v in GEOMETRY.items()}[self._m.geometry]

    @geometry.setter
    def geometry(self, g: str):
        self._m.geometry = GEOMETRY[g]

    @property
    def n_colours(self):
        return self._m.n_colours

    @property
    def n_negative(self):
        return self._m.n_negative

    @property
    def n_blocks(self):
        return self._m.n_blocks

    @property
    def n_occ(self):
        return self._m.n_occ

    def ref(self):
        return C.byref(self._m)

    def workspace(self, n_samples: int) -> torch.Tensor:
        """Zero-filled per-call workspace, cached per sample count (pfem_workspace_bytes)."""
        ws = self._ws.get(n_samples)
        if ws is None:
            nb = L.load().pfem_workspace_bytes(self.ref(), n_samples)
            ws = torch.zeros(max(nb, 1), dtype=torch.uint8, device=self.coords.device)
            self._ws[n_samples] = ws
        return ws

    def cg_workspace(self) -> torch.Tensor:
        ws = self._ws.get("cg")
        if ws is None:
            nb = L.load().pfem_cg_workspace_bytes(self.ref())
            ws = torch.zeros(max(nb, 1), dtype=torch.uint8, device=self.coords.device)
            self._ws["cg"] = ws
        return ws

    def newton_workspace(self) -> torch.Tensor:
        ws = self._ws.get("newton")
        if ws is None:
            nb = L.load().pfem_newton_workspace_bytes(self.ref())
            ws = torch.zeros(max(nb, 1), dtype=torch.uint8, device=self.coords.device)
            self._ws["newton"] = ws
        return ws

    def plan_export(self):
        """Host copies of the assembly plan (tests)."""
        import numpy as np
        nb, no = self.n_blocks, self.n_occ
        be = np.zeros(nb + 1, np.int32)
        bo = np.zeros(nb + 1, np.int32)
        on = np.zeros(no, np.int32)
        oe = np.zeros(no + 1, np.int32)
        le = np.zeros(self.n_elems * (self.dim + 1), np.uint16)
        pm = np.zeros(self.n_elems, np.int32)
        torch.cuda.synchronize()
        L.check(L.load().pfem_plan_export(self.ref(), be.ctypes.data, bo.ctypes.data, on.ctypes.data,
                                          oe.ctypes.data, le.ctypes.data, pm.ctypes.data))
        return {"blk_elem": be, "blk_occ": bo, "occ_node": on, "occ_ent_ptr": oe, "loc_ent": le, "elem_perm": pm}

    def release(self):
        if getattr(self, "_m", None) is not None and self._m.plan:
            L.load().pfem_mesh_release(C.byref(self._m))

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


@dataclass
class Material:
    """pfem_material: per-element (or uniform, numel 1) parameter tensors."""
    model: str
    kind: str
    p0: torch.Tensor
    p1: torch.Tensor

    def c(self):
        m = L.pfem_material()
        m.model = MODELS[self.model]
        m.kind = KINDS[self.kind]
        m.p0, m.p1 = self.p0.data_ptr(), self.p1.data_ptr()
        m.stride0 = 0 if self.p0.numel() == 1 else 1
        m.stride1 = 0 if self.p1.numel() == 1 else 1
        return m


def _field(mesh: Mesh, t: torch.Tensor):
    if t.dtype != mesh.dtype:
        raise TypeError(f"field dtype {t.dtype} != mesh dtype {mesh.dtype}")
    _require_cuda(t)
    t = t.contiguous()
    if t.dim() == 2:
        t = t.unsqueeze(0)
    return t


def lame(kind: str, p0: torch.Tensor, p1: torch.Tensor, n: int):
    """pfem_lame: (mu, lambda) per element on the GPU."""
    _require_cuda(p0, p1)
    mu = torch.empty(n, dtype=p0.dtype, device=p0.device)
    lam = torch.empty_like(mu)
    L.check(L.load().pfem_lame(_DT[p0.dtype], KINDS[kind], n, _ptr(p0), 0 if p0.numel() == 1 else 1, _ptr(p1),
                               0 if p1.numel() == 1 else 1, _ptr(mu), _ptr(lam), _stream()))
    return mu, lam


def energy(mesh: Mesh, mat: Material, u: torch.Tensor, f_ext=None, elem_energy=False, residual=False,
           mode: str = "csr", flags=None, out=None):
    """pfem_energy: totals [S, K] (and W_e [S, E], residual [S, N, d] if requested)."""
    u = _field(mesh, u)
    S = u.shape[0]
    dev = u.device
    totals = torch.empty((S, mesh.n_parts), dtype=mesh.dtype, device=dev) if out is None else out[0]
    W = (torch.empty((S, mesh.n_elems), dtype=mesh.dtype, device=dev) if elem_energy else None)
    r = torch.empty_like(u) if residual else None
    if out is not None:
        W = out[1] if elem_energy else None
        r = out[2] if residual else None
    ws = mesh.workspace(S)
    mc = mat.c()
    L.check(L.load().pfem_energy(mesh.ref(), C.byref(mc), S, _ptr(u), u[0].numel(), _ptr(f_ext), _ptr(W),
                                 _ptr(totals), _ptr(r), MODES[mode], _ptr(flags), _ptr(ws), ws.numel(),
                                 _stream()))
    return totals, W, r


def pretrain_loss(mesh: Mesh, mat: Material, H: torch.Tensor, phi=None, f_ext=None, mode: str = "csr",
                  flags=None, out=None):
    """pfem_pretrain_loss: (loss [device double scalar], Pi totals [S, K], grad [S, N, d], u) of the
    energy loss through the ansatz u = phi (.) H (u is H itself when phi is None)."""
    H = _field(mesh, H)
    S = H.shape[0]
    dev = H.device
    if out is None:
        totals = torch.empty((S, mesh.n_parts), dtype=mesh.dtype, device=dev)
        grad = torch.empty_like(H)
        u = torch.empty_like(H) if phi is not None else None
        loss = torch.empty((), dtype=torch.float64, device=dev)
    else:
        loss, totals, grad, u = out
    ws = mesh.workspace(S)
    mc = mat.c()
    L.check(L.load().pfem_pretrain_loss(mesh.ref(), C.byref(mc), S, _ptr(H), H[0].numel(), _ptr(phi), _ptr(f_ext),
                                        _ptr(u), _ptr(totals), _ptr(grad), _ptr(loss), MODES[mode], _ptr(flags),
                                        _ptr(ws), ws.numel(), _stream()))
    return loss, totals, grad, (u if phi is not None else H)


def heat(mesh: Mesh, k: torch.Tensor, T: torch.Tensor, f=None, elem_energy=True, totals=True, flux=True,
         geometry_on_the_fly: bool = False):
    """pfem_heat: steady heat conduction on the prepared mesh.  T: [S, N] (or [N]); k: per element
    or numel 1.  Returns (W_e [S, E] or None, totals [S, K] or None, flux [S, N] or None)."""
    _require_cuda(T, k)
    if T.dtype != mesh.dtype or k.dtype != mesh.dtype or (f is not None and f.dtype != mesh.dtype):
        raise TypeError(f"heat: T, k and f must have the mesh dtype {mesh.dtype}")
    if k.numel() not in (1, mesh.n_elems):
        raise ValueError(f"heat: k must have 1 or n_elems = {mesh.n_elems} entries, got {k.numel()}")
    if T.numel() % mesh.n_nodes != 0:
        raise ValueError("heat: T must be [S, n_nodes] or [n_nodes]")
    if f is not None:
        if f.numel() != mesh.n_nodes:
            raise ValueError(f"heat: f must have n_nodes = {mesh.n_nodes} entries")
        _require_cuda(f)
        f = f.contiguous()
    k = k.contiguous()
    T = T.reshape(-1, mesh.n_nodes).contiguous()
    S = T.shape[0]
    dev = T.device
    W = torch.empty((S, mesh.n_elems), dtype=mesh.dtype, device=dev) if (elem_energy or totals) else None
    tot = torch.empty((S, mesh.n_parts), dtype=mesh.dtype, device=dev) if totals else None
    r = torch.empty_like(T) if flux else None
    nb = L.load().pfem_heat_workspace_bytes(mesh.ref(), S)
    ws = mesh._ws.get(("heat", S))
    if ws is None:
        ws = torch.zeros(max(nb, 1), dtype=torch.uint8, device=dev)   # zero-filled before first use
        mesh._ws[("heat", S)] = ws
    L.check(L.load().pfem_heat(mesh.ref(), _ptr(k), 0 if k.numel() == 1 else 1, S, _ptr(T), T.shape[1], _ptr(f),
                               _ptr(W), _ptr(tot), _ptr(r), 1 if geometry_on_the_fly else 0, _ptr(ws), ws.numel(),
                               _stream()))
    return W, tot, r


def residual(mesh: Mesh, mat: Material, u: torch.Tensor, mode: str = "csr", flags=None, out=None):
    """pfem_residual: internal force f_int(u) [S, N, d]."""
    u = _field(mesh, u)
    S = u.shape[0]
    r = torch.empty_like(u) if out is None else out
    ws = mesh.workspace(S)
    mc = mat.c()
    L.check(L.load().pfem_residual(mesh.ref(), C.byref(mc), S, _ptr(u), u[0].numel(), _ptr(r), MODES[mode],
                                   _ptr(flags), _ptr(ws), ws.numel(), _stream()))
    return r


def tangent_apply(mesh: Mesh, mat: Material, v: torch.Tensor, u=None, mask=None, mode: str = "csr",
                  flags=None, out=None):
    """pfem_tangent_apply: K(u) v [S, N, d]; with mask: (I-M) K (I-M) v + M v."""
    v = _field(mesh, v)
    S = v.shape[0]
    if u is not None:
        u = _field(mesh, u)
    Kv = torch.empty_like(v) if out is None else out
    ws = mesh.workspace(S)
    mc = mat.c()
    L.check(L.load().pfem_tangent_apply(mesh.ref(), C.byref(mc), S, _ptr(u), _ptr(v), _ptr(Kv), v[0].numel(),
                                        _ptr(mask), MODES[mode], _ptr(flags), _ptr(ws), ws.numel(), _stream()))
    return Kv


PRECONDS = {None: 0, "none": 0, "jacobi": 1}


def tangent_diag(mesh: Mesh, mat: Material, u_state=None, mask=None, out=None):
    """pfem_tangent_diag: diagonal [N][d] of the masked tangent (Jacobi preconditioner)."""
    if u_state is not None:
        u_state = _field(mesh, u_state)[0]
    if out is None:
        out = torch.empty((mesh.n_nodes, mesh.dim), dtype=mesh.dtype, device=mesh.coords.device)
    mc = mat.c()
    L.check(L.load().pfem_tangent_diag(mesh.ref(), C.byref(mc), _ptr(u_state), _ptr(out), _ptr(mask), _stream()))
    return out


def cg(mesh: Mesh, mat: Material, f: torch.Tensor, x0: torch.Tensor, mask=None, tol: float = 1e-8,
       max_iter: int = 50000, u_state=None, mode: str = "csr", history: bool = True, precond=None):
    """pfem_cg (precond None) / pfem_pcg (precond "jacobi"): warm-started CG; returns
    (x, report dict with history)."""
    f = _field(mesh, f)[0]
    x = _field(mesh, x0)[0].clone()
    if u_state is not None:
        u_state = _field(mesh, u_state)[0]
    hist = torch.zeros(max_iter + 1, dtype=torch.float64, device=x.device) if history else None
    rep = L.pfem_cg_report()
    ws = mesh.cg_workspace()
    mc = mat.c()
    if precond is None:
        st = L.load().pfem_cg(mesh.ref(), C.byref(mc), _ptr(u_state), _ptr(f), _ptr(mask), _ptr(x), tol,
                              max_iter, MODES[mode], _ptr(hist), C.byref(rep), _ptr(ws), ws.numel(), _stream())
    else:
        st = L.load().pfem_pcg(mesh.ref(), C.byref(mc), _ptr(u_state), _ptr(f), _ptr(mask), PRECONDS[precond],
                               _ptr(x), tol, max_iter, MODES[mode], _ptr(hist), C.byref(rep), _ptr(ws),
                               ws.numel(), _stream())
    report = {"status": st, "iterations": rep.iterations, "converged": bool(rep.converged),
              "rel_res0": rep.rel_res0, "rel_res_final": rep.rel_res_final,
              "true_rel_res_final": rep.true_rel_res_final, "bnorm": rep.bnorm,
              "history": None if hist is None else hist[: rep.iterations + 1].cpu().numpy()}
    if st not in (L.PFEM_OK, -4, -5):
        L.check(st)
    return x, report


def newton(mesh: Mesh, mat: Material, u0: torch.Tensor, f_ext=None, mask=None, tol: float = 1e-8,
           max_newton: int = 20, cg_tol: float = 1e-10, cg_max_iter: int = 50000, mode: str = "csr"):
    """pfem_newton: Newton-Raphson from u0 (constrained entries = prescribed values);
    returns (u, report dict with the residual-norm history)."""
    import numpy as np
    u = _field(mesh, u0)[0].clone()
    f = None if f_ext is None else _field(mesh, f_ext)[0]
    hist = np.zeros(max_newton + 1, np.float64)
    rep = L.pfem_newton_report()
    ws = mesh.newton_workspace()
    mc = mat.c()
    st = L.load().pfem_newton(mesh.ref(), C.byref(mc), _ptr(u), _ptr(f), _ptr(mask), tol, max_newton, cg_tol,
                              cg_max_iter, MODES[mode], hist.ctypes.data, C.byref(rep), _ptr(ws), ws.numel(),
                              _stream())
    report = {"status": st, "iterations": rep.iterations, "converged": bool(rep.converged),
              "exit": rep.status, "cg_iterations": rep.cg_iterations, "res0": rep.res0,
              "res_final": rep.res_final, "history": hist[: rep.iterations + 1].copy()}
    if st not in (L.PFEM_OK, -4, -5):
        L.check(st)
    return u, report


def launch_count(reset: bool = False) -> int:
    return int(L.load().pfem_launch_count(1 if reset else 0))


FMA_KINDS = {"ffma": 0, "ffma2": 1, "dfma": 2}


def fma_peak(kind: str = "ffma2", iters: int = 4096) -> float:
    """pfem_fma_peak: measured FMA-pipe peak of the current device in lane FMAs per second
    (kind: 'ffma' fp32, 'ffma2' fp32 packed pairs, 'dfma' fp64)."""
    out = C.c_double(0.0)
    L.check(L.load().pfem_fma_peak(FMA_KINDS[kind], int(iters), C.byref(out), _stream()))
    return float(out.value)
