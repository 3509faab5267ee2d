"""ctypes wrapper of the plain-C fp64 oracle (oracle/pfem_oracle.c).

TEST INFRASTRUCTURE ONLY — only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this module.  It shares no
code with the CUDA path.  Every function follows PAPER.md as cited in
pfem_oracle.c; numpy is used only for argument marshalling.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pfem_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, ERR_ARG, ERR_DEGENERATE, ERR_INVERTED, ERR_NOT_CONVERGED, ERR_BREAKDOWN, ERR_CAPACITY = \
    0, -1, -2, -3, -4, -5, -6
MODELS = {"linear": 0, "neohookean": 1}
PARAM_KINDS = {"lame": 0, "young_poisson": 1, "young_poisson_plane_stress": 2}


class OracleError(RuntimeError):
    def __init__(self, status, index, what):
        super().__init__(f"oracle {what}: status {status}, index {index}")
        self.status = status
        self.index = index


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2 -ffp-contract=off: no FMA contraction, plain)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = f"{_LIB}.{os.getpid()}.tmp"
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared",
               "-fPIC", "-std=c11", "-o", tmp, _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB)   # atomic: a process that has the old library mapped keeps it
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB)
        _lib.oracle_last_error_index.restype = C.c_int64
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _check(st, what):
    if st != OK:
        raise OracleError(st, lib().oracle_last_error_index(), what)


I64 = C.c_int64


def set_threads(n: int = 0):
    """OpenMP threads of the oracle (0 = all); results do not depend on it."""
    lib().oracle_set_threads(C.c_int(n))


def set_tangent_form(form: int = 0):
    """Association of the element tangent product: 0 = B^T (D (B v)), 1 = formed K_e then K_e v."""
    lib().oracle_set_tangent_form(C.c_int(form))


def dot(a, b, order: int = 0) -> float:
    """The CG dot product of the oracle under order 0 (ascending), 1 (descending), 2 (pairwise),
    3 (1024-blocked) or 4 (Kahan) — reading R18's orders."""
    a = _f64(a).ravel()
    b = _f64(b).ravel()
    f = lib().oracle_dot
    f.restype = C.c_double
    return float(f(C.c_int(order), I64(len(a)), _p(a), _p(b)))


def lame(kind: str, p0, p1, n: int):
    """(mu, lambda) per element from (E, nu) or (mu, lambda); uniform arrays of length 1 broadcast."""
    p0 = _f64(np.atleast_1d(p0))
    p1 = _f64(np.atleast_1d(p1))
    mu = np.empty(n)
    lam = np.empty(n)
    st = lib().oracle_lame(C.c_int(PARAM_KINDS[kind]), I64(n), _p(p0), I64(0 if len(p0) == 1 else 1),
                           _p(p1), I64(0 if len(p1) == 1 else 1), _p(mu), _p(lam))
    _check(st, "lame")
    return mu, lam


def geometry(coords, conn):
    """grad [E, d, d] (grad[e, a-1, j] = dN_a/dX_j, a = 1..d), vol [E], sign [E]."""
    coords = _f64(coords)
    conn = _i32(conn)
    N, d = coords.shape
    E = conn.shape[0]
    grad = np.zeros((E, d, d))
    vol = np.zeros(E)
    sign = np.zeros(E, np.int32)
    st = lib().oracle_geometry(C.c_int(d), I64(N), I64(E), _p(coords), _p(conn), _p(grad), _p(vol), _p(sign))
    _check(st, "geometry")
    return grad, vol, sign


def csr(conn, n_nodes: int):
    conn = _i32(conn)
    E, nv = conn.shape
    ptr = np.zeros(n_nodes + 1, np.int32)
    ent = np.zeros(E * nv, np.int32)
    _check(lib().oracle_csr(C.c_int(nv - 1), I64(n_nodes), I64(E), _p(conn), _p(ptr), _p(ent)), "csr")
    return ptr, ent


def colour(conn, n_nodes: int, ptr, ent, max_colours: int = 256):
    conn = _i32(conn)
    E, nv = conn.shape
    col = np.zeros(E, np.int32)
    nc = C.c_int32(0)
    st = lib().oracle_colour(C.c_int(nv - 1), I64(n_nodes), I64(E), _p(conn), _p(_i32(ptr)),
                             _p(_i32(ent)), _p(col), C.c_int32(max_colours), C.byref(nc))
    _check(st, "colour")
    return col, nc.value


def colour_sort(col, n_colours: int):
    col = _i32(col)
    elems = np.zeros(len(col), np.int32)
    cptr = np.zeros(n_colours + 1, np.int32)
    _check(lib().oracle_colour_sort(I64(len(col)), _p(col), C.c_int32(n_colours), _p(elems), _p(cptr)),
           "colour_sort")
    return elems, cptr


@dataclass
class Mesh:
    """Oracle-side prepared mesh (fp64 geometry + per-element Lame parameters)."""
    coords: np.ndarray
    conn: np.ndarray
    grad: np.ndarray
    vol: np.ndarray
    mu: np.ndarray
    lam: np.ndarray
    model: str
    part_elem: np.ndarray
    part_node: np.ndarray

    @property
    def dim(self):
        return self.coords.shape[1]

    @property
    def n_nodes(self):
        return self.coords.shape[0]

    @property
    def n_elems(self):
        return self.conn.shape[0]

    def _args(self):
        return (C.c_int(self.dim), I64(self.n_nodes), I64(self.n_elems), _p(self.conn),
                _p(self.grad), _p(self.vol), C.c_int(MODELS[self.model]), _p(self.mu), _p(self.lam))

    def energy(self, u, f_ext=None, want_elem=True):
        """(W_e [S, E] or None, totals [S, K])."""
        u = _f64(u).reshape(-1, self.n_nodes, self.dim)
        S = u.shape[0]
        K = len(self.part_elem) - 1
        W = np.zeros((S, self.n_elems)) if want_elem else None
        tot = np.zeros((S, K))
        fe = None if f_ext is None else _f64(f_ext)
        a = self._args()
        st = lib().oracle_energy(a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8],
                                 C.c_int(S), _p(u), C.c_int(K), _p(self.part_elem), _p(self.part_node),
                                 _p(fe), _p(W), _p(tot))
        _check(st, "energy")
        return W, tot

    def residual(self, u):
        """internal force f_int(u) [S, N, d]."""
        u = _f64(u).reshape(-1, self.n_nodes, self.dim)
        r = np.zeros_like(u)
        st = lib().oracle_residual(*self._args(), C.c_int(u.shape[0]), _p(u), _p(r))
        _check(st, "residual")
        return r

    def pretrain_loss(self, H, phi=None, f_ext=None):
        """Energy-based pretraining loss and its gradient w.r.t. the network output (SURVEY §8(f)
        row f2; P:518-541 linear, P:700-723 Neo-Hookean; reading R28):
            u = phi (.) H                                   (hard-BC ansatz u = (x/L) (.) H_theta)
            Pi_{s,k} = W_{s,k}(u) - f_ext . u               (discrete L of P:518-524 per sample / part)
            loss = mean over (s, k) of Pi_{s,k}             (batch mean, Eq. 2)
            dloss/dH = phi (.) (f_int(u) - f_ext) / (S K)   (chain rule; f_int = dW/du, App. B)
        H [S, N, d]; phi [N, d] or None (= 1); returns (loss, Pi [S, K], grad [S, N, d], u)."""
        H = _f64(H).reshape(-1, self.n_nodes, self.dim)
        ph = np.ones((self.n_nodes, self.dim)) if phi is None else _f64(phi).reshape(self.n_nodes, self.dim)
        fe = np.zeros((self.n_nodes, self.dim)) if f_ext is None else _f64(f_ext).reshape(self.n_nodes, self.dim)
        u = ph[None] * H
        _, Pi = self.energy(u, f_ext=fe, want_elem=False)
        S, K = Pi.shape
        loss = float(Pi.sum()) / (S * K)
        grad = ph[None] * (self.residual(u) - fe[None]) / (S * K)
        return loss, Pi, grad, u

    def heat(self, T, k, f=None):
        """Steady heat conduction: (W_e [S, E],
        totals [S, K] = sum W_e - f.T per part, r [S, N] = dW/dT).  k: per element or length 1."""
        T = _f64(T).reshape(-1, self.n_nodes)
        S = T.shape[0]
        K = len(self.part_elem) - 1
        k = _f64(np.atleast_1d(k))
        W = np.zeros((S, self.n_elems))
        tot = np.zeros((S, K))
        r = np.zeros((S, self.n_nodes))
        fe = None if f is None else _f64(f).reshape(self.n_nodes)
        st = lib().oracle_heat(C.c_int(self.dim), I64(self.n_nodes), I64(self.n_elems), _p(self.conn),
                               _p(self.grad), _p(self.vol), _p(k), I64(0 if len(k) == 1 else 1), C.c_int(S),
                               _p(T), C.c_int(K), _p(self.part_elem), _p(self.part_node), _p(fe), _p(W),
                               _p(tot), _p(r))
        _check(st, "heat")
        return W, tot, r

    def tangent(self, v, u=None, mask=None):
        """K(u) v  [S, N, d]; with mask: (I-M) K (I-M) v + M v."""
        v = _f64(v).reshape(-1, self.n_nodes, self.dim)
        uu = None if u is None else _f64(u).reshape(v.shape)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        out = np.zeros_like(v)
        st = lib().oracle_tangent(*self._args(), C.c_int(v.shape[0]), _p(uu), _p(v), _p(m), _p(out))
        _check(st, "tangent")
        return out

    def cg(self, f, mask, x0, tol=1e-8, max_iter=50000, u_state=None, history=True, dot_order=0):
        """Warm-started masked CG; returns (x, report dict).  dot_order 0/1/2 = ascending /
        descending / pairwise sums in the dot products (reading R18: the oracle's own spread)."""
        lib().oracle_set_dot_order(C.c_int(dot_order))
        x = _f64(x0).copy().reshape(-1)
        f = _f64(f).reshape(-1)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8).reshape(-1)
        us = None if u_state is None else _f64(u_state).reshape(-1)
        hist = np.zeros(max_iter + 1) if history else None
        it = C.c_int32(0)
        r0, rf, tr = C.c_double(0), C.c_double(0), C.c_double(0)
        st = lib().oracle_cg(*self._args(), _p(us), _p(f), _p(m), _p(x), C.c_double(tol),
                             C.c_int32(max_iter), _p(hist), C.byref(it), C.byref(r0), C.byref(rf),
                             C.byref(tr))
        rep = {"status": st, "iterations": it.value, "converged": st == OK, "rel_res0": r0.value,
               "rel_res_final": rf.value, "true_rel_res_final": tr.value,
               "history": None if hist is None else hist[: it.value + 1].copy()}
        lib().oracle_set_dot_order(C.c_int(0))
        return x.reshape(np.shape(x0)), rep

    def newton(self, u0, f_ext=None, mask=None, tol=1e-8, max_newton=20, cg_tol=1e-12, cg_max_iter=50000):
        """Newton-Raphson, App. B, one load step with dead loads (K^ext = 0):
            r(U_k) = f_int(U_k) - f_ext                      (free DOFs)
            stop when ||r|| <= tol                             (absolute 2-norm)
            dU = -(K^geo + K^mat)^{-1} r(U_k)                  (oracle masked CG, rel. tol cg_tol)
            U_{k+1} = U_k + dU
        Constrained DOFs keep their values from u0.  Returns (U, report with the history of
        ||r(U_k)||)."""
        u = _f64(u0).reshape(self.n_nodes, self.dim).copy()
        fe = np.zeros_like(u) if f_ext is None else _f64(f_ext).reshape(u.shape)
        free = np.ones(u.size, bool) if mask is None else np.asarray(mask).reshape(-1) == 0
        hist, cg_its, status = [], 0, 1
        for k in range(max_newton + 1):
            r = (self.residual(u)[0] - fe).reshape(-1)
            r[~free] = 0.0
            nr = float(np.sqrt(r @ r))
            hist.append(nr)
            if not np.isfinite(nr):
                status = 3
                break
            if nr <= tol:
                status = 0
                break
            if k == max_newton:
                break
            du, rep = self.cg(-r.reshape(u.shape), mask, np.zeros_like(u), tol=cg_tol, max_iter=cg_max_iter,
                              u_state=u if self.model == "neohookean" else None, history=False)
            cg_its += rep["iterations"]
            if rep["status"] == ERR_BREAKDOWN:
                status = 2
                break
            u = u + du.reshape(u.shape)
        return u, {"iterations": len(hist) - 1, "converged": status == 0, "exit": status, "history": np.array(hist),
                   "cg_iterations": cg_its}

    def tangent_diag(self, u=None, mask=None):
        """Diagonal of A = (I-M) K(u) (I-M) + M: textbook element tangents' diagonals assembled
        in ascending (e, a) order, 1 on constrained DOFs."""
        d = np.zeros(self.n_nodes * self.dim)
        us = None if u is None else _f64(u).reshape(-1)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8).reshape(-1)
        st = lib().oracle_tangent_diag(*self._args(), _p(us), _p(m), _p(d))
        _check(st, "tangent_diag")
        return d.reshape(self.n_nodes, self.dim)

    def pcg(self, f, mask, x0, tol=1e-8, max_iter=50000, u_state=None, precond=1, history=True, dot_order=0):
        """Jacobi-preconditioned CG (reading R27), same stop test as cg(); precond=0 is plain CG.
        dot_order as in cg() (reading R18)."""
        lib().oracle_set_dot_order(C.c_int(dot_order))
        x = _f64(x0).copy().reshape(-1)
        f = _f64(f).reshape(-1)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8).reshape(-1)
        us = None if u_state is None else _f64(u_state).reshape(-1)
        hist = np.zeros(max_iter + 1) if history else None
        it = C.c_int32(0)
        r0, rf, tr = C.c_double(0), C.c_double(0), C.c_double(0)
        st = lib().oracle_pcg(*self._args(), _p(us), _p(f), _p(m), C.c_int(precond), _p(x), C.c_double(tol),
                              C.c_int32(max_iter), _p(hist), C.byref(it), C.byref(r0), C.byref(rf),
                              C.byref(tr))
        rep = {"status": st, "iterations": it.value, "converged": st == OK, "rel_res0": r0.value,
               "rel_res_final": rf.value, "true_rel_res_final": tr.value,
               "history": None if hist is None else hist[: it.value + 1].copy()}
        lib().oracle_set_dot_order(C.c_int(0))
        return x.reshape(np.shape(x0)), rep

    def pcg_spread(self, f, mask, x0, tol=1e-8, max_iter=50000, u_state=None, forms=(0, 1)):
        """Iteration counts of the oracle Jacobi PCG under the five dot-product orders and both
        tangent associations (R18)."""
        out = []
        for form in forms:
            set_tangent_form(form)
            out += [self.pcg(f, mask, x0, tol, max_iter, u_state, history=False, dot_order=o)[1]["iterations"]
                    for o in (0, 1, 2, 3, 4)]
        set_tangent_form(0)
        return out

    def cg_spread(self, f, mask, x0, tol=1e-8, max_iter=50000, u_state=None, forms=(0, 1)):
        """Iteration counts of the oracle CG under the five dot-product orders and both
        associations of the element tangent product (reading R18: valid re-orderings)."""
        out = []
        for form in forms:
            set_tangent_form(form)
            out += [self.cg(f, mask, x0, tol, max_iter, u_state, history=False, dot_order=o)[1]["iterations"]
                    for o in (0, 1, 2, 3, 4)]
        set_tangent_form(0)
        return out


def prepare(coords, conn, model: str, param_kind: str, p0, p1, part_elem=None, part_node=None) -> Mesh:
    coords = _f64(coords)
    conn = _i32(conn)
    grad, vol, _ = geometry(coords, conn)
    mu, lam = lame(param_kind, p0, p1, conn.shape[0])
    pe = _i32(part_elem if part_elem is not None else [0, conn.shape[0]])
    pn = _i32(part_node if part_node is not None else [0, coords.shape[0]])
    return Mesh(coords, conn, grad, vol, mu, lam, model, pe, pn)


def prepare_problem(prob) -> Mesh:
    """Oracle mesh for a pfem_gen.Problem."""
    pe, pn = prob.parts()
    return prepare(prob.coords, prob.conn, prob.model, prob.param_kind, prob.p0, prob.p1, pe, pn)


# ------------------------------------------------------------------ quadrilaterals (§8(f) row f4)
QUAD_TYPES = {"q4": 1, "q8": 2}


def quad_shape(kind: str, xi: float, eta: float):
    """Shape functions N [nv] and reference derivatives dN [nv, 2] of a Q4 / Q8 element."""
    nv = 4 if kind == "q4" else 8
    N = np.zeros(nv)
    dN = np.zeros((nv, 2))
    _check(lib().oracle_quad_shape(C.c_int(QUAD_TYPES[kind]), C.c_double(xi), C.c_double(eta), _p(N), _p(dN)),
           "quad_shape")
    return N, dN


def quad_rule(kind: str):
    """Gauss points [nq, 2] and weights [nq] (2 x 2 for Q4, 3 x 3 for Q8)."""
    pts = np.zeros((9, 2))
    w = np.zeros(9)
    n = lib().oracle_quad_rule(C.c_int(QUAD_TYPES[kind]), _p(pts), _p(w))
    return pts[:n].copy(), w[:n].copy()


@dataclass
class QuadMesh:
    """Oracle-side Q4 / Q8 mesh (2-D, plane strain): geometry is formed per quadrature point."""
    kind: str
    coords: np.ndarray
    conn: np.ndarray
    mu: np.ndarray
    lam: np.ndarray
    model: str
    part_elem: np.ndarray
    part_node: np.ndarray

    dim = 2

    @property
    def n_nodes(self):
        return self.coords.shape[0]

    @property
    def n_elems(self):
        return self.conn.shape[0]

    def _args(self):
        return (C.c_int(QUAD_TYPES[self.kind]), I64(self.n_nodes), I64(self.n_elems), _p(self.coords),
                _p(self.conn), C.c_int(MODELS[self.model]), _p(self.mu), _p(self.lam))

    def energy(self, u, f_ext=None, want_elem=True):
        u = _f64(u).reshape(-1, self.n_nodes, 2)
        S = u.shape[0]
        K = len(self.part_elem) - 1
        W = np.zeros((S, self.n_elems)) if want_elem else None
        tot = np.zeros((S, K))
        fe = None if f_ext is None else _f64(f_ext)
        st = lib().oracle_quad_energy(*self._args(), C.c_int(S), _p(u), C.c_int(K), _p(self.part_elem),
                                      _p(self.part_node), _p(fe), _p(W), _p(tot))
        _check(st, "quad energy")
        return W, tot

    def residual(self, u):
        u = _f64(u).reshape(-1, self.n_nodes, 2)
        r = np.zeros_like(u)
        _check(lib().oracle_quad_residual(*self._args(), C.c_int(u.shape[0]), _p(u), _p(r)), "quad residual")
        return r

    def tangent(self, v, u=None, mask=None):
        v = _f64(v).reshape(-1, self.n_nodes, 2)
        uu = None if u is None else _f64(u).reshape(v.shape)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        out = np.zeros_like(v)
        _check(lib().oracle_quad_tangent(*self._args(), C.c_int(v.shape[0]), _p(uu), _p(v), _p(m), _p(out)),
               "quad tangent")
        return out

    def cg(self, f, mask, x0, tol=1e-8, max_iter=50000, u_state=None, history=True, dot_order=0):
        lib().oracle_set_dot_order(C.c_int(dot_order))
        x = _f64(x0).copy().reshape(-1)
        f = _f64(f).reshape(-1)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8).reshape(-1)
        us = None if u_state is None else _f64(u_state).reshape(-1)
        hist = np.zeros(max_iter + 1) if history else None
        it = C.c_int32(0)
        r0, rf, tr = C.c_double(0), C.c_double(0), C.c_double(0)
        st = lib().oracle_quad_cg(*self._args(), _p(us), _p(f), _p(m), _p(x), C.c_double(tol), C.c_int32(max_iter),
                                  _p(hist), C.byref(it), C.byref(r0), C.byref(rf), C.byref(tr))
        lib().oracle_set_dot_order(C.c_int(0))
        rep = {"status": st, "iterations": it.value, "converged": st == OK, "rel_res0": r0.value,
               "rel_res_final": rf.value, "true_rel_res_final": tr.value,
               "history": None if hist is None else hist[: it.value + 1].copy()}
        return x.reshape(np.shape(x0)), rep

    newton = Mesh.newton


def prepare_quad(kind: str, coords, conn, model: str, param_kind: str, p0, p1, part_elem=None,
                 part_node=None) -> QuadMesh:
    coords = _f64(coords)
    conn = _i32(conn)
    md = C.c_double(0)
    _check(lib().oracle_quad_check(C.c_int(QUAD_TYPES[kind]), I64(len(coords)), I64(len(conn)), _p(coords),
                                   _p(conn), C.byref(md)), "quad check")
    mu, lam = lame(param_kind, p0, p1, conn.shape[0])
    pe = _i32(part_elem if part_elem is not None else [0, conn.shape[0]])
    pn = _i32(part_node if part_node is not None else [0, coords.shape[0]])
    return QuadMesh(kind, coords, conn, mu, lam, model, pe, pn)
