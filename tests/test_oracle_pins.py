"""Pins of the CPU oracle to what the paper and the mathematics fix (no GPU).

Each test names the passage it follows.  The pins are chosen so that a plausible
mistake (dropped term, wrong sign/index, transposed operand, wrong Lame constant)
fails at least one of them:

* single-element hand-derived values (tests/golden/single_element.json) fix the
  constitutive constants and the force formula;
* affine patch tests fix geometry + integration (discrete W = psi(A) |Omega|);
* central finite differences tie the residual to the energy and the tangent to
  the residual (catches transposes / sign errors in P, S, C^SE, B0, G0);
* NH(eps A) - linear(eps A) = O(eps^3) ties Neo-Hookean to linear elasticity;
* brute force (CSR, colouring, dense Cholesky vs CG) on tiny meshes.
"""
import json
import os

import numpy as np
import pytest

from pfem_gen import config1, kuhn_cube, plate_with_holes, square_t3

GOLD = os.path.join(os.path.dirname(__file__), "golden", "single_element.json")


@pytest.fixture(scope="module")
def gold():
    with open(GOLD) as f:
        return json.load(f)


def rel(a, b):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def jittered_square(n, seed, jit=0.25):
    coords, conn = square_t3(n, n)
    rng = np.random.default_rng(seed)
    h = 1.0 / (n - 1)
    inner = (coords[:, 0] > 0) & (coords[:, 0] < 1) & (coords[:, 1] > 0) & (coords[:, 1] < 1)
    coords = coords + rng.uniform(-jit * h, jit * h, coords.shape) * inner[:, None]
    return coords, conn


def jittered_cube(n, seed, jit=0.15):
    coords, conn = kuhn_cube(n)
    rng = np.random.default_rng(seed)
    h = 1.0 / (n - 1)
    inner = np.all((coords > 0) & (coords < 1), axis=1)
    coords = coords + rng.uniform(-jit * h, jit * h, coords.shape) * inner[:, None]
    return coords, conn


MESHES = {
    "t3": lambda: jittered_square(5, 11),
    "t4": lambda: jittered_cube(4, 12),
}


# ---------------------------------------------------------------- material
def test_lame_pins(orc, gold):
    """P:729-730 (and SPEC S:344): lam = nu E/((1+nu)(1-2nu)), mu = E/(2(1+nu))."""
    for E, nu, lam_ref, mu_ref in gold["lame"]["cases"]:
        mu, lam = orc.lame("young_poisson", [E], [nu], 1)
        assert abs(mu[0] - mu_ref) <= 1e-15 * mu_ref and abs(lam[0] - lam_ref) <= 1e-15 * lam_ref
    mu, lam = orc.lame("young_poisson_plane_stress", [1.0], [0.3], 1)
    assert abs(lam[0] - gold["lame"]["plane_stress_lam_E1_nu03"]) < 1e-15
    # plane stress lam* = nu E/(1-nu^2) (textbook identity, independent form)
    assert abs(lam[0] - 0.3 / (1 - 0.09)) < 1e-15
    mu, lam = orc.lame("lame", [0.4], [0.6], 3)
    assert np.all(mu == 0.4) and np.all(lam == 0.6)


# ---------------------------------------------------------------- geometry
def test_geometry_reference_triangle_and_tet(orc):
    """grad N of the reference simplex are the unit vectors (barycentric coordinates)."""
    g, v, s = orc.geometry(np.array([[0., 0], [1, 0], [0, 1]]), np.array([[0, 1, 2]]))
    assert np.allclose(g[0], np.eye(2), atol=0, rtol=0) and v[0] == 0.5 and s[0] == 1
    g, v, s = orc.geometry(np.array([[0., 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]]), np.array([[0, 1, 2, 3]]))
    assert np.array_equal(g[0], np.eye(3)) and abs(v[0] - 1 / 6) < 1e-17
    # reversed orientation: same volume, negative sign, gradients still reproduce linear fields
    g, v, s = orc.geometry(np.array([[0., 0], [0, 1], [1, 0]]), np.array([[0, 1, 2]]))
    assert v[0] == 0.5 and s[0] == -1


@pytest.mark.parametrize("kind", ["t3", "t4"])
def test_geometry_identities(orc, kind):
    """sum_a X_a (x) grad N_a = I and sum_e V_e = |Omega| = 1 (unit square / cube)."""
    coords, conn = MESHES[kind]()
    g, v, _ = orc.geometry(coords, conn)
    d = coords.shape[1]
    g0 = -g.sum(axis=1)                                      # grad N_0
    X = coords[conn]                                          # [E, d+1, d]
    I = np.einsum("ei,ej->eij", X[:, 0], g0) + np.einsum("eai,eaj->eij", X[:, 1:], g)
    assert np.max(np.abs(I - np.eye(d))) < 1e-13
    assert abs(v.sum() - 1.0) < 1e-13


def test_geometry_regular_grid_volumes(orc):
    """Regular grids: V = h^2/2 (T3), h^3/6 (T4)."""
    c, t = square_t3(6, 6)
    _, v, _ = orc.geometry(c, t)
    assert np.allclose(v, 0.5 / 25, rtol=1e-14)
    c, t = kuhn_cube(4)
    _, v, s = orc.geometry(c, t)
    assert np.allclose(v, 1 / 27 / 6, rtol=1e-13) and np.all(s == 1)


def test_geometry_degenerate(orc):
    """Collinear triangle -> PFEM degenerate error with the element index."""
    coords = np.array([[0., 0], [1, 0], [0, 1], [2, 0]])
    with pytest.raises(orc.OracleError) as ei:
        orc.geometry(coords, np.array([[0, 1, 2], [0, 1, 3]]))
    assert ei.value.status == orc.ERR_DEGENERATE and ei.value.index == 1


# ---------------------------------------------------------------- CSR / colouring
def brute_csr(conn, n):
    nv = conn.shape[1]
    rows = [[] for _ in range(n)]
    for e in range(conn.shape[0]):
        for a in range(nv):
            rows[conn[e, a]].append(e * nv + a)
    ptr = np.cumsum([0] + [len(r) for r in rows])
    return ptr, np.array([x for r in rows for x in sorted(r)], dtype=np.int64)


def brute_greedy(conn):
    E = conn.shape[0]
    col = -np.ones(E, int)
    sets = [set(c) for c in conn.tolist()]
    for e in range(E):
        used = {col[f] for f in range(e) if sets[e] & sets[f]}
        c = 0
        while c in used:
            c += 1
        col[e] = c
    return col


@pytest.mark.parametrize("kind", ["t3", "t4", "plate"])
def test_csr_and_colouring_brute_force(orc, kind):
    if kind == "plate":
        coords, conn, _ = plate_with_holes(14, np.random.default_rng(5), r_range=(0.1, 0.2))
    else:
        coords, conn = MESHES[kind]()
    n = coords.shape[0]
    ptr, ent = orc.csr(conn, n)
    bp, be = brute_csr(conn, n)
    assert np.array_equal(ptr, bp) and np.array_equal(ent, be)
    assert ptr[-1] == conn.size
    col, nc = orc.colour(conn, n, ptr, ent)
    assert np.array_equal(col, brute_greedy(conn))
    # proper colouring: no node shared within a colour
    for c in range(nc):
        nodes = conn[col == c].ravel()
        assert len(nodes) == len(np.unique(nodes))
    # n_colours <= max element degree + 1
    nv = conn.shape[1]
    deg = max(len(set().union(*[set((ent[ptr[v]:ptr[v + 1]] // nv).tolist()) for v in conn[e]]) - {e})
              for e in range(conn.shape[0]))
    assert nc <= deg + 1
    elems, cptr = orc.colour_sort(col, nc)
    order = np.lexsort((np.arange(len(col)), col))
    assert np.array_equal(elems, order) and cptr[-1] == len(col)


# ---------------------------------------------------------------- single elements
def test_single_element_linear(orc, gold):
    g = gold["t3_linear"]
    m = orc.prepare(np.array(g["coords"], float), np.array(g["conn"]), "linear", "young_poisson",
                    [g["E"]], [g["nu"]])
    u = np.array(g["u"], float)[None]
    W, tot = m.energy(u)
    assert abs(W[0, 0] - g["W"]) < 1e-15 * g["W"] and abs(tot[0, 0] - g["W"]) < 1e-15 * g["W"]
    r = m.residual(u)[0]
    assert np.max(np.abs(r - np.array(g["f"]))) < 1e-15


def test_single_element_neohookean(orc, gold):
    for key, d in (("t3_neohookean", 2), ("t4_neohookean", 3)):
        g = gold[key]
        m = orc.prepare(np.array(g["coords"], float), np.array(g["conn"]), "neohookean", "lame",
                        [g["mu"]], [g["lam"]])
        u = np.array(g["u"], float)[None]
        W, _ = m.energy(u)
        assert abs(W[0, 0] - g["W"]) < 1e-13 * g["W"], key
        r = m.residual(u)[0]
        assert np.max(np.abs(r[1] - np.array(g["f1"]))) < 1e-14, key
        if "f2" in g:
            assert np.max(np.abs(r[2] - np.array(g["f2"]))) < 1e-14


# ---------------------------------------------------------------- energy
def psi_lin(A, mu, lam):
    """mu eps:eps + lam/2 tr(eps)^2 (same law as P:527-536, written in Lame form)."""
    eps = 0.5 * (A + A.T)
    return mu * np.sum(eps * eps) + 0.5 * lam * np.trace(eps) ** 2


def psi_nh(F, mu, lam):
    d = F.shape[0]
    J = np.linalg.det(F)
    return 0.5 * lam * np.log(J) ** 2 - mu * np.log(J) + 0.5 * mu * (np.sum(F * F) - d)


@pytest.mark.parametrize("kind", ["t3", "t4"])
@pytest.mark.parametrize("model", ["linear", "neohookean"])
def test_energy_affine_patch(orc, kind, model):
    """Affine u = A X + c => grad u = A on every element => W_total = psi(A) |Omega|
    (classical patch test; exact for P1)."""
    coords, conn = MESHES[kind]()
    d = coords.shape[1]
    rng = np.random.default_rng(3)
    A = 0.05 * rng.standard_normal((d, d))
    u = coords @ A.T + rng.standard_normal(d)
    m = orc.prepare(coords, conn, model, "lame", [0.4], [0.6])
    W, tot = m.energy(u[None])
    ref = (psi_lin(A, 0.4, 0.6) if model == "linear" else psi_nh(np.eye(d) + A, 0.4, 0.6))
    assert abs(tot[0, 0] - ref) < 1e-13 * abs(ref)
    _, vol, _ = orc.geometry(coords, conn)
    assert np.max(np.abs(W[0] - ref * vol)) < 1e-13 * abs(ref) * vol.max()


@pytest.mark.parametrize("kind", ["t3", "t4"])
def test_energy_rigid_motions(orc, kind):
    """Translation: W = 0, r = 0 (both models).  Linear + infinitesimal rotation (skew A):
    eps = 0.  NH + finite rotation R: psi = 0, P = 0 (frame indifference)."""
    coords, conn = MESHES[kind]()
    d = coords.shape[1]
    c = np.arange(1, d + 1) * 0.3
    for model in ("linear", "neohookean"):
        m = orc.prepare(coords, conn, model, "lame", [0.4], [0.6])
        u = np.tile(c, (len(coords), 1))[None]
        W, tot = m.energy(u)
        assert np.max(np.abs(W)) < 1e-28 if model == "linear" else np.max(np.abs(W)) < 1e-15
        assert np.max(np.abs(m.residual(u))) < 1e-14
    skew = np.zeros((d, d))
    skew[0, 1], skew[1, 0] = 0.02, -0.02
    m = orc.prepare(coords, conn, "linear", "lame", [0.4], [0.6])
    W, _ = m.energy((coords @ skew.T)[None])
    assert np.max(np.abs(W)) < 1e-30
    assert np.max(np.abs(m.residual((coords @ skew.T)[None]))) < 1e-14
    th = 0.7
    R = np.eye(d)
    R[0, 0], R[0, 1], R[1, 0], R[1, 1] = np.cos(th), -np.sin(th), np.sin(th), np.cos(th)
    m = orc.prepare(coords, conn, "neohookean", "lame", [0.4], [0.6])
    u = (coords @ (R - np.eye(d)).T)[None]
    W, _ = m.energy(u)
    assert np.max(np.abs(W)) < 1e-14
    assert np.max(np.abs(m.residual(u))) < 1e-13


def test_energy_sign_and_small_strain_limit(orc):
    """W_e >= 0; |W_NH(eps A) - W_lin(eps A)| / eps^3 bounded as eps -> 0 (NH linearises to
    the linear law with the same Lame constants, P:709-732 vs P:527-536)."""
    coords, conn = MESHES["t4"]()
    rng = np.random.default_rng(7)
    field = rng.standard_normal(coords.shape)
    lin = orc.prepare(coords, conn, "linear", "lame", [0.4], [0.6])
    nh = orc.prepare(coords, conn, "neohookean", "lame", [0.4], [0.6])
    ratios = []
    for eps in (1e-3, 5e-4, 2.5e-4):
        Wl, tl = lin.energy(eps * field[None])
        Wn, tn = nh.energy(eps * field[None])
        assert Wl.min() >= 0 and Wn.min() >= -1e-18
        ratios.append(abs(tn[0, 0] - tl[0, 0]) / eps ** 3)
        assert abs(tn[0, 0] - tl[0, 0]) < 0.05 * tl[0, 0]
    # (W_NH - W_lin)/eps^3 converges to a constant (3rd-order term); an O(eps^2) mismatch
    # (wrong constant) would make it grow like 1/eps
    assert abs(ratios[-1] - ratios[-2]) < 0.1 * abs(ratios[-1])
    assert abs(ratios[-1]) < 4 * abs(ratios[0]) + 1e-12


def test_energy_parts_and_potential(orc):
    """Per-part totals and Pi = W - f_ext.u: two disjoint copies of a mesh in
    two parts have identical W; with f_ext the totals drop by f.u."""
    c1, t1 = MESHES["t3"]()
    coords = np.concatenate([c1, c1 + 2.0])
    conn = np.concatenate([t1, t1 + len(c1)])
    pe = np.array([0, len(t1), 2 * len(t1)])
    pn = np.array([0, len(c1), 2 * len(c1)])
    m = orc.prepare(coords, conn, "linear", "young_poisson", [1.0], [0.3], pe, pn)
    rng = np.random.default_rng(1)
    u1 = 0.01 * rng.standard_normal(c1.shape)
    u = np.concatenate([u1, u1])[None]
    _, tot = m.energy(u)
    assert abs(tot[0, 0] - tot[0, 1]) < 1e-18
    f = rng.standard_normal(coords.shape)
    _, tot2 = m.energy(u, f_ext=f)
    assert abs(tot[0, 0] - tot2[0, 0] - np.sum(f[:len(c1)] * u1)) < 1e-14
    assert abs(tot[0, 1] - tot2[0, 1] - np.sum(f[len(c1):] * u1)) < 1e-14


def test_energy_inversion_reported(orc):
    """NH with J <= 0: element inversion error with the element id."""
    coords = np.array([[0., 0], [1, 0], [0, 1], [1, 1]])
    conn = np.array([[0, 1, 2], [1, 3, 2]])
    m = orc.prepare(coords, conn, "neohookean", "lame", [0.4], [0.6])
    u = np.zeros((1, 4, 2))
    u[0, 3] = [-1.5, -1.5]            # node 3 pushed across edge 1-2: element 1 inverts
    with pytest.raises(orc.OracleError) as ei:
        m.energy(u)
    assert ei.value.status == orc.ERR_INVERTED and ei.value.index == 1


# ---------------------------------------------------------------- residual
@pytest.mark.parametrize("kind", ["t3", "t4"])
@pytest.mark.parametrize("model", ["linear", "neohookean"])
def test_residual_is_energy_gradient(orc, kind, model):
    """f_int = dW/du (P:1083-1096 derived from the energy of P:518-536 / P:700-722):
    central finite difference per DOF; residuals sum to zero; linear u.r = 2W."""
    coords, conn = MESHES[kind]()
    rng = np.random.default_rng(2)
    u = 0.05 * rng.standard_normal(coords.shape)
    m = orc.prepare(coords, conn, model, "lame", [0.4], [0.6])
    r = m.residual(u[None])[0]
    assert np.max(np.abs(r.sum(axis=0))) < 1e-14
    h = 1e-6
    fd = np.zeros_like(u)
    for n in range(u.shape[0]):
        for i in range(u.shape[1]):
            up, um = u.copy(), u.copy()
            up[n, i] += h
            um[n, i] -= h
            fd[n, i] = (m.energy(up[None], want_elem=False)[1][0, 0]
                        - m.energy(um[None], want_elem=False)[1][0, 0]) / (2 * h)
    assert rel(fd, r) < 1e-8
    if model == "linear":
        W = m.energy(u[None])[1][0, 0]
        assert abs(np.sum(u * r) - 2 * W) < 1e-13 * W


@pytest.mark.parametrize("kind", ["t3", "t4"])
@pytest.mark.parametrize("model", ["linear", "neohookean"])
def test_residual_affine_patch(orc, kind, model):
    """Constant stress => interior nodal forces vanish; boundary nodes carry
    sum over boundary facets of P n |f| / d (classical patch test)."""
    coords, conn = MESHES[kind]()
    d = coords.shape[1]
    A = 0.04 * np.random.default_rng(9).standard_normal((d, d))
    m = orc.prepare(coords, conn, model, "lame", [0.4], [0.6])
    r = m.residual((coords @ A.T)[None])[0]
    F = np.eye(d) + A
    if model == "linear":
        eps = 0.5 * (A + A.T)
        P = 2 * 0.4 * eps + 0.6 * np.trace(eps) * np.eye(d)
    else:
        Fi = np.linalg.inv(F).T
        P = 0.4 * (F - Fi) + 0.6 * np.log(np.linalg.det(F)) * Fi
    expect = np.zeros_like(coords)
    # boundary facets of the box [0,1]^d: outward normal +-e_k
    from pfem_gen import boundary_faces_on_plane
    for k in range(d):
        for val, sgn in ((0.0, -1.0), (1.0, 1.0)):
            fac = boundary_faces_on_plane(conn, coords, k, val)
            p = coords[fac]
            if d == 2:
                meas = np.linalg.norm(p[:, 1] - p[:, 0], axis=1)
            else:
                meas = 0.5 * np.linalg.norm(np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), axis=1)
            nvec = np.zeros(d)
            nvec[k] = sgn
            t = P @ nvec
            for a in range(d):
                np.add.at(expect, fac[:, a], (meas / d)[:, None] * t[None, :])
    assert np.max(np.abs(r - expect)) < 1e-13 * np.max(np.abs(expect))


# ---------------------------------------------------------------- tangent
@pytest.mark.parametrize("kind", ["t3", "t4"])
def test_tangent_linear_equals_residual_and_symmetric(orc, kind):
    """Linear: K v = f_int(v) (f_int linear in u); v.Kw = w.Kv; K.translation = 0;
    K.(infinitesimal rotation) = 0."""
    coords, conn = MESHES[kind]()
    d = coords.shape[1]
    m = orc.prepare(coords, conn, "linear", "young_poisson", [1.0], [0.3])
    rng = np.random.default_rng(4)
    v = rng.standard_normal((2,) + coords.shape)
    Kv = m.tangent(v)
    assert rel(Kv, m.residual(v)) < 1e-14
    assert abs(np.sum(v[0] * Kv[1]) - np.sum(v[1] * Kv[0])) < 1e-13 * np.abs(Kv).max()
    t = np.tile(np.arange(1.0, d + 1), (len(coords), 1))
    assert np.max(np.abs(m.tangent(t[None]))) < 1e-13
    skew = np.zeros((d, d))
    skew[0, 1], skew[1, 0] = 1.0, -1.0
    assert np.max(np.abs(m.tangent((coords @ skew.T)[None]))) < 1e-13


@pytest.mark.parametrize("kind", ["t3", "t4"])
def test_tangent_nh_finite_difference(orc, kind):
    """NH: K(u) v = d/dt f_int(u + t v) (P:1104-1115 consistent linearisation): central FD;
    K(0) = K_linear; symmetric; K_geo(0)=0 is implied by K(0)=K_lin."""
    coords, conn = MESHES[kind]()
    rng = np.random.default_rng(5)
    u = 0.05 * rng.standard_normal(coords.shape)
    v = rng.standard_normal(coords.shape)
    w = rng.standard_normal(coords.shape)
    m = orc.prepare(coords, conn, "neohookean", "lame", [0.4], [0.6])
    Kv = m.tangent(v[None], u=u[None])[0]
    h = 1e-6
    fd = (m.residual((u + h * v)[None])[0] - m.residual((u - h * v)[None])[0]) / (2 * h)
    assert rel(fd, Kv) < 1e-8
    Kw = m.tangent(w[None], u=u[None])[0]
    assert abs(np.sum(w * Kv) - np.sum(v * Kw)) < 1e-12 * np.abs(Kv).max()
    lin = orc.prepare(coords, conn, "linear", "lame", [0.4], [0.6])
    K0 = m.tangent(v[None], u=np.zeros_like(u)[None])
    assert rel(K0, lin.tangent(v[None])) < 1e-14


def test_tangent_mask(orc):
    """(I-M) K (I-M) v + M v (reading R9)."""
    p = config1()
    m = orc.prepare_problem(p)
    rng = np.random.default_rng(6)
    v = rng.standard_normal((1, p.n_nodes, 2))
    mask = p.mask.reshape(p.n_nodes, 2)
    vf = v * (1 - mask)
    ref = m.tangent(vf) * (1 - mask) + v * mask
    assert rel(m.tangent(v, mask=p.mask), ref) < 1e-15


# ---------------------------------------------------------------- CG
def dense_K(m, n_dof, mask=None):
    K = np.zeros((n_dof, n_dof))
    for i in range(n_dof):
        e = np.zeros(n_dof)
        e[i] = 1.0
        K[:, i] = m.tangent(e.reshape(1, m.n_nodes, m.dim), mask=mask).ravel()
    return K


def test_cg_matches_dense_cholesky(orc):
    """Config 1 (tiny): dense K from columns K e_i + Cholesky vs CG at tol 1e-12
     -> rel error <= 1e-9; also SPD of the masked operator."""
    p = config1()
    m = orc.prepare_problem(p)
    n = p.n_nodes * 2
    A = dense_K(m, n, mask=p.mask)
    assert np.max(np.abs(A - A.T)) < 1e-14
    L = np.linalg.cholesky(A)
    b = p.f_ext.ravel() * (1 - p.mask)
    x_ref = np.linalg.solve(L.T, np.linalg.solve(L, b))
    x, rep = m.cg(p.f_ext, p.mask, np.zeros(n), tol=1e-12)
    assert rep["converged"] and rep["iterations"] > 10
    assert rel(x, x_ref) < 1e-9
    assert rep["true_rel_res_final"] < 1e-11
    # exact initial guess: skip rule -> 0 iterations
    x2, rep2 = m.cg(p.f_ext, p.mask, x_ref, tol=1e-8)
    assert rep2["iterations"] == 0 and rep2["converged"]


def test_cg_patch_test_affine_dirichlet(orc):
    """Affine Dirichlet data on the whole boundary, f = 0 => the discrete solution is the
    affine field at every interior node (classical patch test)."""
    coords, conn = MESHES["t3"]()
    A = np.array([[0.01, 0.02], [-0.03, 0.005]])
    exact = coords @ A.T
    bnd = (coords[:, 0] < 1e-12) | (coords[:, 0] > 1 - 1e-12) | (coords[:, 1] < 1e-12) | (coords[:, 1] > 1 - 1e-12)
    mask = np.repeat(bnd, 2).astype(np.uint8)
    x0 = np.where(np.repeat(bnd, 2), exact.ravel(), 0.0)
    m = orc.prepare(coords, conn, "linear", "young_poisson", [1.0], [0.3])
    x, rep = m.cg(np.zeros_like(coords), mask, x0, tol=1e-13)
    assert rep["converged"]
    assert np.max(np.abs(x.ravel() - exact.ravel())) < 1e-12


def test_cg_a_norm_error_monotone_and_warm_start(orc):
    """A-norm error is non-increasing along CG iterates; a perturbed-exact warm
    start needs fewer iterations than a zero start at a loose tolerance."""
    p = config1()
    m = orc.prepare_problem(p)
    n = p.n_nodes * 2
    A = dense_K(m, n, mask=p.mask)
    b = p.f_ext.ravel() * (1 - p.mask)
    xs = np.linalg.solve(A, b)
    errs = []
    for k in range(1, 40):
        x, rep = m.cg(p.f_ext, p.mask, np.zeros(n), tol=1e-30, max_iter=k, history=False)
        e = x.ravel() - xs
        errs.append(e @ A @ e)
    assert all(errs[i + 1] <= errs[i] * (1 + 1e-12) for i in range(len(errs) - 1))
    _, rz = m.cg(p.f_ext, p.mask, np.zeros(n), tol=1e-3)
    from pfem_gen import warm_start
    x0 = warm_start(xs.reshape(-1, 2), p.mask, seed=1004)
    _, rw = m.cg(p.f_ext, p.mask, x0, tol=1e-3)
    assert rw["iterations"] < rz["iterations"]


def test_cg_history_and_breakdown_conventions(orc):
    """History[0] = initial relative residual; each history entry < tol only at the end;
    iteration count = number of A p products (reading R11)."""
    p = config1()
    m = orc.prepare_problem(p)
    x, rep = m.cg(p.f_ext, p.mask, np.zeros(p.n_nodes * 2), tol=1e-6)
    h = rep["history"]
    assert len(h) == rep["iterations"] + 1
    assert abs(h[0] - 1.0) < 1e-15                      # zero start: r0 = b
    assert h[-1] < 1e-6 and np.all(h[:-1] >= 1e-6)


@pytest.mark.parametrize("order", [0, 1, 2, 3, 4])
def test_dot_orders_pinned_to_exact_dot(orc, order):
    """The five CG dot-product orders of reading R18 (ascending, descending, pairwise,
    1024-blocked, Kahan) are sums of the same n products (P:1021-1036 CG).  Pinned against an
    exact dot: (i) small-integer vectors, where every partial sum is an integer below 2^53 and so
    every order must give the exact value bit for bit (a dropped, repeated or misindexed term
    fails); (ii) random floats against math.fsum of the rounded products, within the
    order-independent bound n eps sum|a_i b_i| (Kahan: 2 eps sum|a_i b_i|)."""
    import math
    rng = np.random.default_rng(1800 + order)
    for n in (1, 2, 7, 8, 9, 1023, 1024, 1025, 5000):
        a = rng.integers(-1000, 1001, n).astype(np.float64)
        b = rng.integers(-1000, 1001, n).astype(np.float64)
        exact = int(np.dot(a.astype(np.int64), b.astype(np.int64)))
        assert orc.dot(a, b, order) == float(exact), (order, n)
    eps = np.finfo(np.float64).eps
    for n in (3, 1000, 4099, 100000):
        a = rng.standard_normal(n) * np.exp(rng.uniform(-5, 5, n))
        b = rng.standard_normal(n)
        prods = a * b
        ref = math.fsum(prods.tolist())
        bound = (2.0 if order == 4 else n) * eps * float(np.sum(np.abs(prods)))
        assert abs(orc.dot(a, b, order) - ref) <= bound, (order, n)


# ---------------------------------------------------------------- Newton (§8(f) row f1)
def _potential(m, u, f):
    """Pi(U) = W(U) - f.U (App. B / P:164, the energy the residual differentiates)."""
    _, tot = m.energy(u.reshape(1, m.n_nodes, m.dim), f_ext=f, want_elem=False)
    return float(tot.sum())


def test_newton_linear_is_one_step(orc):
    """K does not depend on U for the linear model, so Newton from U_0 = 0
    lands on the dense solution in one step (config 1, dense Cholesky of the masked K)."""
    p = config1()
    m = orc.prepare_problem(p)
    n = p.n_nodes * 2
    A = dense_K(m, n, mask=p.mask)
    b = p.f_ext.ravel() * (1 - p.mask)
    xs = np.linalg.solve(A, b)
    tol = 1e-9 * np.linalg.norm(b)
    u, rep = m.newton(np.zeros_like(p.coords), p.f_ext, p.mask, tol=tol, cg_tol=1e-13)
    assert rep["converged"] and rep["iterations"] == 1
    assert rel(u.ravel(), xs) < 1e-9
    assert abs(rep["history"][0] - np.linalg.norm(b)) < 1e-14 * np.linalg.norm(b)


def test_newton_neohookean_quadratic_and_stationary(orc):
    """Neo-Hookean block under shear + tension: (i) quadratic convergence of the residual
    norms in the asymptotic range, e_{k+1} <= 10 e_k^2 (a wrong tangent converges at best
    linearly and fails it); (ii) the converged U makes the potential stationary: central
    difference of Pi along a random free direction ~ 0, while at U_0 = 0 it is -f.v."""
    from pfem_gen import newton_block
    p = newton_block(5, traction=(0.05, 0.0, 0.02))
    m = orc.prepare_problem(p)
    u, rep = m.newton(p.u[0], p.f_ext, p.mask, tol=1e-11, cg_tol=1e-13)
    assert rep["converged"] and 3 <= rep["iterations"] <= 8
    e = rep["history"] / rep["history"][0]
    checked = 0
    for k in range(len(e) - 1):
        if e[k] < 1e-2 and e[k + 1] > 1e-12:
            assert e[k + 1] <= 10 * e[k] ** 2, (k, e)
            checked += 1
    assert checked >= 1
    rng = np.random.default_rng(3)
    v = rng.standard_normal(u.shape) * (1 - p.mask.reshape(u.shape))
    eps = 1e-5
    g = (_potential(m, u + eps * v, p.f_ext) - _potential(m, u - eps * v, p.f_ext)) / (2 * eps)
    g0 = (_potential(m, eps * v, p.f_ext) - _potential(m, -eps * v, p.f_ext)) / (2 * eps)
    scale = np.linalg.norm(p.f_ext) * np.linalg.norm(v)
    assert abs(g0 + float(np.sum(p.f_ext * v))) < 1e-6 * scale
    assert abs(g) < 1e-7 * scale


def test_newton_small_load_limit_and_warm_start(orc):
    """Small loads: the Neo-Hookean solution tends to the linear one with the same (mu, lambda),
    the gap shrinking linearly with the load; a perturbed-exact start needs fewer Newton steps
    than a zero start (the warm-start claim)."""
    from pfem_gen import newton_block, warm_start
    gaps = []
    for s in (1e-3, 1e-4):
        p = newton_block(4, traction=(0.05 * s, 0.0, 0.02 * s))
        nh = orc.prepare_problem(p)
        lin = orc.prepare(p.coords, p.conn, "linear", "lame", p.p0, p.p1)
        un, rn = nh.newton(p.u[0], p.f_ext, p.mask, tol=1e-9 * np.linalg.norm(p.f_ext), cg_tol=1e-13)
        ul, _ = lin.cg(p.f_ext, p.mask, np.zeros_like(p.coords), tol=1e-13)
        assert rn["converged"]
        gaps.append(rel(un, ul))
    assert gaps[0] < 1e-2 and 0.05 < gaps[1] / gaps[0] < 0.2
    p = newton_block(5, traction=(0.05, 0.0, 0.02))
    m = orc.prepare_problem(p)
    us, _ = m.newton(p.u[0], p.f_ext, p.mask, tol=1e-12, cg_tol=1e-13)
    _, rz = m.newton(p.u[0], p.f_ext, p.mask, tol=1e-9, cg_tol=1e-12)
    _, rw = m.newton(warm_start(us, p.mask, seed=77), p.f_ext, p.mask, tol=1e-9, cg_tol=1e-12)
    assert rw["iterations"] < rz["iterations"]


# ---------------------------------------------------------------- Jacobi PCG (§8(f) row f3)
@pytest.mark.parametrize("kind", ["t3", "t4"])
@pytest.mark.parametrize("model", ["linear", "neohookean"])
def test_tangent_diag_is_operator_diagonal(orc, kind, model):
    """diag(A) of A = (I-M) K(u) (I-M) + M equals the brute-force diagonal e_i . A e_i of the
    matrix-free operator (reading R27; P:1104-1115 for K), mask rows 1."""
    coords, conn = MESHES[kind]()
    d = coords.shape[1]
    m = orc.prepare(coords, conn, model, "lame", [0.4], [0.6])
    rng = np.random.default_rng(5)
    u = 0.05 * rng.standard_normal(coords.shape) if model == "neohookean" else None
    mask = (rng.random(coords.size) < 0.2).astype(np.uint8)
    n = coords.size
    diag_bf = np.empty(n)
    for i in range(n):
        e = np.zeros(n)
        e[i] = 1.0
        us = None if u is None else u.reshape(1, -1, d)
        diag_bf[i] = m.tangent(e.reshape(1, -1, d), u=us, mask=mask).ravel()[i]
    dg = m.tangent_diag(u=u, mask=mask).ravel()
    assert rel(dg, diag_bf) < 1e-14
    assert np.all(dg[mask == 1] == 1.0) and np.all(dg > 0)


def test_tangent_diag_closed_form_single_element(orc):
    """Reference T3 / T4, linear law: the diagonal of V B^T D B is
    V [(lam + 2 mu) g_ai^2 + mu sum_{j != i} g_aj^2] (textbook isotropic stiffness);
    Neo-Hookean at F = I has the same diagonal (K(0) = K_lin)."""
    mu, lam = 0.4, 0.6
    for coords in (np.array([[0., 0], [1, 0], [0, 1]]), np.array([[0., 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]])):
        d = coords.shape[1]
        V = 1.0 / (2 if d == 2 else 6)
        g = np.vstack([-np.ones(d), np.eye(d)])          # grad N_a of the reference simplex
        ref = np.array([[V * ((lam + 2 * mu) * g[a, i] ** 2 + mu * (g[a] @ g[a] - g[a, i] ** 2)) for i in range(d)]
                        for a in range(d + 1)])
        conn = np.arange(d + 1)[None, :]
        for model in ("linear", "neohookean"):
            m = orc.prepare(coords, conn, model, "lame", [mu], [lam])
            u0 = np.zeros_like(coords) if model == "neohookean" else None
            assert rel(m.tangent_diag(u=u0), ref) < 1e-15


def _dense_cg(A, b, k):
    """Textbook Hestenes-Stiefel CG, k steps from 0 (numpy, dense)."""
    x = np.zeros_like(b)
    r = b.copy()
    p = r.copy()
    rho = r @ r
    for _ in range(k):
        q = A @ p
        a = rho / (p @ q)
        x += a * p
        r -= a * q
        rn = r @ r
        p = r + (rn / rho) * p
        rho = rn
    return x


def test_pcg_is_cg_on_the_jacobi_scaled_system(orc):
    """Jacobi PCG iterates are x_k = D^-1/2 y_k with y_k the CG iterates of
    (D^-1/2 A D^-1/2) y = D^-1/2 b (the classical equivalence of split preconditioning);
    PCG solves to the dense Cholesky solution; precond 0 is plain CG bit for bit; an exact
    initial guess takes 0 iterations."""
    p = config1()
    m = orc.prepare_problem(p)
    n = p.n_nodes * 2
    A = dense_K(m, n, mask=p.mask)
    b = p.f_ext.ravel() * (1 - p.mask)
    dg = m.tangent_diag(mask=p.mask).ravel()
    assert rel(dg, np.diag(A)) < 1e-15
    s = 1.0 / np.sqrt(dg)
    Ah = A * s[:, None] * s[None, :]
    for k in (1, 3, 10, 25):
        xk, _ = m.pcg(p.f_ext, p.mask, np.zeros(n), tol=1e-30, max_iter=k, history=False)
        assert rel(xk.ravel(), s * _dense_cg(Ah, s * b, k)) < 1e-10
    x_ref = np.linalg.solve(A, b)
    x, rep = m.pcg(p.f_ext, p.mask, np.zeros(n), tol=1e-12)
    assert rep["converged"] and rel(x, x_ref) < 1e-9 and rep["true_rel_res_final"] < 1e-11
    xc, rc = m.cg(p.f_ext, p.mask, np.zeros(n), tol=1e-8)
    x0, r0 = m.pcg(p.f_ext, p.mask, np.zeros(n), tol=1e-8, precond=0)
    assert r0["iterations"] == rc["iterations"] and np.array_equal(r0["history"], rc["history"])
    assert np.array_equal(x0, xc)
    _, rs = m.pcg(p.f_ext, p.mask, x_ref, tol=1e-8)
    assert rs["iterations"] == 0 and rs["converged"]


# ---------------------------------------------------------------- pretraining loss (§8(f) row f2)
@pytest.mark.parametrize("model", ["linear", "neohookean"])
def test_pretrain_loss_gradient_is_finite_difference(orc, model):
    """dloss/dH of the energy loss through the hard-BC ansatz u = phi (.) H
    equals the central finite difference of the loss (two parts, two samples: the batch mean
    divides by S K); phi = 0 rows (the clamped edge) have zero gradient."""
    ca, ta = jittered_square(4, 31)
    cb, tb = jittered_square(3, 32)
    coords = np.concatenate([ca, cb + 2.0])
    conn = np.concatenate([ta, tb + len(ca)])
    pe = np.array([0, len(ta), len(conn)], np.int32)
    pn = np.array([0, len(ca), len(coords)], np.int32)
    m = orc.prepare(coords, conn, model, "lame", [0.4], [0.6], pe, pn)
    rng = np.random.default_rng(4)
    phi = (coords[:, :1] - np.where(np.arange(len(coords)) < len(ca), 0.0, 2.0)[:, None]) * np.ones((1, 2))
    f = 0.01 * rng.standard_normal(coords.shape)
    H = 0.05 * rng.standard_normal((2,) + coords.shape)
    loss, Pi, grad, u = m.pretrain_loss(H, phi, f)
    assert Pi.shape == (2, 2) and abs(loss - Pi.mean()) < 1e-15
    # Pi = W - f.u per part, W from energy() without f
    _, W = m.energy(u, want_elem=False)
    fu = np.stack([[np.sum(f[pn[k]:pn[k + 1]] * u[s, pn[k]:pn[k + 1]]) for k in range(2)] for s in range(2)])
    assert np.max(np.abs(Pi - (W - fu))) < 1e-15
    h = 1e-6
    idx = [(0, 1, 0), (1, 3, 1), (0, len(ca) + 4, 0), (1, len(coords) - 1, 1), (0, 0, 1)]
    for s, n, i in idx:
        Hp, Hm = H.copy(), H.copy()
        Hp[s, n, i] += h
        Hm[s, n, i] -= h
        fd = (m.pretrain_loss(Hp, phi, f)[0] - m.pretrain_loss(Hm, phi, f)[0]) / (2 * h)
        assert abs(fd - grad[s, n, i]) < 1e-8 * max(1.0, abs(grad).max()), (s, n, i, fd, grad[s, n, i])
    assert np.all(grad[:, phi[:, 0] == 0] == 0)
    # phi = 1: the gradient is the potential's gradient f_int - f_ext over S K
    _, _, g1, _ = m.pretrain_loss(H, None, f)
    assert rel(g1, (m.residual(H) - f[None]) / 4) < 1e-15


# ---------------------------------------------------------------- heat conduction (§8(f) row f4)
@pytest.mark.parametrize("kind", ["t3", "t4"])
def test_heat_patch_rigid_and_gradient(orc, kind):
    """Scalar heat conduction (energy form P:249-284): an affine field T = g.x + c
    has W = 1/2 k |g|^2 |Omega| (|Omega| = 1) and zero interior residual (patch test); a
    constant field has W = 0 and r = 0 exactly; r is the central finite difference of W
    (exact up to rounding: W is quadratic) and T.r(T) = 2W; r is linear and symmetric."""
    coords, conn = MESHES[kind]()
    d = coords.shape[1]
    rng = np.random.default_rng(6)
    kk = rng.uniform(0.5, 2.0, len(conn))
    m = orc.prepare(coords, conn, "linear", "lame", [1.0], [1.0])
    g = rng.standard_normal(d)
    W, tot, r = m.heat((coords @ g + 0.7)[None], [1.3])
    assert abs(tot[0, 0] - 0.5 * 1.3 * g @ g) < 1e-13
    interior = np.all((coords > 1e-9) & (coords < 1 - 1e-9), axis=1)
    assert np.max(np.abs(r[0, interior])) < 1e-13
    W0, tot0, r0 = m.heat(np.full((1, len(coords)), 3.25), kk)
    assert np.all(W0 == 0) and np.all(r0 == 0)
    T = rng.standard_normal((2, len(coords)))
    W, tot, r = m.heat(T, kk)
    h = 1e-6
    for s, n in [(0, 1), (1, 5), (0, len(coords) - 1)]:
        Tp, Tm = T.copy(), T.copy()
        Tp[s, n] += h
        Tm[s, n] -= h
        fd = (m.heat(Tp, kk)[1][s, 0] - m.heat(Tm, kk)[1][s, 0]) / (2 * h)
        assert abs(fd - r[s, n]) < 1e-7 * max(1.0, np.abs(r).max())
    assert abs(T[0] @ r[0] - 2 * tot[0, 0]) < 1e-12 * abs(tot[0, 0])
    v, w = rng.standard_normal((2, len(coords)))
    Kv, Kw = m.heat(v[None], kk)[2][0], m.heat(w[None], kk)[2][0]
    assert abs(w @ Kv - v @ Kw) < 1e-12 * abs(w @ Kv)
    # nodal loads enter the totals as - f.T
    f = rng.standard_normal(len(coords))
    _, totf, _ = m.heat(T[:1], kk, f=f)
    assert abs(totf[0, 0] - (tot[0, 0] - f @ T[0])) < 1e-12


def test_heat_single_element_closed_form(orc):
    """Reference T3 with T = (0, 1, 0): grad T = (1, 0), W = 1/2 k V = k / 4; the nodal fluxes
    are k V grad N_a . (1, 0) = k/2 (-1, 1, 0)."""
    m = orc.prepare(np.array([[0., 0], [1, 0], [0, 1]]), np.array([[0, 1, 2]]), "linear", "lame", [1.0], [1.0])
    W, tot, r = m.heat(np.array([[0.0, 1.0, 0.0]]), [2.0])
    assert abs(W[0, 0] - 0.5) < 1e-16 and np.allclose(r[0], [-1.0, 1.0, 0.0], atol=1e-16, rtol=0)
