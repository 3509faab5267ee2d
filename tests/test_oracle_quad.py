"""Pins of the oracle's Q4 / Q8 elements (beam P:774, Cook P:846) to what the
isoparametric formulation and the mathematics fix (no GPU): shape-function identities, Gauss-rule
exactness, geometry (areas, det J of an affine map), the affine patch test for energy and
residual, rigid translations, residual = finite difference of the energy, tangent = finite
difference of the residual and symmetric, CG vs a dense solve, Newton's quadratic convergence."""
import numpy as np
import pytest

from pfem_gen import beam_q4, cook_q8, quad_grid

KINDS = ["q4", "q8"]
REF = {"q4": [(-1, -1), (1, -1), (1, 1), (-1, 1)],
       "q8": [(-1, -1), (1, -1), (1, 1), (-1, 1), (0, -1), (1, 0), (0, 1), (-1, 0)]}


def jittered_quads(kind, n=4, seed=3, corners=((0, 0), (2, 0), (2.2, 1.3), (-0.1, 1.0))):
    """A small distorted (but valid) quad mesh: a bilinear map of a trapezoid, interior corner nodes
    jittered (Q4 only: Q8 midsides must stay on straight edges for the exactness pins)."""
    c, t = quad_grid(n, n, kind, corners=corners)
    if kind == "q4":
        rng = np.random.default_rng(seed)
        inner = np.ones(len(c), bool)
        for k in range(2):
            inner &= (c[:, k] > c[:, k].min() + 1e-9) & (c[:, k] < c[:, k].max() - 1e-9)
        c = c + 0.08 * rng.uniform(-1, 1, c.shape) * inner[:, None]
    return c, t


def qmesh(orc, kind, model="neohookean", mu=0.4, lam=0.6, **kw):
    c, t = jittered_quads(kind, **kw)
    return orc.prepare_quad(kind, c, t, model, "lame", [mu], [lam]), c, t


def area_of(c, t, kind):
    """Polygon area of each element's boundary (corners + midsides in order), shoelace formula."""
    if kind == "q4":
        ring = t
    else:
        ring = t[:, [0, 4, 1, 5, 2, 6, 3, 7]]
    x, y = c[ring, 0], c[ring, 1]
    return 0.5 * np.sum(x * np.roll(y, -1, 1) - np.roll(x, -1, 1) * y, axis=1)


@pytest.mark.parametrize("kind", KINDS)
def test_shape_functions_identities(orc, kind):
    """Kronecker property at the nodes, partition of unity, derivatives sum to zero, and the
    derivatives equal central finite differences of N (SPEC-style pins; Q4 centre = 1/4 each)."""
    nodes = REF[kind]
    for b, (xb, yb) in enumerate(nodes):
        N, _ = orc.quad_shape(kind, xb, yb)
        assert np.allclose(N, np.eye(len(nodes))[b], atol=1e-15)
    if kind == "q4":
        N, _ = orc.quad_shape(kind, 0.0, 0.0)
        assert np.allclose(N, 0.25, atol=1e-16)
    rng = np.random.default_rng(1)
    for _ in range(5):
        xi, eta = rng.uniform(-1, 1, 2)
        N, dN = orc.quad_shape(kind, xi, eta)
        assert abs(N.sum() - 1) < 1e-15 and np.all(np.abs(dN.sum(0)) < 1e-15)
        h = 1e-6
        fd_x = (orc.quad_shape(kind, xi + h, eta)[0] - orc.quad_shape(kind, xi - h, eta)[0]) / (2 * h)
        fd_y = (orc.quad_shape(kind, xi, eta + h)[0] - orc.quad_shape(kind, xi, eta - h)[0]) / (2 * h)
        assert np.allclose(dN[:, 0], fd_x, atol=1e-9) and np.allclose(dN[:, 1], fd_y, atol=1e-9)


@pytest.mark.parametrize("kind,deg", [("q4", 3), ("q8", 5)])
def test_gauss_rule_exactness(orc, kind, deg):
    """m x m Gauss-Legendre integrates xi^a eta^b exactly for a, b <= 2m - 1 (int_{-1}^{1} x^k =
    2/(k+1) for even k, 0 for odd k) and is not exact one degree above."""
    pts, w = orc.quad_rule(kind)
    exact1 = lambda k: 0.0 if k % 2 else 2.0 / (k + 1)
    for a in range(deg + 1):
        for b in range(deg + 1):
            num = np.sum(w * pts[:, 0] ** a * pts[:, 1] ** b)
            assert abs(num - exact1(a) * exact1(b)) < 1e-14, (a, b)
    num = np.sum(w * pts[:, 0] ** (deg + 1))
    assert abs(num - exact1(deg + 1)) > 1e-3


@pytest.mark.parametrize("kind", KINDS)
def test_affine_patch_energy_and_residual(orc, kind):
    """Affine u = A X + c: grad u = A at every quadrature point, so W = psi(A) |Omega| exactly
    (both models), and the interior nodes' residual vanishes (patch test)."""
    A = np.array([[0.02, -0.01], [0.015, 0.03]])
    for model in ("linear", "neohookean"):
        m, c, t = qmesh(orc, kind, model=model)
        u = (c @ A.T + np.array([0.3, -0.1]))[None]
        W, tot = m.energy(u)
        area = area_of(c, t, kind).sum()
        mu, lam = 0.4, 0.6
        eps = 0.5 * (A + A.T)
        if model == "linear":
            psi = mu * np.sum(eps * eps) + 0.5 * lam * np.trace(eps) ** 2
        else:
            F = np.eye(2) + A
            J = np.linalg.det(F)
            psi = 0.5 * lam * np.log(J) ** 2 - mu * np.log(J) + 0.5 * mu * (np.sum(F * F) - 2)
        assert abs(tot[0, 0] - psi * area) < 1e-13 * psi * area
        r = m.residual(u)[0]
        # interior nodes: corners shared by 4 elements (and Q8 midsides shared by 2)
        counts = np.bincount(t[:, :4].ravel(), minlength=len(c))
        interior = counts == 4 if kind == "q4" else np.zeros(len(c), bool)
        if kind == "q8":   # corner nodes shared by 4 elements and midsides shared by 2
            mids = np.bincount(t[:, 4:].ravel(), minlength=len(c))
            interior = (counts == 4) | (mids == 2)
        assert np.max(np.abs(r[interior])) < 1e-13 * np.max(np.abs(r))
        assert np.max(np.abs(r.sum(0))) < 1e-13 * np.max(np.abs(r))


@pytest.mark.parametrize("kind", KINDS)
def test_rigid_translation_and_geometry(orc, kind):
    """A rigid translation gives W = 0 and r = 0; the element areas by quadrature (the sum over
    the Gauss points of w det J, read through the linear energy of u = (s x, 0) with lam = 0 and
    mu = 1 / (2 s^2), where psi = mu s^2 = 1/2) match the shoelace areas of the elements."""
    m, c, t = qmesh(orc, kind, model="neohookean")
    u = np.tile([0.7, -0.4], (len(c), 1))[None]
    W, tot = m.energy(u)
    assert np.all(np.abs(W) < 1e-15) and np.max(np.abs(m.residual(u))) < 1e-15
    s = 1e-2
    ml = orc.prepare_quad(kind, c, t, "linear", "lame", [1.0 / (2 * s * s)], [0.0])
    W, _ = ml.energy((c * np.array([s, 0.0]))[None])       # psi = mu s^2 = 1/2 per unit area
    assert np.allclose(2 * W[0], area_of(c, t, kind), rtol=1e-13)


@pytest.mark.parametrize("kind", KINDS)
def test_residual_and_tangent_finite_differences(orc, kind):
    """r = central FD of W and K v = central FD of r along v; K is
    symmetric; linear model: K v = r(v)."""
    m, c, t = qmesh(orc, kind, n=2)
    rng = np.random.default_rng(7)
    u = 0.03 * rng.standard_normal((1,) + c.shape)
    r = m.residual(u)[0].ravel()
    h = 1e-6
    fd = np.zeros_like(r)
    for k in range(len(fd)):
        up, um = u.copy().reshape(-1), u.copy().reshape(-1)
        up[k] += h
        um[k] -= h
        fd[k] = (m.energy(up.reshape(u.shape))[1][0, 0] - m.energy(um.reshape(u.shape))[1][0, 0]) / (2 * h)
    assert np.max(np.abs(fd - r)) < 1e-8 * np.max(np.abs(r))
    v, w = rng.standard_normal((2,) + u.shape)
    Kv = m.tangent(v, u=u)
    fdk = (m.residual(u + h * v) - m.residual(u - h * v)) / (2 * h)
    assert np.max(np.abs(fdk - Kv)) < 1e-7 * np.max(np.abs(Kv))
    assert abs(np.sum(w * m.tangent(v, u=u)) - np.sum(v * m.tangent(w, u=u))) < 1e-12 * np.sum(np.abs(w * Kv))
    ml = orc.prepare_quad(kind, c, t, "linear", "lame", [0.4], [0.6])
    assert np.max(np.abs(ml.tangent(v) - ml.residual(v))) < 1e-14 * np.max(np.abs(ml.residual(v)))


@pytest.mark.parametrize("kind", KINDS)
def test_cg_dense_and_newton_quadratic(orc, kind):
    """CG on a small clamped quad mesh vs a dense solve of the masked operator, and the
    Newton iteration's quadratic convergence on the NH problem (App. B)."""
    m, c, t = qmesh(orc, kind, n=3, model="linear")
    n = 2 * len(c)
    mask = np.zeros((len(c), 2), np.uint8)
    mask[np.abs(c[:, 0] + 0.1 * c[:, 1]) < 1e-9] = 1       # the left edge (0,0)-(-0.1,1) clamped
    mask = mask.ravel()
    f = np.zeros((len(c), 2))
    f[c[:, 0] > c[:, 0].max() - 0.3, 1] = -1e-3
    K = np.zeros((n, n))
    for i in range(n):
        e = np.zeros(n)
        e[i] = 1
        K[:, i] = m.tangent(e.reshape(1, -1, 2), mask=mask).ravel()
    b = f.ravel() * (1 - mask)
    xs = np.linalg.solve(K, b)
    x, rep = m.cg(f, mask, np.zeros(n), tol=1e-13)
    assert rep["converged"] and np.linalg.norm(x - xs) < 1e-10 * np.linalg.norm(xs)
    p = (beam_q4 if kind == "q4" else cook_q8)(n_cells=6)
    mq = orc.prepare_quad(p.elem, p.coords, p.conn, p.model, p.param_kind, p.p0, p.p1)
    U, rep = mq.newton(p.u[0], p.f_ext, p.mask, tol=1e-10 * np.linalg.norm(p.f_ext), cg_tol=1e-13)
    h = rep["history"] / rep["history"][0]
    assert rep["converged"] and rep["iterations"] >= 2
    # quadratic: once in the asymptotic region, ||r_{k+1}|| <= 100 ||r_k||^2 (relative to ||r_0||),
    # checked while well above the rounding floor (1e-10 relative)
    steps = [(h[k], h[k + 1]) for k in range(len(h) - 1) if h[k] < 0.2 and h[k + 1] > 1e-10]
    assert steps and all(b <= 100.0 * a * a for a, b in steps), h
