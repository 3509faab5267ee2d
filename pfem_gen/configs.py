"""The five BASELINE.json configs (and reduced-size variants) as concrete seeded
synthetic inputs.  Recipe: SURVEY.md §8(d1), readings in DESIGN.md §"Input recipe".

Seeds: config c uses 1000*c + {1: mesh, 2: material, 3: displacement,
4: warm-start noise}.  Everything is generated in float64; fp32 runs round the
float64 fields (RN) and both the oracle and the GPU path see the rounded values.

No method arithmetic lives here (no gradients, strains, stresses, energies):
``f_ext`` is an INPUT of the method (App. B, "F is the nodal
external force vector"), built as the consistent nodal load of a uniform
traction on flat facets: every facet node receives t * |facet| / n_facet_nodes,
with |facet| the facet's length (2-D) or area (3-D) on a structured boundary.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .meshes import (boundary_faces_on_plane, fourier_field, kuhn_cube,
                     plate_with_holes, quad_grid, square_t3)


@dataclass
class Problem:
    name: str
    dim: int
    coords: np.ndarray                  # [N, d] float64
    conn: np.ndarray                    # [E, d+1] int32
    model: str                          # "linear" | "neohookean"
    param_kind: str                     # "young_poisson" | "lame" | "young_poisson_plane_stress"
    p0: np.ndarray                      # per-element [E] or uniform [1]
    p1: np.ndarray
    u: np.ndarray                       # [S, N, d] float64
    dtype: str = "f64"                  # arithmetic type of the GPU run
    part_elem: np.ndarray | None = None  # [K+1] int32
    part_node: np.ndarray | None = None  # [K+1] int32
    f_ext: np.ndarray | None = None     # [N, d] float64
    mask: np.ndarray | None = None      # [N*d] uint8, 1 = Dirichlet DOF
    meta: dict = field(default_factory=dict)
    elem: str = "simplex"               # "simplex" (T3 / T4) | "q4" | "q8"

    @property
    def n_nodes(self):
        return self.coords.shape[0]

    @property
    def n_elems(self):
        return self.conn.shape[0]

    @property
    def n_samples(self):
        return self.u.shape[0]

    @property
    def n_parts(self):
        return 1 if self.part_elem is None else len(self.part_elem) - 1

    def parts(self):
        """(part_elem, part_node) offsets, defaulting to one part."""
        pe = self.part_elem if self.part_elem is not None else np.array([0, self.n_elems], np.int32)
        pn = self.part_node if self.part_node is not None else np.array([0, self.n_nodes], np.int32)
        return pe.astype(np.int32), pn.astype(np.int32)


def _facet_measure(coords, facets):
    p = coords[facets]
    if facets.shape[1] == 2:
        return np.linalg.norm(p[:, 1] - p[:, 0], axis=1)
    return 0.5 * np.linalg.norm(np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), axis=1)


def traction_load(coords, facets, traction):
    """Consistent nodal load of a uniform traction on flat facets (input data):
    each facet node gets traction * |facet| / (#facet nodes)."""
    f = np.zeros_like(coords)
    meas = _facet_measure(coords, facets)
    k = facets.shape[1]
    for a in range(k):
        np.add.at(f, facets[:, a], (meas / k)[:, None] * np.asarray(traction)[None, :])
    return f


def config1(seed_base: int = 1000, n_nodes: int = 16) -> Problem:
    """Config 1: unit square, 16x16 nodes, 450 T3, linear plane strain E=1 nu=0.3,
    S=1, u ~ N(0, 0.01^2); clamp x=0, traction (1e-2, 0) on x=1 (for the tiny CG)."""
    coords, conn = square_t3(n_nodes, n_nodes)
    rng = np.random.default_rng(seed_base + 3)
    u = rng.normal(0.0, 0.01, size=(1, len(coords), 2))
    right = boundary_faces_on_plane(conn, coords, 0, 1.0)
    f_ext = traction_load(coords, right, (1e-2, 0.0))
    mask = np.zeros((len(coords), 2), np.uint8)
    mask[np.abs(coords[:, 0]) < 1e-12, :] = 1
    return Problem("config1", 2, coords, conn, "linear", "young_poisson",
                   np.array([1.0]), np.array([0.3]), u, "f64",
                   f_ext=f_ext, mask=mask.ravel())


def config2(seed_base: int = 2000, n_cells: int = 200, n_samples: int = 32,
            dtype: str = "f32") -> Problem:
    """Config 2: unit plate with 3 holes, 200x200 cells, jitter U[+-0.2h], ~67-75k T3;
    per-element E = lognormal(0, 0.5), nu = 0.3 (plane strain, reading R1);
    32 fields u ~ N(0, 0.01^2)."""
    coords, conn, holes = plate_with_holes(n_cells, np.random.default_rng(seed_base + 1))
    rng_m = np.random.default_rng(seed_base + 2)
    E = np.exp(0.5 * rng_m.standard_normal(len(conn)))
    rng_u = np.random.default_rng(seed_base + 3)
    u = rng_u.normal(0.0, 0.01, size=(n_samples, len(coords), 2))
    return Problem("config2", 2, coords, conn, "linear", "young_poisson", E, np.array([0.3]),
                   u, dtype, meta={"holes": holes})


def config3(seed_base: int = 3000, n_nodes: int = 64, n_samples: int = 4,
            brick: int | None = 8) -> Problem:
    """Config 3: unit cube 64^3 nodes Kuhn T4 (1,500,282 tets), Neo-Hookean mu=0.4,
    lambda=0.6 uniform, u_s = 0.1 Phi_s(X) + eta, eta ~ N(0, (1e-4)^2) (std reading,
    DESIGN.md R19), S=4, fp32."""
    coords, conn = kuhn_cube(n_nodes, brick=brick)
    rng = np.random.default_rng(seed_base + 3)
    u = np.empty((n_samples, len(coords), 3))
    for s in range(n_samples):
        u[s] = 0.1 * fourier_field(coords, rng) + rng.normal(0.0, 1e-4, size=(len(coords), 3))
    return Problem("config3", 3, coords, conn, "neohookean", "lame",
                   np.array([0.4]), np.array([0.6]), u, "f32")


def config4(seed_base: int = 4000, n_nodes: int = 80, brick: int | None = 8,
            n_spheres: int = 20) -> Problem:
    """Config 4: unit cube 80^3 nodes Kuhn T4 (2,958,234 tets), linear, E = 10 inside
    any of 20 seeded spheres (centres U[0,1]^3, radii U[0.05,0.15]) else 1, nu = 0.3;
    bottom face z=0 clamped, top face z=1 traction (0,0,1e-3); fp64, S=1.
    ``u`` holds one random probe field for K.v (N(0, 0.01^2))."""
    coords, conn = kuhn_cube(n_nodes, brick=brick)
    rng_m = np.random.default_rng(seed_base + 2)
    centres = rng_m.uniform(0.0, 1.0, size=(n_spheres, 3))
    radii = rng_m.uniform(0.05, 0.15, size=n_spheres)
    cen = coords[conn].mean(axis=1)
    inside = np.zeros(len(conn), dtype=bool)
    for c, r in zip(centres, radii):
        inside |= np.sum((cen - c) ** 2, axis=1) < r * r
    E = np.where(inside, 10.0, 1.0)
    top = boundary_faces_on_plane(conn, coords, 2, 1.0)
    f_ext = traction_load(coords, top, (0.0, 0.0, 1e-3))
    mask = np.zeros((len(coords), 3), np.uint8)
    mask[np.abs(coords[:, 2]) < 1e-12, :] = 1
    rng_u = np.random.default_rng(seed_base + 3)
    u = rng_u.normal(0.0, 0.01, size=(1, len(coords), 3))
    return Problem("config4", 3, coords, conn, "linear", "young_poisson", E, np.array([0.3]),
                   u, "f64", f_ext=f_ext, mask=mask.ravel(),
                   meta={"spheres": np.concatenate([centres, radii[:, None]], 1)})


def config5(seed_base: int = 5000, n_meshes: int = 64, cells_range=(128, 176),
            amp: float = 0.05) -> Problem:
    """Config 5: 64 independent plates as in config 2 with per-mesh n_m ~ U{128..176}
    cells per axis (ragged), concatenated as 64 parts (contiguous nodes and elements);
    Neo-Hookean mu, lambda ~ U[0.3, 1.0] per element; u = 0.05 Phi (2-D); S=1, fp32."""
    rng_mesh = np.random.default_rng(seed_base + 1)
    rng_m = np.random.default_rng(seed_base + 2)
    rng_u = np.random.default_rng(seed_base + 3)
    coords_l, conn_l, us = [], [], []
    pe, pn = [0], [0]
    for _ in range(n_meshes):
        nc = int(rng_mesh.integers(cells_range[0], cells_range[1] + 1))
        c, t, _h = plate_with_holes(nc, rng_mesh)
        conn_l.append(t + pn[-1])
        coords_l.append(c)
        us.append(amp * fourier_field(c, rng_u))
        pe.append(pe[-1] + len(t))
        pn.append(pn[-1] + len(c))
    coords = np.concatenate(coords_l)
    conn = np.concatenate(conn_l).astype(np.int32)
    mu = rng_m.uniform(0.3, 1.0, size=len(conn))
    lam = rng_m.uniform(0.3, 1.0, size=len(conn))
    u = np.concatenate(us)[None]
    return Problem("config5", 2, coords, conn, "neohookean", "lame", mu, lam, u, "f32",
                   part_elem=np.array(pe, np.int32), part_node=np.array(pn, np.int32))


def warm_start(u_star: np.ndarray, mask: np.ndarray, seed: int, rel: float = 0.01):
    """Perturbed-exact warm start x0 = u* + rel * rms(u*) * xi on free DOFs
    (xi ~ N(0,1)); constrained DOFs keep u*'s (prescribed) values."""
    rng = np.random.default_rng(seed)
    flat = u_star.reshape(-1)
    free = mask.reshape(-1) == 0
    rms = np.sqrt(np.mean(flat[free] ** 2))
    x0 = flat.copy()
    x0[free] += rel * rms * rng.standard_normal(int(free.sum()))
    return x0.reshape(u_star.shape)


def smooth_warm_start(u_star: np.ndarray, coords: np.ndarray, mask: np.ndarray, seed: int, rel: float = 0.01):
    """Perturbed-exact warm start with a SMOOTH error, the shape of a network prediction's error:
    x0 = u* + rel * rms(u*) * Phi(X) / rms(Phi) on free DOFs, Phi a seeded smooth Fourier field
    over the bounding box (white noise on a slender mesh makes the Neo-Hookean tangent
    indefinite at x0, which no network prediction does)."""
    rng = np.random.default_rng(seed)
    lo, hi = coords.min(0), coords.max(0)
    phi = fourier_field((coords - lo) / np.maximum(hi - lo, 1e-300), rng).reshape(-1)
    flat = u_star.reshape(-1)
    free = mask.reshape(-1) == 0
    rms = np.sqrt(np.mean(flat[free] ** 2))
    rphi = np.sqrt(np.mean(phi[free] ** 2))
    x0 = flat.copy()
    x0[free] += rel * rms * phi[free] / rphi
    return x0.reshape(u_star.shape)


def small_cube_problem(n_nodes: int = 12, seed_base: int = 4000, brick: int | None = None,
                       n_spheres: int = 20) -> Problem:
    """Config-4 recipe at reduced size (n_nodes^3), for CG iteration-count parity."""
    return config4(seed_base=seed_base, n_nodes=n_nodes, brick=brick, n_spheres=n_spheres)


def newton_block(n_nodes: int = 9, traction=(0.02, 0.0, 0.01), mu: float = 0.4, lam: float = 0.6,
                 dtype: str = "f64", brick: int | None = None) -> Problem:
    """Nonlinear warm-start workload (§8(f) row f1; the paper's hyperelastic cantilever /
    Cook-type rows): unit cube of n_nodes^3 nodes, Kuhn T4, compressible
    Neo-Hookean (mu, lambda uniform), bottom face z = 0 clamped, uniform dead traction on the
    top face z = 1 (shear + tension, large enough that Newton needs several steps).  S = 1;
    ``u`` holds the zero start."""
    coords, conn = kuhn_cube(n_nodes, brick=brick)
    top = boundary_faces_on_plane(conn, coords, 2, 1.0)
    f_ext = traction_load(coords, top, traction)
    mask = np.zeros((len(coords), 3), np.uint8)
    mask[np.abs(coords[:, 2]) < 1e-12, :] = 1
    u = np.zeros((1,) + coords.shape)
    return Problem("newton_block", 3, coords, conn, "neohookean", "lame", np.array([mu]), np.array([lam]),
                   u, dtype, f_ext=f_ext, mask=mask.ravel())


def _edge_loads(coords, nodes, traction_y):
    """Nodal loads on a straight boundary edge (input data, no shape-function arithmetic): each
    edge node receives t_y(y_n) times its tributary length (half the distance to each neighbour
    along the edge), in the y direction."""
    ys = coords[nodes, 1]
    order = np.argsort(ys)
    nodes, ys = nodes[order], ys[order]
    trib = np.zeros(len(nodes))
    gaps = np.diff(ys)
    trib[:-1] += 0.5 * gaps
    trib[1:] += 0.5 * gaps
    f = np.zeros_like(coords)
    f[nodes, 1] = traction_y(ys) * trib * np.hypot(1.0, 0.0)
    return f


def beam_q4(n_cells: int = 50, seed_base: int = 6000, t_scale: float = 1e-3, dtype: str = "f64") -> Problem:
    """Hyperelastic beam (§4.2): W x H = 4 x 1, uniform n x n Q4 mesh (50 x 50 = 2500
    elements), compressible Neo-Hookean, plane strain; left end x = 0 clamped; downward
    traction t_y(y) on the right end x = 4 as nodal loads; E and nu per element from smooth
    random fields (stand-ins for the paper's Gaussian random fields): E = 1 + 0.5 tanh(Phi_1),
    nu = 0.3 + 0.05 tanh(Phi_2) at the element centroid; t_y = -t_scale (1 + 0.5 tanh(Phi_3(y))).
    S = 1; ``u`` is the zero start."""
    coords, conn = quad_grid(n_cells, n_cells, "q4", corners=((0, 0), (4, 0), (4, 1), (0, 1)))
    rng = np.random.default_rng(seed_base + 2)
    cen = coords[conn].mean(axis=1)
    E = 1.0 + 0.5 * np.tanh(fourier_field(cen / 4.0, rng)[:, 0] * 4.0)
    nu = 0.3 + 0.05 * np.tanh(fourier_field(cen / 4.0, rng)[:, 0] * 4.0)
    phi3 = fourier_field(np.stack([np.zeros(len(coords)), coords[:, 1]], 1), rng)[:, 1]
    right = np.where(np.abs(coords[:, 0] - 4.0) < 1e-12)[0]
    tvals = dict(zip(coords[right, 1], -t_scale * (1.0 + 0.5 * np.tanh(4.0 * phi3[right]))))
    f_ext = _edge_loads(coords, right, lambda ys: np.array([tvals[y] for y in ys]))
    mask = np.zeros((len(coords), 2), np.uint8)
    mask[np.abs(coords[:, 0]) < 1e-12, :] = 1
    u = np.zeros((1,) + coords.shape)
    return Problem("beam_q4", 2, coords, conn, "neohookean", "young_poisson", E, nu, u, dtype, f_ext=f_ext,
                   mask=mask.ravel(), elem="q4")


def cook_q8(n_cells: int = 30, seed_base: int = 7000, t_scale: float = 2e-3, dtype: str = "f64") -> Problem:
    """Hyperelastic Cook's membrane (§4.2): the classical tapered panel with corners
    (0, 0), (48, 44), (48, 60), (0, 44), uniform n x n Q8 serendipity mesh (30 x 30 = 900
    elements), compressible Neo-Hookean, plane strain; left edge x = 0 clamped; traction
    t_y on the right edge x = 48 as nodal loads; E, nu per element from smooth random fields
    (E = 1 + 0.5 tanh(Phi_1), nu = 0.3 + 0.05 tanh(Phi_2)); t_y = t_scale (1 + 0.5 tanh(Phi_3(y))).
    S = 1; ``u`` is the zero start."""
    coords, conn = quad_grid(n_cells, n_cells, "q8", corners=((0, 0), (48, 44), (48, 60), (0, 44)))
    rng = np.random.default_rng(seed_base + 2)
    cen = coords[conn[:, :4]].mean(axis=1)
    E = 1.0 + 0.5 * np.tanh(fourier_field(cen / 60.0, rng)[:, 0] * 4.0)
    nu = 0.3 + 0.05 * np.tanh(fourier_field(cen / 60.0, rng)[:, 0] * 4.0)
    phi3 = fourier_field(np.stack([np.zeros(len(coords)), coords[:, 1] / 60.0], 1), rng)[:, 1]
    right = np.where(np.abs(coords[:, 0] - 48.0) < 1e-9)[0]
    tvals = dict(zip(coords[right, 1], t_scale * (1.0 + 0.5 * np.tanh(4.0 * phi3[right]))))
    f_ext = _edge_loads(coords, right, lambda ys: np.array([tvals[y] for y in ys]))
    mask = np.zeros((len(coords), 2), np.uint8)
    mask[np.abs(coords[:, 0]) < 1e-12, :] = 1
    u = np.zeros((1,) + coords.shape)
    return Problem("cook_q8", 2, coords, conn, "neohookean", "young_poisson", E, nu, u, dtype, f_ext=f_ext,
                   mask=mask.ravel(), elem="q8")


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}
