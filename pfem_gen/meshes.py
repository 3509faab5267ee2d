"""Seeded synthetic meshes and fields — the input generators shared by tests,
bench and smoke.

This module holds NO arithmetic of the PFEM method (no shape-function
gradients, strains, energies, stresses, forces or solves): only mesh topology,
node coordinates, random fields and boundary data, so that the oracle and the
CUDA path receive identical inputs without sharing any method code (task rule
③; DESIGN.md §"Input recipe").

All randomness is numpy PCG64 ``default_rng(seed)``.  Node ids of structured
meshes are x-fastest then y then z unless a brick ordering is requested.
"""
from __future__ import annotations

import itertools

import numpy as np


# --------------------------------------------------------------------------
# 2-D structured triangle meshes (T3)
# --------------------------------------------------------------------------
def square_t3(nx_nodes: int, ny_nodes: int, lx: float = 1.0, ly: float = 1.0):
    """Structured T3 mesh of [0,lx]x[0,ly] with nx_nodes x ny_nodes nodes.

    Each cell (i,j) is split along (i,j)-(i+1,j+1):
    T_a = (n00, n10, n11), T_b = (n00, n11, n01) — both counter-clockwise.
    Returns coords [N,2] float64, conn [E,3] int32.
    """
    xs = np.linspace(0.0, lx, nx_nodes)
    ys = np.linspace(0.0, ly, ny_nodes)
    X, Y = np.meshgrid(xs, ys, indexing="xy")          # [ny, nx], x fastest
    coords = np.stack([X.ravel(), Y.ravel()], axis=1)
    i, j = np.meshgrid(np.arange(nx_nodes - 1), np.arange(ny_nodes - 1), indexing="xy")
    n00 = (j * nx_nodes + i).ravel()
    n10, n01, n11 = n00 + 1, n00 + nx_nodes, n00 + nx_nodes + 1
    ta = np.stack([n00, n10, n11], axis=1)
    tb = np.stack([n00, n11, n01], axis=1)
    conn = np.stack([ta, tb], axis=1).reshape(-1, 3)   # cell order, T_a then T_b
    return coords, conn.astype(np.int32)


def plate_with_holes(n_cells: int, rng: np.random.Generator, n_holes: int = 3,
                     jitter: float = 0.2, r_range=(0.05, 0.15), c_range=(0.2, 0.8)):
    """Unit plate, n_cells x n_cells cells (h = 1/n_cells), interior nodes jittered
    by U[-jitter*h, +jitter*h] per coordinate (boundary nodes fixed), n_holes circular
    holes (centres U[c_range]^2, radii U[r_range]).  A triangle is removed if its
    centroid lies strictly inside a hole; orphan nodes are dropped and the rest
    renumbered in their original (x-fastest) order.

    Stands in for the paper's GRF-hole plates (§4.1).
    Returns coords [N,2] float64, conn [E,3] int32, holes [n_holes,3] (cx, cy, r).
    """
    n = n_cells
    h = 1.0 / n
    coords, conn = square_t3(n + 1, n + 1)
    ij = np.stack(np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="xy"), -1).reshape(-1, 2)
    interior = (ij[:, 0] > 0) & (ij[:, 0] < n) & (ij[:, 1] > 0) & (ij[:, 1] < n)
    jit = rng.uniform(-jitter * h, jitter * h, size=coords.shape)
    coords = coords + jit * interior[:, None]
    centres = rng.uniform(c_range[0], c_range[1], size=(n_holes, 2))
    radii = rng.uniform(r_range[0], r_range[1], size=n_holes)
    cen = coords[conn].mean(axis=1)
    keep = np.ones(len(conn), dtype=bool)
    for c, r in zip(centres, radii):
        keep &= np.sum((cen - c) ** 2, axis=1) >= r * r
    conn = conn[keep]
    used = np.zeros(len(coords), dtype=bool)
    used[conn.ravel()] = True
    new_id = np.cumsum(used) - 1
    coords = coords[used]
    conn = new_id[conn].astype(np.int32)
    holes = np.concatenate([centres, radii[:, None]], axis=1)
    return coords, conn, holes


# --------------------------------------------------------------------------
# 3-D Kuhn tetrahedral cube (T4)
# --------------------------------------------------------------------------
def _brick_rank(idx: np.ndarray, dims, brick: int) -> np.ndarray:
    """Rank of each multi-index (rows of idx, columns x,y,z) under brick ordering:
    bricks of brick^3 points ordered z,y,x-major (x fastest), points inside a brick
    x-fastest.  Returns new_id[old_id]."""
    b = idx // brick
    l = idx % brick
    nb = [(d + brick - 1) // brick for d in dims]
    bid = (b[:, 2] * nb[1] + b[:, 1]) * nb[0] + b[:, 0]
    lid = (l[:, 2] * brick + l[:, 1]) * brick + l[:, 0]
    order = np.lexsort((lid, bid))          # primary bid, secondary lid
    rank = np.empty(len(idx), dtype=np.int64)
    rank[order] = np.arange(len(idx))
    return rank


def kuhn_cube(n_nodes: int, brick: int | None = None, length: float = 1.0):
    """Unit cube with n_nodes^3 nodes (h = length/(n_nodes-1)), each cell split into
    6 tetrahedra along the (0,0,0)-(1,1,1) diagonal (Kuhn / Freudenthal split, one
    tet per axis permutation: v0 = 000, v1 = e_a, v2 = e_a + e_b, v3 = 111).
    The split is conforming.  Tets are emitted positively oriented (v1,v2 swapped
    for odd permutations).  With ``brick``, nodes and cells are renumbered in brick
    order (locality for the block-partitioned assembly, DESIGN.md §"Mesh order").
    Returns coords [N,3] float64, conn [E,4] int32.
    """
    n = n_nodes
    m = n - 1
    h = length / m
    g = np.arange(n)
    K, J, I = np.meshgrid(g, g, g, indexing="ij")         # z slowest, x fastest
    nidx = np.stack([I.ravel(), J.ravel(), K.ravel()], axis=1)
    coords = nidx.astype(np.float64) * h
    gc = np.arange(m)
    Kc, Jc, Ic = np.meshgrid(gc, gc, gc, indexing="ij")
    cidx = np.stack([Ic.ravel(), Jc.ravel(), Kc.ravel()], axis=1)

    def nid(off):   # node id of cell corner offset off (3-tuple of 0/1)
        q = cidx + np.asarray(off)[None, :]
        return (q[:, 2] * n + q[:, 1]) * n + q[:, 0]

    tets = []
    for perm in itertools.permutations(range(3)):
        e = np.eye(3, dtype=np.int64)
        v0 = (0, 0, 0)
        v1 = tuple(e[perm[0]])
        v2 = tuple(e[perm[0]] + e[perm[1]])
        v3 = (1, 1, 1)
        # parity of the permutation: odd permutations give negative volume
        inv = sum(1 for a in range(3) for b in range(a + 1, 3) if perm[a] > perm[b])
        if inv % 2 == 1:
            v1, v2 = v2, v1
        tets.append(np.stack([nid(v0), nid(v1), nid(v2), nid(v3)], axis=1))
    conn = np.stack(tets, axis=1).reshape(-1, 4)          # cell-major, 6 tets per cell
    if brick:
        node_rank = _brick_rank(nidx, (n, n, n), brick)
        cell_rank = _brick_rank(cidx, (m, m, m), brick)
        new_coords = np.empty_like(coords)
        new_coords[node_rank] = coords
        coords = new_coords
        conn = node_rank[conn]
        cell_order = np.argsort(cell_rank, kind="stable")
        conn = conn.reshape(m ** 3, 6, 4)[cell_order].reshape(-1, 4)
    return coords, conn.astype(np.int32)


def boundary_faces_on_plane(conn: np.ndarray, coords: np.ndarray, axis: int, value: float,
                            tol: float = 1e-12) -> np.ndarray:
    """Faces (node triples / pairs) of simplices lying on the plane coords[:,axis]==value.
    Pure topology + coordinate test; returns [F, d] int32 node ids."""
    d = conn.shape[1] - 1
    on = np.abs(coords[:, axis] - value) < tol
    faces = []
    for drop in range(d + 1):
        f = np.delete(conn, drop, axis=1)
        sel = np.all(on[f], axis=1)
        faces.append(f[sel])
    return np.concatenate(faces, axis=0).astype(np.int32)


# --------------------------------------------------------------------------
# Smooth random fields
# --------------------------------------------------------------------------
def fourier_field(X: np.ndarray, rng: np.random.Generator, n_modes: int = 8, kmax: int = 2):
    """Phi_c(X) = sum_m a_cm sin(2 pi k_m.X + phi_cm) / (2 pi |k_m|), per component c,
    with k_m uniform on {-kmax..kmax}^d minus 0, a ~ N(0,1)/sqrt(n_modes),
    phi ~ U[0, 2 pi).  Its gradient has O(1) magnitude.  Returns [N, d]."""
    N, d = X.shape
    ks = np.array([k for k in itertools.product(range(-kmax, kmax + 1), repeat=d) if any(k)])
    kk = ks[rng.integers(0, len(ks), size=n_modes)].astype(np.float64)       # [M, d]
    a = rng.standard_normal((d, n_modes)) / np.sqrt(n_modes)
    ph = rng.uniform(0.0, 2 * np.pi, size=(d, n_modes))
    knorm = np.linalg.norm(kk, axis=1)
    arg = 2 * np.pi * (X @ kk.T)                                              # [N, M]
    out = np.empty((N, d))
    for c in range(d):
        out[:, c] = (np.sin(arg + ph[c][None, :]) * (a[c] / (2 * np.pi * knorm))[None, :]).sum(1)
    return out


# --------------------------------------------------------------------------
# 2-D structured quadrilateral meshes (Q4 / Q8), §8(f) row f4
# --------------------------------------------------------------------------
def quad_grid(nx: int, ny: int, kind: str = "q4", corners=((0.0, 0.0), (1.0, 0.0), (1.0, 1.0), (0.0, 1.0))):
    """Structured nx x ny quadrilateral mesh of the bilinear map of the unit square onto the
    quadrilateral `corners` (counter-clockwise A, B, C, D: (s,t) -> (1-s)(1-t)A + s(1-t)B + stC
    + (1-s)tD).  kind "q4": (nx+1)(ny+1) nodes x-fastest, element (i, j) = (n00, n10, n11, n01),
    counter-clockwise.  kind "q8": serendipity — the (2nx+1)(2ny+1) half-step grid without the
    cell centres, renumbered in x-fastest order ((2nx+1)(2ny+1) - nx ny nodes); element nodes
    are the four corners (counter-clockwise) then the midsides of edges 01, 12, 23, 30.  Every
    cell edge is straight (the map is linear along s and t), so midside nodes are edge
    midpoints.  Returns coords [N,2] float64, conn [E,4|8] int32."""
    A, B, Cc, D = (np.asarray(c, np.float64) for c in corners)

    def emap(s, t):
        return ((1 - s) * (1 - t))[:, None] * A + (s * (1 - t))[:, None] * B + (s * t)[:, None] * Cc + \
            ((1 - s) * t)[:, None] * D

    if kind == "q4":
        i, j = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), indexing="xy")
        coords = emap(i.ravel() / nx, j.ravel() / ny)
        ci, cj = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
        n00 = (cj * (nx + 1) + ci).ravel()
        conn = np.stack([n00, n00 + 1, n00 + nx + 2, n00 + nx + 1], axis=1)
        return coords, conn.astype(np.int32)
    if kind != "q8":
        raise ValueError(kind)
    mx, my = 2 * nx + 1, 2 * ny + 1
    i, j = np.meshgrid(np.arange(mx), np.arange(my), indexing="xy")
    i, j = i.ravel(), j.ravel()
    keep = ~((i % 2 == 1) & (j % 2 == 1))
    new_id = np.full(mx * my, -1, np.int64)
    new_id[keep] = np.arange(int(keep.sum()))
    coords = emap(i[keep] / (2 * nx), j[keep] / (2 * ny))
    ci, cj = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    ci, cj = 2 * ci.ravel(), 2 * cj.ravel()

    def g(a, b):
        return new_id[b * mx + a]

    conn = np.stack([g(ci, cj), g(ci + 2, cj), g(ci + 2, cj + 2), g(ci, cj + 2),
                     g(ci + 1, cj), g(ci + 2, cj + 1), g(ci + 1, cj + 2), g(ci, cj + 1)], axis=1)
    return coords, conn.astype(np.int32)
