"""GPU parity: the CUDA path (through the C-ABI) vs the fp64 CPU oracle on the same
seeded inputs.  Bars (BASELINE.json north star): bit-exact CSR / colouring; rel-L2 <= 1e-12
(fp64) and <= 2e-5 (fp32) for energies, residuals and K.v."""
import numpy as np
import pytest
import torch

from helpers import TOL, assert_field, assert_totals, gpu_problem, max_rel, oracle_problem, rel_l2, rounded
from pfem_gen import (config1, config2, config3, config4, config5, fourier_field, kuhn_cube, plate_with_holes,
                      square_t3)
from pfem_gen.configs import Problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_03086_b200 as pf
    pf.load()


def small_problems():
    """Several tiles + ragged tails, both dims, both models, multi-part."""
    rng = np.random.default_rng(77)
    c, t, _ = plate_with_holes(40, np.random.default_rng(3))
    u = rng.normal(0, 0.02, (3,) + c.shape)
    yield Problem("plate40-lin-f64", 2, c, t, "linear", "young_poisson",
                  np.exp(0.5 * rng.standard_normal(len(t))), np.array([0.3]), u, "f64")
    un = np.stack([0.05 * fourier_field(c, rng) for _ in range(3)])
    yield Problem("plate40-nh-f32", 2, c, t, "neohookean", "lame", rng.uniform(0.3, 1, len(t)),
                  rng.uniform(0.3, 1, len(t)), un, "f32")
    c3, t3 = kuhn_cube(13, brick=4)
    u3 = rng.normal(0, 0.01, (5,) + c3.shape)
    u3n = np.stack([0.1 * fourier_field(c3, rng) + rng.normal(0, 1e-3, c3.shape) for _ in range(5)])
    yield Problem("cube13-nh-f32", 3, c3, t3, "neohookean", "lame", np.array([0.4]), np.array([0.6]), u3n, "f32")
    yield Problem("cube13-lin-f64", 3, c3, t3, "linear", "young_poisson", rng.uniform(1, 10, len(t3)),
                  np.array([0.3]), u3[:2], "f64")
    # two parts (ragged), NH 2-D
    ca, ta = square_t3(23, 17)
    cb, tb = square_t3(9, 31)
    coords = np.concatenate([ca, cb + 3.0])
    conn = np.concatenate([ta, tb + len(ca)]).astype(np.int32)
    up = 0.003 * rng.standard_normal((1,) + coords.shape)
    yield Problem("two-parts-nh-f64", 2, coords, conn, "neohookean", "lame", np.array([0.4]), np.array([0.6]),
                  up, "f64", part_elem=np.array([0, len(ta), len(conn)], np.int32),
                  part_node=np.array([0, len(ca), len(coords)], np.int32))


SMALL = list(small_problems())


# ------------------------------------------------------------------ prep
FULL = {2: lambda: config2(dtype="f32"), "2d": lambda: config2(dtype="f64"), 3: config3, 4: config4, 5: config5}


@pytest.mark.parametrize("prob", SMALL + [config1()] + [pytest.param(k, id=f"config{k}-full") for k in FULL])
def test_prepare_bitexact(orc, prob):
    """Preparation is bit-exact against the oracle (north star): the CSR (ptr, ent), the greedy
    colouring, the colour-sorted element list and its offsets; geometry within rounding.  Every
    BASELINE config at full size (configs 2 fp32 / fp64, 3, 4, 5) plus the small meshes."""
    if not isinstance(prob, Problem):
        prob = FULL[prob]()
    mesh, _, _ = gpu_problem(prob)
    ptr, ent = orc.csr(prob.conn, prob.n_nodes)
    assert np.array_equal(mesh.csr_ptr.cpu().numpy(), ptr)
    assert np.array_equal(mesh.csr_ent.cpu().numpy(), ent)
    col, nc = orc.colour(prob.conn, prob.n_nodes, ptr, ent)
    assert mesh.n_colours == nc
    assert np.array_equal(mesh.colour.cpu().numpy(), col)
    elems, cptr = orc.colour_sort(col, nc)
    assert np.array_equal(mesh.colour_elems.cpu().numpy(), elems)
    assert np.array_equal(mesh.colour_ptr[: nc + 1].cpu().numpy(), cptr)
    g, v, sgn = orc.geometry(prob.coords, prob.conn)
    d = prob.dim
    G = mesh.grad.double().cpu().numpy().reshape(d, d, -1).transpose(2, 0, 1)
    tol = 1e-14 if prob.dtype == "f64" else 1e-7
    assert rel_l2(G, g) < tol and rel_l2(mesh.vol.double().cpu().numpy(), v) < tol
    assert mesh.n_negative == int((sgn < 0).sum())


@pytest.mark.parametrize("order", ["input", "locality"])
@pytest.mark.parametrize("prob", SMALL[:3], ids=lambda p: p.name)
def test_plan_is_a_partition_of_the_csr(orc, prob, order):
    """Every (element, slot) entry appears exactly once, under the occurrence of its own
    node, inside its own block; occurrences of a block are sorted by node; exactly one
    owner per node (the block of its highest element position).  Blocks hold plan
    positions; elem_perm maps them to input elements (a permutation inside each part)."""
    mesh, _, _ = gpu_problem(prob, block_elems=97, elem_order=order)    # small blocks -> many boundaries
    P = mesh.plan_export()
    nv = prob.dim + 1
    be, bo, on, oe, le, pm = (P["blk_elem"], P["blk_occ"], P["occ_node"], P["occ_ent_ptr"], P["loc_ent"],
                              P["elem_perm"])
    assert np.array_equal(np.sort(pm), np.arange(prob.n_elems))
    if order == "input":
        assert np.array_equal(pm, np.arange(prob.n_elems))
    pe, _ = prob.parts()
    part_of = np.searchsorted(pe, np.arange(prob.n_elems), side="right") - 1
    assert np.array_equal(part_of[pm], part_of)          # positions stay inside their part
    seen = np.zeros(prob.n_elems * nv, np.int32)
    owners = np.zeros(prob.n_nodes, np.int32)
    for b in range(len(be) - 1):
        nodes = on[bo[b]:bo[b + 1]] & 0x1FFFFFFF
        assert np.all(np.diff(nodes) > 0)
        for o in range(bo[b], bo[b + 1]):
            n = on[o] & 0x1FFFFFFF
            if not (on[o] & 0x40000000):
                owners[n] += 1
            ents = le[oe[o]:oe[o + 1]].astype(np.int64)
            assert np.all(np.diff(ents) > 0)
            pos = be[b] * nv + ents
            assert np.all(pos < be[b + 1] * nv)
            glob = pm[pos // nv].astype(np.int64) * nv + pos % nv      # input (element, slot)
            assert np.all(prob.conn.reshape(-1)[glob] == n)
            seen[glob] += 1
    assert np.all(seen == 1)
    used = np.unique(prob.conn)
    assert np.all(owners[used] == 1)


@pytest.mark.parametrize("order", ["input", "locality"])
@pytest.mark.parametrize("prob", SMALL, ids=lambda p: p.name)
def test_element_order_energy_residual_tangent(orc, prob, order):
    """Both plan element orders give the oracle's W_e (in input element order), totals,
    residual and K.v, with element-wise materials gathered through the permutation."""
    import paper_2601_03086_b200 as pf
    mesh, mat, u = gpu_problem(prob, block_elems=61, elem_order=order)
    om = oracle_problem(orc, prob)
    ur = rounded(prob.u, prob.dtype)
    W_ref, tot_ref = om.energy(ur)
    r_ref = om.residual(ur)
    tot, W, r = pf.energy(mesh, mat, u, elem_energy=True, residual=True)
    v = rounded(np.random.default_rng(11).standard_normal(prob.u.shape) * 1e-2, prob.dtype)
    kv_ref = om.tangent(v, u=ur if prob.model == "neohookean" else None)
    kv = pf.tangent_apply(mesh, mat, torch.as_tensor(v, dtype=u.dtype, device="cuda"),
                          u=u if prob.model == "neohookean" else None)
    torch.cuda.synchronize()
    assert_field(W.cpu().numpy(), W_ref, prob.dtype, "W_e")
    assert_totals(tot.cpu().numpy(), tot_ref, np.abs(tot_ref), prob.dtype)
    assert_field(r.cpu().numpy(), r_ref, prob.dtype, "residual")
    assert_field(kv.cpu().numpy(), kv_ref, prob.dtype, "Kv")


# ------------------------------------------------------------------ energy / residual
def check_energy(orc, prob, mode, block_elems=0, f_ext=None):
    mesh, mat, u = gpu_problem(prob, block_elems=block_elems)
    om = oracle_problem(orc, prob)
    ur = rounded(prob.u, prob.dtype)
    fe = None if f_ext is None else rounded(f_ext, prob.dtype)
    W_ref, tot_ref = om.energy(ur, f_ext=fe)
    _, w_ref = om.energy(ur, want_elem=False) if fe is not None else (None, tot_ref)
    r_ref = om.residual(ur)
    import paper_2601_03086_b200 as pf
    ft = None if fe is None else torch.as_tensor(fe, dtype=u.dtype, device="cuda")
    tot, W, r = pf.energy(mesh, mat, u, f_ext=ft, elem_energy=True, residual=True, mode=mode)
    torch.cuda.synchronize()
    tol = TOL[prob.dtype]
    assert_field(W.cpu().numpy(), W_ref, prob.dtype, "W_e")
    # Pi = W - f.u: scale |W| + |f.u| (reading R32)
    assert_totals(tot.cpu().numpy(), tot_ref, np.abs(w_ref) + np.abs(w_ref - tot_ref), prob.dtype)
    assert_field(r.cpu().numpy(), r_ref, prob.dtype, "residual")
    r2 = pf.residual(mesh, mat, u, mode=mode)
    torch.cuda.synchronize()
    assert torch.equal(r2, r) or rel_l2(r2.cpu().numpy(), r_ref) < tol
    return mesh, mat, u


@pytest.mark.parametrize("mode", ["csr", "colour"])
@pytest.mark.parametrize("prob", SMALL + [config1()], ids=lambda p: p.name)
def test_energy_residual_small(orc, prob, mode):
    rng = np.random.default_rng(5)
    f = rng.standard_normal(prob.coords.shape) * 1e-2
    check_energy(orc, prob, mode, f_ext=f)
    check_energy(orc, prob, mode, block_elems=61)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_config2_full(orc, dtype):
    p = config2(dtype=dtype)
    check_energy(orc, p, "csr")


def test_config3_full(orc):
    check_energy(orc, config3(), "csr")


def test_config5_full(orc):
    check_energy(orc, config5(), "csr")


def test_config5_colour(orc):
    check_energy(orc, config5(), "colour")


# ------------------------------------------------------------------ tangent
def check_tangent(orc, prob, mode, mask=None, seed=9, block_elems=0):
    import paper_2601_03086_b200 as pf
    mesh, mat, u = gpu_problem(prob, block_elems=block_elems)
    om = oracle_problem(orc, prob)
    rng = np.random.default_rng(seed)
    v = rounded(rng.standard_normal(prob.u.shape), prob.dtype)
    ur = rounded(prob.u, prob.dtype)
    ref = om.tangent(v, u=ur if prob.model == "neohookean" else None, mask=mask)
    vt = torch.as_tensor(v, dtype=u.dtype, device="cuda")
    mt = None if mask is None else torch.as_tensor(mask, dtype=torch.uint8, device="cuda")
    Kv = pf.tangent_apply(mesh, mat, vt, u=u if prob.model == "neohookean" else None, mask=mt, mode=mode)
    torch.cuda.synchronize()
    assert_field(Kv.cpu().numpy(), ref, prob.dtype, "Kv")


@pytest.mark.parametrize("mode", ["csr", "colour"])
@pytest.mark.parametrize("prob", SMALL, ids=lambda p: p.name)
def test_tangent_small(orc, prob, mode):
    check_tangent(orc, prob, mode)
    check_tangent(orc, prob, mode, block_elems=53)
    mask = (np.random.default_rng(2).random(prob.n_nodes * prob.dim) < 0.2).astype(np.uint8)
    check_tangent(orc, prob, mode, mask=mask)


def test_config4_tangent_full(orc):
    p = config4()
    check_tangent(orc, p, "csr")
    check_tangent(orc, p, "csr", mask=p.mask)


def test_config3_tangent_full(orc):
    check_tangent(orc, config3(), "csr")


# ------------------------------------------------------------------ on-the-fly geometry (§8(f) row f4)
@pytest.mark.parametrize("prob", SMALL + [config1()], ids=lambda p: p.name)
def test_geometry_on_the_fly_small(orc, prob):
    """PFEM_GEOMETRY_ON_THE_FLY: grad N_a and V_e formed in fp64 from the coordinates inside the
    element pass (the prepare formula) give the oracle's W_e, totals, residual and
    K.v within the north-star bars, with element-wise materials, parts and masks."""
    import paper_2601_03086_b200 as pf
    mesh, mat, u = gpu_problem(prob)
    mesh.geometry = "on_the_fly"
    om = oracle_problem(orc, prob)
    ur = rounded(prob.u, prob.dtype)
    W_ref, tot_ref = om.energy(ur)
    tot, W, r = pf.energy(mesh, mat, u, elem_energy=True, residual=True)
    v = rounded(np.random.default_rng(12).standard_normal(prob.u.shape), prob.dtype)
    mask = (np.random.default_rng(4).random(prob.n_nodes * prob.dim) < 0.2).astype(np.uint8)
    kv_ref = om.tangent(v, u=ur if prob.model == "neohookean" else None, mask=mask)
    kv = pf.tangent_apply(mesh, mat, torch.as_tensor(v, dtype=u.dtype, device="cuda"),
                          u=u if prob.model == "neohookean" else None, mask=torch.as_tensor(mask, device="cuda"))
    torch.cuda.synchronize()
    assert_field(W.cpu().numpy(), W_ref, prob.dtype, "W_e otf")
    assert_totals(tot.cpu().numpy(), tot_ref, np.abs(tot_ref), prob.dtype)
    assert_field(r.cpu().numpy(), om.residual(ur), prob.dtype, "residual otf")
    assert_field(kv.cpu().numpy(), kv_ref, prob.dtype, "Kv otf")


@pytest.mark.parametrize("cfg", [4, 5])
def test_geometry_on_the_fly_full(orc, cfg):
    """On-the-fly geometry at full size: config-4 masked K.v (fp64) and config-5 fused E+R over
    64 parts (fp32) against the oracle."""
    if cfg == 4:
        p = config4()
        mesh, mat, u = gpu_problem(p)
        mesh.geometry = "on_the_fly"
        import paper_2601_03086_b200 as pf
        om = oracle_problem(orc, p)
        v = rounded(np.random.default_rng(9).standard_normal(p.u.shape), p.dtype)
        ref = om.tangent(v, mask=p.mask)
        kv = pf.tangent_apply(mesh, mat, torch.as_tensor(v, device="cuda"), mask=torch.as_tensor(p.mask, device="cuda"))
        torch.cuda.synchronize()
        assert_field(kv.cpu().numpy(), ref, p.dtype, "Kv otf config 4")
    else:
        p = config5()
        mesh, mat, u = gpu_problem(p)
        mesh.geometry = "on_the_fly"
        import paper_2601_03086_b200 as pf
        om = oracle_problem(orc, p)
        ur = rounded(p.u, p.dtype)
        W_ref, tot_ref = om.energy(ur)
        tot, W, r = pf.energy(mesh, mat, u, elem_energy=True, residual=True)
        torch.cuda.synchronize()
        assert_field(W.cpu().numpy(), W_ref, p.dtype, "W_e otf config 5")
        assert_totals(tot.cpu().numpy(), tot_ref, np.abs(tot_ref), p.dtype)
        assert_field(r.cpu().numpy(), om.residual(ur), p.dtype, "residual otf config 5")


# ------------------------------------------------------------------ determinism, flags
@pytest.mark.parametrize("mode", ["csr", "colour"])
def test_bitwise_deterministic(mode):
    import paper_2601_03086_b200 as pf
    p = SMALL[2]
    mesh, mat, u = gpu_problem(p, block_elems=100)
    outs = []
    for _ in range(3):
        tot, W, r = pf.energy(mesh, mat, u, elem_energy=True, residual=True, mode=mode)
        Kv = pf.tangent_apply(mesh, mat, u, u=u, mode=mode)
        torch.cuda.synchronize()
        outs.append((tot.clone(), W.clone(), r.clone(), Kv.clone()))
    for o in outs[1:]:
        for a, b in zip(o, outs[0]):
            assert torch.equal(a, b)


def test_inversion_flags():
    import paper_2601_03086_b200 as pf
    coords = np.array([[0., 0], [1, 0], [0, 1], [1, 1]])
    conn = np.array([[0, 1, 2], [1, 3, 2]], np.int32)
    u = np.zeros((1, 4, 2))
    u[0, 3] = [-1.5, -1.5]
    p = Problem("inv", 2, coords, conn, "neohookean", "lame", np.array([0.4]), np.array([0.6]), u, "f64")
    mesh, mat, ut = gpu_problem(p)
    flags = torch.zeros(4, dtype=torch.int32, device="cuda")
    tot, W, r = pf.energy(mesh, mat, ut, elem_energy=True, residual=True, flags=flags)
    torch.cuda.synchronize()
    f = flags.cpu().numpy()
    assert f[0] == 1 and f[1] == 1
    assert not np.isfinite(W[0, 1].item())
    # a following clean call reports zero
    tot, W, r = pf.energy(mesh, mat, torch.zeros_like(ut), residual=True, flags=flags)
    torch.cuda.synchronize()
    assert flags.cpu().numpy()[0] == 0 and flags.cpu().numpy()[1] == -1


# ------------------------------------------------------------------ invariants through the GPU path
def test_gpu_invariants_translation_and_patch():
    import paper_2601_03086_b200 as pf
    c3, t3 = kuhn_cube(9, brick=4)
    u = np.tile([0.3, -0.2, 0.1], (len(c3), 1))[None]
    p = Problem("tr", 3, c3, t3, "neohookean", "lame", np.array([0.4]), np.array([0.6]), u, "f64")
    mesh, mat, ut = gpu_problem(p)
    tot, W, r = pf.energy(mesh, mat, ut, elem_energy=True, residual=True)
    torch.cuda.synchronize()
    assert torch.all(W == 0) and torch.all(r == 0)
    A = np.array([[0.01, 0.02, 0.0], [-0.01, 0.03, 0.005], [0.0, 0.01, -0.02]])
    ua = torch.as_tensor((c3 @ A.T)[None], device="cuda")
    tot, W, r = pf.energy(mesh, mat, ua, residual=True)
    torch.cuda.synchronize()
    F = np.eye(3) + A
    J = np.linalg.det(F)
    psi = 0.3 * np.log(J) ** 2 - 0.4 * np.log(J) + 0.2 * (np.sum(F * F) - 3)
    assert abs(tot.item() - psi) < 1e-13 * psi
    rs = r[0].cpu().numpy()
    assert np.max(np.abs(rs.sum(0))) < 1e-15
    interior = np.all((c3 > 1e-9) & (c3 < 1 - 1e-9), axis=1)
    assert np.max(np.abs(rs[interior])) < 1e-15


# ------------------------------------------------------------------ CG
def test_cg_tiny_matches_oracle_and_dense(orc):
    import paper_2601_03086_b200 as pf
    p = config1()
    mesh, mat, _ = gpu_problem(p)
    om = oracle_problem(orc, p)
    f = torch.as_tensor(p.f_ext, device="cuda")
    mask = torch.as_tensor(p.mask, device="cuda")
    x0 = torch.zeros_like(f)
    for tol in (1e-8, 1e-12):
        x, rep = pf.cg(mesh, mat, f, x0, mask=mask, tol=tol)
        xo, ro = om.cg(p.f_ext, p.mask, np.zeros_like(p.f_ext), tol=tol)
        assert rep["converged"] and abs(rep["iterations"] - ro["iterations"]) <= 1
        assert rel_l2(x.cpu().numpy(), xo) < 10 * tol
        h = rep["history"]
        assert np.max(np.abs(h[:20] - ro["history"][:20]) / ro["history"][:20]) < 1e-6
    # exact start -> 0 iterations (skip rule)
    x1, rep1 = pf.cg(mesh, mat, f, x, mask=mask, tol=1e-8)
    assert rep1["iterations"] == 0 and rep1["converged"]


def assert_cg_count(rep, ro, spread):
    """Reading R18: |dk| <= 1 vs the default oracle, or inside the oracle's own spread over
    5 valid dot-product orderings (+-1); first 50 residual-history entries agree to 1e-6."""
    k = rep["iterations"]
    ok = abs(k - ro["iterations"]) <= 1 or (min(spread) - 1 <= k <= max(spread) + 1)
    assert ok, (k, ro["iterations"], spread)
    h, ho = rep["history"], ro["history"]
    m = min(50, len(h), len(ho))
    assert np.max(np.abs(h[:m] - ho[:m]) / ho[:m]) < 1e-6


@pytest.mark.parametrize("n", [12, 20])
def test_cg_config4_scaled(orc, n):
    """Config-4 recipe at n^3 nodes: iteration count vs the oracle (R18), zero and warm start."""
    import paper_2601_03086_b200 as pf
    from pfem_gen import small_cube_problem, warm_start
    p = small_cube_problem(n_nodes=n, brick=4)
    mesh, mat, _ = gpu_problem(p)
    om = oracle_problem(orc, p)
    f = torch.as_tensor(p.f_ext, device="cuda")
    mask = torch.as_tensor(p.mask, device="cuda")
    xs, _ = om.cg(p.f_ext, p.mask, np.zeros_like(p.f_ext), tol=1e-12, history=False)
    x0w = warm_start(xs, p.mask, seed=4004)
    for x0 in (np.zeros_like(p.f_ext), x0w):
        xo, ro = om.cg(p.f_ext, p.mask, x0, tol=1e-8)
        spread = om.cg_spread(p.f_ext, p.mask, x0, tol=1e-8)
        for mode in ("csr", "colour"):   # CSR: the pipelined iteration (§8(f) row f3)
            x, rep = pf.cg(mesh, mat, f, torch.as_tensor(x0, device="cuda"), mask=mask, tol=1e-8, mode=mode)
            assert rep["converged"] and ro["converged"]
            assert_cg_count(rep, ro, spread)
            assert rep["true_rel_res_final"] < 2e-8
            assert rel_l2(x.cpu().numpy(), xo) < 1e-6


def _golden_config4():
    import json
    import os
    g = os.path.join(os.path.dirname(__file__), "golden")
    with open(os.path.join(g, "config4_cg.json")) as fh:
        gold = json.load(fh)
    ustar = np.load(os.path.join(g, "config4_ustar_f32.npz"))["ustar"].astype(np.float64)
    return gold, ustar


@pytest.mark.parametrize("start", ["zero", "warm"])
def test_cg_config4_full_vs_oracle_golden(start):
    """Config 4 at full size (80^3 nodes, 2,958,234 tets, tol 1e-8): the
    GPU CG iteration count against the oracle's, stored by tests/golden/make_config4_cg.py (which
    calls only oracle/): |dk| <= 1 vs dot order 0, or inside the oracle's own spread over three
    dot orders +-1 (reading R18); the first 50 residual-history entries within 1e-6 relative; the
    true residual below the tolerance.  The warm start x0 = u* + 0.01 rms(u*) xi is rebuilt from
    the stored oracle u* (float32) with the same seed on both sides."""
    import paper_2601_03086_b200 as pf
    from pfem_gen import warm_start
    gold, ustar = _golden_config4()
    p = config4()
    mesh, mat, _ = gpu_problem(p)
    x0 = np.zeros_like(p.f_ext) if start == "zero" else warm_start(ustar.reshape(p.f_ext.shape), p.mask, seed=4004)
    f = torch.as_tensor(p.f_ext, device="cuda")
    mask = torch.as_tensor(p.mask, device="cuda")
    x, rep = pf.cg(mesh, mat, f, torch.as_tensor(x0, device="cuda"), mask=mask, tol=gold["tol"])
    g = gold[start]
    r0 = g["runs"]["0"]
    assert rep["converged"]
    k = rep["iterations"]
    lo, hi = g["spread"]
    assert abs(k - r0["iterations"]) <= 1 or lo - 1 <= k <= hi + 1, (k, r0["iterations"], g["spread"])
    h = rep["history"][:50]
    ho = np.asarray(r0["history50"])
    assert np.max(np.abs(h - ho[: len(h)]) / ho[: len(h)]) < 1e-6
    assert rep["true_rel_res_final"] < gold["tol"]
    assert abs(rep["rel_res0"] - r0["rel_res0"]) <= 1e-9 * r0["rel_res0"]


# ------------------------------------------------------------------ Newton (§8(f) row f1)
@pytest.mark.parametrize("order", ["input", "locality"])
def test_newton_matches_oracle(orc, order):
    """pfem_newton vs the oracle's Newton on a Neo-Hookean block (fp64): the same number of
    Newton steps, residual histories within 1e-9 relative while above the rounding floor, and
    the converged U within 1e-9 relative (inner CG at 1e-12)."""
    import paper_2601_03086_b200 as pf
    from pfem_gen import newton_block
    p = newton_block(7, traction=(0.05, 0.0, 0.02))
    mesh, mat, u = gpu_problem(p, elem_order=order)
    om = oracle_problem(orc, p)
    f = torch.as_tensor(p.f_ext, device="cuda")
    mask = torch.as_tensor(p.mask, device="cuda")
    tol = 1e-10
    ug, rg = pf.newton(mesh, mat, u[0], f_ext=f, mask=mask, tol=tol, cg_tol=1e-12)
    uo, ro = om.newton(p.u[0], p.f_ext, p.mask, tol=tol, cg_tol=1e-12)
    assert rg["converged"] and ro["converged"]
    assert rg["iterations"] == ro["iterations"], (rg["history"], ro["history"])
    ho, hg = ro["history"], rg["history"]
    big = ho > 1e-6 * ho[0]
    assert np.max(np.abs(hg[big] - ho[big]) / ho[big]) < 1e-9
    assert rel_l2(ug.cpu().numpy(), uo) < 1e-9
    # warm start from the converged solution: zero Newton steps
    _, r1 = pf.newton(mesh, mat, ug, f_ext=f, mask=mask, tol=10 * tol, cg_tol=1e-12)
    assert r1["iterations"] == 0 and r1["converged"]


def test_newton_linear_one_step_gpu(orc):
    """Linear model: one Newton step reaches the CG solution (config 1)."""
    import paper_2601_03086_b200 as pf
    p = config1()
    mesh, mat, _ = gpu_problem(p)
    f = torch.as_tensor(p.f_ext, device="cuda")
    mask = torch.as_tensor(p.mask, device="cuda")
    b = np.linalg.norm(p.f_ext.ravel() * (1 - p.mask))
    u, rep = pf.newton(mesh, mat, torch.zeros_like(f), f_ext=f, mask=mask, tol=1e-9 * b, cg_tol=1e-13)
    x, _ = pf.cg(mesh, mat, f, torch.zeros_like(f), mask=mask, tol=1e-13)
    assert rep["converged"] and rep["iterations"] == 1
    assert rel_l2(u.cpu().numpy(), x.cpu().numpy()) < 1e-10


def test_empty_and_tiny_parts(orc):
    """Parts with no elements (their nodes, if any, carry no stiffness) get zero totals; a
    one-element part and a large part in the same launch match the oracle (R23)."""
    import paper_2601_03086_b200 as pf
    ca, ta = square_t3(14, 11)
    cb, tb = square_t3(2, 2)
    tb = tb[:1]
    used = np.unique(tb)
    cb = cb[used]
    tb = np.searchsorted(used, tb).astype(np.int32)
    coords = np.concatenate([ca, cb + 2.0])
    conn = np.concatenate([ta, tb + len(ca)]).astype(np.int32)
    E, N = len(conn), len(coords)
    pe = np.array([0, 0, len(ta), len(ta), E, E], np.int32)       # parts 0, 2 and 4 are empty
    pn = np.array([0, 0, len(ca), len(ca), N, N], np.int32)
    rng = np.random.default_rng(9)
    u = 0.01 * rng.standard_normal((2,) + coords.shape)
    prob = Problem("parts-empty", 2, coords, conn, "neohookean", "lame", np.array([0.4]), np.array([0.6]), u,
                   "f64", part_elem=pe, part_node=pn)
    for order in ("input", "locality"):
        mesh, mat, ut = gpu_problem(prob, elem_order=order)
        om = oracle_problem(orc, prob)
        W_ref, tot_ref = om.energy(prob.u)
        tot, W, r = pf.energy(mesh, mat, ut, elem_energy=True, residual=True)
        torch.cuda.synchronize()
        t = tot.cpu().numpy()
        assert t.shape == (2, 5)
        assert np.all(t[:, [0, 2, 4]] == 0.0)
        assert max_rel(t[:, [1, 3]], tot_ref[:, [1, 3]]) < 1e-12
        assert rel_l2(r.cpu().numpy(), om.residual(prob.u)) < 1e-12


# ------------------------------------------------------------------ Jacobi PCG (§8(f) row f3)
@pytest.mark.parametrize("prob", SMALL[:4], ids=lambda p: p.name)
def test_tangent_diag_matches_oracle(orc, prob):
    """pfem_tangent_diag vs the oracle's textbook element-tangent diagonals (reading R27), with
    and without a Dirichlet mask, at the NH state u (first sample)."""
    import paper_2601_03086_b200 as pf
    mesh, mat, u = gpu_problem(prob)
    om = oracle_problem(orc, prob)
    us = u[0] if prob.model == "neohookean" else None
    uo = rounded(prob.u[0], prob.dtype) if prob.model == "neohookean" else None
    rng = np.random.default_rng(9)
    for mk in (None, (rng.random(prob.n_nodes * prob.dim) < 0.1).astype(np.uint8)):
        mt = None if mk is None else torch.as_tensor(mk, device="cuda")
        d = pf.tangent_diag(mesh, mat, u_state=us, mask=mt)
        do = om.tangent_diag(u=uo, mask=mk)
        assert rel_l2(d.cpu().numpy(), do) < TOL[prob.dtype]
        if mk is not None:
            assert np.all(d.cpu().numpy().ravel()[mk == 1] == 1.0)


@pytest.mark.parametrize("n", [12])
def test_pcg_config4_scaled(orc, n):
    """Jacobi PCG on the config-4 recipe at n^3 nodes (fp64) vs the oracle PCG: iteration count
    within +-1 or the R18 spread of the unpreconditioned oracle, histories within 1e-6 over the
    first 50 iterations, true residual below tol; zero and warm start, both assembly modes."""
    import paper_2601_03086_b200 as pf
    from pfem_gen import small_cube_problem, warm_start
    p = small_cube_problem(n_nodes=n, brick=4)
    mesh, mat, _ = gpu_problem(p)
    om = oracle_problem(orc, p)
    f = torch.as_tensor(p.f_ext, device="cuda")
    mask = torch.as_tensor(p.mask, device="cuda")
    xs, _ = om.cg(p.f_ext, p.mask, np.zeros_like(p.f_ext), tol=1e-12, history=False)
    x0w = warm_start(xs, p.mask, seed=4004)
    for x0 in (np.zeros_like(p.f_ext), x0w):
        xo, ro = om.pcg(p.f_ext, p.mask, x0, tol=1e-8)
        assert ro["converged"]
        spread = om.pcg_spread(p.f_ext, p.mask, x0, tol=1e-8)
        for mode in ("csr", "colour"):
            x, rep = pf.cg(mesh, mat, f, torch.as_tensor(x0, device="cuda"), mask=mask, tol=1e-8, mode=mode,
                           precond="jacobi")
            assert rep["converged"]
            # reading R18 with the oracle PCG's own spread over the five dot orders
            assert_cg_count(rep, ro, spread)
            assert rep["true_rel_res_final"] < 2e-8
            assert rel_l2(x.cpu().numpy(), xo) < 1e-6
    # precond "none" through pfem_pcg is pfem_cg
    x1, r1 = pf.cg(mesh, mat, f, torch.zeros_like(f), mask=mask, tol=1e-8, precond="none")
    x2, r2 = pf.cg(mesh, mat, f, torch.zeros_like(f), mask=mask, tol=1e-8)
    assert r1["iterations"] == r2["iterations"] and torch.equal(x1, x2)


def test_pcg_neohookean_state(orc):
    """Jacobi PCG on the NH tangent at a non-trivial state (the Newton inner solve) vs the
    oracle PCG (fp64)."""
    import paper_2601_03086_b200 as pf
    from pfem_gen import newton_block
    p = newton_block(6, traction=(0.05, 0.0, 0.02))
    mesh, mat, _ = gpu_problem(p)
    om = oracle_problem(orc, p)
    rng = np.random.default_rng(21)
    us = 0.02 * fourier_field(p.coords, rng) * (1 - p.mask.reshape(p.coords.shape))
    f = torch.as_tensor(p.f_ext, device="cuda")
    mask = torch.as_tensor(p.mask, device="cuda")
    x, rep = pf.cg(mesh, mat, f, torch.zeros_like(f), mask=mask, tol=1e-10, u_state=torch.as_tensor(us, device="cuda"),
                   precond="jacobi")
    xo, ro = om.pcg(p.f_ext, p.mask, np.zeros_like(p.f_ext), tol=1e-10, u_state=us)
    assert rep["converged"] and ro["converged"]
    assert_cg_count(rep, ro, om.pcg_spread(p.f_ext, p.mask, np.zeros_like(p.f_ext), tol=1e-10, u_state=us))
    assert rel_l2(x.cpu().numpy(), xo) < 1e-8


# ------------------------------------------------------------------ pretraining loss (§8(f) row f2)
@pytest.mark.parametrize("prob", [SMALL[1], SMALL[2], SMALL[4]], ids=lambda p: p.name)
@pytest.mark.parametrize("with_phi", [True, False])
def test_pretrain_loss_matches_oracle(orc, prob, with_phi):
    """pfem_pretrain_loss vs the oracle: u = phi (.) H with phi = x_1 / L (distance to the
    clamped edge x_1 = min, broadcast over components; R28), Pi per (sample, part), the batch
    mean loss and dloss/dH = phi (.) (f_int - f_ext) / (S K)."""
    import paper_2601_03086_b200 as pf
    mesh, mat, H = gpu_problem(prob)
    om = oracle_problem(orc, prob)
    x = prob.coords[:, 0]
    phi = np.repeat(((x - x.min()) / (x.max() - x.min()))[:, None], prob.dim, axis=1) if with_phi else None
    rng = np.random.default_rng(17)
    f = 1e-3 * rng.standard_normal(prob.coords.shape)
    fr, phr = rounded(f, prob.dtype), None if phi is None else rounded(phi, prob.dtype)
    dt = H.dtype
    lo, Po, go, uo = om.pretrain_loss(rounded(prob.u, prob.dtype), phr, fr)
    _, Wo = om.energy(uo, want_elem=False)
    scale = np.abs(Wo) + np.abs(Wo - Po)                      # |W| + |f.u| (reading R32)
    tol = TOL[prob.dtype]
    for mode in ("csr", "colour"):   # CSR: epilogue fused into the assembly writes; COLOUR: own pass
        loss, tot, grad, u = pf.pretrain_loss(mesh, mat, H, mode=mode,
                                              phi=None if phi is None else torch.as_tensor(phr, dtype=dt, device="cuda"),
                                              f_ext=torch.as_tensor(fr, dtype=dt, device="cuda"))
        assert_field(u.cpu().numpy(), uo, prob.dtype, "u")
        assert_totals(tot.cpu().numpy(), Po, scale, prob.dtype, "Pi")
        assert abs(float(loss) - lo) <= tol * float(scale.mean())   # loss = mean of Pi
        assert_field(grad.cpu().numpy(), go, prob.dtype, "dloss/dH")


# ------------------------------------------------------------------ large blocks (direct form)
@pytest.mark.parametrize("prob", SMALL, ids=lambda p: p.name)
def test_large_blocks_direct_form(orc, prob):
    """Blocks above the staged kernel's capacity (T4 > 256, T3 > 512 elements) are served by the
    direct form for every sample count: energy, residual and K.v (masked) still match the oracle."""
    be = 700 if prob.dim == 3 else 1200
    check_energy(orc, prob, "csr", block_elems=be)
    mask = (np.random.default_rng(3).random(prob.n_nodes * prob.dim) < 0.2).astype(np.uint8)
    check_tangent(orc, prob, "csr", mask=mask, block_elems=be)


# ------------------------------------------------------------------ edge cases
def test_prepare_errors_and_single_element(orc):
    """Degenerate element -> PFEM_ERR_DEGENERATE with its index; connectivity out of range ->
    PFEM_ERR_ARG with the element; a one-element mesh matches the oracle (and the golden
    single-element values of tests/golden/single_element.json via the oracle pins)."""
    import paper_2601_03086_b200 as pf
    from paper_2601_03086_b200 import PfemError
    dev = "cuda"
    coords = torch.tensor([[0., 0], [1, 0], [0, 1], [2, 0]], dtype=torch.float64, device=dev)
    bad = torch.tensor([[0, 1, 2], [0, 1, 3]], dtype=torch.int32, device=dev)      # element 1 collinear
    with pytest.raises(PfemError) as ei:
        pf.Mesh(coords, bad)
    assert ei.value.status == -2 and ei.value.index == 1
    oob = torch.tensor([[0, 1, 2], [1, 2, 7]], dtype=torch.int32, device=dev)
    with pytest.raises(PfemError) as ei:
        pf.Mesh(coords, oob)
    assert ei.value.status == -1 and ei.value.index == 1
    # one element, NH fp64, 3 samples (staged) and 1 sample (direct)
    c1 = np.array([[0., 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]])
    t1 = np.array([[0, 1, 2, 3]], np.int32)
    rng = np.random.default_rng(8)
    for S in (3, 1):
        u = 0.05 * rng.standard_normal((S, 4, 3))
        p = Problem("one-tet", 3, c1, t1, "neohookean", "lame", np.array([0.4]), np.array([0.6]), u, "f64")
        check_energy(orc, p, "csr")
        check_tangent(orc, p, "csr")


def test_cg_edge_cases(orc):
    """Zero right-hand side with zero prescribed values -> x = 0 after 0 iterations; every DOF
    constrained -> x = x0 (prescribed) after 0 iterations; max_iter reached ->
    PFEM_ERR_NOT_CONVERGED (status -4) with the partial iterate and a filled report."""
    import paper_2601_03086_b200 as pf
    p = config1()
    mesh, mat, _ = gpu_problem(p)
    f = torch.as_tensor(p.f_ext, device="cuda")
    mask = torch.as_tensor(p.mask, device="cuda")
    x, rep = pf.cg(mesh, mat, torch.zeros_like(f), torch.zeros_like(f), mask=mask, tol=1e-8)
    assert rep["iterations"] == 0 and rep["converged"] and torch.count_nonzero(x) == 0
    allm = torch.ones_like(mask)
    x0 = torch.as_tensor(np.random.default_rng(1).standard_normal(p.f_ext.shape), device="cuda")
    x, rep = pf.cg(mesh, mat, f, x0, mask=allm, tol=1e-8)
    assert rep["iterations"] == 0 and torch.equal(x, x0)
    x, rep = pf.cg(mesh, mat, f, torch.zeros_like(f), mask=mask, tol=1e-12, max_iter=3)
    assert rep["status"] == -4 and not rep["converged"] and rep["iterations"] == 3
    xo, ro = oracle_problem(orc, p).cg(p.f_ext, p.mask, np.zeros_like(p.f_ext), tol=1e-12, max_iter=3)
    assert rel_l2(x.cpu().numpy(), xo) < 1e-10


# ------------------------------------------------------------------ heat conduction (§8(f) row f4)
@pytest.mark.parametrize("prob", SMALL, ids=lambda p: p.name)
def test_heat_matches_oracle(orc, prob):
    """pfem_heat (the paper's scalar example) vs the oracle: W_e, per-part totals with nodal
    loads, and the CSR-ordered fluxes, on the small problems' meshes (one and two parts, T3 /
    T4, fp32 / fp64), three temperature fields with per-element conductivity."""
    import paper_2601_03086_b200 as pf
    mesh, _, _ = gpu_problem(prob)
    om = oracle_problem(orc, prob)
    rng = np.random.default_rng(31)
    T = rounded(np.sin(3 * prob.coords[:, 0])[None] + 0.1 * rng.standard_normal((3, prob.n_nodes)), prob.dtype)
    k = rounded(np.exp(0.5 * rng.standard_normal(prob.n_elems)), prob.dtype)
    f = rounded(0.01 * rng.standard_normal(prob.n_nodes), prob.dtype)
    dt = {"f32": torch.float32, "f64": torch.float64}[prob.dtype]
    W, tot, r = pf.heat(mesh, torch.as_tensor(k, dtype=dt, device="cuda"), torch.as_tensor(T, dtype=dt, device="cuda"),
                        f=torch.as_tensor(f, dtype=dt, device="cuda"))
    Wo, toto, ro = om.heat(T, k, f=f)
    _, wo, _ = om.heat(T, k)
    scale = np.abs(wo) + np.abs(wo - toto)                    # |W| + |f.T| (reading R32)
    tol = TOL[prob.dtype]
    assert_field(W.cpu().numpy(), Wo, prob.dtype, "W_e")
    assert_totals(tot.cpu().numpy(), toto, scale, prob.dtype)
    assert_field(r.cpu().numpy(), ro, prob.dtype, "flux")
    # geometry formed on the fly from the coordinates (f4 variant): same results within the bar
    W2, tot2, r2 = pf.heat(mesh, torch.as_tensor(k, dtype=dt, device="cuda"), torch.as_tensor(T, dtype=dt, device="cuda"),
                           f=torch.as_tensor(f, dtype=dt, device="cuda"), geometry_on_the_fly=True)
    assert_field(W2.cpu().numpy(), Wo, prob.dtype, "W_e otf")
    assert_field(r2.cpu().numpy(), ro, prob.dtype, "flux otf")
    assert_totals(tot2.cpu().numpy(), toto, scale, prob.dtype)
    # uniform conductivity (stride 0)
    W1, _, r1 = pf.heat(mesh, torch.tensor([1.5], dtype=dt, device="cuda"), torch.as_tensor(T, dtype=dt, device="cuda"))
    Wo1, _, ro1 = om.heat(T, [1.5])
    assert rel_l2(r1.cpu().numpy(), ro1) < tol and rel_l2(W1.cpu().numpy(), Wo1) < tol


def test_staged_items_multi_part_ragged_samples(orc):
    """The staged form's (block, sample chunk) items on a two-part mesh with a ragged last chunk
    (S = 6 fp32: chunks of 4 + 2; S = 5 fp64: 2 + 2 + 1): W_e, per-(sample, part) totals with
    nodal loads, the residual and K.v match the oracle."""
    rng = np.random.default_rng(41)
    ca, ta = square_t3(31, 19)
    cb, tb = square_t3(13, 37)
    coords = np.concatenate([ca, cb + 3.0])
    conn = np.concatenate([ta, tb + len(ca)]).astype(np.int32)
    pe = np.array([0, len(ta), len(conn)], np.int32)
    pn = np.array([0, len(ca), len(coords)], np.int32)
    for S, dt in ((6, "f32"), (5, "f64")):
        u = np.stack([0.05 * fourier_field(coords, rng) for _ in range(S)])
        p = Problem(f"two-parts-S{S}-{dt}", 2, coords, conn, "neohookean", "lame", rng.uniform(0.3, 1.0, len(conn)),
                    rng.uniform(0.3, 1.0, len(conn)), u, dt, part_elem=pe, part_node=pn)
        f = rng.standard_normal(coords.shape) * 1e-2
        check_energy(orc, p, "csr", f_ext=f)
        check_tangent(orc, p, "csr")


def test_inversion_flags_staged_items():
    """Inversion counts through the staged (block, sample chunk) items: S = 7 fp32 fields on a
    small T4 block, two of them inverting element 0 (J <= 0): n_inverted counts every
    (element, sample) with J <= 0, first_inverted is element 0, and the non-inverted samples'
    energies stay finite."""
    import paper_2601_03086_b200 as pf
    coords, conn = kuhn_cube(4)
    S = 7
    u = np.zeros((S,) + coords.shape)
    c0 = conn[0]
    for s in (2, 5):   # flatten element 0 through its vertex 1 (beyond the opposite face)
        d = coords[c0[1]] - coords[c0[0]]
        u[s, c0[1]] = -2.0 * d
    p = Problem("inv-staged", 3, coords, conn, "neohookean", "lame", np.array([0.4]), np.array([0.6]), u, "f32")
    mesh, mat, ut = gpu_problem(p)
    flags = torch.zeros(4, dtype=torch.int32, device="cuda")
    tot, W, r = pf.energy(mesh, mat, ut, elem_energy=True, residual=True, flags=flags)
    torch.cuda.synchronize()
    f = flags.cpu().numpy()
    Wn = W.cpu().numpy()
    bad = ~np.isfinite(Wn)
    assert f[0] == int(bad.sum()) and f[0] >= 2 and f[1] == 0
    assert np.all(np.isfinite(Wn[[0, 1, 3, 4, 6]]))


# ------------------------------------------------------------------ Q4 / Q8 elements (§8(f) row f4)
def quad_problem(kind, dtype, model="neohookean", S=3, seed=61, n_cells=None):
    from pfem_gen import beam_q4, cook_q8
    p = (beam_q4 if kind == "q4" else cook_q8)(**({"n_cells": n_cells} if n_cells else {}), dtype=dtype)
    rng = np.random.default_rng(seed)
    L = np.ptp(p.coords, axis=0).max()
    p.u = np.stack([0.02 * L * fourier_field(p.coords / L, rng) for _ in range(S)])
    p.model = model
    return p


def quad_gpu(p, dtype=None):
    import paper_2601_03086_b200 as pf
    dt = {"f32": torch.float32, "f64": torch.float64}[dtype or p.dtype]
    mesh = pf.Mesh(torch.as_tensor(p.coords, device="cuda"), torch.as_tensor(p.conn, device="cuda"), dtype=dt,
                   elem_type=p.elem)
    mat = pf.Material(p.model, p.param_kind, torch.as_tensor(np.asarray(p.p0), dtype=dt, device="cuda"),
                      torch.as_tensor(np.asarray(p.p1), dtype=dt, device="cuda"))
    return mesh, mat, torch.as_tensor(p.u, dtype=dt, device="cuda")


def quad_oracle(orc, p):
    return orc.prepare_quad(p.elem, p.coords, p.conn, p.model, p.param_kind, rounded(p.p0, p.dtype),
                            rounded(p.p1, p.dtype))


@pytest.mark.parametrize("kind", ["q4", "q8"])
def test_quad_prepare_bitexact(orc, kind):
    """Q4 / Q8 meshes: the CSR and the greedy colouring are bit-exact with the oracle's
    definitions (reading R12 with d+1 replaced by the element's node count)."""
    p = quad_problem(kind, "f64")
    mesh, _, _ = quad_gpu(p)
    ptr, ent = orc.csr(p.conn, p.n_nodes)
    assert np.array_equal(mesh.csr_ptr.cpu().numpy(), ptr) and np.array_equal(mesh.csr_ent.cpu().numpy(), ent)
    col, nc = orc.colour(p.conn, p.n_nodes, ptr, ent)
    assert mesh.n_colours == nc and np.array_equal(mesh.colour.cpu().numpy(), col)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("model", ["linear", "neohookean"])
@pytest.mark.parametrize("kind", ["q4", "q8"])
def test_quad_energy_residual_tangent(orc, kind, model, dtype):
    """Beam (50 x 50 Q4) and Cook (30 x 30 Q8) meshes, three displacement fields,
    element-wise (E, nu): W_e, totals with nodal loads, the residual and the masked K.v against the
    Gauss-quadrature oracle within the north-star bars."""
    import paper_2601_03086_b200 as pf
    p = quad_problem(kind, dtype, model)
    mesh, mat, u = quad_gpu(p)
    om = quad_oracle(orc, p)
    ur = rounded(p.u, dtype)
    fe = rounded(p.f_ext, dtype)
    W_ref, tot_ref = om.energy(ur, f_ext=fe)
    _, w_ref = om.energy(ur, want_elem=False)
    tot, W, r = pf.energy(mesh, mat, u, f_ext=torch.as_tensor(fe, dtype=u.dtype, device="cuda"), elem_energy=True,
                          residual=True)
    v = rounded(np.random.default_rng(5).standard_normal(p.u.shape), dtype)
    Kv = pf.tangent_apply(mesh, mat, torch.as_tensor(v, dtype=u.dtype, device="cuda"),
                          u=u if model == "neohookean" else None, mask=torch.as_tensor(p.mask, device="cuda"))
    torch.cuda.synchronize()
    assert_field(W.cpu().numpy(), W_ref, dtype, "W_e")
    assert_totals(tot.cpu().numpy(), tot_ref, np.abs(w_ref) + np.abs(w_ref - tot_ref), dtype)
    assert_field(r.cpu().numpy(), om.residual(ur), dtype, "residual")
    ref = om.tangent(v, u=ur if model == "neohookean" else None, mask=p.mask)
    assert_field(Kv.cpu().numpy(), ref, dtype, "Kv")


@pytest.mark.parametrize("kind", ["q4", "q8"])
def test_quad_newton_matches_oracle(orc, kind):
    """Newton warm start on the hyperelastic beam (Q4) and Cook's membrane (Q8) at reduced size
    (App. B): the same number of Newton steps as the oracle, residual
    histories within 1e-9 above the rounding floor, U within 1e-9; a converged start takes 0 steps."""
    import paper_2601_03086_b200 as pf
    from pfem_gen import beam_q4, cook_q8
    p = (beam_q4 if kind == "q4" else cook_q8)(n_cells=12)
    mesh, mat, u = quad_gpu(p)
    om = quad_oracle(orc, p)
    f = torch.as_tensor(p.f_ext, device="cuda")
    mask = torch.as_tensor(p.mask, device="cuda")
    tol = 1e-10 * float(np.linalg.norm(p.f_ext))
    ug, rg = pf.newton(mesh, mat, u[0], f_ext=f, mask=mask, tol=tol, cg_tol=1e-12)
    uo, ro = om.newton(p.u[0], p.f_ext, p.mask, tol=tol, cg_tol=1e-12)
    assert rg["converged"] and ro["converged"] and rg["iterations"] == ro["iterations"] >= 2
    ho, hg = ro["history"], rg["history"]
    # relative 1e-9, plus the rounding floor of r = f_int - f_ext (1e-11 of the initial residual:
    # the converged entries are rounding noise of a cancellation, ~1e-12 of ||r_0|| on both sides)
    assert np.all(np.abs(hg - ho) <= 1e-9 * ho + 1e-11 * ho[0]), (hg, ho)
    assert rel_l2(ug.cpu().numpy(), uo) < 1e-9
    _, r1 = pf.newton(mesh, mat, ug, f_ext=f, mask=mask, tol=10 * tol, cg_tol=1e-12)
    assert r1["iterations"] == 0


def test_bitwise_deterministic_all_paths():
    """Every kernel family is bitwise reproducible run to run (no float atomics, fixed orders;
    also the race check of the checked-build suite: a data race would perturb the bits): the
    staged form with a ragged sample chunk, the direct form, on-the-fly geometry, the pipelined
    CG (the solution), Jacobi PCG, the pretraining epilogue and the Q4 / Q8 path."""
    import paper_2601_03086_b200 as pf
    from pfem_gen import beam_q4, small_cube_problem
    rng = np.random.default_rng(123)
    c, t, _ = plate_with_holes(30, np.random.default_rng(4))
    mesh = pf.Mesh(torch.as_tensor(c, device="cuda"), torch.as_tensor(t, device="cuda"), dtype=torch.float32,
                   block_elems=150)
    mat = pf.Material("neohookean", "lame", torch.as_tensor(rng.uniform(0.3, 1, len(t)), dtype=torch.float32, device="cuda"),
                      torch.as_tensor(rng.uniform(0.3, 1, len(t)), dtype=torch.float32, device="cuda"))
    u5 = torch.as_tensor(np.stack([0.05 * fourier_field(c, rng) for _ in range(5)]), dtype=torch.float32, device="cuda")
    f = torch.as_tensor(0.01 * rng.standard_normal(c.shape), dtype=torch.float32, device="cuda")
    p4 = small_cube_problem(n_nodes=10, brick=4)
    m4, mat4, _ = gpu_problem(p4)
    f4, mk4 = torch.as_tensor(p4.f_ext, device="cuda"), torch.as_tensor(p4.mask, device="cuda")
    pq = beam_q4(n_cells=10)
    mq = pf.Mesh(torch.as_tensor(pq.coords, device="cuda"), torch.as_tensor(pq.conn, device="cuda"), elem_type="q4")
    matq = pf.Material(pq.model, pq.param_kind, torch.as_tensor(pq.p0, device="cuda"), torch.as_tensor(pq.p1, device="cuda"))
    uq = torch.as_tensor(0.01 * rng.standard_normal((2,) + pq.coords.shape), device="cuda")

    def run():
        out = []
        out += list(pf.energy(mesh, mat, u5, f_ext=f, elem_energy=True, residual=True))
        out += list(pf.energy(mesh, mat, u5[:1], elem_energy=True, residual=True))
        mesh.geometry = "on_the_fly"
        out += list(pf.energy(mesh, mat, u5[:1], elem_energy=True, residual=True))
        mesh.geometry = "stored"
        out.append(pf.tangent_apply(mesh, mat, u5, u=u5))
        out += list(pf.pretrain_loss(mesh, mat, u5, f_ext=f)[:3])
        out.append(pf.cg(m4, mat4, f4, torch.zeros_like(f4), mask=mk4, tol=1e-8)[0])
        out.append(pf.cg(m4, mat4, f4, torch.zeros_like(f4), mask=mk4, tol=1e-8, precond="jacobi")[0])
        out += list(pf.energy(mq, matq, uq, elem_energy=True, residual=True))
        out.append(pf.tangent_apply(mq, matq, uq, u=uq))
        torch.cuda.synchronize()
        return [o.clone() for o in out]

    ref = run()
    for _ in range(2):
        for a, b in zip(run(), ref):
            assert torch.equal(a, b)


def test_fma_peak_diagnostic():
    """pfem_fma_peak: the measured FMA-pipe rates are positive and below what
    148 SMs x 128 lanes at 2.2 GHz could issue; the packed FFMA2 form is at least as fast as the
    scalar FFMA form (measured on B200: both reach the same ~36 T lane-FMA/s, FFMA2 in half the
    issue slots); fp64 runs at about half the fp32 rate."""
    import paper_2601_03086_b200 as pf
    p1, p2, p64 = pf.fma_peak("ffma"), pf.fma_peak("ffma2"), pf.fma_peak("dfma")
    cap = 148 * 128 * 2.2e9
    assert 1e12 < p1 < cap and 1e12 < p2 < cap * 1.01
    assert 0.9 < p2 / p1 < 2.5
    assert 1e11 < p64 <= p1 * 1.05
