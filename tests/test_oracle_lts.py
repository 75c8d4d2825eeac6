"""Pins for the FB-LTS oracle (P1-P5, P14, P16, P21, P22, P23)."""
import collections
import json
import os

import numpy as np
import pytest

from inputs.configs import config1, small_shelf
from inputs.hexmesh import build_periodic_hex_mesh
from oracle import diagnostics as dg
from oracle import fbrk32, lts

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


@pytest.fixture(scope="module")
def cfg1():
    c = config1(dt=80.0)
    return c, lts.label_regions(c.mesh, c.fine_mask)


@pytest.fixture(scope="module")
def shelf():
    c = small_shelf(nx=40, ny=36, dt=12.0)
    return c, lts.label_regions(c.mesh, c.fine_mask)


def phys_of(c, slow=True):
    return fbrk32.Phys(g=c.g, beta=c.beta, slow=slow, tau_n=c.tau_n, rho0=c.rho0)


# ---------------------------------------------------------------- P1, P2
@pytest.mark.parametrize("which", ["cfg1", "shelf"])
def test_M1_equals_global_bitwise(which, cfg1, shelf):
    """P1: with M = 1 the predictions are exactly the coarse data, so FB-LTS is FB-RK(3,2)
    (reading Q13: bitwise) -- on any labels."""
    c, lab = cfg1 if which == "cfg1" else shelf
    phys = phys_of(c)
    h, u = c.h0.copy(), c.u0.copy()
    hg, ug = c.h0.copy(), c.u0.copy()
    for _ in range(5):
        h, u = lts.fblts_step(c.mesh, lab, h, u, c.dt, 1, phys)
        hg, ug = fbrk32.fbrk32_step(c.mesh, hg, ug, c.dt, phys)
    assert np.array_equal(h, hg) and np.array_equal(u, ug)


def test_no_fine_cells_equals_global_bitwise(cfg1):
    """P2: an empty fine region labels everything C^int; the step is global FB-RK(3,2)."""
    c, _ = cfg1
    lab = lts.label_regions(c.mesh, np.zeros(c.mesh.nCells, bool))
    assert np.all(lab.cell == lts.INT) and np.all(lab.edge == lts.INT)
    phys = phys_of(c)
    h, u = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 4, phys, 3)
    hg, ug = c.h0.copy(), c.u0.copy()
    for _ in range(3):
        hg, ug = fbrk32.fbrk32_step(c.mesh, hg, ug, c.dt, phys)
    assert np.array_equal(h, hg) and np.array_equal(u, ug)


# ---------------------------------------------------------------- P3, P4
@pytest.mark.parametrize("M", [1, 2, 3, 4, 8])
def test_predictor_exact_for_linear_data(M):
    """P3: data sampled from p(t) = al + be t reproduce p at t^{n,k}, t^{n,k+1/3}, t^{n,k+1/2}
    (eq. preds; App. A derivation P:L60-222), coefficients sum to 1."""
    dt = 7.0
    al, be = np.array([3.0, -1.25]), np.array([0.5, 2.0])
    p = lambda t: al + be * t
    for k in range(M + 1):
        co = lts.pred_coeffs(min(k, M - 1), M)
        lvl = lts.predict_level(co, p(dt), p(0.0), k)
        np.testing.assert_allclose(lvl, p(k * dt / M), rtol=4e-16 * 4, atol=4e-16 * 8)
        if k < M:
            assert co["a"] + co["b"] + co["c"] == pytest.approx(1.0, abs=1e-15)
            s1 = lts.predict_stage(co, p(dt), p(dt / 3), p(0.0))
            s2 = lts.predict_stage(co, p(dt), p(dt / 2), p(0.0))
            np.testing.assert_allclose(s1, p((k + 1 / 3) * dt / M), rtol=1e-15, atol=1e-14)
            np.testing.assert_allclose(s2, p((k + 1 / 2) * dt / M), rtol=1e-15, atol=1e-14)


def test_predictor_worked_examples():
    """M = 4, k = 2 -> level (1/2, 1/2), stage (1/2, 1/4, 1/4); M = 1 is the identity;
    h* = b1 * 2 + (1 - b1) * 1 = 1.531 (eq. hstar_preds)."""
    g = GOLD["predict_M4_k2"]
    co = lts.pred_coeffs(g["k"], g["M"])
    assert [co["a"], co["b"], co["c"]] == g["stage"]
    assert [g["k"] / g["M"], 1.0 - g["k"] / g["M"]] == g["level"]
    co1 = lts.pred_coeffs(0, 1)
    x = np.array([1.7, -2.3])
    assert np.array_equal(lts.predict_stage(co1, x + 5, x, x - 9), x)
    assert np.array_equal(lts.predict_level(co1, x + 5, x, 0), x)
    assert np.array_equal(lts.predict_level(co1, x + 5, x, 1), x + 5)
    hs = GOLD["hstar"]
    assert hs["beta1"] * hs["pred"] + (1 - hs["beta1"]) * hs["base"] == pytest.approx(hs["hstar"], abs=1e-15)


def test_prediction_gap_second_order(shelf):
    """P4: the gap between the predicted IF data (from coarse stage data) and the stage values a
    fine-step FB-RK(3,2) actually computes shrinks like dt^2 (App. A: second-order predictor)."""
    c, _ = shelf
    phys = phys_of(c, slow=False)
    m = c.mesh
    h, u = c.h0.copy(), c.u0.copy()
    for _ in range(10):
        h, u = fbrk32.fbrk32_step(m, h, u, 10.0, phys)
    M = 4
    gaps = []
    for dt in (2.0, 1.0, 0.5):
        _, _, st = fbrk32.fbrk32_step(m, h, u, dt, phys, stages=True)
        hk, uk = h.copy(), u.copy()
        gap = 0.0
        for k in range(M):
            co = lts.pred_coeffs(k, M)
            hn, un, fs = fbrk32.fbrk32_step(m, hk, uk, dt / M, phys, stages=True)
            gap = max(gap,
                      np.max(np.abs(lts.predict_level(co, st["h3"], h, k) - hk)),
                      np.max(np.abs(lts.predict_stage(co, st["h3"], st["h1"], h) - fs["h1"])),
                      np.max(np.abs(lts.predict_stage(co, st["h3"], st["h2"], h) - fs["h2"])),
                      np.max(np.abs(lts.predict_stage(co, st["u3"], st["u2"], u) - fs["u2"])))
            hk, uk = hn, un
        gaps.append(gap)
    r1, r2 = gaps[0] / gaps[1], gaps[1] / gaps[2]
    assert 3.4 < r1 < 4.6 and 3.4 < r2 < 4.6, gaps


# ---------------------------------------------------------------- P5
@pytest.mark.parametrize("M", [1, 2, 4])
@pytest.mark.parametrize("which", ["cfg1", "shelf"])
def test_mass_conservation(which, M, cfg1, shelf):
    """P5 / Theorem 1: sum_i A_i h_i is constant to roundoff for any M and labels;
    the diagnostic absolute vorticity (Theorem 2 statement) likewise."""
    c, lab = cfg1 if which == "cfg1" else shelf
    phys = phys_of(c)
    m = c.mesh
    m0, G0 = dg.total_mass(m, c.h0), dg.total_abs_vorticity(m, c.u0)
    h, u = lts.run(m, lab, c.h0, c.u0, c.dt, M, phys, 40)
    assert np.all(np.isfinite(h)) and np.all(np.isfinite(u))
    assert abs(dg.total_mass(m, h) - m0) <= 1e-13 * m0
    fscale = np.sum(m.areaTriangle * np.abs(m.fVertex))
    assert abs(dg.total_abs_vorticity(m, u) - G0) <= 1e-13 * fscale


# ---------------------------------------------------------------- P14
@pytest.mark.parametrize("which", ["cfg1", "shelf"])
def test_widened_extents_change_nothing(which, cfg1, shelf):
    """P14: running every coarse stage on all of F (the MPAS simplification) gives
    bit-identical results to the paper's shrinking extents F^5/F^4/F^3/F^2/F^1."""
    c, lab = cfg1 if which == "cfg1" else shelf
    phys = phys_of(c)
    a = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 4, phys, 3, extents="paper")
    b = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 4, phys, 3, extents="all_fine")
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# ---------------------------------------------------------------- P16
def test_temporal_convergence_second_order():
    """P16: gravity-wave model (slow terms off, eq. grav_wave_model), M = 4, errors vs an
    RK4 reference at a much smaller step (E_RMS, eq. rmse) fall with slope 2 -- globally and on IF-1."""
    c = config1(nx=24, ny=24)
    m = c.mesh
    lab = lts.label_regions(m, c.fine_mask)
    phys = phys_of(c, slow=False)
    T = 8 * 40.0
    dts = [40.0, 20.0, 10.0, 5.0]
    h_ref, u_ref = c.h0.copy(), c.u0.copy()
    n_ref = int(round(T / 0.5))
    for _ in range(n_ref):
        h_ref, u_ref = fbrk32.rk4_step(m, h_ref, u_ref, T / n_ref, phys)
    eh, eu, eif = [], [], []
    for dt in dts:
        h, u = lts.run(m, lab, c.h0, c.u0, dt, 4, phys, int(round(T / dt)))
        eh.append(dg.rms_error(h_ref, h))
        eu.append(dg.rms_error(u_ref, u))
        eif.append(dg.rms_error(h_ref[lab.IF1()], h[lab.IF1()]))
    for e in (eh, eu, eif):
        slopes = np.log2(np.array(e[:-1]) / np.array(e[1:]))
        assert np.all((slopes > 1.8) & (slopes < 2.25)), slopes


# ---------------------------------------------------------------- P21
def _bfs(mesh, src):
    d = np.full(mesh.nCells, -1)
    q = collections.deque()
    for i in np.nonzero(src)[0]:
        d[i] = 0
        q.append(i)
    while q:
        i = q.popleft()
        for j in range(mesh.nEdgesOnCell[i]):
            nb = mesh.cellsOnCell[i, j]
            if d[nb] < 0:
                d[nb] = d[i] + 1
                q.append(nb)
    return d


def test_labels_strip_example():
    """S:L320 / P:L416-426: 40x4 periodic strip, fine = columns 0-19, r = 2 -> IF-1 = columns 20-21 and
    38-39, IF-2 = 22-23 and 36-37, int = 24-35; F/IF-1 edges belong to F_E (closest-to-fine rule)."""
    m = build_periodic_hex_mesh(40, 4, 1000.0)
    col = np.arange(m.nCells) % 40
    lab = lts.label_regions(m, col < 20)
    exp = np.where(col < 20, -1, np.where(np.isin(col, [20, 21, 38, 39]), lts.IF1,
                   np.where(np.isin(col, [22, 23, 36, 37]), lts.IF2, lts.INT)))
    assert np.array_equal(lab.cell[col >= 20], exp[col >= 20])
    c0, c1 = m.cellsOnEdge[:, 0], m.cellsOnEdge[:, 1]
    fi = (lab.F()[c0] & lab.IF1()[c1]) | (lab.F()[c1] & lab.IF1()[c0])
    assert np.all(lab.edge[fi] >= lts.FINE_MIN)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_labels_are_function_of_hop_distance(seed):
    """P21: region labels equal a pure function of brute-force BFS hop distance; edge labels follow
    the closest-to-fine rule; F^l_E = edges touching F^l (reading Q7)."""
    m = build_periodic_hex_mesh(30, 24, 1000.0)
    rng = np.random.default_rng(seed)
    fine = np.zeros(m.nCells, bool)
    for _ in range(3):
        cx, cy, rad = rng.uniform(0, m.Lx), rng.uniform(0, m.Ly), rng.uniform(3e3, 7e3)
        fine |= (m.xCell - cx) ** 2 + (m.yCell - cy) ** 2 < rad ** 2
    lab = lts.label_regions(m, fine)
    dF, dC = _bfs(m, fine), _bfs(m, ~fine)
    r = 2
    for i in range(m.nCells):
        if fine[i]:
            l = min(-(-dC[i] // r), 6)
            assert lab.cell[i] == 2 + l
        else:
            exp = lts.IF1 if dF[i] <= r else (lts.IF2 if dF[i] <= 2 * r else lts.INT)
            assert lab.cell[i] == exp
    rank = {lts.INT: 0, lts.IF2: 1, lts.IF1: 2}
    for e in range(m.nEdges):
        a, b = lab.cell[m.cellsOnEdge[e]]
        fa, fb = a >= 3, b >= 3
        if fa or fb:
            exp = min([x for x, f in ((a, fa), (b, fb)) if f])
        else:
            exp = a if rank[a] >= rank[b] else b
        assert lab.edge[e] == exp


def test_validate_labels_rejects_thin_interface():
    """thinning IF-1 to nothing (an int cell touching F) violates the stencil assumption."""
    m = build_periodic_hex_mesh(40, 4, 1000.0)
    col = np.arange(m.nCells) % 40
    lab = lts.label_regions(m, col < 20)
    bad = lts.Labels(cell=lab.cell.copy(), edge=lab.edge.copy(), r=2)
    bad.cell[col == 20] = lts.INT
    with pytest.raises(ValueError):
        lts.validate_labels(m, bad)


# ---------------------------------------------------------------- P22, P23
def test_fblts_limit_below_global(cfg1):
    """P22 / reading Q12: the FB-LTS stability limit on config 1 lies below the global FB-RK(3,2)
    bound nu_max = 1.5767: stable at nu_loc = 1.0, unstable at nu_loc = 1.5 within 300 steps."""
    c, lab = cfg1
    m = c.mesh
    phys = phys_of(c)
    nu1 = dg.rest_courant(m, lab, 1.0, c.M, c.g)           # nu_loc per second of coarse step
    res = {}
    for nu in (1.0, 1.5):
        dt = nu / nu1
        h, u = c.h0.copy(), c.u0.copy()
        with np.errstate(all="ignore"):
            for _ in range(300):
                h, u = lts.fblts_step(m, lab, h, u, dt, c.M, phys)
                if not np.all(np.isfinite(u)) or np.max(np.abs(u)) > 5.0:
                    break
        res[nu] = bool(np.all(np.isfinite(u)) and np.max(np.abs(u)) <= 5.0)
    assert res[1.0] and not res[1.5]


def test_speedup_arithmetic():
    """P23 / eq. speedup: Table 3 CPU-times 26.07, 5.86, 2.59 s."""
    g = GOLD["speedup"]
    assert round(dg.speedup(g["rk4"], g["fblts"]), 2) == g["vs_rk4"]
    assert round(dg.speedup(g["lts3"], g["fblts"]), 2) == g["vs_lts3"]
    with pytest.raises(ValueError):
        dg.speedup(1.0, 0.0)
