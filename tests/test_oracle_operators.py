"""Oracle operator pins (P6, P8, P9, P10, P11, P12) and SPEC worked examples.

Each test checks oracle/trisk.py against a closed form, an invariant or a
number the paper/SPEC prints -- never against a retyped copy of its formula.
"""
import json
import math
import os

import numpy as np
import pytest

from inputs.hexmesh import build_periodic_hex_mesh
from oracle import fbrk32, lts, trisk
from oracle import diagnostics as dg

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


def hexmesh(nx=12, ny=10, dc=3000.0, H=100.0, f=1e-4):
    m = build_periodic_hex_mesh(nx, ny, dc)
    m.bottomDepth = np.full(m.nCells, H) if np.isscalar(H) else H
    m.fVertex = np.full(m.nVertices, f)
    return m


def unwrapped(m, mask_e):
    """Edges whose two cells are not split by the periodic wrap."""
    dx = np.abs(m.xCell[m.cellsOnEdge[:, 1]] - m.xCell[m.cellsOnEdge[:, 0]])
    dy = np.abs(m.yCell[m.cellsOnEdge[:, 1]] - m.yCell[m.cellsOnEdge[:, 0]])
    return mask_e & (dx < m.Lx / 2) & (dy < m.Ly / 2)


def test_single_edge_thickness_tendency():
    """one edge, F = 1, l = 1000, A = 8.6602540e5, n = +1 -> dh = -1.1547005e-3 (sign: outward flux drains)."""
    g = GOLD["single_edge_dh"]
    m = hexmesh(4, 4, 1000.0)
    e = 5
    c0, c1 = m.cellsOnEdge[e]
    m.dvEdge = m.dvEdge.copy()
    m.dvEdge[e] = g["l"]
    m.areaCell = np.full(m.nCells, g["A"])
    u = np.zeros(m.nEdges)
    u[e] = g["F"]
    h = np.ones(m.nCells)
    psi = trisk.thickness_tendency(m, u, h, np.array([c0, c1]))
    assert psi[0] == pytest.approx(g["dh"], rel=1e-7)
    assert psi[1] == pytest.approx(-g["dh"], rel=1e-7)


def test_thickness_tendency_conserves_and_kills_uniform_flow():
    """P10: sum_i A_i Psi_i = 0 for random (u, h) (Thm 1 mechanism);
    Psi = 0 for uniform h and uniform flow (discrete divergence of a constant field)."""
    m = hexmesh()
    rng = np.random.default_rng(3)
    cells = np.arange(m.nCells)
    for _ in range(4):
        u = rng.standard_normal(m.nEdges)
        h = 100.0 + rng.random(m.nCells)
        psi = trisk.thickness_tendency(m, u, h, cells)
        terms = m.areaCell * psi
        assert abs(math.fsum(terms)) <= 1e-13 * np.sum(np.abs(terms))
    U = np.array([0.7, -0.3, 0.0])
    psi = trisk.thickness_tendency(m, m.edgeNormal @ U, np.full(m.nCells, 50.0), cells)
    assert np.max(np.abs(psi)) <= 1e-13 * 50.0 * np.linalg.norm(U) / 3000.0


def test_fast_momentum_linear_ssh():
    """P11: for eta = a x + b y (flat bottom), Phi^fast_e = -g grad(eta) . n_e exactly."""
    m = hexmesh(12, 10, 3000.0, H=0.0)
    a, b = 2.5e-6, -1.5e-6
    x0, y0 = m.xCell[0], m.yCell[0]
    h = a * (m.xCell - x0) + b * (m.yCell - y0)
    ok = unwrapped(m, np.ones(m.nEdges, bool))
    e = np.nonzero(ok)[0]
    phi = trisk.fast_momentum(m, h, 9.81, e)
    exact = -9.81 * (a * m.edgeNormal[e, 0] + b * m.edgeNormal[e, 1])
    np.testing.assert_allclose(phi, exact, atol=1e-14 * 9.81 * math.hypot(a, b) * 10)


def test_vorticity_of_linear_field_and_circulation_sum():
    """P12: zeta_v of a linear velocity field equals its curl (interior vertices, regular hex);
    sum_v circulation = 0 for any u (each u_e enters twice with opposite t_{e,v}; Thm 2 mechanism)."""
    m = hexmesh(12, 10, 3000.0)
    al, be = 3e-5, -2e-5                               # U = (al (y - y0), be (x - x0)) -> curl = be - al
    x0, y0 = m.Lx / 2, m.Ly / 2
    xe, ye = m.edgePoint[:, 0], m.edgePoint[:, 1]
    U = np.stack([al * (ye - y0), be * (xe - x0)], axis=1)
    u = U[:, 0] * m.edgeNormal[:, 0] + U[:, 1] * m.edgeNormal[:, 1]
    zeta = trisk.relative_vorticity(m, u)
    # vertices whose three edges are all away from the wrap
    ok_e = unwrapped(m, np.ones(m.nEdges, bool)) & (np.abs(xe - x0) < m.Lx / 3) & (np.abs(ye - y0) < m.Ly / 3)
    ok_v = np.all(ok_e[m.edgesOnVertex], axis=1)
    assert np.count_nonzero(ok_v) > 20
    np.testing.assert_allclose(zeta[ok_v], be - al, rtol=1e-12)
    rng = np.random.default_rng(4)
    circ = trisk.circulation(m, rng.standard_normal(m.nEdges))
    assert abs(math.fsum(circ.tolist())) <= 1e-14 * np.sum(np.abs(circ))


def test_kinetic_energy_uniform_flow_exact():
    """P9: uniform flow on a regular hex gives K_i = |U|^2/2 exactly (reading Q18; SPEC's 2 % is loose)."""
    m = hexmesh()
    U = np.array([1.3, -0.4, 0.0])
    K = trisk.kinetic_energy(m, m.edgeNormal @ U)
    np.testing.assert_allclose(K, 0.5 * U @ U, rtol=1e-15 * 8)
    # quadratic form: K(2u) = 4 K(u) exactly
    rng = np.random.default_rng(5)
    u = rng.standard_normal(m.nEdges)
    assert np.array_equal(trisk.kinetic_energy(m, 2 * u), 4 * trisk.kinetic_energy(m, u))


def test_lake_at_rest():
    """P6: u = 0, h + z_b = const over random bathymetry, f != 0, slow terms on.
    Operator level, bit for bit: Phi^fast = 0 (the (h + z_b)-per-cell form, Q15),
    Psi = 0 and S = 0.  Step level: the literal FB average b h1 + (1 - b) h^n rounds,
    so the state may move only at roundoff (|u| <= 1e-12 m/s, |dh| <= 1e-13 h) -- see DESIGN.md."""
    m = hexmesh(16, 12, 2000.0)
    rng = np.random.default_rng(6)
    H = np.round(50.0 + 3000.0 * rng.random(m.nCells))          # integer depths: h = H + 1 exactly
    m.bottomDepth = H
    h = H + 1.0
    u = np.zeros(m.nEdges)
    e = np.arange(m.nEdges)
    assert np.all(trisk.fast_momentum(m, h, 9.81, e) == 0.0)
    assert np.all(trisk.thickness_tendency(m, u, h, np.arange(m.nCells)) == 0.0)
    phys = fbrk32.Phys(tau_n=np.zeros(m.nEdges))
    assert np.all(trisk.slow_tendency(m, u, h, phys) == 0.0)
    lab = lts.label_regions(m, H > 1500.0)
    h1, u1 = lts.run(m, lab, h, u, 10.0, 4, phys, 5)     # nu_loc < 1
    assert np.max(np.abs(u1)) <= 1e-12
    assert np.max(np.abs(h1 - h) / h) <= 1e-13


@pytest.mark.parametrize("M", [1, 2, 4])
def test_inertial_oscillation_split(M):
    """P8 split: uniform h and U on an f-plane; the split step adds dt*S once, so
    (u, v) <- (u + f dt v, v - f dt u) per coarse step, for every M and labelling."""
    m = hexmesh(16, 12, 2000.0, H=100.0, f=1e-4)
    fine = (m.xCell > m.Lx / 2)
    lab = lts.label_regions(m, fine)
    phys = fbrk32.Phys(tau_n=np.zeros(m.nEdges))
    U = np.array([0.4, -0.2])
    dt = 40.0
    h = np.full(m.nCells, 100.0)
    u = m.edgeNormal[:, :2] @ U
    for n in range(3):
        h, u = lts.fblts_step(m, lab, h, u, dt, M, phys)
        U = np.array([U[0] + 1e-4 * dt * U[1], U[1] - 1e-4 * dt * U[0]])
        np.testing.assert_allclose(u, m.edgeNormal[:, :2] @ U, atol=1e-13 * np.linalg.norm(U))
    np.testing.assert_allclose(h, 100.0, rtol=1e-15)


def test_inertial_oscillation_unsplit_rk3_polynomial():
    """P8 unsplit, global: Psi = 0 reduces FB-RK(3,2) to R(z) = 1 + z + z^2/2 + z^3/6 with
    z = -i f dt acting on w = u + i v (the momentum equation's -f k x u)."""
    m = hexmesh(12, 10, 3000.0, H=100.0, f=1e-4)
    phys = fbrk32.Phys(tau_n=np.zeros(m.nEdges))
    dt = 500.0
    w = complex(0.3, 0.5)
    h = np.full(m.nCells, 100.0)
    u = m.edgeNormal[:, :2] @ np.array([w.real, w.imag])
    z = -1j * 1e-4 * dt
    R = 1 + z + z * z / 2 + z ** 3 / 6
    for _ in range(3):
        h, u = fbrk32.fbrk32_step(m, h, u, dt, phys, split=False)
        w = R * w
        np.testing.assert_allclose(u, m.edgeNormal[:, :2] @ np.array([w.real, w.imag]), atol=1e-13 * abs(w))


def test_abs_vorticity_fplane_example():
    """eta = f = 1e-4 on dual area 1.38564065e7 m^2 -> Gamma = 1385.64065 m^2/s."""
    g = GOLD["abs_vorticity_fplane"]
    m = hexmesh(4, 4, 1000.0, f=g["f"])
    assert dg.total_abs_vorticity(m, np.zeros(m.nEdges)) == pytest.approx(g["Gamma"], rel=1e-8)


def test_courant_and_rms_examples():
    """S:L270 (nu = 0.31321) and S:L496 (rms = 1.41421356)."""
    g = GOLD["courant"]
    m = hexmesh(4, 4, g["d"])
    nu = dg.courant_numbers(m, None, np.full(m.nCells, g["h"]), np.zeros(m.nEdges), g["dt"], 1, g["g"])
    np.testing.assert_allclose(nu, g["nu"], rtol=2e-5)
    r = GOLD["rms"]
    assert dg.rms_error(r["s"], r["m"]) == pytest.approx(r["rms"], rel=1e-8)
    with pytest.raises(ValueError):
        dg.rms_error([1.0], [1.0, 2.0])


def test_vertex_thickness_linear_field_on_hex():
    """h_v on the regular hex: the three kites of a vertex are equal (A_v/3, P19), so
    h_v is the mean of the three cell values, which for a LINEAR h is h at the triangle's centroid --
    the vertex itself.  Checked with h = b + a.x on every vertex whose three cells are not wrapped by
    the periodicity; then q_v = f / h(x_v) at rest."""
    m = build_periodic_hex_mesh(12, 10, 10e3)
    a, b = np.array([3.0e-3, -2.0e-3]), 1000.0
    H = b + a[0] * m.xCell + a[1] * m.yCell
    hv = trisk.vertex_thickness(m, H)
    cx = m.xCell[m.cellsOnVertex]
    cy = m.yCell[m.cellsOnVertex]
    ok = (np.max(np.abs(cx - m.xVertex[:, None]), axis=1) < 2e4) & (np.max(np.abs(cy - m.yVertex[:, None]), axis=1) < 2e4)
    assert ok.sum() > 0.5 * m.nVertices
    exact = b + a[0] * m.xVertex + a[1] * m.yVertex
    np.testing.assert_allclose(hv[ok], exact[ok], rtol=1e-13)
    f = np.full(m.nVertices, 1e-4)
    m.fVertex = f
    q = trisk.potential_vorticity(m, np.zeros(m.nEdges), H)
    np.testing.assert_allclose(q[ok], f[ok] / exact[ok], rtol=1e-13)


def _mesh_with_unequal_kites():
    from inputs.icosmesh import build_icosahedral_mesh
    return build_icosahedral_mesh(3)


def test_vertex_thickness_integral_identity_nonuniform_kites():
    """sum_v A_v h_v = sum_v sum_j kite_{v,j} h_{c_j} = sum_i h_i (sum of the kites of cell i) = sum_i A_i h_i
    for ANY h, because the kites of a cell tile it (P:L1150-1151 with P19's sum of kites).  On a mesh
    whose kites differ (icosahedral level 3: pentagons, distorted triangles) this pins the kite <-> cell
    pairing of the oracle's h_v: pairing a kite with a neighbouring cell breaks it by O(1e-3).  Then
    q_v at rest: sum_v A_v h_v q_v = sum_v A_v f_v exactly in real arithmetic."""
    m = _mesh_with_unequal_kites()
    rng = np.random.default_rng(3)
    kites = m.kiteAreasOnVertex
    assert np.ptp(kites) > 1e-3 * np.mean(kites)                  # the kites really differ
    H = 4000.0 + 500.0 * rng.standard_normal(m.nCells)
    hv = trisk.vertex_thickness(m, H)
    lhs = float(np.sum(m.areaTriangle * hv))
    rhs = float(np.sum(m.areaCell * H))
    assert abs(lhs - rhs) <= 1e-13 * abs(rhs)
    # the same sum with the kites rotated one slot against cellsOnVertex fails
    bad = np.sum(np.roll(kites, 1, axis=1) * H[m.cellsOnVertex], axis=1)
    assert abs(float(np.sum(bad)) - rhs) > 1e-9 * abs(rhs)
    m.fVertex = 1e-4 * m.zVertex / m.radius
    q = trisk.potential_vorticity(m, np.zeros(m.nEdges), H)
    fsum = float(np.sum(m.areaTriangle * m.fVertex))
    scale = float(np.sum(m.areaTriangle * np.abs(m.fVertex)))
    assert abs(float(np.sum(m.areaTriangle * hv * q)) - fsum) <= 1e-13 * scale
