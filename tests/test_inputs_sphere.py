"""Pins for the spherical (icosahedral-dual) mesh input of config 3 (SURVEY c.5 P19/P20, P7 on the sphere)."""
import numpy as np
import pytest

from inputs.icosmesh import EARTH_R, build_icosahedral_mesh


@pytest.fixture(scope="module")
def m3():
    return build_icosahedral_mesh(3)


@pytest.mark.parametrize("level", [0, 1, 2, 4])
def test_counts_closed_form(level):
    """P20: level L gives 10*4^L + 2 cells, 30*4^L edges, 20*4^L vertices, exactly 12 pentagons;
    Euler characteristic of the sphere V - E + C = 2 (P19)."""
    m = build_icosahedral_mesh(level)
    assert (m.nCells, m.nEdges, m.nVertices) == (10 * 4 ** level + 2, 30 * 4 ** level, 20 * 4 ** level)
    assert np.count_nonzero(m.nEdgesOnCell == 5) == 12 and np.all(m.nEdgesOnCell >= 5)
    assert m.nVertices - m.nEdges + m.nCells == 2


def test_level8_counts_match_baseline():
    """BASELINE config 3: 655,362 cells, 1,966,080 edges (and 1,310,720 vertices)."""
    assert (10 * 4 ** 8 + 2, 30 * 4 ** 8, 20 * 4 ** 8) == (655362, 1966080, 1310720)


def test_areas_tile_the_sphere(m3):
    """P19: sum A_i = sum A_v = sum kites = 4 pi R^2."""
    S = 4 * np.pi * EARTH_R ** 2
    assert np.sum(m3.areaCell) == pytest.approx(S, rel=1e-13)
    assert np.sum(m3.areaTriangle) == pytest.approx(S, rel=1e-13)
    assert np.sum(m3.kiteAreasOnVertex) == pytest.approx(S, rel=1e-13)


def test_orientation(m3):
    """n_e is tangent at the edge point and points from c0 to c1; v1 lies on the +t_e = k x n_e side."""
    m = m3
    p = m.edgePoint / np.linalg.norm(m.edgePoint, axis=1, keepdims=True)
    assert np.max(np.abs(np.sum(m.edgeNormal * p, axis=1))) < 1e-12
    c0 = np.stack([m.xCell, m.yCell, m.zCell], 1)[m.cellsOnEdge[:, 0]]
    c1 = np.stack([m.xCell, m.yCell, m.zCell], 1)[m.cellsOnEdge[:, 1]]
    assert np.all(np.sum((c1 - c0) * m.edgeNormal, axis=1) > 0)
    t = np.cross(p, m.edgeNormal)
    v1 = np.stack([m.xVertex, m.yVertex, m.zVertex], 1)[m.verticesOnEdge[:, 1]]
    v0 = np.stack([m.xVertex, m.yVertex, m.zVertex], 1)[m.verticesOnEdge[:, 0]]
    assert np.all(np.sum((v1 - v0) * t, axis=1) > 0)


def test_weights_antisymmetry_and_pv_consistency(m3):
    """P7 on the sphere (reading Q6): l_e d_e W_{e,e'} = -l_e' d_e' W_{e',e}, and the dual divergence
    of F_perp equals the kite average of the primal divergence (S:L77(b))."""
    m = m3
    Wd = {}
    for e in range(m.nEdges):
        for j in range(m.nEdgesOnEdge[e]):
            Wd[(e, m.edgesOnEdge[e, j])] = m.weightsOnEdge[e, j]
    scale = np.max(np.abs(m.weightsOnEdge)) * np.max(m.dvEdge * m.dcEdge)
    for (e, ep), w in Wd.items():
        assert abs(m.dvEdge[e] * m.dcEdge[e] * w + m.dvEdge[ep] * m.dcEdge[ep] * Wd.get((ep, e), 0.0)) <= 1e-13 * scale
    rng = np.random.default_rng(2)
    F = rng.standard_normal(m.nEdges)
    Fp = np.zeros(m.nEdges)
    for j in range(m.maxEdges2):
        Fp += np.where(j < m.nEdgesOnEdge, m.weightsOnEdge[:, j] * F[np.maximum(m.edgesOnEdge[:, j], 0)], 0.0)
    div = np.zeros(m.nCells)
    for c in range(m.nCells):
        for j in range(m.nEdgesOnCell[c]):
            e = m.edgesOnCell[c, j]
            div[c] += (1.0 if m.cellsOnEdge[e, 0] == c else -1.0) * m.dvEdge[e] * F[e]
    div /= m.areaCell
    lhs = np.zeros(m.nVertices)
    rhs = np.zeros(m.nVertices)
    for v in range(m.nVertices):
        for k in range(3):
            e = m.edgesOnVertex[v, k]
            lhs[v] += (1.0 if m.verticesOnEdge[e, 1] == v else -1.0) * m.dcEdge[e] * Fp[e]
            rhs[v] -= m.kiteAreasOnVertex[v, k] * div[m.cellsOnVertex[v, k]]
    np.testing.assert_allclose(lhs, rhs, atol=1e-12 * np.max(np.abs(lhs)))


def test_oracle_conserves_on_sphere():
    """Theorems 1-2 on the closed sphere (no boundary): mass and diagnostic absolute vorticity
    conserved by global FB-RK(3,2) steps with full Coriolis (config-3 recipe, level 4)."""
    from inputs import configs
    from oracle import diagnostics as dg
    from oracle import fbrk32, lts
    c = configs.config3(level=4, dt=300.0, n_steps=20)
    m = c.mesh
    lab = lts.label_regions(m, c.fine_mask)
    h, u = lts.run(m, lab, c.h0, c.u0, c.dt, 1, fbrk32.Phys(tau_n=c.tau_n), 20)
    m0 = dg.total_mass(m, c.h0)
    assert abs(dg.total_mass(m, h) - m0) <= 1e-13 * m0
    G0 = dg.total_abs_vorticity(m, c.u0)
    assert abs(dg.total_abs_vorticity(m, u) - G0) <= 1e-13 * np.sum(m.areaTriangle * np.abs(m.fVertex))
    assert np.max(np.abs(u)) > 0.01
