"""Pins for the variable-resolution spherical centroidal Voronoi input of config 4 (inputs/scvt.py,
SURVEY 8(d) config-4 row, reading Q24), on the dx_scale = 8 reduction of the recipe (~12 k cells):
closed-sphere topology and areas (P19), orientation and the weightsOnEdge identities (P7), the
refinement the recipe asks for, the centroidal property Lloyd's iteration converges to, and
conservation by the oracle's FB-LTS step with M = 8 on this mesh (Theorems 1-2)."""
import numpy as np
import pytest

from inputs import configs, scvt
from inputs.icosmesh import EARTH_R


@pytest.fixture(scope="module")
def c4():
    return configs.config4(dx_scale=8, dt=400.0)


def _xyz(m, kind="Cell"):
    return np.stack([getattr(m, "x" + kind), getattr(m, "y" + kind), getattr(m, "z" + kind)], 1)


def test_topology_and_areas(c4):
    """P19: V - E + C = 2 on the sphere; every vertex has 3 cells; sum A_i = sum A_v = sum kites = 4 pi R^2."""
    m = c4.mesh
    assert m.nVertices - m.nEdges + m.nCells == 2
    assert 2 * m.nEdges == int(np.sum(m.nEdgesOnCell)) and 2 * m.nEdges == 3 * m.nVertices
    S = 4 * np.pi * EARTH_R ** 2
    assert np.sum(m.areaCell) == pytest.approx(S, rel=1e-12)
    assert np.sum(m.areaTriangle) == pytest.approx(S, rel=1e-12)
    assert np.all(m.areaCell > 0) and np.all(m.kiteAreasOnVertex > 0)


def test_orientation(c4):
    m = c4.mesh
    p = m.edgePoint / np.linalg.norm(m.edgePoint, axis=1, keepdims=True)
    assert np.max(np.abs(np.sum(m.edgeNormal * p, axis=1))) < 1e-12
    c = _xyz(m)
    assert np.all(np.sum((c[m.cellsOnEdge[:, 1]] - c[m.cellsOnEdge[:, 0]]) * m.edgeNormal, axis=1) > 0)
    v = _xyz(m, "Vertex")
    t = np.cross(p, m.edgeNormal)
    assert np.all(np.sum((v[m.verticesOnEdge[:, 1]] - v[m.verticesOnEdge[:, 0]]) * t, axis=1) > 0)


def test_weights_identities(c4):
    """P7 on the variable-resolution sphere: antisymmetry of l d W and PV consistency (S:L77(b))."""
    m = c4.mesh
    eoe, W, n = m.edgesOnEdge, m.weightsOnEdge, m.nEdgesOnEdge
    e_idx = np.repeat(np.arange(m.nEdges), m.maxEdges2).reshape(m.nEdges, -1)
    valid = np.arange(m.maxEdges2)[None, :] < n[:, None]
    a, b, w = e_idx[valid], eoe[valid], W[valid]
    lhs = m.dvEdge[a] * m.dcEdge[a] * w
    key = a.astype(np.int64) * m.nEdges + b
    rkey = b.astype(np.int64) * m.nEdges + a
    order = np.argsort(key)
    pos = np.searchsorted(key[order], rkey)
    assert np.all(key[order][pos] == rkey)
    rhs = -(m.dvEdge[b] * m.dcEdge[b] * w[order][pos])
    assert np.max(np.abs(lhs - rhs)) <= 1e-13 * np.max(np.abs(lhs))
    rng = np.random.default_rng(4)
    F = rng.standard_normal(m.nEdges)
    Fp = np.sum(np.where(valid, W * F[np.maximum(eoe, 0)], 0.0), axis=1)
    sgn = np.where(m.cellsOnEdge[m.edgesOnCell, 0] == np.arange(m.nCells)[:, None], 1.0, -1.0)
    cvalid = np.arange(m.maxEdges)[None, :] < m.nEdgesOnCell[:, None]
    div = np.sum(np.where(cvalid, sgn * m.dvEdge[m.edgesOnCell] * F[m.edgesOnCell], 0.0), axis=1) / m.areaCell
    ev = m.edgesOnVertex
    s = np.where(m.verticesOnEdge[ev, 1] == np.arange(m.nVertices)[:, None], 1.0, -1.0)
    lhs_v = np.sum(s * m.dcEdge[ev] * Fp[ev], axis=1)
    rhs_v = -np.sum(m.kiteAreasOnVertex * div[m.cellsOnVertex], axis=1)
    np.testing.assert_allclose(lhs_v, rhs_v, atol=1e-12 * np.max(np.abs(lhs_v)))


def test_refinement_follows_the_density(c4):
    """The local cell size follows dx(x) = dx_f rho^(-1/4): cells deep inside the disk ~ 16 km and far
    from it ~ 240 km at dx_scale = 8 (ratio 15, as 2 km / 30 km in the full recipe), within 25 %;
    the cell count is the recipe's N = int dA / ((sqrt 3/2) dx^2)."""
    m = c4.mesh
    rng = np.random.default_rng(4)
    centre = rng.standard_normal(3)
    ref = scvt.Refinement(centre, dx_coarse=240e3, dx_fine=16e3)
    x = _xyz(m) / m.radius
    d = ref.dist(x)
    size = np.sqrt(m.areaCell / (0.5 * np.sqrt(3.0)))            # hexagon-equivalent spacing
    inner, outer = d < 100e3, d > 3000e3
    assert inner.sum() > 50 and outer.sum() > 1000
    assert np.median(size[inner]) == pytest.approx(16e3, rel=0.25)
    assert np.median(size[outer]) == pytest.approx(240e3, rel=0.25)
    assert m.nCells == ref.n_points()
    assert np.count_nonzero(c4.fine_mask) > 500 and c4.M == 8


def test_generators_are_centroidal():
    """After the Lloyd iterations a further Lloyd step moves every generator by a small fraction of
    its local spacing (the centroidal fixed point; an unweighted or mis-signed centroid would not
    converge to this): max move < 5 % and mean move < 0.5 % of dx(x)."""
    rng = np.random.default_rng(11)
    ref = scvt.Refinement(rng.standard_normal(3), dx_coarse=480e3, dx_fine=32e3)
    mesh, p = scvt.build_scvt(ref, rng, n_lloyd=50)
    q = scvt.lloyd_step(p, scvt.delaunay(p), ref)
    move = ref.R * np.arccos(np.clip(np.sum(p * q, axis=1), -1.0, 1.0)) / ref.dx(p)
    assert np.max(move) < 0.05 and np.mean(move) < 0.005, (np.max(move), np.mean(move))


def test_deterministic():
    a = configs.config4(dx_scale=16, dt=800.0, n_lloyd=5)
    b = configs.config4(dx_scale=16, dt=800.0, n_lloyd=5)
    assert np.array_equal(a.mesh.xCell, b.mesh.xCell) and np.array_equal(a.h0, b.h0)


def test_oracle_conserves_config4(c4):
    """Theorems 1-2 through FB-LTS with M = 8 on the variable-resolution sphere."""
    from oracle import diagnostics as dg
    from oracle import fbrk32, lts
    m = c4.mesh
    lab = lts.label_regions(m, c4.fine_mask)
    h, u = lts.run(m, lab, c4.h0, c4.u0, c4.dt, c4.M, fbrk32.Phys(tau_n=c4.tau_n), 5)
    m0 = dg.total_mass(m, c4.h0)
    assert abs(dg.total_mass(m, h) - m0) <= 1e-13 * m0
    G0 = dg.total_abs_vorticity(m, c4.u0)
    assert abs(dg.total_abs_vorticity(m, u) - G0) <= 1e-13 * np.sum(m.areaTriangle * np.abs(m.fVertex))
    assert np.max(np.abs(u)) > 1e-4
