"""Pins for the shared mesh input.

These check the generated TRiSK mesh against closed forms and invariants, so
that neither the oracle nor the CUDA path inherits a silently wrong mesh.
"""
import json
import os

import numpy as np
import pytest

from inputs.hexmesh import build_periodic_hex_mesh, build_periodic_hex_mesh_fast

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))
SQ3 = np.sqrt(3.0)


BUILDERS = {"generic": build_periodic_hex_mesh, "lattice": build_periodic_hex_mesh_fast}


@pytest.fixture(scope="module", params=sorted(BUILDERS))
def m4(request):
    g = GOLD["hex4x4"]
    return BUILDERS[request.param](g["nx"], g["ny"], g["dc"])


@pytest.fixture(scope="module", params=sorted(BUILDERS))
def m12(request):
    return BUILDERS[request.param](12, 10, 3000.0)


def test_hex4x4_counts_and_areas(m4):
    """16 cells, 48 edges, 32 vertices; A_i = (sqrt3/2) dc^2; sums agree."""
    g = GOLD["hex4x4"]
    assert (m4.nCells, m4.nEdges, m4.nVertices) == (g["nCells"], g["nEdges"], g["nVertices"])
    assert m4.nVertices - m4.nEdges + m4.nCells == 0           # torus Euler characteristic
    np.testing.assert_allclose(m4.areaCell, g["areaCell"], rtol=1e-7)
    np.testing.assert_allclose(m4.areaCell, SQ3 / 2 * 1000.0 ** 2, rtol=1e-14)
    s_cell = np.sum(m4.areaCell)
    np.testing.assert_allclose(s_cell, g["areaSum"], rtol=1e-8)
    np.testing.assert_allclose(np.sum(m4.areaTriangle), s_cell, rtol=1e-14)
    np.testing.assert_allclose(np.sum(m4.kiteAreasOnVertex), s_cell, rtol=1e-14)


def test_regular_hex_geometry(m12):
    """P19: l = dc/sqrt3, d = dc, A_v = (sqrt3/4) dc^2, kite = A_v/3."""
    dc = 3000.0
    np.testing.assert_allclose(m12.dcEdge, dc, rtol=1e-14)
    np.testing.assert_allclose(m12.dvEdge, dc / SQ3, rtol=1e-14)
    np.testing.assert_allclose(m12.areaTriangle, SQ3 / 4 * dc * dc, rtol=1e-14)
    np.testing.assert_allclose(m12.kiteAreasOnVertex, SQ3 / 12 * dc * dc, rtol=1e-14)


def test_connectivity_invariants(m12):
    """each edge sits in edgesOnCell of exactly its two cells, with n-sign product -1;
    t-sign product -1; vertices of an edge are the ends of the shared primal edge."""
    m = m12
    count = np.zeros(m.nEdges, dtype=int)
    sign_prod = np.ones(m.nEdges)
    for c in range(m.nCells):
        for j in range(m.nEdgesOnCell[c]):
            e = m.edgesOnCell[c, j]
            count[e] += 1
            sign_prod[e] *= 1.0 if m.cellsOnEdge[e, 0] == c else -1.0
            assert c in m.cellsOnEdge[e]
            assert m.cellsOnCell[c, j] == (m.cellsOnEdge[e, 1] if m.cellsOnEdge[e, 0] == c else m.cellsOnEdge[e, 0])
    assert np.all(count == 2) and np.all(sign_prod == -1.0)
    for v in range(m.nVertices):
        for k in range(3):
            e = m.edgesOnVertex[v, k]
            assert v in m.verticesOnEdge[e]
            # edgesOnVertex[k] joins cellsOnVertex[k] and cellsOnVertex[k+1]
            assert set(m.cellsOnEdge[e]) == {m.cellsOnVertex[v, k], m.cellsOnVertex[v, (k + 1) % 3]}


def _tangent(m):
    n = m.edgeNormal
    return np.stack([-n[:, 1], n[:, 0], np.zeros(m.nEdges)], axis=1)   # t_e = k x n_e


def test_weights_reconstruct_uniform_flow(m12):
    """P7 (reading Q6): sum_j W_{e,j} (U . n_{eoe_j}) = U . t_e for uniform U."""
    m = m12
    rng = np.random.default_rng(0)
    for _ in range(5):
        U = np.array([*rng.standard_normal(2), 0.0])
        un = m.edgeNormal @ U
        rec = np.zeros(m.nEdges)
        for j in range(m.maxEdges2):
            rec += np.where(j < m.nEdgesOnEdge, m.weightsOnEdge[:, j] * un[np.maximum(m.edgesOnEdge[:, j], 0)], 0.0)
        np.testing.assert_allclose(rec, _tangent(m) @ U, atol=1e-14 * np.linalg.norm(U))


def test_weights_antisymmetry(m12):
    """P7 / reading Q6: l_e d_e W_{e,e'} = -l_{e'} d_{e'} W_{e',e} (SPEC S:L40 form corrected)."""
    m = m12
    Wd = {}
    for e in range(m.nEdges):
        for j in range(m.nEdgesOnEdge[e]):
            Wd[(e, m.edgesOnEdge[e, j])] = m.weightsOnEdge[e, j]
    scale = np.max(np.abs(m.weightsOnEdge)) * np.max(m.dvEdge * m.dcEdge)
    for (e, ep), w in Wd.items():
        wt = Wd.get((ep, e), 0.0)
        lhs = m.dvEdge[e] * m.dcEdge[e] * w
        rhs = -m.dvEdge[ep] * m.dcEdge[ep] * wt
        assert abs(lhs - rhs) <= 1e-14 * scale


def test_weights_pv_consistency(m12):
    """P7 / S:L77(b): dual divergence of F_perp equals the kite average of the primal divergence,
    (1/A_v) sum_e t_{e,v} d_e F_perp_e = -(1/A_v) sum_i kite_{v,i} [(1/A_i) sum_e n_{e,i} l_e F_e]."""
    m = m12
    rng = np.random.default_rng(1)
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
            t = 1.0 if m.verticesOnEdge[e, 1] == v else -1.0
            lhs[v] += t * m.dcEdge[e] * Fp[e]
            rhs[v] -= m.kiteAreasOnVertex[v, k] * div[m.cellsOnVertex[v, k]]
    scale = np.max(np.abs(lhs))
    np.testing.assert_allclose(lhs, rhs, atol=1e-13 * scale)


@pytest.mark.parametrize("builder", sorted(BUILDERS))
def test_mesh_deterministic(builder):
    """same (nx, ny, dc) -> bit-identical mesh."""
    a = BUILDERS[builder](8, 6, 1234.5)
    b = BUILDERS[builder](8, 6, 1234.5)
    for k, v in a.arrays().items():
        if isinstance(v, np.ndarray):
            assert np.array_equal(v, getattr(b, k)), k


def test_lattice_builder_matches_generic():
    """The lattice builder describes the same mesh as the generic one: same cells, positions,
    cell adjacency, and per-cell/per-edge geometry up to the edge/vertex numbering and rounding."""
    a = build_periodic_hex_mesh(10, 8, 2000.0)
    b = build_periodic_hex_mesh_fast(10, 8, 2000.0)
    assert (a.nCells, a.nEdges, a.nVertices) == (b.nCells, b.nEdges, b.nVertices)
    assert np.array_equal(a.cellsOnCell, b.cellsOnCell)
    np.testing.assert_allclose(a.xCell, b.xCell, atol=1e-9)
    np.testing.assert_allclose(a.areaCell, b.areaCell, rtol=1e-14)
    pa = {tuple(sorted(p)): i for i, p in enumerate(a.cellsOnEdge.tolist())}
    for e in range(b.nEdges):
        ea = pa[tuple(sorted(b.cellsOnEdge[e].tolist()))]
        assert abs(a.dvEdge[ea] - b.dvEdge[e]) <= 1e-12 * b.dvEdge[e]
        sgn = 1.0 if a.cellsOnEdge[ea, 0] == b.cellsOnEdge[e, 0] else -1.0
        np.testing.assert_allclose(sgn * a.edgeNormal[ea], b.edgeNormal[e], atol=1e-14)


def test_rejects_small_or_odd():
    with pytest.raises(ValueError):
        build_periodic_hex_mesh(3, 4, 1.0)
    with pytest.raises(ValueError):
        build_periodic_hex_mesh(4, 5, 1.0)
