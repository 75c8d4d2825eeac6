"""Pins for the energy-conserving PV flux variant (the alternative to reading Q2):
    PV_e = sum_j W_{e,j} F_{e_j} (q_hat_e + q_hat_{e_j}) / 2   instead of   q_hat_e F_perp_e.
With l_e d_e W_{e,e'} antisymmetric (pin P7), the symmetric pairwise PV average makes the PV term
do no work: sum_e l_e d_e F_e PV_e = 0 for ANY state -- the TRiSK energy-conservation identity
(the paper's TRiSK reference).  The centred variant does not satisfy it, so the
identity tells the two apart; uniform PV makes them agree; conservation (Theorems 1-2) and the
M = 1 reduction hold for the variant as for the default."""
import dataclasses
import math

import numpy as np
import pytest

from inputs import configs
from inputs.hexmesh import build_periodic_hex_mesh
from inputs.icosmesh import build_icosahedral_mesh
from oracle import diagnostics as dg
from oracle import fbrk32, lts, trisk


def random_state(m, seed):
    rng = np.random.default_rng(seed)
    H = 100.0 + 20.0 * rng.random(m.nCells)
    U = rng.standard_normal(m.nEdges)
    return U, H


def pv_terms(m, U, H):
    e = np.arange(m.nEdges)
    F = trisk.edge_flux(m, U, H, e)
    q = trisk.potential_vorticity(m, U, H)
    q_hat = 0.5 * (q[m.verticesOnEdge[:, 0]] + q[m.verticesOnEdge[:, 1]])
    return F, q_hat, trisk.pv_flux_energy(m, F, q_hat, e), q_hat * trisk.perp_flux(m, F, e)


def work(m, F, PV):
    w = m.dvEdge * m.dcEdge * F * PV
    return abs(np.sum(w)) / np.sum(np.abs(w))


@pytest.mark.parametrize("mesh", ["hex", "icos"])
def test_pv_term_does_no_work(mesh):
    """sum_e l_e d_e F_e PV_e = 0 to roundoff for random u, h (energy form); the centred form does
    work (relative size O(1e-2) or larger)."""
    m = build_periodic_hex_mesh(16, 12, 2000.0) if mesh == "hex" else build_icosahedral_mesh(3)
    if mesh == "hex":
        m.fVertex = np.full(m.nVertices, 1e-4)
    for seed in (1, 2):
        U, H = random_state(m, seed)
        F, _, pe, pc = pv_terms(m, U, H)
        assert work(m, F, pe) < 1e-13
        assert work(m, F, pc) > 1e-4


def test_uniform_pv_variants_agree():
    """f-plane at rest (zeta = 0, uniform h): q_hat = f / h everywhere, so (q_e + q_e')/2 = q_hat and
    the two forms are sum_j W F q vs q sum_j W F -- equal up to rounding."""
    m = build_periodic_hex_mesh(16, 12, 2000.0)
    m.fVertex = np.full(m.nVertices, 1e-4)
    rng = np.random.default_rng(3)
    H = np.full(m.nCells, 80.0)
    e = np.arange(m.nEdges)
    F = rng.standard_normal(m.nEdges)                 # any flux field; q from the state at rest
    q = trisk.potential_vorticity(m, np.zeros(m.nEdges), H)
    np.testing.assert_allclose(q, 1e-4 / 80.0, rtol=1e-15)      # uniform up to the kite-sum rounding
    q_hat = 0.5 * (q[m.verticesOnEdge[:, 0]] + q[m.verticesOnEdge[:, 1]])
    pe = trisk.pv_flux_energy(m, F, q_hat, e)
    pc = q_hat * trisk.perp_flux(m, F, e)
    scale = q_hat[0] * np.sum(np.abs(m.weightsOnEdge), axis=1) * np.max(np.abs(F))
    assert np.all(np.abs(pe - pc) <= 1e-14 * scale)


def test_single_pair_closed_form():
    """One nonzero flux F_{e'} = 1: PV_e = W_{e,e'} (q_e + q_e') / 2 exactly on every edge e that has
    e' in its edgesOnEdge (all other slots contribute +0.0)."""
    m = build_periodic_hex_mesh(8, 6, 2000.0)
    rng = np.random.default_rng(4)
    q_hat = rng.standard_normal(m.nEdges)
    ep = 17
    F = np.zeros(m.nEdges)
    F[ep] = 1.0
    pe = trisk.pv_flux_energy(m, F, q_hat, np.arange(m.nEdges))
    for e in range(m.nEdges):
        want = 0.0
        for j in range(m.nEdgesOnEdge[e]):
            if m.edgesOnEdge[e, j] == ep:
                want = m.weightsOnEdge[e, j] * 1.0 * (0.5 * (q_hat[e] + q_hat[ep]))
        assert pe[e] == want


@pytest.mark.parametrize("M", [1, 4])
def test_conservation_and_M1_with_energy_pv(M):
    """FB-LTS with the energy form conserves mass and the diagnostic absolute vorticity to 1e-13
    (Theorems 1-2 do not depend on q_hat), and M = 1 is global FB-RK(3,2) bitwise (P1)."""
    c = configs.small_shelf(nx=32, ny=28, dt=5.0 * M)
    phys = fbrk32.Phys(g=c.g, beta=c.beta, tau_n=c.tau_n, rho0=c.rho0, pv="energy")
    lab = lts.label_regions(c.mesh, c.fine_mask)
    h, u = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, M, phys, 10)
    m0, g0 = dg.total_mass(c.mesh, c.h0), dg.total_abs_vorticity(c.mesh, c.u0)
    assert abs(dg.total_mass(c.mesh, h) - m0) <= 1e-13 * m0
    assert abs(dg.total_abs_vorticity(c.mesh, u) - g0) <= 1e-13 * abs(g0)
    hc, uc = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, M, dataclasses.replace(phys, pv="centered"), 10)
    assert not np.array_equal(uc, u)                  # the variant changes the solution
    if M == 1:
        hh, uu = c.h0.copy(), c.u0.copy()
        for _ in range(10):
            hh, uu = fbrk32.fbrk32_step(c.mesh, hh, uu, c.dt, phys)
        assert np.array_equal(hh, h) and np.array_equal(uu, u)


def test_pv_volume_integral():
    """Remark rmk:volume_conservation_pv: sum_v A_v h_v q_v = sum_v A_v eta_v = Gamma
    (to rounding) for any state; with uniform q = 1 (eta_v = h_v) it is sum_v A_v h_v; and it is
    conserved by FB-LTS steps as Gamma is (Theorem 2)."""
    c = configs.small_shelf(nx=32, ny=28, dt=20.0)
    rng = np.random.default_rng(5)
    h = c.h0 * (1.0 + 0.1 * rng.random(c.mesh.nCells))
    u = rng.standard_normal(c.mesh.nEdges)
    pv, gam = dg.total_pv_volume(c.mesh, h, u), dg.total_abs_vorticity(c.mesh, u)
    scale = math.fsum(np.abs(dg.vertex_abs_vorticity_integrals(c.mesh, u)).tolist())
    assert abs(pv - gam) <= 1e-14 * scale
    m = build_periodic_hex_mesh(8, 6, 2000.0)          # uniform q = 1: f_v = h_v, u = 0
    hh = 50.0 + 10.0 * rng.random(m.nCells)
    m.fVertex = trisk.vertex_thickness(m, hh)
    want = math.fsum((m.areaTriangle * trisk.vertex_thickness(m, hh)).tolist())
    assert abs(dg.total_pv_volume(m, hh, np.zeros(m.nEdges)) - want) <= 1e-14 * want
    lab = lts.label_regions(c.mesh, c.fine_mask)
    h1, u1 = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, c.M, fbrk32.Phys(tau_n=c.tau_n), 10)
    p0, p1 = dg.total_pv_volume(c.mesh, c.h0, c.u0), dg.total_pv_volume(c.mesh, h1, u1)
    assert abs(p1 - p0) <= 1e-13 * max(abs(p0), scale * 1e-3)
    with pytest.raises(ValueError):
        dg.total_pv_volume(m, -hh, np.zeros(m.nEdges))
