"""Pins for the hurricane-model terms (eq. hurricane_model and
hurricane_fast_terms) with a synthetic wind field: closed forms for bottom drag and
wind stress on uniform states (the split step is forward Euler in S, P8), the SAL coefficient as
g (1 - beta) in the fast term, reduction to the plain model when the terms are off, and mass
conservation (the terms act on the momentum only)."""
import numpy as np
import pytest

from inputs import configs
from inputs.hexmesh import build_periodic_hex_mesh
from oracle import diagnostics as dg
from oracle import fbrk32, lts, trisk


def flat(nx=16, ny=12, f=0.0):
    m = build_periodic_hex_mesh(nx, ny, 2000.0)
    m.bottomDepth = np.full(m.nCells, 50.0)
    m.fVertex = np.full(m.nVertices, f)
    return m


def test_tangential_reconstruction_uniform_flow():
    """v_e = sum W u = U . t_e for a uniform U on the regular hex (P7 applied to u)."""
    m = flat()
    U = np.array([0.7, -0.4])
    u = m.edgeNormal[:, :2] @ U
    t = np.stack([-m.edgeNormal[:, 1], m.edgeNormal[:, 0]], axis=1)
    np.testing.assert_allclose(trisk.tangential_velocity(m, u), t @ U, atol=1e-14)


@pytest.mark.parametrize("M", [1, 3])
def test_bottom_drag_closed_form(M):
    """f = 0, uniform h and U, no wind: S_e = -C_D |U| (U . n_e) / h, so one coarse step is
    U <- U - dt C_D |U| U / h for every edge and every M (the fine subcycles add dt/M S M times)."""
    m = flat()
    lab = lts.label_regions(m, m.xCell > m.Lx / 2)
    U = np.array([0.8, 0.3])
    h0 = np.full(m.nCells, 50.0)
    u0 = m.edgeNormal[:, :2] @ U
    z = np.zeros(m.nEdges)
    phys = fbrk32.Phys(tau_n=z, cd=2.5e-3, cw=0.0, uw_n=z, uw_t=z)
    dt = 60.0
    h1, u1 = lts.fblts_step(m, lab, h0, u0, dt, M, phys)
    V = U - dt * 2.5e-3 * np.linalg.norm(U) * U / 50.0
    np.testing.assert_allclose(u1, m.edgeNormal[:, :2] @ V, atol=1e-14)
    np.testing.assert_allclose(h1, 50.0, rtol=1e-15)


def test_wind_closed_form():
    """f = 0, fluid at rest, uniform wind U_W: S_e = C_W |U_W| (U_W . n_e) / h -> after one coarse
    step u = dt C_W |U_W| U_W . n_e / h."""
    m = flat()
    lab = lts.label_regions(m, m.xCell > m.Lx / 2)
    UW = np.array([30.0, -10.0])
    t = np.stack([-m.edgeNormal[:, 1], m.edgeNormal[:, 0]], axis=1)
    phys = fbrk32.Phys(tau_n=np.zeros(m.nEdges), cd=2.5e-3, cw=1.8e-6, uw_n=m.edgeNormal[:, :2] @ UW, uw_t=t @ UW)
    h0 = np.full(m.nCells, 50.0)
    dt = 60.0
    h1, u1 = lts.fblts_step(m, lab, h0, np.zeros(m.nEdges), dt, 2, phys)
    expect = dt * 1.8e-6 * np.linalg.norm(UW) * (m.edgeNormal[:, :2] @ UW) / 50.0
    np.testing.assert_allclose(u1, expect, atol=1e-15)


def test_sal_is_reduced_gravity_in_the_fast_term():
    """-g grad(xi - beta xi) = -g (1 - beta) grad(xi): a step with (g, sal) equals one with
    (g (1 - sal), 0) -- the slow terms have no g -- bit for bit."""
    c = configs.small_shelf(nx=32, ny=24, dt=20.0)
    lab = lts.label_regions(c.mesh, c.fine_mask)
    a = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 4, fbrk32.Phys(g=9.81, sal=0.1, tau_n=c.tau_n), 5)
    b = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 4, fbrk32.Phys(g=9.81 * (1.0 - 0.1), tau_n=c.tau_n), 5)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_terms_off_is_the_plain_model():
    c = configs.small_shelf(nx=32, ny=24, dt=20.0)
    lab = lts.label_regions(c.mesh, c.fine_mask)
    a = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 4, fbrk32.Phys(tau_n=c.tau_n), 5)
    b = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 4, fbrk32.Phys(tau_n=c.tau_n, sal=0.0), 5)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_hurricane_case_conserves_mass_and_spins_up():
    c = configs.hurricane_case(nx=48, ny=36)
    lab = lts.label_regions(c.mesh, c.fine_mask)
    phys = fbrk32.Phys(g=c.g, beta=c.beta, tau_n=c.tau_n, rho0=c.rho0, **c.hurricane)
    h, u = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, c.M, phys, 20)
    m0 = dg.total_mass(c.mesh, c.h0)
    assert abs(dg.total_mass(c.mesh, h) - m0) <= 1e-13 * m0
    assert np.all(np.isfinite(u)) and np.max(np.abs(u)) > 1e-3
