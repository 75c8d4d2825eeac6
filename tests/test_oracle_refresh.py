"""Pins for the slow-term refresh variant of FB-LTS (the paper's proposal
P:L1427-1431: slow tendencies evaluated at t^{n,k} and used while advancing on fine cells;
reading in DESIGN.md section 3).  What fixes it without an implementation to compare against:
special cases that reduce to the frozen-S scheme bit for bit, conservation of mass (the slow
terms act only on u), the finite-stencil property (the NaN-poisoned views stay finite on F_E), and
a closed form: on an f-plane with uniform h and U the refreshed scheme rotates the deep fine
velocity by M forward-Euler steps of dt/M, the frozen one by a single step of dt."""
import numpy as np
import pytest

from inputs.configs import config1, small_shelf
from inputs.hexmesh import build_periodic_hex_mesh
from oracle import diagnostics as dg
from oracle import fbrk32, lts


def phys_of(c, slow=True):
    return fbrk32.Phys(g=c.g, beta=c.beta, slow=slow, tau_n=c.tau_n, rho0=c.rho0)


@pytest.fixture(scope="module")
def shelf():
    c = small_shelf(nx=40, ny=36, dt=12.0)
    return c, lts.label_regions(c.mesh, c.fine_mask)


def test_M1_refresh_is_frozen_scheme(shelf):
    """M = 1: the only level is k = 0, whose state is (h^n, u^n) on every view -> S^0 = S bitwise."""
    c, lab = shelf
    a = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 1, phys_of(c), 5)
    b = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 1, phys_of(c), 5, slow_refresh=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_gravity_wave_model_unchanged(shelf):
    """Slow terms off: nothing to refresh, bitwise equal for any M."""
    c, lab = shelf
    a = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 4, phys_of(c, slow=False), 5)
    b = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 4, phys_of(c, slow=False), 5, slow_refresh=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_no_fine_cells_unchanged():
    c = config1(dt=60.0)
    lab = lts.label_regions(c.mesh, np.zeros(c.mesh.nCells, dtype=bool))
    a = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 4, phys_of(c), 5)
    b = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 4, phys_of(c), 5, slow_refresh=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("M", [2, 4])
def test_refresh_conserves_mass_and_stays_finite(shelf, M):
    """Theorem 1 is untouched (S enters only the momentum equation); the refreshed S^k stencil
    stays inside the views (no NaN reaches a fine edge); the result differs from the frozen scheme."""
    c, lab = shelf
    h, u = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, M, phys_of(c), 20, slow_refresh=True)
    assert np.all(np.isfinite(h)) and np.all(np.isfinite(u))
    m0 = dg.total_mass(c.mesh, c.h0)
    assert abs(dg.total_mass(c.mesh, h) - m0) <= 1e-13 * m0
    hf, uf = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, M, phys_of(c), 20)
    assert np.max(np.abs(u - uf)) > 1e-9


def test_inertial_rotation_closed_form():
    """f-plane, uniform h and U (M = 2, one coarse step): Phi^fast = 0 exactly and S = f (U . t_e).
    Refreshed: the fine edges whose slow stencil holds only fine data (both cells at hop >= 2 from
    C) take two forward-Euler rotations of dt/2, (u, v) <- (u + f dt/2 v, v - f dt/2 u) twice;
    frozen: one rotation of dt on every edge (P8).  The two differ at O((f dt)^2) -- checked."""
    m = build_periodic_hex_mesh(24, 20, 2000.0)
    m.bottomDepth = np.full(m.nCells, 100.0)
    m.fVertex = np.full(m.nVertices, 1e-4)
    fine = m.xCell > m.Lx / 2
    lab = lts.label_regions(m, fine)
    phys = fbrk32.Phys(tau_n=np.zeros(m.nEdges))
    U = np.array([0.4, -0.2])
    dt, f = 400.0, 1e-4
    h0 = np.full(m.nCells, 100.0)
    u0 = m.edgeNormal[:, :2] @ U
    h1, u1 = lts.fblts_step(m, lab, h0, u0, dt, 2, phys, slow_refresh=True)
    hf, uf = lts.fblts_step(m, lab, h0, u0, dt, 2, phys)
    rho = lts.hop_distance(m, ~fine, 20)
    deep = (rho[m.cellsOnEdge[:, 0]] >= 2) & (rho[m.cellsOnEdge[:, 1]] >= 2)
    assert deep.sum() > 100
    V = U.copy()
    for _ in range(2):
        V = np.array([V[0] + f * (dt / 2) * V[1], V[1] - f * (dt / 2) * V[0]])
    W = np.array([U[0] + f * dt * U[1], U[1] - f * dt * U[0]])
    np.testing.assert_allclose(u1[deep], (m.edgeNormal[:, :2] @ V)[deep], atol=1e-14 * np.linalg.norm(U))
    np.testing.assert_allclose(uf[deep], (m.edgeNormal[:, :2] @ W)[deep], atol=1e-14 * np.linalg.norm(U))
    assert np.max(np.abs(V - W)) > 1e-4 * np.linalg.norm(U)
    # near the interface the refreshed fine velocities differ from the predicted IF-1 ones at
    # O((f dt)^2), so the thickness moves there -- conservatively (with the frozen S only at roundoff)
    np.testing.assert_allclose(hf, 100.0, rtol=1e-12)
    assert np.max(np.abs(h1 - 100.0)) > 1e-9
    assert abs(dg.total_mass(m, h1) - dg.total_mass(m, h0)) <= 1e-13 * dg.total_mass(m, h0)
