"""Pins for the unsplit FB-LTS oracle (the scheme of P:L468-787 with the full
Phi(U, HS) = Phi^fast(HS) + Phi^slow(U, HS) in every velocity update, reading Q16).  Fixed without an
implementation to compare against: the special cases that reduce to global unsplit FB-RK(3,2)
 or to the split scheme (slow terms off, P17) bit for bit; the paper's shrinking extents
being exactly sufficient (NaN-poisoned arrays outside every extent stay out of the result);
Theorems 1-2 (mass and absolute vorticity); and the inertial-oscillation closed form of the
unsplit scheme on the deep fine edges (M steps of the RK3 polynomial at dt/M, P8)."""
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


def global_unsplit(c, n, dt):
    h, u = c.h0.copy(), c.u0.copy()
    for _ in range(n):
        h, u = fbrk32.fbrk32_step(c.mesh, h, u, dt, phys_of(c), split=False)
    return h, u


def test_M1_unsplit_is_global_unsplit_fbrk32(shelf):
    c, lab = shelf
    a = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 1, phys_of(c), 5, split=False)
    b = global_unsplit(c, 5, c.dt)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_no_fine_cells_unsplit_is_global():
    c = config1(dt=60.0)
    lab = lts.label_regions(c.mesh, np.zeros(c.mesh.nCells, dtype=bool))
    a = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 4, phys_of(c), 5, split=False)
    b = global_unsplit(c, 5, c.dt)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_without_slow_terms_unsplit_is_split(shelf):
    c, lab = shelf
    a = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 4, phys_of(c, slow=False), 5, split=False)
    b = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, 4, phys_of(c, slow=False), 5)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("M", [2, 4])
def test_extents_suffice_and_theorems_hold(shelf, M):
    """Every array is NaN outside the extent that computes it: a finite result proves the slow
    stencils of Y1/Y2/Y3 stay inside X1/X2/X3 and the fine ones inside the views.  Mass and the
    diagnostic absolute vorticity are conserved to roundoff (Theorems 1-2)."""
    c, lab = shelf
    h, u = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, M, phys_of(c), 20, split=False)
    assert np.all(np.isfinite(h)) and np.all(np.isfinite(u))
    m0 = dg.total_mass(c.mesh, c.h0)
    assert abs(dg.total_mass(c.mesh, h) - m0) <= 1e-13 * m0
    G0 = dg.total_abs_vorticity(c.mesh, c.u0)
    fscale = float(np.sum(c.mesh.areaTriangle * np.abs(c.mesh.fVertex)))
    assert abs(dg.total_abs_vorticity(c.mesh, u) - G0) <= 1e-13 * fscale
    hs, us = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, M, phys_of(c), 20)
    assert np.max(np.abs(u - us)) > 1e-9          # the unsplit scheme is a different scheme


def test_inertial_oscillation_deep_fine_edges():
    """f-plane, uniform h and U, one coarse step, M = 2: Psi = 0 and Phi^fast = 0 exactly while the
    field is uniform, so far from the interface the unsplit fine subcycles apply the RK3 polynomial
    R(z) = 1 + z + z^2/2 + z^3/6, z = -i f dt/M, twice to w = u + i v, and the interior coarse edges
    R(-i f dt) once (P8 unsplit); edges near the interface see predicted values and differ."""
    m = build_periodic_hex_mesh(96, 8, 2000.0)
    m.bottomDepth = np.full(m.nCells, 100.0)
    m.fVertex = np.full(m.nVertices, 1e-4)
    fine = m.xCell > m.Lx / 2
    lab = lts.label_regions(m, fine)
    phys = fbrk32.Phys(tau_n=np.zeros(m.nEdges))
    dt, f = 600.0, 1e-4
    w = complex(0.4, -0.2)
    h0 = np.full(m.nCells, 100.0)
    u0 = m.edgeNormal[:, :2] @ np.array([w.real, w.imag])
    h1, u1 = lts.fblts_step(m, lab, h0, u0, dt, 2, phys, split=False)
    R = lambda z: 1 + z + z * z / 2 + z ** 3 / 6
    wf = R(-1j * f * dt / 2) ** 2 * w
    wc = R(-1j * f * dt) * w
    rho = lts.hop_distance(m, ~fine, 40)
    dF = lts.hop_distance(m, fine, 40)
    c0, c1 = m.cellsOnEdge[:, 0], m.cellsOnEdge[:, 1]
    deep_f = (np.minimum(rho[c0], rho[c1]) >= 16)
    deep_c = (np.minimum(dF[c0], dF[c1]) >= 16)
    assert deep_f.sum() > 50 and deep_c.sum() > 50
    un = lambda ww: m.edgeNormal[:, :2] @ np.array([ww.real, ww.imag])
    np.testing.assert_allclose(u1[deep_f], un(wf)[deep_f], atol=1e-14)
    np.testing.assert_allclose(u1[deep_c], un(wc)[deep_c], atol=1e-14)
    assert abs(wf - wc) > 1e-7                   # O((f dt)^4): far above the 1e-14 tolerance
