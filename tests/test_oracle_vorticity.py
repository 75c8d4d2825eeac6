"""Pins of the prognostic absolute-vorticity companion (Theorem 2; SPEC
step_prognostic_vorticity S:L472-480): oracle/lts.py fblts_step(eta=...) and
oracle/trisk.py vorticity_update.

What fixes it, independently of the companion's own code:
* Theorem 2: the total sum_v A_v eta_v is conserved to roundoff by FB-LTS, unsplit and split, any M;
* Ringler et al. 2010: the prognostically advanced eta equals the diagnostic
  eta = curl u + f of the advanced velocity "up to machine precision" when the velocity update has no
  rotational forcing (its gradient terms have zero discrete curl in exact arithmetic) -- a dropped PV
  term, a wrong t_{e,v} sign or a wrong stage would show as an O(1) difference;
* M = 1 reduces it to the global FB-RK(3,2) companion eta + dt Theta(u_bar^{n+1/2}, h***),
  built here from the oracle's global stages.
"""
import numpy as np
import pytest

from inputs import configs
from oracle import fbrk32, lts, trisk


def phys_of(c, **kw):
    return fbrk32.Phys(g=c.g, beta=c.beta, slow=c.slow, tau_n=c.tau_n, rho0=c.rho0, **kw)


def eta_diag(mesh, u):
    return trisk.relative_vorticity(mesh, u) + mesh.fVertex


def spin_up(c, n=3):
    """A state with velocity: a few split steps from the case's initial bump."""
    lab = lts.label_regions(c.mesh, c.fine_mask)
    h, u = lts.run(c.mesh, lab, c.h0, c.u0, c.dt, c.M, phys_of(c), n)
    return lab, h, u


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("which", ["config1", "shelf"])
def test_theorem2_total_conserved(which, split):
    c = configs.config1() if which == "config1" else configs.small_shelf(nx=40, ny=36, dt=20.0)
    lab, h, u = spin_up(c)
    m = c.mesh
    eta = eta_diag(m, u)
    tot0 = float(np.sum(m.areaTriangle * eta))
    scale = float(np.sum(m.areaTriangle * np.abs(eta)))
    out = lts.run(m, lab, h, u, c.dt, c.M, phys_of(c), 10, split=split, eta=eta)
    tot1 = float(np.sum(m.areaTriangle * out[2]))
    assert np.all(np.isfinite(out[2]))
    assert abs(tot1 - tot0) <= 1e-13 * scale, (tot1 - tot0) / scale
    assert np.max(np.abs(out[2] - eta)) > 1e-12 * np.max(np.abs(eta))       # it does evolve


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("M", [1, 4])
def test_prognostic_equals_diagnostic_without_forcing(split, M):
    """No wind forcing (its curl is the only rotational term besides the PV flux): after 10 FB-LTS
    steps the prognostic eta equals curl u + f of the stepped velocity to roundoff, on every vertex --
    including the vertices on the fine / IF-1 / IF-2 / interior boundaries, whose edges take their
    fluxes from the subcycles, the correction and the coarse stage respectively."""
    c = configs.config1()
    c.M = M
    lab, h, u = spin_up(c)
    m = c.mesh
    eta = eta_diag(m, u)
    h1, u1, eta1 = lts.run(m, lab, h, u, c.dt, M, phys_of(c), 10, split=split, eta=eta)
    diag = eta_diag(m, u1)
    err = np.max(np.abs(eta1 - diag)) / np.max(np.abs(diag - m.fVertex))
    assert err <= 1e-11, err          # observed ~1e-13
    # and the companion is not trivially equal to its start
    assert np.max(np.abs(eta1 - eta)) > 1e-3 * np.max(np.abs(diag - m.fVertex))


def test_m1_companion_is_global_fbrk32_companion():
    """M = 1: eta^{n+1} = eta^n + dt Theta(u_bar^{n+1/2}, h***) of global unsplit FB-RK(3,2), bitwise."""
    c = configs.config1()
    lab, h, u = spin_up(c)
    m = c.mesh
    phys = phys_of(c)
    eta = eta_diag(m, u)
    _, _, eta1 = lts.fblts_step(m, lab, h, u, c.dt, 1, phys, split=False, eta=eta)
    _, _, st = fbrk32.fbrk32_step(m, h, u, c.dt, phys, split=False, stages=True)
    b1, b2, b3 = phys.beta
    hs3 = b3 * st["h3"] + (1.0 - 2.0 * b3) * st["h2"] + b3 * h
    dP = c.dt * trisk.pv_flux(m, st["u2"], hs3, phys)
    ref = trisk.vorticity_update(m, eta, dP)
    assert np.array_equal(eta1, ref)


def test_zero_flux_leaves_eta_unchanged():
    """At rest with uniform thickness the PV flux vanishes: eta is unchanged bit for bit."""
    c = configs.config1()
    m = c.mesh
    c.slow = True
    lab = lts.label_regions(m, c.fine_mask)
    h = np.full(m.nCells, 1000.0)
    m.bottomDepth = np.full(m.nCells, 1000.0)
    u = np.zeros(m.nEdges)
    eta = eta_diag(m, u)
    _, _, eta1 = lts.fblts_step(m, lab, h, u, c.dt, c.M, phys_of(c), split=False, eta=eta)
    assert np.array_equal(eta1, eta)
