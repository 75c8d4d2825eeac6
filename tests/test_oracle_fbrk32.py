"""Pins for the global integrators (P13, P17, P18, P22; RK4 scalar)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from inputs.configs import small_shelf
from inputs.hexmesh import build_periodic_hex_mesh
from oracle import fbrk32

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fbrk32_scalar.json")))


def poly(coeffs, z):
    return sum(float(Fraction(str(c))) * z ** p for p, c in coeffs)


def G_closed(z):
    g = GOLD["G"]
    return np.array([[poly(g["uu"], z), poly(g["uh"], z)], [poly(g["hu"], z), poly(g["hh"], z)]])


def oscillator_step(u, h, dt):
    return fbrk32.fbrk32_generic(lambda u, h: -h, lambda u, h: u, u, h, dt, fbrk32.BETA_PAPER)


def test_scalar_oscillator_example():
    """P13: u' = -h, h' = u, dt = 0.1, (0, 1) -> (-0.09978130516916667, 0.995004425) (eq. fbrk32)."""
    ex = GOLD["example"]
    u1, h1 = oscillator_step(ex["u0"], ex["h0"], ex["dt"])
    assert abs(u1 - ex["u1"]) <= 2 * np.spacing(abs(ex["u1"]))
    assert abs(h1 - ex["h1"]) <= 2 * np.spacing(abs(ex["h1"]))


@pytest.mark.parametrize("z", [0.05, 0.3, 1.0, 2.5, 3.8])
def test_scalar_oscillator_matches_closed_form(z):
    """P13: the step equals the exact rational amplification matrix G(z) to a few ulp."""
    G = G_closed(z)
    for col, (u0, h0) in enumerate([(1.0, 0.0), (0.0, 1.0)]):
        u1, h1 = oscillator_step(u0, h0, z)
        np.testing.assert_allclose([u1, h1], G[:, col], rtol=0, atol=8 * np.spacing(np.max(np.abs(G))))


def test_stability_limit_and_weights():
    """P13: FB-RK(3,2) with the paper's weights is stable on the oscillator iff z <= 3.8621532;
    and it is second order (local error O(z^3))."""
    zmax = GOLD["stability_limit_z"]
    rho = lambda z: np.max(np.abs(np.linalg.eigvals(G_closed(z))))
    assert rho(zmax - 1e-6) <= 1.0 + 1e-12
    assert rho(zmax + 1e-5) > 1.0
    assert all(rho(z) <= 1.0 + 1e-12 for z in np.linspace(0.01, zmax - 1e-5, 200))
    # local error vs the exact rotation: ratio 8 per halving of z -> third-order local error
    err = []
    for z in (0.02, 0.01):
        u1, h1 = oscillator_step(0.0, 1.0, z)
        err.append(np.hypot(u1 + np.sin(z), h1 - np.cos(z)))
    assert 7.0 < err[0] / err[1] < 9.0


def test_rk4_scalar():
    """Classical RK4 on h' = -h, dt = 0.1 -> 0.9048375."""
    r = GOLD["rk4_exp"]
    y = fbrk32.rk4_generic(lambda y: -y, 1.0, r["dt"])
    assert y == pytest.approx(r["factor"], abs=1e-15)


def test_split_equals_unsplit_without_slow_terms():
    """P17: with the slow terms disabled (gravity-wave model) the split and
    unsplit FB-RK(3,2) steps are bit-identical."""
    c = small_shelf(nx=24, ny=20, forcing=False)
    phys = fbrk32.Phys(slow=False, tau_n=c.tau_n)
    m = c.mesh
    h, u = c.h0.copy(), c.u0.copy()
    for _ in range(3):
        h, u = fbrk32.fbrk32_step(m, h, u, 5.0, phys, split=True)
    h2, u2 = c.h0.copy(), c.u0.copy()
    for _ in range(3):
        h2, u2 = fbrk32.fbrk32_step(m, h2, u2, 5.0, phys, split=False)
    assert np.array_equal(h, h2) and np.array_equal(u, u2)


def test_split_error_is_second_order_locally():
    """P18: with forcing and rotation on, the one-step split - unsplit gap shrinks ~4x per halving of dt
    (first-order Lie-Trotter splitting)."""
    c = small_shelf(nx=24, ny=20)
    m = c.mesh
    phys = fbrk32.Phys(tau_n=c.tau_n)
    h, u = c.h0.copy(), c.u0.copy()
    for _ in range(40):                                    # spin up a nonzero flow (global nu ~ 0.5)
        h, u = fbrk32.fbrk32_step(m, h, u, 5.0, phys)
    gaps = []
    for dt in (10.0, 5.0, 2.5):
        hs, us = fbrk32.fbrk32_step(m, h, u, dt, phys, split=True)
        hu, uu = fbrk32.fbrk32_step(m, h, u, dt, phys, split=False)
        gaps.append(np.max(np.abs(us - uu)))
    r1, r2 = gaps[0] / gaps[1], gaps[1] / gaps[2]
    assert 3.4 < r1 < 4.6 and 3.4 < r2 < 4.6, gaps


@pytest.mark.parametrize("factor,grows", [(0.99, False), (1.05, True)])
def test_global_cfl_limit_on_hex(factor, grows):
    """P22: global FB-RK(3,2), gravity-wave model, tiny amplitude on a regular hex with nx, ny multiples
    of 6: stable at 0.99 nu_max, unstable at 1.05 nu_max with nu_max = 3.8621532/sqrt(6) (eq. cfl, P:L9-16;
    sqrt(6) c/d is the largest TRiSK gravity-wave frequency on a regular hex, reading Q12)."""
    m = build_periodic_hex_mesh(12, 12, 1000.0)
    H = 100.0
    m.bottomDepth = np.full(m.nCells, H)
    m.fVertex = np.zeros(m.nVertices)
    phys = fbrk32.Phys(slow=False, tau_n=np.zeros(m.nEdges))
    nu = factor * GOLD["stability_limit_z"] / np.sqrt(6.0)
    dt = nu * 1000.0 / np.sqrt(phys.g * H)
    rng = np.random.default_rng(11)
    h = H + 1e-6 * rng.standard_normal(m.nCells)
    u = np.zeros(m.nEdges)
    a0 = np.max(np.abs(h - H))
    with np.errstate(all="ignore"):
        for _ in range(300):
            h, u = fbrk32.fbrk32_step(m, h, u, dt, phys)
        a1 = np.max(np.abs(h - H))
    if grows:
        assert not np.isfinite(a1) or a1 > 100 * a0
    else:
        assert a1 < 2 * a0
