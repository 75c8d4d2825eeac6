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


def test_rk32_scalar_oscillator_closed_form():
    """True RK(3,2) (Wicker-Skamarock) on u' = -h, h' = u: with A = [[0, -1], [1, 0]]
    (A^2 = -I, A^3 = -A) the step is R(zA) = (1 - z^2/2) I + (z - z^3/6) A, written out here by hand;
    so (0, 1) at z = 0.1 -> (-(0.1 - 0.001/6), 0.995), exact in rationals."""
    z = Fraction(1, 10)
    u1, h1 = fbrk32.rk32_generic(lambda u, h: -h, lambda u, h: u, Fraction(0), Fraction(1), z)
    assert u1 == -(z - z ** 3 / 6) and h1 == 1 - z ** 2 / 2
    assert float(u1) == pytest.approx(-0.09983333333333333, abs=1e-17) and float(h1) == 0.995
    for zf in (0.05, 0.7, 1.7):
        for col, (u0, h0) in enumerate([(1.0, 0.0), (0.0, 1.0)]):
            u1, h1 = fbrk32.rk32_generic(lambda u, h: -h, lambda u, h: u, u0, h0, zf)
            a, b = 1 - zf ** 2 / 2, zf - zf ** 3 / 6
            G = np.array([[a, -b], [b, a]])
            np.testing.assert_allclose([u1, h1], G[:, col], rtol=0, atol=8 * np.spacing(1.0))


def test_rk32_imaginary_axis_limit_is_sqrt3():
    """|R(iz)|^2 = (1 - z^2/2)^2 + (z - z^3/6)^2 = 1 - z^4/12 + z^6/36 <= 1 iff z <= sqrt(3): the
    amplification of one oracle step on the oscillator (its growth factor per step, measured by
    stepping) is <= 1 just below sqrt(3) and > 1 just above -- the CFL gap FB-RK(3,2) closes
    (3.8621532 / sqrt(3) = 2.23, P:L299-300 'between factors of 1.6 and 2.2')."""
    def growth(z):
        u, h = 0.0, 1.0
        for _ in range(2000):
            u, h = fbrk32.rk32_generic(lambda u, h: -h, lambda u, h: u, u, h, z)
        return np.hypot(u, h) ** (1 / 2000)
    s3 = np.sqrt(3.0)
    assert growth(s3 * (1 - 1e-3)) <= 1.0
    assert growth(s3 * (1 + 1e-3)) > 1.0
    # on LINEAR problems R(z) matches exp(z) through z^3 (Wicker-Skamarock: third order for linear,
    # second for nonlinear), so the local error vs the exact rotation is O(z^4): ratio 16 per halving
    err = []
    for z in (0.02, 0.01):
        u1, h1 = fbrk32.rk32_generic(lambda u, h: -h, lambda u, h: u, 0.0, 1.0, z)
        err.append(np.hypot(u1 + np.sin(z), h1 - np.cos(z)))
    assert 15.0 < err[0] / err[1] < 17.0
    # scalar decay y' = -y: R(-z) = 1 - z + z^2/2 - z^3/6 (z = 0.1 -> 0.9048333...)
    y = fbrk32.rk32_generic(lambda u, h: -u, lambda u, h: 0.0 * h, 1.0, 0.0, 0.1)[0]
    assert y == pytest.approx(1 - 0.1 + 0.005 - 0.001 / 6, abs=1e-16)


def test_rk32_conserves_mass_on_mesh():
    """RK(3,2) on the TRiSK mesh (unsplit, global): mass sum A_i h_i is conserved to roundoff
    (Theorem 1's argument holds for any explicit RK combination of Psi)."""
    c = small_shelf(nx=24, ny=20)
    phys = fbrk32.Phys(tau_n=c.tau_n)
    h, u = c.h0.copy(), c.u0.copy()
    m0 = float(np.sum(c.mesh.areaCell * h))
    for _ in range(10):
        h, u = fbrk32.rk32_step(c.mesh, h, u, 4.0, phys)
    assert abs(float(np.sum(c.mesh.areaCell * h)) - m0) <= 1e-13 * m0
    assert np.all(np.isfinite(u)) and np.max(np.abs(u)) > 0


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


def _standing_wave(eps, n_steps, slow):
    """Global FB-RK(3,2) on a flat 24 x 24 periodic hex (H = 100 m, f = 0) started from
    h = H + eps cos(k.x), u = 0, k = 2 pi (3/L_x, 2/L_y); returns the measured mode amplitudes
    (A_n of h - H on c = cos(k.x), B_n of u on p = D c / kappa) and the linear prediction.
    dt is 0.8 of the stability limit of the fastest (K-point) grid mode, z = omega dt ~ 1."""
    nx = ny = 24
    dc, H, g = 10e3, 100.0, 9.81
    m = build_periodic_hex_mesh(nx, ny, dc)
    m.bottomDepth = np.full(m.nCells, H)
    m.fVertex = np.zeros(m.nVertices)
    Lx, Ly = nx * dc, ny * dc * np.sqrt(3.0) / 2.0
    k = 2.0 * np.pi * np.array([3.0 / Lx, 2.0 / Ly])
    c = np.cos(k[0] * m.xCell + k[1] * m.yCell)
    # P15: kappa^2 = (2 / (3 d^2)) sum_j (1 - cos k.delta_j) over the 6 neighbour offsets of the hex
    delta = dc * np.array([[np.cos(a), np.sin(a)] for a in np.arange(6) * np.pi / 3.0])
    kappa = np.sqrt(2.0 / (3.0 * dc * dc) * np.sum(1.0 - np.cos(delta @ k)))
    c0, c1 = m.cellsOnEdge[:, 0], m.cellsOnEdge[:, 1]
    p = (c[c1] - c[c0]) / m.dcEdge / kappa
    omega = np.sqrt(g * H) * kappa
    dt = 0.8 * 3.8621532 / (np.sqrt(g * H) * np.sqrt(6.0) / dc)    # 0.8 of the grid-scale (K-point) limit
    z = omega * dt
    phys = fbrk32.Phys(g=g, slow=slow)
    h, u = H + eps * c, np.zeros(m.nEdges)
    for _ in range(n_steps):
        h, u = fbrk32.fbrk32_step(m, h, u, dt, phys)
    A = np.dot(h - H, c) / np.dot(c, c)
    B = np.dot(u, p) / np.dot(p, p)
    # linear prediction: (b, a) = (B sqrt(H), A sqrt(g)) obey b' = -omega a, a' = omega b, i.e. the
    # scalar oscillator of P13 with z = omega dt
    y = np.array([0.0, eps * np.sqrt(g)])
    Gz = G_closed(z)
    for _ in range(n_steps):
        y = Gz @ y
    return A, B, y[1] / np.sqrt(g), y[0] / np.sqrt(H), h, u, c, p


@pytest.mark.parametrize("slow", [False, True])
def test_standing_wave_mode_follows_G(slow):
    """P15: a tiny standing wave on the flat regular hex evolves, mode by mode, as the
    scalar FB-RK(3,2) amplification G(omega dt)^n of P13 with the discrete frequency
    omega^2 = g H (2/(3 d^2)) sum_j (1 - cos k.delta_j), and the state stays in the mode.  With the
    slow terms the deviation is their O(eps^2) nonlinearity (O(eps) relative: 1e-3 vs 1e-4); in the
    gravity-wave model the mode follows G to the mesh-geometry rounding (< 1e-8).  A wrong sign, a
    dropped factor or a transposed operand in Psi, Phi^fast or the FB stages changes omega or G."""
    dev = []
    for eps in (1e-3, 1e-4):
        A, B, A_lin, B_lin, h, u, c, p = _standing_wave(eps, 10, slow)
        scale = np.hypot(A_lin, B_lin * np.sqrt(100.0 / 9.81))
        dev.append(max(abs(A - A_lin), abs(B - B_lin) * np.sqrt(100.0 / 9.81)) / scale)
        assert np.max(np.abs(h - 100.0 - A * c)) <= 1e-2 * eps      # no other mode excited (O(eps^2))
        assert np.max(np.abs(u - B * p)) <= 1e-2 * np.max(np.abs(B * p)) + 1e-12
    if slow:        # q_hat F_perp - grad K is O(eps^2): the mode deviates at O(eps) relative
        assert dev[0] < 1e-3 and dev[1] < 1e-4
        assert 5.0 < dev[0] / dev[1] < 20.0
    else:           # gravity-wave model: h_e u is the only nonlinearity and it feeds other modes only
        assert dev[0] < 1e-8 and dev[1] < 1e-8
