"""Global time integrators: FB-RK(3,2) and classical RK4 (oracle; test infrastructure only)."""
from __future__ import annotations

import dataclasses

import numpy as np

from . import trisk

# FB weights (beta1, beta2, beta3) = (0.531, 0.531, 0.313).
BETA_PAPER = (0.531, 0.531, 0.313)


@dataclasses.dataclass
class Phys:
    """Physics of the split shallow-water model.

    g: gravity (9.81, reading Q28); beta: FB weights; slow: whether the
    slow terms are on (False = gravity-wave model);
    tau_n: per-edge wind-stress projection tau . n_e (N m^-2, reading Q19);
    rho0: reference density (kg m^-3).
    Hurricane-model terms (eq. hurricane_model, synthetic forcing):
    sal: self-attraction-and-loading coefficient beta of the fast term -g grad(xi - beta xi)
    (eq. hurricane_fast_terms), evaluated with g_fast = g (1 - sal);
    cd: bottom-drag coefficient C_D; cw: wind coefficient C_W; uw_n, uw_t: per-edge normal and
    tangential components of the wind velocity u_W (None: no drag / wind terms).
    pv: the PV flux term of the slow tendency -- "centered": q_hat_e F_perp_e with
    q_hat_e = (q_v0 + q_v1) / 2 (reading Q2, the paper's symbol); "energy": the
    energy-conserving TRiSK form sum_j W_{e,j} F_{e_j} (q_hat_e + q_hat_{e_j}) / 2.
    """
    g: float = 9.81
    beta: tuple = BETA_PAPER
    slow: bool = True
    tau_n: np.ndarray | None = None
    rho0: float = 1000.0
    sal: float = 0.0
    cd: float = 0.0
    cw: float = 0.0
    uw_n: np.ndarray | None = None
    uw_t: np.ndarray | None = None
    pv: str = "centered"

    def g_fast(self):
        """g (1 - beta_SAL): the gravity of the fast term -g grad(xi - beta xi)."""
        return self.g * (1.0 - self.sal)

    def hurricane(self):
        return self.uw_n is not None

    def with_tau(self, mesh):
        if self.tau_n is None:
            self.tau_n = np.zeros(mesh.nEdges)
        return self


def fbrk32_generic(Phi, Psi, u, h, dt, beta, stages=False):
    """One FB-RK(3,2) step of u' = Phi(u, h), h' = Psi(u, h)  (eq. fbrk32).

    Stage 1:  h1 = h^n + dt/3 Psi(u^n, h^n);   h*  = b1 h1 + (1-b1) h^n;   u1 = u^n + dt/3 Phi(u^n, h*)
    Stage 2:  h2 = h^n + dt/2 Psi(u1, h1);     h** = b2 h2 + (1-b2) h^n;   u2 = u^n + dt/2 Phi(u1, h**)
    Stage 3:  h3 = h^n + dt Psi(u2, h2);       h*** = b3 h3 + (1-2 b3) h2 + b3 h^n;  u3 = u^n + dt Phi(u2, h***)
    Each h-update precedes its u-update (the forward-backward order).
    Works on numpy arrays or on exact fractions (for closed-form pins).
    """
    b1, b2, b3 = beta
    one = b1 - b1 + 1  # 1 in the number type of beta (float or Fraction)
    omb1 = one - b1
    omb2 = one - b2
    om2b3 = one - 2 * b3
    c1 = dt / 3
    c2 = dt / 2
    c3 = dt
    h1 = h + c1 * Psi(u, h)
    hs1 = b1 * h1 + omb1 * h
    u1 = u + c1 * Phi(u, hs1)
    h2 = h + c2 * Psi(u1, h1)
    hs2 = b2 * h2 + omb2 * h
    u2 = u + c2 * Phi(u1, hs2)
    h3 = h + c3 * Psi(u2, h2)
    hs3 = b3 * h3 + om2b3 * h2 + b3 * h
    u3 = u + c3 * Phi(u2, hs3)
    if stages:
        return u3, h3, {"h1": h1, "h2": h2, "h3": h3, "u1": u1, "u2": u2, "u3": u3}
    return u3, h3


def mesh_tendencies(mesh, phys, S=None):
    """(Phi, Psi) closures on the whole mesh.

    Split mode (S given): Phi(u, h_FB) = Phi^fast(h_FB) + S.
    Unsplit (S None, reading Q16): Phi(u, h_FB) = Phi^fast(h_FB) + Phi^slow(u, h_FB).
    Psi(u, h) = trisk thickness tendency (no split in the thickness equation).
    """
    cells = np.arange(mesh.nCells)
    edges = np.arange(mesh.nEdges)
    phys.with_tau(mesh)

    def Psi(u, h):
        return trisk.thickness_tendency(mesh, u, h, cells)

    if S is not None:
        def Phi(u, h):
            return trisk.fast_momentum(mesh, h, phys.g_fast(), edges) + S
    else:
        def Phi(u, h):
            f = trisk.fast_momentum(mesh, h, phys.g_fast(), edges)
            if not phys.slow:
                return f + np.zeros(mesh.nEdges)
            return f + trisk.slow_momentum(mesh, u, h, phys.tau_n, phys.rho0, phys)
    return Phi, Psi


def fbrk32_step(mesh, h, u, dt, phys, split=True, stages=False):
    """Global FB-RK(3,2) on the whole mesh (the M = 1 / no-fine-cells case)."""
    phys.with_tau(mesh)
    S = trisk.slow_tendency(mesh, u, h, phys) if split else None
    Phi, Psi = mesh_tendencies(mesh, phys, S)
    out = fbrk32_generic(Phi, Psi, u, h, dt, phys.beta, stages=stages)
    if stages:
        return out[1], out[0], out[2]
    return out[1], out[0]


def rk32_generic(Phi, Psi, u, h, dt):
    """One step of RK(3,2), the three-stage second-order Runge-Kutta scheme of Wicker & Skamarock
    (2002) that FB-RK(3,2) extends (subsec. fbrk32): every stage evaluates both
    tendencies at the previous stage's (u, h), no forward-backward averaging:
        stage 1:  h1 = h^n + dt/3 Psi(u^n, h^n);  u1 = u^n + dt/3 Phi(u^n, h^n)
        stage 2:  h2 = h^n + dt/2 Psi(u1, h1);    u2 = u^n + dt/2 Phi(u1, h1)
        stage 3:  h3 = h^n + dt   Psi(u2, h2);    u3 = u^n + dt   Phi(u2, h2)
    For y' = lambda y the step multiplies by R(z) = 1 + z + z^2/2 + z^3/6 (z = lambda dt): stable on
    the imaginary axis iff |z| <= sqrt(3).  Works on numpy arrays or exact fractions."""
    c1 = dt / 3
    c2 = dt / 2
    c3 = dt
    h1 = h + c1 * Psi(u, h)
    u1 = u + c1 * Phi(u, h)
    h2 = h + c2 * Psi(u1, h1)
    u2 = u + c2 * Phi(u1, h1)
    h3 = h + c3 * Psi(u2, h2)
    u3 = u + c3 * Phi(u2, h2)
    return u3, h3


def rk32_step(mesh, h, u, dt, phys):
    """RK(3,2) on the unsplit system (u, h), global (the baseline FB-RK(3,2) extends, P:L283-285;
    the Table-1 analogue's third scheme)."""
    Phi, Psi = mesh_tendencies(mesh, phys, None)
    u3, h3 = rk32_generic(Phi, Psi, u, h, dt)
    return h3, u3


def rk4_generic(f, y, dt):
    """Classical four-stage RK4 ("classical, four-stage, fourth order")."""
    k1 = f(y)
    k2 = f(y + (dt / 2) * k1)
    k3 = f(y + (dt / 2) * k2)
    k4 = f(y + dt * k3)
    return y + (dt / 6) * (k1 + 2 * k2 + 2 * k3 + k4)


def rk4_step(mesh, h, u, dt, phys):
    """RK4 on the unsplit system (u, h) (convergence reference)."""
    Phi, Psi = mesh_tendencies(mesh, phys, None)
    nC = mesh.nCells

    def f(y):
        hh, uu = y[:nC], y[nC:]
        return np.concatenate([Psi(uu, hh), Phi(uu, hh)])

    y = rk4_generic(f, np.concatenate([h, u]), dt)
    return y[:nC].copy(), y[nC:].copy()
