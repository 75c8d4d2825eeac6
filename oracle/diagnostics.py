"""Diagnostics: conserved integrals, Courant numbers, RMS error (oracle; test infrastructure only)."""
from __future__ import annotations

import math

import numpy as np

from . import trisk


def total_mass(mesh, h):
    """sum_i A_i h_i (Theorem 1), correctly rounded sum of the products."""
    return math.fsum((mesh.areaCell * h).tolist())


def vertex_abs_vorticity_integrals(mesh, u):
    """Per vertex: circulation + A_v f_v = A_v (zeta_v + f_v) = A_v eta_v."""
    return trisk.circulation(mesh, u) + mesh.areaTriangle * mesh.fVertex


def total_abs_vorticity(mesh, u):
    """Gamma = sum_v A_v eta_v (Theorem 2), diagnostic form."""
    return math.fsum(vertex_abs_vorticity_integrals(mesh, u).tolist())


def total_pv_volume(mesh, h, u):
    """Volume integral of PV, sum_v A_v h_v q_v (Remark rmk:volume_conservation_pv, eq.
    vol_integral_pv): h_v the kite-weighted dual-cell thickness, q_v = eta_v / h_v.
    Equal to Gamma = sum_v A_v eta_v up to rounding (the identity the remark uses), so FB-LTS
    conserves it wherever Theorem 2 holds.  Raises if some h_v <= 0 (q undefined)."""
    hv = trisk.vertex_thickness(mesh, h)
    if np.any(~(hv > 0.0)):
        raise ValueError("total_pv_volume: dual-cell thickness h_v <= 0")
    q = trisk.potential_vorticity(mesh, u, h)
    return math.fsum((mesh.areaTriangle * hv * q).tolist())


def courant_numbers(mesh, lab, h, u, dt, M, g):
    """nu_e = (|u_e| + sqrt(g h_e)) dt_e / d_e with dt_e = dt/M on F_E, else dt  (eq. cfl)."""
    c0, c1 = mesh.cellsOnEdge[:, 0], mesh.cellsOnEdge[:, 1]
    h_e = 0.5 * (h[c0] + h[c1])
    dte = np.where(lab.F_E(), dt / M, dt) if lab is not None else np.full(mesh.nEdges, float(dt))
    return (np.abs(u) + np.sqrt(g * h_e)) * dte / mesh.dcEdge


def rest_courant(mesh, lab, dt, M, g):
    """nu_loc = max_e sqrt(g max(H_c0, H_c1)) dt_e / d_e  (reading Q12, at rest)."""
    H = mesh.bottomDepth
    c = np.sqrt(g * np.maximum(H[mesh.cellsOnEdge[:, 0]], H[mesh.cellsOnEdge[:, 1]]))
    dte = np.where(lab.F_E(), dt / M, dt)
    return float(np.max(c * dte / mesh.dcEdge))


def rms_error(s, m):
    """E_RMS = sqrt(sum (s_i - m_i)^2 / N)  (eq. rmse)."""
    s = np.asarray(s, dtype=np.float64)
    m = np.asarray(m, dtype=np.float64)
    if s.shape != m.shape:
        raise ValueError("rms_error: length mismatch")
    return float(np.sqrt(np.sum((s - m) ** 2) / s.size))


def diagnostics(mesh, lab, h, u, dt, M, g):
    """(mass, Gamma, min h, max nu) -- the four numbers fblts_diagnostics reports."""
    return (total_mass(mesh, h), total_abs_vorticity(mesh, u), float(np.min(h)),
            float(np.max(courant_numbers(mesh, lab, h, u, dt, M, g))))


def speedup(baseline_seconds, candidate_seconds):
    """speedup = baseline CPU-time / FB-LTS CPU-time  (eq. speedup)."""
    if candidate_seconds <= 0 or baseline_seconds <= 0:
        raise ValueError("speedup: times must be positive")
    return baseline_seconds / candidate_seconds
