"""TRiSK spatial operators, literal fp64 numpy (oracle; test infrastructure only).

Notation: h_i at cell centres, u_e normal velocity at edges
(eq. semi_discrete_sys).  ``cells``/``edges`` arguments restrict the
evaluation to an index subset (the LTS phases evaluate on region subsets); the
result has the length of the subset.
"""
from __future__ import annotations

import numpy as np


def n_sign(mesh, cells, j):
    """n_{e,i} for slot j of the given cells: +1 if the cell is cellsOnEdge[e][0].

    P:L961: n_{e,i} in {1,-1} such that n_{e,i} n_e is the outward normal of i;
    n_e points from cellsOnEdge[e][0] to cellsOnEdge[e][1] (SURVEY c.1).
    """
    e = mesh.edgesOnCell[cells, j]
    return np.where(mesh.cellsOnEdge[e, 0] == cells, 1.0, -1.0)


def edge_flux(mesh, U, H, edges):
    """F_e = h_e u_e with h_e = 0.5 (h[c0] + h[c1]).

    P:L962 ("F_e is the signed value of the thickness flux"); the edge-thickness
    closure (centred mean) is the reading Q1 (SURVEY c.4).
    """
    c0 = mesh.cellsOnEdge[edges, 0]
    c1 = mesh.cellsOnEdge[edges, 1]
    h_e = 0.5 * (H[c0] + H[c1])
    return h_e * U[edges]


def thickness_tendency(mesh, U, H, cells):
    """Psi_i(u, h) = -(1/A_i) sum_{e in E_i} n_{e,i} l_e F_e  (eq. trisk_thickness).

    Evaluated as  -(sum_j n_{e_j,i} * l_{e_j} * F_{e_j}) / A_i,  sum sequential in
    edgesOnCell slot order from +0.0.
    """
    cells = np.asarray(cells)
    acc = np.zeros(cells.size)
    nE = mesh.nEdgesOnCell[cells]
    for j in range(mesh.maxEdges):
        act = j < nE
        if not np.any(act):
            break
        c = cells[act]
        e = mesh.edgesOnCell[c, j]
        F = edge_flux(mesh, U, H, e)
        term = n_sign(mesh, c, j) * mesh.dvEdge[e] * F
        acc[act] = acc[act] + term
    return -acc / mesh.areaCell[cells]


def fast_momentum(mesh, H, g, edges):
    """Phi^fast_e = -g grad(h + z_b) . n_e  (eq. fast_terms).

    Evaluated as  -g * ((h[c1] + z_b[c1]) - (h[c0] + z_b[c0])) / d_e  with
    z_b = -bottomDepth and d_e = dcEdge (reading Q3, Q15: (h + z_b) per cell first,
    then the difference; never fold -g grad z_b into a separate term).
    """
    c0 = mesh.cellsOnEdge[edges, 0]
    c1 = mesh.cellsOnEdge[edges, 1]
    zb = -mesh.bottomDepth
    t1 = H[c1] + zb[c1]
    t0 = H[c0] + zb[c0]
    return -g * (t1 - t0) / mesh.dcEdge[edges]


def relative_vorticity(mesh, U):
    """zeta_v = (1/A_v) sum_{e in E_v} t_{e,v} d_e u_e on every vertex.

    Circulation on the dual cell ("eta = k . curl u + f");
    t_{e,v} = +1 if v = verticesOnEdge[e][1] (the +t_e side), else -1 (SURVEY c.1,
    reading Q4).  Sum sequential in edgesOnVertex order.
    """
    acc = np.zeros(mesh.nVertices)
    v = np.arange(mesh.nVertices)
    for k in range(3):
        e = mesh.edgesOnVertex[:, k]
        s = np.where(mesh.verticesOnEdge[e, 1] == v, 1.0, -1.0)
        acc = acc + s * mesh.dcEdge[e] * U[e]
    return acc / mesh.areaTriangle


def circulation(mesh, U):
    """sum_{e in E_v} t_{e,v} d_e u_e (un-normalised; used by the Gamma diagnostic)."""
    acc = np.zeros(mesh.nVertices)
    v = np.arange(mesh.nVertices)
    for k in range(3):
        e = mesh.edgesOnVertex[:, k]
        s = np.where(mesh.verticesOnEdge[e, 1] == v, 1.0, -1.0)
        acc = acc + s * mesh.dcEdge[e] * U[e]
    return acc


def vertex_thickness(mesh, H):
    """h_v = (1/A_v) sum_i kite_{v,i} h_i  (dual thickness by interpolation)."""
    acc = np.zeros(mesh.nVertices)
    for k in range(3):
        acc = acc + mesh.kiteAreasOnVertex[:, k] * H[mesh.cellsOnVertex[:, k]]
    return acc / mesh.areaTriangle


def potential_vorticity(mesh, U, H):
    """q_v = (zeta_v + f_v) / h_v  (q = eta / h)."""
    return (relative_vorticity(mesh, U) + mesh.fVertex) / vertex_thickness(mesh, H)


def perp_flux(mesh, F_all, edges):
    """F_perp_e = M_e(F) = sum_j W_{e,j} F_{eoe_j}  (MPAS normalisation, Q6)."""
    edges = np.asarray(edges)
    acc = np.zeros(edges.size)
    nE2 = mesh.nEdgesOnEdge[edges]
    for j in range(mesh.maxEdges2):
        act = j < nE2
        if not np.any(act):
            break
        e = edges[act]
        acc[act] = acc[act] + mesh.weightsOnEdge[e, j] * F_all[mesh.edgesOnEdge[e, j]]
    return acc


def pv_flux_energy(mesh, F_all, q_hat, edges):
    """Energy-conserving PV flux term sum_j W_{e,j} F_{eoe_j} (q_hat_e + q_hat_{eoe_j}) / 2: the
    symmetric pairwise PV average inside the F_perp sum (the variant of reading Q2).
    With l_e d_e W_{e,e'} antisymmetric (pin P7) the term does no work on the flow:
    sum_e l_e d_e F_e PV_e = 0.  Evaluated per slot as (W * F) * (0.5 * (q_e + q_e')), summed
    sequentially in slot order from +0.0."""
    edges = np.asarray(edges)
    acc = np.zeros(edges.size)
    nE2 = mesh.nEdgesOnEdge[edges]
    for j in range(mesh.maxEdges2):
        act = j < nE2
        if not np.any(act):
            break
        e = edges[act]
        ej = mesh.edgesOnEdge[e, j]
        acc[act] = acc[act] + mesh.weightsOnEdge[e, j] * F_all[ej] * (0.5 * (q_hat[e] + q_hat[ej]))
    return acc


def kinetic_energy(mesh, U):
    """K_i = (1/A_i) sum_{e in E_i} (l_e d_e / 4) u_e^2 on every cell.

    P:L1213 ("K = |u|^2/2"); quadrature reading Q18.  Evaluated as
    (sum_j 0.25 * l_e * d_e * u_e * u_e) / A_i, left to right.
    """
    acc = np.zeros(mesh.nCells)
    nE = mesh.nEdgesOnCell
    for j in range(mesh.maxEdges):
        act = j < nE
        if not np.any(act):
            break
        e = mesh.edgesOnCell[act, j]
        acc[act] = acc[act] + 0.25 * mesh.dvEdge[e] * mesh.dcEdge[e] * U[e] * U[e]
    return acc / mesh.areaCell


def tangential_velocity(mesh, U):
    """v_e = sum_j W_{e,j} u_{eoe_j}: the TRiSK reconstruction of the velocity along +t_e with the
    same weightsOnEdge as F_perp (Thuburn et al. 2009; exact for uniform flow on the regular hex,
    pin P7), sequential in slot order from +0.0 (hurricane drag / wind terms, reading in DESIGN.md)."""
    return perp_flux(mesh, U, np.arange(mesh.nEdges))


def hurricane_terms(mesh, U, h_e, phys):
    """Bottom drag and wind terms of eq. hurricane_model on every edge:
        D_e = C_D |u|_e u_e / h_e,   W_e = C_W |u_W - u|_e (u_W,n - u_e) / h_e,
    |u|_e = sqrt(u_e^2 + v_e^2), |u_W - u|_e = sqrt((u_W,n - u_e)^2 + (u_W,t - v_e)^2),
    v_e the tangential reconstruction; returns (D, W) (the slow tendency subtracts D, adds W)."""
    v = tangential_velocity(mesh, U)
    speed = np.sqrt(U * U + v * v)
    D = phys.cd * speed * U / h_e
    dn = phys.uw_n - U
    dt = phys.uw_t - v
    ws = np.sqrt(dn * dn + dt * dt)
    W = phys.cw * ws * dn / h_e
    return D, W


def pv_flux(mesh, U, H, phys=None):
    """PV_e = q_hat_e F_perp_e on every edge: the absolute-vorticity flux of the momentum equation
    (eq. trisk_vorticity, the term whose curl is Theta_v), q_hat_e = 0.5 (q[v0] + q[v1])
    (reading Q2); phys.pv == "energy": the energy-conserving pv_flux_energy."""
    e = np.arange(mesh.nEdges)
    F = edge_flux(mesh, U, H, e)
    q = potential_vorticity(mesh, U, H)
    v0 = mesh.verticesOnEdge[:, 0]
    v1 = mesh.verticesOnEdge[:, 1]
    q_hat = 0.5 * (q[v0] + q[v1])
    if phys is not None and phys.pv == "energy":
        return pv_flux_energy(mesh, F, q_hat, e)
    return q_hat * perp_flux(mesh, F, e)


def vorticity_update(mesh, eta, dP):
    """Prognostic absolute vorticity on the dual cells (eq. trisk_vorticity):
    eta_v^{n+1} = eta_v^n + (sum_j t_{e_j,v} d_{e_j} dP_{e_j}) / A_v  over edgesOnVertex in slot order,
    with dP_e the time-integrated PV flux the step applied to edge e (lts.fblts_step(eta=...)) and
    t_{e,v} = +1 if v = verticesOnEdge[e][1] (the +t_e side) else -1 -- the circulation sign, so that
    the prognostic eta tracks the diagnostic (curl u + f) (Ringler et al. 2010)."""
    acc = np.zeros(mesh.nVertices)
    v = np.arange(mesh.nVertices)
    for k in range(3):
        e = mesh.edgesOnVertex[:, k]
        s = np.where(mesh.verticesOnEdge[e, 1] == v, 1.0, -1.0)
        acc = acc + s * mesh.dcEdge[e] * dP[e]
    return eta + acc / mesh.areaTriangle


def slow_momentum(mesh, U, H, tau_n, rho0, phys=None):
    """Phi^slow_e(u, h) on every edge: the non-gravity-wave momentum terms.

    Split per P:L1548-1561 (the fast part is only -g grad(h + z_b)).  From
    eq. nonlinear_swe: -(curl u + f k) x u - grad K, written in TRiSK form
     as  q_hat_e F_perp_e - (K[c1] - K[c0]) / d_e   (sign reading Q5:
    F_perp along +t_e, so the PV term enters with +), plus the wind-stress-like
    forcing G_e = (tau . n_e) / (rho0 h_e) (reading Q19; config 2 and 5).
    q_hat_e = 0.5 (q[v0] + q[v1]) (reading Q2); phys.pv == "energy" replaces q_hat_e F_perp_e by
    the energy-conserving pv_flux_energy.
    Evaluated as  (PV_e - (K1 - K0) / d_e) + G_e,  PV_e = q_hat * F_perp (centred).
    """
    PV = pv_flux(mesh, U, H, phys)
    K = kinetic_energy(mesh, U)
    c0 = mesh.cellsOnEdge[:, 0]
    c1 = mesh.cellsOnEdge[:, 1]
    h_e = 0.5 * (H[c0] + H[c1])
    G = tau_n / (rho0 * h_e)
    S = PV - (K[c1] - K[c0]) / mesh.dcEdge + G
    if phys is not None and phys.hurricane():
        D, W = hurricane_terms(mesh, U, h_e, phys)
        S = S - D + W
    return S


def slow_tendency(mesh, U, H, phys):
    """S_e = Phi^slow_e(u^n, h^n), frozen for the coarse step (Q17).

    ``phys.slow`` False disables every slow term (gravity-wave model,
    eq. grav_wave_model; "all the slow terms disabled").
    """
    if not phys.slow:
        return np.zeros(mesh.nEdges)
    return slow_momentum(mesh, U, H, phys.tau_n, phys.rho0, phys)
