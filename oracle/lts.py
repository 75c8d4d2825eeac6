"""FB-LTS: region labelling and the literal four-phase step (oracle; test infrastructure only).

Region codes (cells and edges), shared by the tests and the C-ABI's
``fblts_get_labels`` (a documented output format, not shared code):
    0 = C^int, 1 = C^IF-2, 2 = C^IF-1,
    2 + l  (l = 1..5) = F^l minus F^(l-1)  (3..7),   8 = F minus F^5.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from . import trisk

INT, IF2, IF1 = 0, 1, 2
FINE_MIN = 3
BIG = np.iinfo(np.int32).max


def hop_distance(mesh, src_mask, max_depth):
    """Multi-source breadth-first hop distance over cellsOnCell, capped at max_depth+1."""
    d = np.where(src_mask, 0, BIG).astype(np.int64)
    nb = mesh.cellsOnCell
    valid = np.arange(mesh.maxEdges)[None, :] < mesh.nEdgesOnCell[:, None]
    for depth in range(1, max_depth + 1):
        front = d == depth - 1
        adj = np.zeros(mesh.nCells, dtype=bool)
        for j in range(mesh.maxEdges):
            adj |= valid[:, j] & front[np.where(valid[:, j], nb[:, j], 0)]
        d[(d == BIG) & adj] = depth
    d[d == BIG] = max_depth + 1
    return d


@dataclasses.dataclass
class Labels:
    cell: np.ndarray  # int8 region code per cell
    edge: np.ndarray  # int8 region code per edge
    r: int

    # --- cell sets ---
    def F(self):
        return self.cell >= FINE_MIN

    def Fl(self, l):
        """F^l_P: fine cells within l*r hops of the coarse region."""
        return (self.cell >= FINE_MIN) & (self.cell <= 2 + l)

    def C(self):
        return self.cell < FINE_MIN

    def IF1(self):
        return self.cell == IF1

    def IF2(self):
        return self.cell == IF2

    def INT(self):
        return self.cell == INT

    # --- edge sets (F^l_E per reading Q7) ---
    def F_E(self):
        return self.edge >= FINE_MIN

    def Fl_E(self, l):
        return (self.edge >= FINE_MIN) & (self.edge <= 2 + l)

    def C_E(self):
        return self.edge < FINE_MIN

    def IF1_E(self):
        return self.edge == IF1

    def IF2_E(self):
        return self.edge == IF2

    def INT_E(self):
        return self.edge == INT


def label_regions(mesh, fine_mask, r=2):
    """LTS regions from a fine-cell mask (reading Q7/Q8).

    Coarse cells with hop distance d to F: IF-1 = {1 <= d <= r}, IF-2 = {r < d <= 2r},
    int = {d > 2r}.  Fine cells with hop distance rho to C: F^l = {rho <= l r}.
    Edge rule: an edge between regions belongs to the one closest to
    the fine region; F^l_E = edges with at least one cell in F^l_P.
    """
    fine = np.asarray(fine_mask, dtype=bool)
    dF = hop_distance(mesh, fine, 2 * r)
    rho = hop_distance(mesh, ~fine, 5 * r)
    cell = np.empty(mesh.nCells, dtype=np.int8)
    cell[~fine & (dF > 2 * r)] = INT
    cell[~fine & (dF > r) & (dF <= 2 * r)] = IF2
    cell[~fine & (dF >= 1) & (dF <= r)] = IF1
    layer = np.minimum((rho + r - 1) // r, 6)           # ceil(rho / r), 6 = beyond F^5
    cell[fine] = (2 + layer[fine]).astype(np.int8)
    a = cell[mesh.cellsOnEdge[:, 0]].astype(np.int64)
    b = cell[mesh.cellsOnEdge[:, 1]].astype(np.int64)
    fa, fb = a >= FINE_MIN, b >= FINE_MIN
    both = fa & fb
    edge = np.where(both, np.minimum(a, b),
                    np.where(fa, a, np.where(fb, b, np.maximum(a, b)))).astype(np.int8)
    lab = Labels(cell=cell, edge=edge, r=r)
    validate_labels(mesh, lab)
    return lab


def region_class(code):
    """F -> 3, IF-1 -> 2, IF-2 -> 1, int -> 0."""
    return np.minimum(code.astype(np.int64), 3)


def validate_labels(mesh, lab):
    """Stencil assumption: neighbouring cells are at most one region apart
    in the chain F - IF-1 - IF-2 - int.  Raises ValueError naming the first offender."""
    cls = region_class(lab.cell)
    a = cls[mesh.cellsOnEdge[:, 0]]
    b = cls[mesh.cellsOnEdge[:, 1]]
    bad = np.nonzero(np.abs(a - b) > 1)[0]
    if bad.size:
        e = int(bad[0])
        raise ValueError(f"labels: edge {e} joins regions {int(a[e])} and {int(b[e])} (stencil assumption)")
    return True


def pred_coeffs(k, M):
    """Prediction coefficients of eq. preds, derived in App. A:
    a = k/M, b = 1/M, c = 1 - (k+1)/M; levels use (a_k, 1 - a_k) for k = 0..M."""
    return {"M": M, "a": k / M, "b": 1.0 / M, "c": 1.0 - (k + 1) / M}


def predict_level(co, x_new, x_n, k):
    """x^{n,k} = (k/M) x~^{n+1} + (1 - k/M) x^n  (subeqn pred_old; k = M allowed)."""
    a = k / co["M"]
    return a * x_new + (1.0 - a) * x_n


def predict_stage(co, x_new, x_stage, x_n):
    """x-bar^{n,k+1/m} = (k/M) x~^{n+1} + (1/M) x~^{n+1/m} + (1 - (k+1)/M) x^n  (pred_s1 / pred_s2)."""
    return co["a"] * x_new + co["b"] * x_stage + co["c"] * x_n


def fblts_step(mesh, lab, h, u, dt, M, phys, extents="paper", slow_refresh=False, split=True, eta=None):
    """One FB-LTS coarse step in split mode, literal (P:L551-787 inside P:L1548-1561).

    slow_refresh=True: the variant the paper proposes to lift the splitting's coarse-step cap
    (SURVEY 8(f) N2): "calculate the slow tendencies at times t^{n,k} for
    k = 0, ..., M-1 and use these values while advancing on fine cells".  Reading:
    S^k = Phi^slow(u^{n,k}, h^{n,k}) on F_E, its stencil (edges F_E u IF-1_E, cells F u IF-1 u IF-2)
    taking the fine data on F / F_E and the level-k prediction (eq. pred_old) on IF-1 / IF-1_E and
    on IF-2 (the same formula from the tilde coarse data); S^k replaces S in the three fine
    velocity stages on F_E; everything on C (coarse stages, predictions, correction summands)
    keeps the frozen S.

    split=False: the unsplit FB-LTS of P:L468-787: every velocity update uses the
    full Phi(U, HS) = Phi^fast(HS) + Phi^slow(U, HS) (reading Q16: the FB-averaged thickness for every
    h-dependence), with U the stage's velocity views -- coarse: u^n, u~1, u~2 on the paper's extents
    Y1 = C_E u F^4_E, Y2 = C_E u F^2_E, Y3 = IF-1_E u int_E (whose slow stencils stay inside
    X1 = C u F^5, X2 = C u F^3, X3 = C u F^1); fine: U0, U1, U2 of the view table;
    correction summand Phi(U2, HS3) on the IF edges.

    eta (vertex array, optional): the prognostic absolute vorticity companion (Theorem 2, P:L1038-1137;
    SPEC step_prognostic_vorticity S:L472-480) advanced with the step: every velocity update's PV-flux
    term PV_e = q_hat_e F_perp_e (trisk.pv_flux; inside S in split mode, at each stage's (U, HS) in
    unsplit mode) is integrated per edge exactly as the velocity integrates it -- int_E: dt PV(coarse
    stage 3); F_E: sum_k dt/M PV^k (fine velocity stage 3 of every subcycle, ascending k); IF-1_E and
    IF-2_E: dt/M sum_k PV^k (the correction's sum, reading Q14) -- and eta_v += (sum_j t d dP) / A_v
    (trisk.vorticity_update).  One dP per edge, shared by its two dual cells with opposite t_{e,v}: the
    total sum_v A_v eta_v is conserved (Theorem 2).  Then returns (h^{n+1}, u^{n+1}, eta^{n+1}).

    extents="paper": the shrinking F^5/F^4/F^3/F^2/F^1 extents of P:L557-661.
    extents="all_fine": the MPAS simplification of P:L1284-1286 (every coarse
    stage also on all of F); results on C must not change (pin P14).
    Arrays are NaN outside the extent a phase computes, so any read outside the
    stated domain of dependence poisons the result.
    Returns (h^{n+1}, u^{n+1}).
    """
    nC, nE = mesh.nCells, mesh.nEdges
    g = phys.g_fast()
    b1, b2, b3 = phys.beta
    omb1, omb2, om2b3 = 1.0 - b1, 1.0 - b2, 1.0 - 2.0 * b3
    c1, c2, c3 = dt / 3.0, dt / 2.0, dt
    c1f, c2f, c3f = dt / (3.0 * M), dt / (2.0 * M), dt / M
    nan_c = lambda: np.full(nC, np.nan)
    nan_e = lambda: np.full(nE, np.nan)

    C, F = lab.C(), lab.F()
    IF1, IF2, INTc = lab.IF1(), lab.IF2(), lab.INT()
    C_E, F_E = lab.C_E(), lab.F_E()
    IF1_E, IF2_E, INT_E = lab.IF1_E(), lab.IF2_E(), lab.INT_E()
    if extents == "paper":
        X1, Y1, X2, Y2, X3 = C | lab.Fl(5), C_E | lab.Fl_E(4), C | lab.Fl(3), C_E | lab.Fl_E(2), C | lab.Fl(1)
    else:
        X1 = X2 = X3 = np.ones(nC, dtype=bool)
        Y1 = Y2 = np.ones(nE, dtype=bool)
    Y3 = IF1_E | INT_E                      # velocity stage 3: IF-2_E skipped as written (Q10)

    def Psi(U, H, mask):
        idx = np.nonzero(mask)[0]
        return idx, trisk.thickness_tendency(mesh, U, H, idx)

    def PhiF(H, mask):
        idx = np.nonzero(mask)[0]
        return idx, trisk.fast_momentum(mesh, H, g, idx)

    # ---------- slow terms at t^n, frozen for the whole coarse step ----------
    S = trisk.slow_tendency(mesh, u, h, phys) if split else None
    track = eta is not None

    def PVf(U, HS, mask):
        """PV-flux part of the slow term on the edges of mask (0 with the slow terms off)."""
        if not phys.slow:
            return np.zeros(int(np.count_nonzero(mask)))
        with np.errstate(invalid="ignore"):
            return trisk.pv_flux(mesh, U, HS, phys)[mask]

    PS = trisk.pv_flux(mesh, u, h, phys) if (track and split and phys.slow) else np.zeros(nE)

    def Slow(U, HS, mask):
        """Phi^slow(U, HS) on the edges of mask (unsplit); NaN in the views poisons misuse."""
        if not phys.slow:
            return np.zeros(int(np.count_nonzero(mask)))
        with np.errstate(invalid="ignore"):
            return trisk.slow_momentum(mesh, U, HS, phys.tau_n, phys.rho0, phys)[mask]

    # ---------- Phase 1: Coarse Advancement ----------
    h1, hs1, h2, hs2, h3, hs3 = nan_c(), nan_c(), nan_c(), nan_c(), nan_c(), nan_c()
    u1, u2, u3 = nan_e(), nan_e(), nan_e()
    i, psi = Psi(u, h, X1)                                   # thickness stage 1 (eq. if_h_s1 / coarse_h_s1)
    h1[i] = h[i] + c1 * psi
    hs1[i] = b1 * h1[i] + omb1 * h[i]
    e, phi = PhiF(hs1, Y1)                                   # velocity stage 1 (eq. if_u_s1 / coarse_u_s1)
    u1[e] = u[e] + c1 * (phi + (S[e] if split else Slow(u, hs1, Y1)))
    i, psi = Psi(u1, h1, X2)                                 # thickness stage 2 (eq. if_h_s2 / coarse_h_s2)
    h2[i] = h[i] + c2 * psi
    hs2[i] = b2 * h2[i] + omb2 * h[i]
    e, phi = PhiF(hs2, Y2)                                   # velocity stage 2 (eq. if_u_s2 / coarse_u_s2)
    u2[e] = u[e] + c2 * (phi + (S[e] if split else Slow(u1, hs2, Y2)))
    i, psi = Psi(u2, h2, X3)                                 # thickness stage 3 (eq. if_h_s3 / coarse_h_s3)
    h3[i] = h[i] + c3 * psi
    hs3[i] = b3 * h3[i] + om2b3 * h2[i] + b3 * h[i]
    e, phi = PhiF(hs3, Y3)                                   # velocity stage 3
    u3[e] = u[e] + c3 * (phi + (S[e] if split else Slow(u2, hs3, Y3)))

    h_new, u_new = nan_c(), nan_e()
    h_new[INTc] = h3[INTc]                                   # interior coarse data is final
    u_new[INT_E] = u3[INT_E]
    if track:                                                # eta companion: int_E from coarse stage 3
        dP = nan_e()
        dP[INT_E] = c3 * (PS[INT_E] if split else PVf(u2, hs3, INT_E))
        dPF = np.where(F_E, 0.0, np.nan)
        accP = np.where(IF1_E | IF2_E, 0.0, np.nan)

    # ---------- Phases 2 + 3: Interface Prediction per k and Fine Advancement ----------
    hk, uk = nan_c(), nan_e()
    hk[F] = h[F]
    uk[F_E] = u[F_E]
    IFc = IF1 | IF2
    IFe = IF1_E | IF2_E
    accH = np.where(IFc, 0.0, np.nan)
    accU = np.where(IFe, 0.0, np.nan)
    for k in range(M):
        co = pred_coeffs(k, M)
        hP0, hP0n, hP1, hP2 = nan_c(), nan_c(), nan_c(), nan_c()
        hsP1, hsP2, hsP3 = nan_c(), nan_c(), nan_c()
        hP0[IF1] = predict_level(co, h3[IF1], h[IF1], k)                # pred_old, k
        hP0n[IF1] = predict_level(co, h3[IF1], h[IF1], k + 1)           # pred_old, k+1 (k = M extra)
        hP1[IF1] = predict_stage(co, h3[IF1], h1[IF1], h[IF1])         # pred_s1
        hP2[IF1] = predict_stage(co, h3[IF1], h2[IF1], h[IF1])         # pred_s2
        hsP1[IF1] = b1 * hP1[IF1] + omb1 * hP0[IF1]                    # eq. hstar_preds
        hsP2[IF1] = b2 * hP2[IF1] + omb2 * hP0[IF1]
        hsP3[IF1] = b3 * hP0n[IF1] + om2b3 * hP2[IF1] + b3 * hP0[IF1]
        uP0, uP1, uP2 = nan_e(), nan_e(), nan_e()
        uP0[IF1_E] = predict_level(co, u3[IF1_E], u[IF1_E], k)
        uP1[IF1_E] = predict_stage(co, u3[IF1_E], u1[IF1_E], u[IF1_E])
        uP2[IF1_E] = predict_stage(co, u3[IF1_E], u2[IF1_E], u[IF1_E])

        # views (reading Q11): F -> fine data, IF-1 -> predicted,
        # IF-2 -> tilde coarse data, int -> bar coarse data
        def cview(fine, pred, coarse):
            return np.where(F, fine, np.where(IF1, pred, coarse))

        def eview(fine, pred, coarse):
            return np.where(F_E, fine, np.where(IF1_E, pred, coarse))

        if slow_refresh and split:
            # S^k on F_E from the state at t^{n,k} (NaN outside the stencil region poisons misuse)
            Hk = np.where(F, hk, np.where(IF1 | IF2, predict_level(co, h3, h, k), np.nan))
            Uk = np.where(F_E, uk, np.where(IF1_E, uP0, np.nan))
            Sk = nan_e()
            with np.errstate(invalid="ignore"):
                Sk[F_E] = trisk.slow_tendency(mesh, Uk, Hk, phys)[F_E]
        else:
            Sk = S

        hk1, hsk1, hk2, hsk2, hkn, hs3k = nan_c(), nan_c(), nan_c(), nan_c(), nan_c(), nan_c()
        uk1, uk2, ukn = nan_e(), nan_e(), nan_e()
        H0 = cview(hk, hP0, h)
        U0 = eview(uk, uP0, u)
        i, psi = Psi(U0, H0, F)                                         # eq. fine_s1
        hk1[i] = hk[i] + c1f * psi
        hsk1[i] = b1 * hk1[i] + omb1 * hk[i]
        HS1 = cview(hsk1, hsP1, hs1)
        e, phi = PhiF(HS1, F_E)
        uk1[e] = uk[e] + c1f * (phi + (Sk[e] if split else Slow(U0, HS1, F_E)))
        U1 = eview(uk1, uP1, u1)
        H1 = cview(hk1, hP1, h1)
        i, psi = Psi(U1, H1, F)                                         # eq. fine_s2
        hk2[i] = hk[i] + c2f * psi
        hsk2[i] = b2 * hk2[i] + omb2 * hk[i]
        HS2 = cview(hsk2, hsP2, hs2)
        e, phi = PhiF(HS2, F_E)
        uk2[e] = uk[e] + c2f * (phi + (Sk[e] if split else Slow(U1, HS2, F_E)))
        U2 = eview(uk2, uP2, u2)
        H2 = cview(hk2, hP2, h2)
        i, psi = Psi(U2, H2, IFc)                                       # correction summand (eq. if_correction)
        accH[i] = accH[i] + psi
        i, psi = Psi(U2, H2, F)                                         # eq. fine_s3
        hkn[i] = hk[i] + c3f * psi
        hs3k[i] = b3 * hkn[i] + om2b3 * hk2[i] + b3 * hk[i]
        HS3 = cview(hs3k, hsP3, hs3)
        e, phi = PhiF(HS3, F_E)
        ukn[e] = uk[e] + c3f * (phi + (Sk[e] if split else Slow(U2, HS3, F_E)))
        e, phi = PhiF(HS3, IFe)                                         # correction summand (eq. if_correction)
        accU[e] = accU[e] + (phi + (S[e] if split else Slow(U2, HS3, IFe)))
        if track:
            if split:
                PkF = PVf(Uk, Hk, F_E) if slow_refresh else PS[F_E]
                PkI = PS[IFe]
            else:
                PkF, PkI = PVf(U2, HS3, F_E), PVf(U2, HS3, IFe)
            dPF[F_E] = dPF[F_E] + c3f * PkF
            accP[IFe] = accP[IFe] + PkI
        hk, uk = hkn, ukn

    h_new[F] = hk[F]                                                    # h^{n+1} := h^{n,M}
    u_new[F_E] = uk[F_E]

    # ---------- Phase 4: Interface Correction (reading Q14) ----------
    h_new[IFc] = h[IFc] + c3f * accH[IFc]
    u_new[IFe] = u[IFe] + c3f * accU[IFe]
    if track:
        dP[F_E] = dPF[F_E]
        dP[IFe] = c3f * accP[IFe]
        return h_new, u_new, trisk.vorticity_update(mesh, eta, dP)
    return h_new, u_new


def run(mesh, lab, h, u, dt, M, phys, n_steps, extents="paper", slow_refresh=False, split=True, eta=None):
    for _ in range(n_steps):
        out = fblts_step(mesh, lab, h, u, dt, M, phys, extents, slow_refresh=slow_refresh, split=split, eta=eta)
        h, u = out[0], out[1]
        if eta is not None:
            eta = out[2]
    return (h, u) if eta is None else (h, u, eta)
