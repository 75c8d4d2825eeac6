// kernels.cu -- sm_100a fp64 kernels of the FB-LTS hot path (split mode).
//
// Every kernel evaluates the paper's formulas in the canonical order listed in
// DESIGN.md ("Canonical arithmetic"): sums sequential in slot order from +0.0,
// left-to-right products, IEEE division, no FMA contraction (--fmad=false), so
// the results agree bit for bit with a literal implementation of the paper.
//
// Thread mapping: one thread per cell (cell kernels) or per
// edge (edge kernels), 256-thread blocks over a contiguous index range.  A cell
// fetches its (edge, neighbour) row with 16-byte vector loads and the slot loop is
// unrolled to G >= maxEdges with predication, so every gather of the cell can be
// in flight at once.
//
// Band / deep split: cells are ordered [int | IF-2 | IF-1 | F^1 | F^2 .. | F\F^5]
// and edges likewise.  Only the "band" [IF-2, F^1] can see a neighbour of another
// region; a cell of F\F^1 has only fine neighbours (its hop distance to C is >= 3)
// and an edge of F_E\F^1_E has two fine cells.  Every fine kernel is therefore
// launched twice: a BAND instance with the region views and a DEEP instance with
// none (no class tests, fewer registers).
//
// Fusion: in split mode Phi^fast_e depends only on cell data, so the stage-s
// velocity  u_bar_{s-1,e} = u_base,e + c_{s-1} (Phi^fast_e(h_FB) + S_e)  is
// recomputed inside the stage-s cell kernel from the two cells of e instead of
// being stored; the FB averages h*, h**, h*** and the IF-1 predictions (eq. preds,
// P:L683-742) are likewise recomputed from the stored stage thicknesses.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "fblts_internal.h"

namespace fblts {

constexpr int TPB = 256;
// min resident blocks per SM requested for the register-heavy stage kernels (occupancy knob)
#ifndef FBLTS_MINB
#define FBLTS_MINB 6
#endif
// band fine stage kernels (k_fine_s2 / k_fine_s3 BAND): 64 registers, 4 CTAs per SM (config 5: fine_s3
// 1.795 -> 1.759 ms per step against 76 registers / 3 CTAs; 5 CTAs no better)
#ifndef FBLTS_BAND_MINB
#define FBLTS_BAND_MINB 4
#endif
#ifndef FBLTS_TILE_MINB
#define FBLTS_TILE_MINB 2
#endif
#ifndef FBLTS_TILE_NBUF
#define FBLTS_TILE_NBUF 2
#endif
constexpr int NBUF = FBLTS_TILE_NBUF;   // tile buffers of the staged kernel's pipeline
static_assert(NBUF == 2, "k_stage_tiled is a two-buffer pipeline (3 buffers measured slower)");
constexpr int TREC = 16;                // ints per tile-record slot in shared memory (the record + the next one)
#ifndef FBLTS_TILE_NTHR
#define FBLTS_TILE_NTHR 256
#endif
constexpr int NTHR = FBLTS_TILE_NTHR;   // threads per tile CTA (>= TILE)
static_assert(NTHR >= TILE, "one thread per tile cell in the cell phase");

static inline unsigned nblocks(long n) { return (unsigned)((n + TPB - 1) / TPB); }

// cell class: 2 = F, 1 = IF-1, 0 = other coarse (IF-2 or int); the boundary [0, nB), interior
// [nB, nOwnC) and halo [nOwnC, nC) blocks are each region-major
__device__ __forceinline__ int ccls(const DevMesh &m, int x) {
    const Bounds &b = x < m.nB ? m.cb : (x < m.nOwnC ? m.cbI : m.cbh);
    return x >= b.f ? 2 : (x >= b.if1 ? 1 : 0);
}
// edge class: 3 = F_E, 2 = IF-1_E, 1 = IF-2_E, 0 = int_E
__device__ __forceinline__ int ecls(const Bounds &b, int e) {
    return e >= b.f ? 3 : (e >= b.if1 ? 2 : (e >= b.if2 ? 1 : 0));
}

__device__ __forceinline__ void report(DevError *err, int kind, int k, int i, double v) {
    if (atomicCAS(&err->flag, 0, 1) == 0) {
        err->kind = kind;
        err->k = k;
        err->index = i;
        err->value = v;
    }
}

// Phi^fast_e = -g ((h_c1 + z_b,c1) - (h_c0 + z_b,c0)) / d_e   (eq. fast_terms; Q15)
__device__ __forceinline__ double phi_fast(double g, double hs0, double zb0, double hs1, double zb1, double dc) {
    const double t1 = hs1 + zb1;
    const double t0 = hs0 + zb0;
    return -g * (t1 - t0) / dc;
}

__device__ __forceinline__ int decode(int es, bool &pos) {
    pos = es >= 0;
    return pos ? es : ~es;
}

// One slot of Psi_i: the signed term n_{e,i} l_e F_e with F_e = (0.5 (H_c0 + H_c1)) u_e.
__device__ __forceinline__ double psi_term(bool pos, double Hi, double Hn, double ue, double l) {
    const double Fe = (0.5 * (Hi + Hn)) * ue;
    const double t = l * Fe;
    return pos ? t : -t;
}

// (edge, neighbour) row of cell i with G/2 16-byte loads (row stride G, 16-B aligned)
template <int G>
__device__ __forceinline__ void load_row(const DevMesh &m, int i, int2 (&r)[G]) {
    const int4 *p = reinterpret_cast<const int4 *>(m.ec + (size_t)i * G);
#pragma unroll
    for (int q = 0; q < G / 2; ++q) {
        const int4 v = p[q];
        r[2 * q] = make_int2(v.x, v.y);
        r[2 * q + 1] = make_int2(v.z, v.w);
    }
}

// ---------------------------------------------------------------- slow terms
// One launch, three index spaces: vertices (q_v), cells (K_i), edges (F_e).
// q_v = (zeta_v + f_v) / h_v,  zeta_v = (sum t d u)/A_v,  h_v = (sum kite h)/A_v
// K_i = (sum 0.25 l d u u) / A_i   (Q18);   F_e = (0.5 (h_c0 + h_c1)) u_e   (Q1)
// VF (DevMesh::vF, full sweeps): the vertex role also writes F_e for the edges e = eov[k][v] with
// v = voe[e][1]; their cells are the kite cells k, k+1 whose h it has loaded, so F costs no extra
// reads and the edge role is not launched ((0.5 (h_a + h_b)) u_e: the same bits in either cell order).
template <int G, bool VF>
__global__ void __launch_bounds__(TPB) k_slow_pre(DevMesh m, const double *__restrict__ h,
                                                  const double *__restrict__ u, double *__restrict__ q,
                                                  double *__restrict__ K, double *__restrict__ F,
                                                  unsigned nbV, unsigned nbC, int v0, int c0, int e0) {
    const unsigned b = blockIdx.x;
    if (b < nbV) {
        const int v = v0 + b * TPB + threadIdx.x;
        if (v >= m.nV) return;
        const double A = m.areaTri[v], fv = m.fV[v];       // independent loads first
        int ev[3];
        bool pv[3];
        double uk[3], hk[3], circ = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            ev[k] = decode(m.eov[k * m.strideV + v], pv[k]);
            uk[k] = u[ev[k]];
            const double t = m.dc[ev[k]] * uk[k];
            circ = circ + (pv[k] ? t : -t);
        }
        double hv = 0.0;                                   // (its gathers before the first division)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            hk[k] = h[m.cov[k * m.strideV + v]];
            hv = hv + m.kite[k * m.strideV + v] * hk[k];
        }
        if (VF) {
#pragma unroll
            for (int k = 0; k < 3; ++k)
                if (pv[k]) F[ev[k]] = (0.5 * (hk[k] + hk[(k + 1) % 3])) * uk[k];
        }
        const double zeta = circ / A;
        hv = hv / A;
        q[v] = (zeta + fv) / hv;
    } else if (b < nbV + nbC) {
        const int i = c0 + (b - nbV) * TPB + threadIdx.x;
        if (i >= m.nC) return;
        int2 r[G];
        load_row<G>(m, i, r);
        const int n = m.nEoC[i];
        const double Ai = m.areaCell[i];
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < G; ++j) {
            if (j < n) {
                bool pos;
                const int e = decode(r[j].x, pos);
                const double ue = u[e];
                acc = acc + 0.25 * m.dv[e] * m.dc[e] * ue * ue;
            }
        }
        K[i] = acc / Ai;
    } else {
        const int e = e0 + (b - nbV - nbC) * TPB + threadIdx.x;
        if (e >= m.nE) return;
        const int2 c = m.coe[e];
        F[e] = (0.5 * (h[c.x] + h[c.y])) * u[e];
    }
}

// S_e = q_hat_e F_perp_e - (K_c1 - K_c0) / d_e + G_e   (Q2, Q5, Q19)
#ifndef FBLTS_SLOW_CHUNK
#define FBLTS_SLOW_CHUNK 5
#endif
#ifndef FBLTS_SLOW_MINB
#define FBLTS_SLOW_MINB 5
#endif
// PVE (energy-conserving PV flux): the term q_hat_e F_perp_e becomes
// sum_j (W_j F_eoe_j) (0.5 (q_hat_e + q_hat_eoe_j)) with q_hat per edge from k_qhat (oracle
// trisk.pv_flux_energy); it does no work on the flow (sum_e l_e d_e F_e PV_e = 0).
// VEL (unsplit FB-LTS): the stage's velocity update follows in the same thread (see
// VelFuse) instead of a store of S_e and a separate k_un_vel sweep; h is then the stage's HS view.
template <int MAXE2, bool HUR, bool PVE, bool VEL>
__global__ void __launch_bounds__(TPB, FBLTS_SLOW_MINB) k_slow_edge(DevMesh m, const double *__restrict__ h,
                                                   const double *__restrict__ q, const double *__restrict__ K,
                                                   const double *__restrict__ F, const double *__restrict__ u,
                                                   const double *__restrict__ qe,
                                                   double *__restrict__ S, double *__restrict__ pvout,
                                                   double rho0, double cd, double cw, int e0, int e1,
                                                   VelFuse vf, double g) {
    const int e = e0 + blockIdx.x * TPB + threadIdx.x;
    if (e >= e1) return;
    const int2 c = m.coe[e];                  // issued first: its gathers (q, K, h) end the chain (measured -3 %)
    const int n = m.nEoE[e];
#ifndef FBLTS_SLOW_HOIST
#define FBLTS_SLOW_HOIST 1   // config 5: slow_edge 1.374 -> 1.328 ms per step (with FBLTS_SLOW_MINB 5)
#endif
    // FBLTS_SLOW_HOIST: the per-edge gathers (q, K, h) and streams (tau, d_e) issued before the slot loop
    double qv0 = 0.0, qv1 = 0.0, K0 = 0.0, K1 = 0.0, h0 = 0.0, h1 = 0.0, tau = 0.0, dce = 0.0;
    if (FBLTS_SLOW_HOIST) {
        if (!PVE) {
            const int2 v = m.voe[e];
            qv0 = q[v.x], qv1 = q[v.y];
        }
        K0 = K[c.x], K1 = K[c.y], h0 = h[c.x], h1 = h[c.y], tau = m.tau[e], dce = m.dc[e];
    }

    // F_perp = sum_j W_j F_eoe_j in slot order, gathered in chunks of CH slots (register budget);
    // with the hurricane terms also v_e = sum_j W_j u_eoe_j (tangential reconstruction)
    constexpr int CH = FBLTS_SLOW_CHUNK < MAXE2 ? FBLTS_SLOW_CHUNK : MAXE2;
    double fp = 0.0, vt = 0.0;
    const double qs = PVE ? qe[e] : 0.0;
#pragma unroll
    for (int j0 = 0; j0 < MAXE2; j0 += CH) {
        double w[CH], f[CH], ut[HUR ? CH : 1], qj[PVE ? CH : 1];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
            if (j0 + j < n && j0 + j < MAXE2) {
                const int ee = m.eoe[(j0 + j) * m.strideE + e];
                w[j] = m.W[(j0 + j) * m.strideE + e];
                f[j] = F[ee];
                if (HUR) ut[HUR ? j : 0] = u[ee];
                if (PVE) qj[PVE ? j : 0] = qe[ee];
            }
        }
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (j0 + j < n && j0 + j < MAXE2) {
                if (PVE) fp = fp + w[j] * f[j] * (0.5 * (qs + qj[PVE ? j : 0]));
                else fp = fp + w[j] * f[j];
                if (HUR) vt = vt + w[j] * ut[HUR ? j : 0];
            }
    }
    // VEL: the update's own loads (z_b, base / accumulator) after the slot loop (not live in it: no
    // spills at 5 CTAs per SM) but before the divisions
    const bool ia = VEL && vf.acc && e >= vf.a0 && e < vf.a1;
    double zb0 = 0.0, zb1 = 0.0, b0 = 0.0;
    if (VEL) {
        zb0 = m.zb[c.x], zb1 = m.zb[c.y];
        b0 = ia ? (vf.first ? 0.0 : vf.acc[e - vf.a0]) : vf.base[e];
    }
    double pv;
    if (PVE) {
        pv = fp;
    } else {
        if (!FBLTS_SLOW_HOIST) {
            const int2 v = m.voe[e];
            qv0 = q[v.x], qv1 = q[v.y];
        }
        const double qh = 0.5 * (qv0 + qv1);
        pv = qh * fp;
    }
    if (pvout) pvout[e] = pv;                 // vorticity companion: the PV-flux part alone
    if (!FBLTS_SLOW_HOIST) K0 = K[c.x], K1 = K[c.y], h0 = h[c.x], h1 = h[c.y], tau = m.tau[e], dce = m.dc[e];
    const double he = 0.5 * (h0 + h1);
    const double G = tau / (rho0 * he);
    double s = pv - (K1 - K0) / dce + G;
    if (HUR) {   // bottom drag and wind (eq. hurricane_model)
        const double ue = u[e];
        const double speed = sqrt(ue * ue + vt * vt);
        const double D = cd * speed * ue / he;
        const double dn = m.uwn[e] - ue, dt = m.uwt[e] - vt;
        const double ws = sqrt(dn * dn + dt * dt);
        const double Wd = cw * ws * dn / he;
        s = s - D + Wd;
    }
    if (VEL) {
        const double phi = phi_fast(g, h0, zb0, h1, zb1, dce);
        if (ia) vf.acc[e - vf.a0] = b0 + (phi + s);
        else vf.out[e] = b0 + vf.c * (phi + s);
    } else {
        S[e] = s;
    }
}

// ---------------------------------------------------------------- coarse stages
// Stage 1 (eq. if_h_s1 / coarse_h_s1): h1 = h^n + dt/3 Psi(u^n, h^n) on C u F^5.
// Stage 2 (eq. if_h_s2 / coarse_h_s2): h2 = h^n + dt/2 Psi(u1, h1) on C u F^3,
//   u1_e = u^n_e + dt/3 (Phi^fast_e(h*) + S_e), h* = b1 h1 + (1-b1) h^n.
// Stage 3 (eq. if_h_s3 / coarse_h_s3): h3 = h^n + dt Psi(u2, h2) on C u F^1,
//   u2_e = u^n_e + dt/2 (Phi^fast_e(h**) + S_e), h** = b2 h2 + (1-b2) h^n.
template <int G, int STAGE>
__global__ void __launch_bounds__(TPB, FBLTS_MINB) k_coarse_stage(DevMesh m, const double *__restrict__ hN,
                                                      const double *__restrict__ hprev,
                                                      const double *__restrict__ uN,
                                                      const double *__restrict__ S, double *__restrict__ out,
                                                      StepConst sc, int begin, int end, DevError *err) {
    const int i = begin + blockIdx.x * TPB + threadIdx.x;
    if (i >= end) return;
    int2 r[G];
    load_row<G>(m, i, r);
    const int n = m.nEoC[i];
    const double cu = STAGE == 2 ? sc.c1 : sc.c2;        // c_{s-1} of the velocity
    const double bb = STAGE == 2 ? sc.b1 : sc.b2;
    const double omb = STAGE == 2 ? sc.omb1 : sc.omb2;
    const double hNi = hN[i];
    const double Hi = STAGE == 1 ? hNi : hprev[i];
    const double HSi = STAGE == 1 ? 0.0 : bb * Hi + omb * hNi;
    const double zbi = STAGE == 1 ? 0.0 : m.zb[i];
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < G; ++j) {
        if (j < n) {
            bool pos;
            const int e = decode(r[j].x, pos);
            const int nb = r[j].y;
            double ue, Hn;
            const double dve = m.dv[e];
            if (STAGE == 1) {
                Hn = hN[nb];
                ue = uN[e];
            } else {
                Hn = hprev[nb];
                const double HSn = bb * Hn + omb * hN[nb];
                const double zbn = m.zb[nb];
                const double dc = m.dc[e];
                const double une = uN[e], se = S[e];        // loaded before the division
                const double phi = pos ? phi_fast(sc.g, HSi, zbi, HSn, zbn, dc) : phi_fast(sc.g, HSn, zbn, HSi, zbi, dc);
                ue = une + cu * (phi + se);
            }
            acc = acc + psi_term(pos, Hi, Hn, ue, dve);
        }
    }
    const double ch = STAGE == 1 ? sc.c1 : (STAGE == 2 ? sc.c2 : sc.c3);
    const double psi = -acc / m.areaCell[i];
    const double v = hNi + ch * psi;
    out[i] = v;
    if (!(v > 0.0)) report(err, STAGE == 1 ? K_COARSE_S1 : (STAGE == 2 ? K_COARSE_S2 : K_COARSE_S3), -1, i, v);
}

// ---------------------------------------------------------------- staged stage sweep (tiles)
// The same arithmetic as k_coarse_stage / the DEEP fine stages, reorganised per tile of TILE
// consecutive cells (fblts_internal.h TileMesh) into an edge phase and a cell phase over shared
// memory, in a persistent double-buffered TMA pipeline:
//   * each CTA walks the tiles tile0 + blockIdx.x + k * gridDim.x; while it computes tile k the
//     other shared buffer fills with tile k+1: one thread issues 1-D bulk copies (TMA,
//     cp.async.bulk, completion counted on the buffer's mbarrier) of the tile's contiguous data
//     -- its own cells, its owned edge run, its local-edge cell pairs -- and every thread adds
//     8-byte asynchronous copies (LDGSTS) of the indexed data, the halo cells and foreign edges,
//     whose index lists were prefetched into registers during the previous tile's compute;
//   * edge phase: every local edge computes its flux term ONCE,
//        T_e = l_e * ((0.5 (H_c0 + H_c1)) * u_bar_e),
//     u_bar_e = u_e (stage 1) or u_e + cu (Phi^fast_e(bb H + omb h_base) + S_e) (stages 2, 3);
//   * cell phase: Psi_i = -(sum_j n_{e_j,i} T_{e_j}) / A_i in slot order, out_i = h_base,i + ch Psi_i.
// Bit-identical to the per-cell evaluation: 0.5 (H_i + H_n) is commutative in IEEE arithmetic and
// Phi^fast_e is always evaluated as (c0, c1), so both cells of an edge see the same T_e; each
// cell's sum keeps its sequential slot order from +0.0.
// Bulk copies need 16-byte aligned source, destination and size: a contiguous double range [a, b)
// is copied from a & ~1 to (b + 1) & ~1 (at most one element of slack at each end, inside the
// 256-byte padded workspace allocation) and addressed in shared memory with offset a & 1.
constexpr int HPT = 2;   // halo-cell indices prefetched per thread (more: loaded synchronously)
constexpr int FPT = 2;   // foreign-edge indices prefetched per thread

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_pending() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    unsigned ok = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok)
                     : "r"(smem_u32(bar)), "r"(parity)
                     : "memory");
    } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// FBLTS_CHECK=1 (debug builds): device-side bounds checks of every shared-memory index the staged
// kernel derives from its tile tables; a violation traps (the launch fails with a CUDA error)
#ifndef FBLTS_CHECK
#define FBLTS_CHECK 0
#endif
#define FBLTS_REQUIRE(cond)                  \
    do {                                     \
        if (FBLTS_CHECK && !(cond)) __trap(); \
    } while (0)

template <int STAGE>
struct TileShape {
    static constexpr int NCA = STAGE == 4 ? 4 : (STAGE > 1 ? 3 : 1);   // cell arrays: hprev (, hbase, z_b (, h2))
    static constexpr int NEA = STAGE > 1 ? 4 : 2;                       // edge arrays: u, l_e (, S, d_e)
};

struct TileRec {
    int c0, c1, h0, h1, eo0, eo1, f0, f1, l0, g0, ge0;
};
__device__ __forceinline__ TileRec load_rec(const TileMesh &t, int tile) {
    const int *p = t.info + (size_t)tile * TINFO;
    TileRec r;
    r.c0 = p[0], r.h0 = p[1], r.eo0 = p[2], r.eo1 = p[3], r.f0 = p[4], r.l0 = p[5], r.g0 = p[6], r.ge0 = p[7];
    r.c1 = p[TINFO + 0], r.h1 = p[TINFO + 1], r.f1 = p[TINFO + 4];
    return r;
}

// Shared buffer of one tile (strides in elements, every array 16-byte aligned):
// cells [NCA][CS2], edges [NEA][ES2] (doubles), cell pairs [ES4] (uint32); the views below are
// shifted by the tile's alignment offsets so that local index 0 is the tile's first cell / edge.
template <int STAGE>
struct TileBuf {
    double *hp, *hb, *z, *h2, *u, *l, *S, *d;
    uint32_t *ecl;
    __device__ __forceinline__ TileBuf(double *B, int CS2, int ES2, const TileRec &r) {
        const int oc = r.c0 & 1, oe = r.eo0 & 1, ol = r.l0 & 3;
        hp = B + oc, hb = B + CS2 + oc, z = B + 2 * CS2 + oc, h2 = B + 3 * CS2 + oc;
        double *E = B + TileShape<STAGE>::NCA * CS2;
        u = E + oe, l = E + ES2 + oe, S = E + 2 * ES2 + oe, d = E + 3 * ES2 + oe;
        ecl = reinterpret_cast<uint32_t *>(E + TileShape<STAGE>::NEA * ES2) + ol;
    }
};

// one elected thread: bulk copies of the tile's contiguous ranges into buffer B, counted on bar
template <int STAGE>
__device__ __forceinline__ void issue_bulk(const DevMesh &m, const StageArgs &a, const TileRec &r, double *B,
                                           int CS2, int ES2, uint64_t *bar) {
    constexpr int NCA = TileShape<STAGE>::NCA, NEA = TileShape<STAGE>::NEA;
    const int ca = r.c0 & ~1, cb = (r.c1 + 1) & ~1;
    const int ea = r.eo0 & ~1, eb = (r.eo1 + 1) & ~1;
    const int nLE = r.eo1 - r.eo0 + r.f1 - r.f0;
    const int la = r.l0 & ~3, lb = (r.l0 + nLE + 3) & ~3;
    const unsigned cbytes = 8u * (cb - ca), ebytes = 8u * (eb - ea), lbytes = 4u * (lb - la);
    // ghosts (TileMesh): the halo cells' z_b and the foreign edges' l_e, d_e, S -- values that do not change
    // during a step -- stored per tile contiguously, so they arrive by bulk copies: halo cell q lands at
    // local HALO0 + q, foreign edge q at nOE + FGAP + q; each ghost range starts at the parity that makes
    // source and destination 16-byte aligned (host layout) and is copied with an even length
    const int oc = r.c0 & 1, pe = r.eo1 & 1;
    const int nH = r.h1 - r.h0, nF = r.f1 - r.f0;
    const int gs = r.g0 - oc, ges = r.ge0 - pe;
    const unsigned hbytes = (STAGE > 1 && nH) ? 8u * ((nH + oc + 1) & ~1) : 0u;
    const unsigned fbytes = nF ? 8u * ((nF + pe + 1) & ~1) : 0u;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic writes of the last use first
    mbar_expect_tx(bar, NCA * cbytes + hbytes + (ebytes ? NEA * ebytes : 0u) + (NEA - 1) * fbytes + lbytes);
    bulk_g2s(B, a.hprev + ca, cbytes, bar);
    if (STAGE > 1) {
        bulk_g2s(B + CS2, a.hbase + ca, cbytes, bar);
        bulk_g2s(B + 2 * CS2, m.zb + ca, cbytes, bar);
    }
    if (STAGE == 4) bulk_g2s(B + 3 * CS2, a.h2 + ca, cbytes, bar);
    FBLTS_REQUIRE(gs >= 0 && HALO0 + (int)(hbytes / 8u) <= CS2);
    if (hbytes) bulk_g2s(B + 2 * CS2 + HALO0, m.tm.Gz + gs, hbytes, bar);
    double *E = B + NCA * CS2;
    if (ebytes) {
        bulk_g2s(E, a.ubase + ea, ebytes, bar);
        bulk_g2s(E + ES2, m.dv + ea, ebytes, bar);
        if (STAGE > 1) {
            bulk_g2s(E + 2 * ES2, a.S + ea, ebytes, bar);
            bulk_g2s(E + 3 * ES2, m.dc + ea, ebytes, bar);
        }
    }
    if (fbytes) {
        const int fo = (r.eo0 & 1) + (r.eo1 - r.eo0) + FGAP - pe;      // even: eo0 + nOE has the parity of eo1
        FBLTS_REQUIRE(ges >= 0 && (fo & 1) == 0 && fo + (int)(fbytes / 8u) <= ES2);
        bulk_g2s(E + ES2 + fo, m.tm.Gl + ges, fbytes, bar);
        if (STAGE > 1) {
            bulk_g2s(E + 2 * ES2 + fo, a.gS + ges, fbytes, bar);
            bulk_g2s(E + 3 * ES2 + fo, m.tm.Gd + ges, fbytes, bar);
        }
    }
    bulk_g2s(E + NEA * ES2, m.tm.ecl + la, lbytes, bar);
}

template <int STAGE>
__device__ __forceinline__ void issue_indexed(const DevMesh &m, const StageArgs &a, const TileRec &r,
                                              const TileBuf<STAGE> &b, int tid, const int (&hx)[HPT],
                                              const int (&fx)[FPT]) {
    const int nH = r.h1 - r.h0, nF = r.f1 - r.f0, nOE = r.eo1 - r.eo0;
    auto halo = [&](int q, int x) {                       // the values that change during a step
        cp_async8(b.hp + HALO0 + q, a.hprev + x);
        if (STAGE > 1) cp_async8(b.hb + HALO0 + q, a.hbase + x);
        if (STAGE == 4) cp_async8(b.h2 + HALO0 + q, a.h2 + x);
    };
    auto foreign = [&](int p, int e) { cp_async8(b.u + p, a.ubase + e); };
#pragma unroll
    for (int k = 0; k < HPT; ++k)
        if (k * NTHR + tid < nH) halo(k * NTHR + tid, hx[k]);
    for (int q = HPT * NTHR + tid; q < nH; q += NTHR) halo(q, m.tm.halo[r.h0 + q]);
#pragma unroll
    for (int k = 0; k < FPT; ++k)
        if (k * NTHR + tid < nF) foreign(nOE + FGAP + k * NTHR + tid, fx[k]);
    for (int q = FPT * NTHR + tid; q < nF; q += NTHR) foreign(nOE + FGAP + q, m.tm.fedge[r.f0 + q]);
}

__device__ __forceinline__ void load_indices(const TileMesh &t, const TileRec &r, int tid, int (&hx)[HPT], int (&fx)[FPT]) {
#pragma unroll
    for (int k = 0; k < HPT; ++k) {
        const int q = k * NTHR + tid;
        hx[k] = q < r.h1 - r.h0 ? t.halo[r.h0 + q] : 0;
    }
#pragma unroll
    for (int k = 0; k < FPT; ++k) {
        const int q = k * NTHR + tid;
        fx[k] = q < r.f1 - r.f0 ? t.fedge[r.f0 + q] : 0;
    }
}

// development probes were removed (round 2); FBLTS_PROBE stays 0 and is reported by fblts_build_info
#ifndef FBLTS_PROBE
#define FBLTS_PROBE 0
#endif
template <int G, int STAGE>
__global__ void __launch_bounds__(NTHR, FBLTS_TILE_MINB) k_stage_tiled(DevMesh m, int tile0, int tile1, int CS2, int ES2,
                                                         StageArgs a, DevError *err) {
    extern __shared__ __align__(16) double smem[];
    constexpr int NCA = TileShape<STAGE>::NCA, NEA = TileShape<STAGE>::NEA;
    const int BUF = NCA * CS2 + NEA * ES2 + ES2 / 2 + 2;   // doubles per buffer (+ ecl, 16-B multiple)
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);    // NBUF mbarriers
    double *buf0 = smem + ((NBUF + 1) & ~1);               // 16-byte aligned after the barriers
    const TileMesh &t = m.tm;
    const int tid = threadIdx.x;
    int tile = tile0 + blockIdx.x;
    if (tile >= tile1) return;
    const int G0 = gridDim.x;
    // tile records in a 4-slot shared-memory ring, fetched three tiles ahead by cp.async (16 ints per slot:
    // the tile's 8-int record and the next one's, whose c0 / h0 / f0 end the tile's ranges), so no tile
    // waits on a dependent global load of its record and index lists can be fetched two tiles ahead
    const int nmine = (tile1 - tile + G0 - 1) / G0;
    const int tfirst = tile;
    int *recs = reinterpret_cast<int *>(buf0 + NBUF * BUF);
    auto fetch_rec = [&](int j) {                         // threads 0..3: one 16-byte copy each
        if (tid < 4 && j < nmine) {
            const int *src = t.info + (size_t)(tfirst + j * G0) * TINFO + tid * 4;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(recs + (j & 3) * TREC + tid * 4)),
                         "l"(src) : "memory");
        }
    };
    if (tid == 0) {
        for (int k = 0; k < NBUF; ++k) mbar_init(&bar[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    fetch_rec(0);
    fetch_rec(1);
    fetch_rec(2);
    cp_async_commit();
    cp_async_wait_pending<0>();
    __syncthreads();
    auto rec = [&](int j) {
        const int *p = recs + (j & 3) * TREC;
        TileRec r;
        r.c0 = p[0], r.h0 = p[1], r.eo0 = p[2], r.eo1 = p[3], r.f0 = p[4], r.l0 = p[5], r.g0 = p[6], r.ge0 = p[7];
        r.c1 = p[8], r.h1 = p[9], r.f1 = p[12];
        return r;
    };
    // Two tile buffers: while tile j is computed the other buffer fills with tile j+1 -- one thread
    // issues its bulk copies at the top of the iteration, every thread its halo / foreign gathers after
    // the edge phase (issued earlier they only slow the edge phase's shared-memory traffic -- measured),
    // from index lists loaded one iteration before (two tiles ahead).  The gathers of a tile form one
    // cp.async group, committed once per iteration (even if empty).
    int hx[HPT], fx[FPT], hx2[HPT], fx2[FPT];
    {
        const TileRec r0 = rec(0);
        if (tid == 0) issue_bulk<STAGE>(m, a, r0, buf0, CS2, ES2, &bar[0]);
        load_indices(t, r0, tid, hx, fx);
        issue_indexed<STAGE>(m, a, r0, TileBuf<STAGE>(buf0, CS2, ES2, r0), tid, hx, fx);
        cp_async_commit();
        if (nmine > 1) load_indices(t, rec(1), tid, hx, fx);
    }
    unsigned phase = 0u;                                   // bit b: parity of buffer b's next completion
    int buf = 0;
    for (int j = 0; j < nmine; ++j, tile += G0, buf ^= 1) {
        const TileRec cur = rec(j);
        const bool more = j + 1 < nmine;
        const TileRec nx = more ? rec(j + 1) : TileRec{};
        mbar_wait(&bar[buf], (phase >> buf) & 1u);
        phase ^= 1u << buf;
        cp_async_wait_pending<0>();
        __syncthreads();                                   // tile `cur` staged; the other buffer is free
        if (j + 2 < nmine) load_indices(t, rec(j + 2), tid, hx2, fx2);   // record j+2 arrived; used next iteration
        double *Bn = buf0 + (buf ^ 1) * BUF;
        if (more && tid == 0) issue_bulk<STAGE>(m, a, nx, Bn, CS2, ES2, &bar[buf ^ 1]);
        const TileBuf<STAGE> bc(buf0 + buf * BUF, CS2, ES2, cur);
        // ---- compute tile `cur`
        const int nOwn = cur.c1 - cur.c0;
        const int i = cur.c0 + tid;
        const bool own = tid < nOwn;
        uint16_t r[G];
        double A = 1.0;
        if (own) {
#pragma unroll
            for (int j = 0; j < G; ++j) r[j] = j < m.maxE ? t.row[(size_t)j * t.strideRow + i] : TILE_SENT;
            A = m.areaCell[i];
        }
        const int nOE = cur.eo1 - cur.eo0, nLE = nOE + cur.f1 - cur.f0;
        FBLTS_REQUIRE(nOwn <= TILE && HALO0 + (cur.h1 - cur.h0) + 1 <= CS2 && nLE + FGAP + 1 <= ES2 && nOE >= 0);
#ifndef FBLTS_EDGE_UNROLL
#define FBLTS_EDGE_UNROLL 1
#endif
        // edge phase: T_e overwrites u_e; EU independent edges per thread in flight (fp64 latency)
        constexpr int EU = FBLTS_EDGE_UNROLL;
        // edge slots are dealt from warp 1 on, warp 0 last: the partial last round of a tile's ~3.4 edges
        // per thread falls on the low slots, so warp 0 -- which also issued the next tile's bulk copies --
        // skips it, evening out the arrival at the barrier below
#ifndef FBLTS_EDGE_ROTATE
#define FBLTS_EDGE_ROTATE 1
#endif
        const int te = FBLTS_EDGE_ROTATE ? (tid >= 32 ? tid - 32 : tid + NTHR - 32) : tid;
        for (int p0 = te; p0 < nLE; p0 += EU * NTHR) {
#pragma unroll
            for (int uu = 0; uu < EU; ++uu) {
                const int p = p0 + uu * NTHR;
                if (p < nLE) {
                    const uint32_t pr = bc.ecl[p];
                    const int q = p < nOE ? p : p + FGAP;
                    const int l0 = pr & 0xFFFF, l1 = pr >> 16;
                    FBLTS_REQUIRE((l0 < nOwn || (l0 >= HALO0 && l0 < HALO0 + cur.h1 - cur.h0)) &&
                                  (l1 < nOwn || (l1 >= HALO0 && l1 < HALO0 + cur.h1 - cur.h0)));
                    const double H0 = bc.hp[l0], H1 = bc.hp[l1];
                    double ue = bc.u[q];
                    const double le = bc.l[q];                   // before the division (see k_fine_vel)
                    if (STAGE == 2 || STAGE == 3) {
                        const double Se = bc.S[q];
                        const double HS0 = a.bb * H0 + a.omb * bc.hb[l0];
                        const double HS1 = a.bb * H1 + a.omb * bc.hb[l1];
                        const double phi = phi_fast(a.g, HS0, bc.z[l0], HS1, bc.z[l1], bc.d[q]);
                        ue = ue + a.cu * (phi + Se);
                    } else if (STAGE == 4) {            // u^{n,k} (fine velocity stage 3, subeqn fine_s3)
                        const double Se = bc.S[q];
                        const double HS0 = a.bb * H0 + a.omb * bc.h2[l0] + a.bb * bc.hb[l0];
                        const double HS1 = a.bb * H1 + a.omb * bc.h2[l1] + a.bb * bc.hb[l1];
                        const double phi = phi_fast(a.g, HS0, bc.z[l0], HS1, bc.z[l1], bc.d[q]);
                        ue = ue + a.cu * (phi + Se);
                        if (p < nOE) a.unew[cur.eo0 + p] = ue;
                    }
                    const double Fe = (0.5 * (H0 + H1)) * ue;
                    bc.u[q] = le * Fe;
                }
            }
        }
        if (more) issue_indexed<STAGE>(m, a, nx, TileBuf<STAGE>(Bn, CS2, ES2, nx), tid, hx, fx);
        fetch_rec(j + 3);                                  // into the slot of tile j - 1 (read at the top)
        cp_async_commit();
#pragma unroll
        for (int q = 0; q < HPT; ++q) hx[q] = hx2[q];
#pragma unroll
        for (int q = 0; q < FPT; ++q) fx[q] = fx2[q];
        if (tid == 0) bc.u[nOE] = 0.0;                    // the gap slot: the term of an unused slot
        __syncthreads();
        if (own) {                                        // cell phase
            const double hbi = (STAGE == 1 || STAGE == 4) ? bc.hp[tid] : bc.hb[tid];
            double acc = 0.0;
            // branch-free slot loop: n_{e,i} applied by flipping the sign bit (exactly -tt); an unused
            // slot (TILE_SENT, sign bit set) reads the gap slot's +0.0 as -0.0, and x + (-0.0) == x for
            // every x, so the sum is bit-identical to the sequential sum over the used slots
#pragma unroll
            for (int j = 0; j < G; ++j) {
                const uint32_t rj = r[j];
                const int q = rj == TILE_SENT ? nOE : (int)(rj & 0x7FFFu);
                FBLTS_REQUIRE(q <= nOE || (q >= nOE + FGAP && q < nLE + FGAP));
                const unsigned long long tb = __double_as_longlong(bc.u[q]) ^ ((unsigned long long)(rj >> 15) << 63);
                acc = acc + __longlong_as_double(tb);
            }
            const double psi = -acc / A;
            const double v = hbi + a.ch * psi;
            a.out[i] = v;
            if (!(v > 0.0)) report(err, a.kind, a.k, i, v);
        }
    }
}

// coarse FB averages (tilde / bar data)
__device__ __forceinline__ double hs2c(const StepConst &sc, const double *h2, const double *hN, int x) {
    return sc.b2 * h2[x] + sc.omb2 * hN[x];
}
__device__ __forceinline__ double hs3c(const StepConst &sc, const double *h3, const double *h2, const double *hN,
                                       int x) {
    return sc.b3 * h3[x] + sc.om2b3 * h2[x] + sc.b3 * hN[x];
}

// Velocity stage 3 on C^int_E: u^{n+1} = u^n + dt (Phi^fast(h***) + S).
// IF-1_E tilde u^{n+1} is never stored: the fine phase recomputes it (Q10).
__global__ void __launch_bounds__(TPB) k_coarse_vel(DevMesh m, const double *__restrict__ hN,
                                                    const double *__restrict__ h2,
                                                    const double *__restrict__ h3, const double *__restrict__ uN,
                                                    const double *__restrict__ S, double *__restrict__ uNew,
                                                    StepConst sc, int end, double *__restrict__ u2o,
                                                    double *__restrict__ u3o, int if1, int fend) {
    const int e = blockIdx.x * TPB + threadIdx.x;
    if (e >= fend) return;
    const int2 c = m.coe[e];
    const double zb0 = m.zb[c.x], zb1 = m.zb[c.y], dc = m.dc[e], un = uN[e], se = S[e];
    if (e < end || e >= if1) {      // u~^{n+1}: int_E -> u^{n+1}; IF-1_E -> u~^{n+1} for the fine phase (Q10)
        const double phi = phi_fast(sc.g, hs3c(sc, h3, h2, hN, c.x), zb0, hs3c(sc, h3, h2, hN, c.y), zb1, dc);
        const double v = un + sc.c3 * (phi + se);
        if (e < end) {
            uNew[e] = v;
            return;
        }
        u3o[e - end] = v;
    }
    // IF-2_E u IF-1_E: u~^{n+1/2} -- the fine stage-3 band sweep's edge velocities on the IF edges (k_fine_s3),
    // which the fine phase never changes: h2, h^n, h3 of IF cells and u^n, S stay as the coarse stages left them
    const double phi2 = phi_fast(sc.g, hs2c(sc, h2, hN, c.x), zb0, hs2c(sc, h2, hN, c.y), zb1, dc);
    u2o[e - end] = un + sc.c2 * (phi2 + se);
}

// ---------------------------------------------------------------- fine subcycles
// Views (reading Q11): F -> fine data, IF-1 -> predicted (eq. preds,
// eq. hstar_preds), IF-2 / int -> coarse tilde / bar data.  In a DEEP instance every
// cell and edge touched is fine, so the views reduce to the fine arrays.
struct FineArrays {
    const double *hN, *h1, *h2, *h3, *hk;   // h3 = coarse stage-3 output (hNew before the correction)
    const double *Sf;                       // slow tendency used on F_E (S, or S^k with the refresh)
    const double *uIF2, *uIF3;              // u~^{n+1/2}, u~^{n+1} on the IF edges (DevState)
};

__device__ __forceinline__ double pred_level(const PredConst &p, const FineArrays &a, int x) {
    return p.a * a.h3[x] + p.oma * a.hN[x];                     // subeqn pred_old, level k
}
__device__ __forceinline__ double pred_level1(const PredConst &p, const FineArrays &a, int x) {
    return p.a1 * a.h3[x] + p.oma1 * a.hN[x];                   // level k+1 (k = M extra)
}
__device__ __forceinline__ double pred_stage(const PredConst &p, const double *h3, const double *hs,
                                             const double *hN, int x) {
    return p.a * h3[x] + p.b * hs[x] + p.c * hN[x];              // subeqn pred_s1 / pred_s2
}

template <bool BAND>
__device__ __forceinline__ int cclass(const DevMesh &m, int x) { return BAND ? ccls(m, x) : 2; }
template <bool BAND>
__device__ __forceinline__ int eclass(const Bounds &b, int e) { return BAND ? ecls(b, e) : 3; }

// view H0 (h^{n,k}) for fine stage 1
template <bool BAND>
__device__ __forceinline__ double view0(const DevMesh &b, const PredConst &p, const FineArrays &a, int x) {
    const int cl = cclass<BAND>(b, x);
    return cl == 2 ? a.hk[x] : (cl == 1 ? pred_level(p, a, x) : a.hN[x]);
}

// view (H1, HS1) for fine stage 2
template <bool BAND>
__device__ __forceinline__ void view1(const DevMesh &b, const StepConst &sc, const PredConst &p, const FineArrays &a,
                                      int x, double &H, double &HS) {
    const int cl = cclass<BAND>(b, x);
    if (cl == 2) {
        H = a.h1[x];
        HS = sc.b1 * H + sc.omb1 * a.hk[x];
    } else if (cl == 1) {
        const double hP0 = pred_level(p, a, x);
        H = pred_stage(p, a.h3, a.h1, a.hN, x);
        HS = sc.b1 * H + sc.omb1 * hP0;
    } else {
        H = a.h1[x];
        HS = sc.b1 * H + sc.omb1 * a.hN[x];
    }
}

// view (H2, HS2) for fine stage 3 / the correction summand
template <bool BAND>
__device__ __forceinline__ void view2(const DevMesh &b, const StepConst &sc, const PredConst &p, const FineArrays &a,
                                      int x, double &H, double &HS) {
    const int cl = cclass<BAND>(b, x);
    if (cl == 2) {
        H = a.h2[x];
        HS = sc.b2 * H + sc.omb2 * a.hk[x];
    } else if (cl == 1) {
        const double hP0 = pred_level(p, a, x);
        H = pred_stage(p, a.h3, a.h2, a.hN, x);
        HS = sc.b2 * H + sc.omb2 * hP0;
    } else {
        H = a.h2[x];
        HS = sc.b2 * H + sc.omb2 * a.hN[x];
    }
}

// view HS3 (h^{***,k}) for the fine velocity stage 3
template <bool BAND>
__device__ __forceinline__ double view3(const DevMesh &b, const StepConst &sc, const PredConst &p,
                                        const FineArrays &a, const double *hnext, int x) {
    const int cl = cclass<BAND>(b, x);
    if (cl == 2) return sc.b3 * hnext[x] + sc.om2b3 * a.h2[x] + sc.b3 * a.hk[x];
    if (cl == 1) {
        const double hP0 = pred_level(p, a, x);
        const double hP0n = pred_level1(p, a, x);
        const double hP2 = pred_stage(p, a.h3, a.h2, a.hN, x);
        return sc.b3 * hP0n + sc.om2b3 * hP2 + sc.b3 * hP0;
    }
    return hs3c(sc, a.h3, a.h2, a.hN, x);
}

// Fine stage 1 (subeqn fine_s1): h_bar^{n,k+1/3} = h^{n,k} + dt/(3M) Psi(u^{n,k}, h^{n,k}) on F.
template <int G, bool BAND>
__global__ void __launch_bounds__(TPB) k_fine_s1(DevMesh m, FineArrays a, const double *__restrict__ uk,
                                                 double *__restrict__ out, StepConst sc, PredConst p, int k,
                                                 int begin, int end, DevError *err) {
    const int i = begin + blockIdx.x * TPB + threadIdx.x;
    if (i >= end) return;
    int2 r[G];
    load_row<G>(m, i, r);
    const int n = m.nEoC[i];
    const double Hi = a.hk[i];
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < G; ++j) {
        if (j < n) {
            bool pos;
            const int e = decode(r[j].x, pos);
            acc = acc + psi_term(pos, Hi, view0<BAND>(m, p, a, r[j].y), uk[e], m.dv[e]);
        }
    }
    const double psi = -acc / m.areaCell[i];
    const double v = Hi + sc.c1f * psi;
    out[i] = v;
    if (!(v > 0.0)) report(err, K_FINE_S1, k, i, v);
}

// Fine stage 2 (subeqn fine_s2): h_bar^{n,k+1/2} = h^{n,k} + dt/(2M) Psi(u_bar^{n,k+1/3}, h_bar^{n,k+1/3}),
// u_bar^{n,k+1/3}_e = u^{n,k}_e + dt/(3M) (Phi^fast_e(h^{*,k}) + S_e) recomputed per edge.
template <int G, bool BAND>
__global__ void __launch_bounds__(TPB, BAND ? FBLTS_BAND_MINB : FBLTS_MINB) k_fine_s2(DevMesh m, FineArrays a, const double *__restrict__ uk,
                                                 const double *__restrict__ S, double *__restrict__ out,
                                                 StepConst sc, PredConst p, int k, int begin, int end,
                                                 DevError *err) {
    const int i = begin + blockIdx.x * TPB + threadIdx.x;
    if (i >= end) return;
    int2 r[G];
    load_row<G>(m, i, r);
    const int n = m.nEoC[i];
    double Hi, HSi;
    view1<BAND>(m, sc, p, a, i, Hi, HSi);
    const double zbi = m.zb[i];
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < G; ++j) {
        if (j < n) {
            bool pos;
            const int e = decode(r[j].x, pos);
            const int nb = r[j].y;
            double Hn, HSn;
            view1<BAND>(m, sc, p, a, nb, Hn, HSn);
            const double zbn = m.zb[nb];
            const double dc = m.dc[e];
            const double uke = uk[e], sfe = a.Sf[e], dve = m.dv[e];  // loaded before the division
            const double phi = pos ? phi_fast(sc.g, HSi, zbi, HSn, zbn, dc) : phi_fast(sc.g, HSn, zbn, HSi, zbi, dc);
            const double ue = uke + sc.c1f * (phi + sfe);           // every edge of a fine cell is F_E
            acc = acc + psi_term(pos, Hi, Hn, ue, dve);
        }
    }
    const double psi = -acc / m.areaCell[i];
    const double v = a.hk[i] + sc.c2f * psi;
    out[i] = v;
    if (!(v > 0.0)) report(err, K_FINE_S2, k, i, v);
}

// Fine stage 3 on F (subeqn fine_s3) fused with the correction summand on IF-1 u IF-2
// (eq. if_correction, "accumulated during the fine advancement step"):
//   F:      h^{n,k+1} = h^{n,k} + dt/M Psi(u_bar^{n,k+1/2}, h_bar^{n,k+1/2})
//   IF:     accH += Psi(u_bar^{n,k+1/2}, h_bar^{n,k+1/2})          (views, reading Q11/Q14)
// Edge velocity u_bar^{n,k+1/2} by edge region: F_E -> u^{n,k} + dt/(2M)(Phi^fast(h^{**,k}) + S);
// IF-1_E -> predicted (k/M) u~^{n+1} + (1/M) u~^{n+1/2} + (1-(k+1)/M) u^n with the tilde data
// recomputed from the coarse thicknesses; IF-2_E / int_E -> coarse u~^{n+1/2}.
template <int G, bool BAND>
__global__ void __launch_bounds__(TPB, BAND ? FBLTS_BAND_MINB : FBLTS_MINB) k_fine_s3(DevMesh m, FineArrays a, const double *__restrict__ uN,
                                                 const double *__restrict__ uk, const double *__restrict__ S,
                                                 double *__restrict__ hnext, double *__restrict__ accH,
                                                 StepConst sc, PredConst p, int k, int begin, int fstart, int end,
                                                 DevError *err) {
    const int i = begin + blockIdx.x * TPB + threadIdx.x;
    if (i >= end) return;
    int2 r[G];
    load_row<G>(m, i, r);
    const int n = m.nEoC[i];
    double Hi, HSi;
    view2<BAND>(m, sc, p, a, i, Hi, HSi);
    const double zbi = m.zb[i];
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < G; ++j) {
        if (j < n) {
            bool pos;
            const int e = decode(r[j].x, pos);
            const int nb = r[j].y;
            double Hn, HSn;
            view2<BAND>(m, sc, p, a, nb, Hn, HSn);
            const double dc = m.dc[e];
            const double dve = m.dv[e];                       // loaded before any division
            double ue;
            const int ec = eclass<BAND>(m.eb, e);
            if (ec == 3) {
                const double zbn = m.zb[nb];
                const double uke = uk[e], sfe = a.Sf[e];
                const double phi = pos ? phi_fast(sc.g, HSi, zbi, HSn, zbn, dc) : phi_fast(sc.g, HSn, zbn, HSi, zbi, dc);
                ue = uke + sc.c2f * (phi + sfe);
            } else if (ec >= 1) {             // IF edges: the coarse stage velocities (k_coarse_vel, once per step)
                const double u2 = a.uIF2[e - m.eb.if2];
                ue = ec == 2 ? p.a * a.uIF3[e - m.eb.if2] + p.b * u2 + p.c * uN[e] : u2;
            } else {                          // int_E edge of an IF-2 cell: u~^{n+1/2}
                const int c0 = pos ? i : nb, c1 = pos ? nb : i;
                const double une = uN[e], se = S[e];
                const double phi2 = phi_fast(sc.g, hs2c(sc, a.h2, a.hN, c0), m.zb[c0], hs2c(sc, a.h2, a.hN, c1), m.zb[c1], dc);
                ue = une + sc.c2 * (phi2 + se);
            }
            acc = acc + psi_term(pos, Hi, Hn, ue, dve);
        }
    }
    const double psi = -acc / m.areaCell[i];
    if (!BAND || i >= fstart) {
        const double v = a.hk[i] + sc.c3f * psi;
        hnext[i] = v;
        if (!(v > 0.0)) report(err, K_FINE_S3, k, i, v);
    } else {
        const double prev = k == 0 ? 0.0 : accH[i];
        accH[i] = prev + psi;
    }
}

// Fine velocity stage 3 (subeqn fine_s3) on F_E fused with the momentum correction summand on
// IF-1_E u IF-2_E (eq. if_correction): F_E: u^{n,k+1} = u^{n,k} + dt/M (Phi^fast(h^{***,k}) + S);
// IF_E: accU += Phi^fast(h^{***,k}) + S.
template <bool BAND>
__global__ void __launch_bounds__(TPB) k_fine_vel(DevMesh m, FineArrays a, const double *__restrict__ hnext,
                                                  const double *__restrict__ uk, const double *__restrict__ S,
                                                  double *__restrict__ unext, double *__restrict__ accU,
                                                  StepConst sc, PredConst p, int k, int begin, int end) {
    const int e = begin + blockIdx.x * TPB + threadIdx.x;
    if (e >= end) return;
    const int2 c = m.coe[e];
    // every load before the division: the compiler does not move a load above the division's slow-path
    // branch, so a load written after it starts only when the division is done (measured on slow_edge)
    const bool fine = !BAND || e >= m.eb.f;
    const int ai = e - m.eb.if2;
    const double base = fine ? uk[e] : (k == 0 ? 0.0 : accU[ai]);
    const double se = fine ? a.Sf[e] : S[e];
    const double phi = phi_fast(sc.g, view3<BAND>(m, sc, p, a, hnext, c.x), m.zb[c.x],
                                view3<BAND>(m, sc, p, a, hnext, c.y), m.zb[c.y], m.dc[e]);
    if (fine) unext[e] = base + sc.c3f * (phi + se);
    else accU[ai] = base + (phi + se);
}

// Interface Correction (eq. if_correction; reading Q14):
// h^{n+1} = h^n + dt/M accH on IF-1 u IF-2, u^{n+1} = u^n + dt/M accU on IF-1_E u IF-2_E.
__global__ void __launch_bounds__(TPB) k_correct(DevMesh m, const double *__restrict__ hN,
                                                 const double *__restrict__ uN, const double *__restrict__ accH,
                                                 const double *__restrict__ accU, double *__restrict__ hNew,
                                                 double *__restrict__ uNew, StepConst sc, int c0, int c1, unsigned nbC,
                                                 DevError *err) {
    if (blockIdx.x < nbC) {
        const int i = c0 + blockIdx.x * TPB + threadIdx.x;
        if (i >= c1) return;
        const double v = hN[i] + sc.c3f * accH[i];
        hNew[i] = v;
        if (!(v > 0.0)) report(err, K_CORRECT, -1, i, v);
    } else {
        const int e = m.eb.if2 + (blockIdx.x - nbC) * TPB + threadIdx.x;
        if (e >= m.eb.f) return;
        uNew[e] = uN[e] + sc.c3f * accU[e - m.eb.if2];
    }
}

// ---------------------------------------------------------------- RK4 reference scheme
// Classical four-stage RK4 on the unsplit system y = (h, u), y' = (Psi(u, h), Phi^fast(h) + Phi^slow(u, h))
// (oracle fbrk32.rk4_step): evaluated as numpy does, k1 + 2 k2 + 2 k3 + k4 left to right.
template <int G>
__global__ void __launch_bounds__(TPB) k_rk4_stage(DevMesh m, int stage, const double *__restrict__ hN,
                                                   const double *__restrict__ uN, const double *__restrict__ hs,
                                                   const double *__restrict__ us, const double *__restrict__ S,
                                                   double *__restrict__ accH, double *__restrict__ accU,
                                                   double *__restrict__ hout, double *__restrict__ uout,
                                                   double cnext, double dt6, double g, unsigned nbC, DevError *err) {
    double kx, base, accv = 0.0;          // base and the running sum loaded before the division (k_fine_vel)
    double *acc, *out;
    int x;
    if (blockIdx.x < nbC) {
        x = blockIdx.x * TPB + threadIdx.x;
        if (x >= m.nOwnC) return;
        base = hN[x];
        if (stage >= 2) accv = accH[x];
        int2 r[G];
        load_row<G>(m, x, r);
        const int n = m.nEoC[x];
        const double Hi = hs[x];
        double a = 0.0;
#pragma unroll
        for (int j = 0; j < G; ++j) {
            if (j < n) {
                bool pos;
                const int e = decode(r[j].x, pos);
                a = a + psi_term(pos, Hi, hs[r[j].y], us[e], m.dv[e]);
            }
        }
        kx = -a / m.areaCell[x];
        acc = accH;
        out = hout;
    } else {
        x = (blockIdx.x - nbC) * TPB + threadIdx.x;
        if (x >= m.nOwnE) return;
        const int2 c = m.coe[x];
        base = uN[x];
        if (stage >= 2) accv = accU[x];
        const double sx = S[x];
        kx = phi_fast(g, hs[c.x], m.zb[c.x], hs[c.y], m.zb[c.y], m.dc[x]) + sx;
        acc = accU;
        out = uout;
    }
    if (stage == 0) {                     // RK(3,2) stage: base + c_s k, no running sum
        const double v = base + cnext * kx;
        out[x] = v;
        if (blockIdx.x < nbC && !(v > 0.0)) report(err, K_RK4_STAGE, stage, x, v);
        return;
    }
    double sum;
    if (stage == 1) sum = kx;
    else if (stage == 4) sum = accv + kx;
    else sum = accv + 2.0 * kx;
    if (stage < 4) {
        acc[x] = sum;
        const double v = base + cnext * kx;
        out[x] = v;
        if (blockIdx.x < nbC && !(v > 0.0)) report(err, K_RK4_STAGE, stage, x, v);
    } else {
        const double v = base + dt6 * sum;
        out[x] = v;
        if (blockIdx.x < nbC && !(v > 0.0)) report(err, K_RK4_STAGE, stage, x, v);
    }
}


// ---------------------------------------------------------------- permutation, diagnostics
__global__ void k_permute_in(const int32_t *__restrict__ old, const double *__restrict__ src,
                             double *__restrict__ dst, int n) {
    const int i = blockIdx.x * TPB + threadIdx.x;
    if (i < n) dst[i] = src[old[i]];
}
// set_state input check on the device: bad[0] = smallest index whose value is not finite (or, with
// positive, not > 0) -- the first offending entry, as a sequential host scan would report it
__global__ void k_validate(const double *__restrict__ v, int n, int positive, int *bad) {
    const int i = blockIdx.x * TPB + threadIdx.x;
    if (i >= n) return;
    const double x = v[i];
    if (!(isfinite(x) && (!positive || x > 0.0))) atomicMin(bad, i);
}
__global__ void k_permute_out(const int32_t *__restrict__ old, const double *__restrict__ src,
                              double *__restrict__ dst, int n) {
    const int i = blockIdx.x * TPB + threadIdx.x;
    if (i < n) dst[old[i]] = src[i];
}

__global__ void k_pack(const int32_t *__restrict__ idx, const double *__restrict__ a, double *__restrict__ buf,
                       int n) {
    const int k = blockIdx.x * TPB + threadIdx.x;
    if (k < n) buf[k] = a[idx[k]];
}
__global__ void k_unpack(const int32_t *__restrict__ idx, const double *__restrict__ buf, double *__restrict__ a,
                         int n) {
    const int k = blockIdx.x * TPB + threadIdx.x;
    if (k < n) a[idx[k]] = buf[k];
}

// double-double accumulation (Knuth TwoSum), deterministic for a fixed launch shape
struct DD {
    double hi, lo;
};
__device__ __forceinline__ void dd_add(DD &a, double x) {
    const double s = a.hi + x;
    const double bb = s - a.hi;
    const double err = (a.hi - (s - bb)) + (x - bb);
    a.hi = s;
    a.lo = a.lo + err;
}
__device__ __forceinline__ DD dd_merge(DD a, DD b) {
    const double s = a.hi + b.hi;
    const double bb = s - a.hi;
    const double err = (a.hi - (s - bb)) + (b.hi - bb) + (a.lo + b.lo);
    DD r;
    r.hi = s + err;
    r.lo = err - (r.hi - s);
    return r;
}

// Deterministic block reduction of the diagnostics record (mass and Gamma as double-double, min h, max
// nu) with warp shuffles: a fixed shuffle-down tree inside each warp (lane i merges lane i + 16, 8, 4,
// 2, 1), the per-warp results through shared memory, then the same tree in warp 0.  Result in thread 0.
struct DiagRec {
    DD mass, gam;
    double hmin, numax;
};
__device__ __forceinline__ DiagRec diag_shfl(const DiagRec &a, int off) {
    DiagRec b;
    b.mass.hi = __shfl_down_sync(0xffffffffu, a.mass.hi, off);
    b.mass.lo = __shfl_down_sync(0xffffffffu, a.mass.lo, off);
    b.gam.hi = __shfl_down_sync(0xffffffffu, a.gam.hi, off);
    b.gam.lo = __shfl_down_sync(0xffffffffu, a.gam.lo, off);
    b.hmin = __shfl_down_sync(0xffffffffu, a.hmin, off);
    b.numax = __shfl_down_sync(0xffffffffu, a.numax, off);
    return b;
}
__device__ __forceinline__ void diag_merge(DiagRec &a, const DiagRec &b) {
    a.mass = dd_merge(a.mass, b.mass);
    a.gam = dd_merge(a.gam, b.gam);
    a.hmin = fmin(a.hmin, b.hmin);
    a.numax = fmax(a.numax, b.numax);
}
__device__ __forceinline__ DiagRec diag_block_reduce(DiagRec r) {
    constexpr int NW = TPB / 32;
    __shared__ DiagRec warp_part[NW];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const DiagRec o = diag_shfl(r, off);
        if (lane < off) diag_merge(r, o);
    }
    if (lane == 0) warp_part[wid] = r;
    __syncthreads();
    if (wid == 0) {
        r = lane < NW ? warp_part[lane] : DiagRec{{0.0, 0.0}, {0.0, 0.0}, (double)INFINITY, 0.0};
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const DiagRec o = diag_shfl(r, off);
            if (lane < off) diag_merge(r, o);
        }
    }
    return r;
}


// Diagnostics, pass 1: three roles by block range -- blocks [0, DIAG_RB) sum A_i h_i and min h over
// the owned cells, [DIAG_RB, 2 DIAG_RB) the absolute circulation of the owned vertices, the rest the
// Courant maximum over the owned edges; each block writes its 6 partials (identities for the
// quantities it does not touch).  Pass 2 merges them in a fixed order, so the result is a
// deterministic function of the state.
__global__ void __launch_bounds__(TPB) k_diag_partial(DevMesh m, const double *__restrict__ h,
                                                      const double *__restrict__ u, StepConst sc,
                                                      double *__restrict__ part, int pvmode) {
    const int role = blockIdx.x / DIAG_RB;
    const int tid = (blockIdx.x - role * DIAG_RB) * TPB + threadIdx.x;
    const int T = DIAG_RB * TPB;
    DD mass{0.0, 0.0}, gam{0.0, 0.0};
    double hmin = (double)INFINITY, numax = 0.0;
    if (role == 0) {
#pragma unroll 4
        for (int i = tid; i < m.nOwnC; i += T) {
            const double hi = h[i];
            dd_add(mass, m.areaCell[i] * hi);
            hmin = fmin(hmin, hi);
        }
    } else if (role == 1) {
#pragma unroll 2
        for (int v = tid; v < m.nV; v += T) {
            if (!m.vOwn[v]) continue;
            double circ = 0.0;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                bool pos;
                const int e = decode(m.eov[k * m.strideV + v], pos);
                const double t = m.dc[e] * u[e];
                circ = circ + (pos ? t : -t);
            }
            if (pvmode) {   // PV volume integral term A_v h_v q_v (Remark rmk:volume_conservation_pv)
                const double A = m.areaTri[v];
                double hv = 0.0;
#pragma unroll
                for (int k = 0; k < 3; ++k) hv = hv + m.kite[k * m.strideV + v] * h[m.cov[k * m.strideV + v]];
                hv = hv / A;
                const double q = (circ / A + m.fV[v]) / hv;
                dd_add(gam, A * hv * q);
            } else {
                dd_add(gam, circ + m.areaTri[v] * m.fV[v]);
            }
        }
    } else {
#pragma unroll 4
        for (int e = tid; e < m.eb.end; e += T) {
            if (!m.eOwn[e]) continue;
            const int2 c = m.coe[e];
            const double he = 0.5 * (h[c.x] + h[c.y]);
            const double dte = e >= m.eb.f ? sc.c3f : sc.c3;
            const double nu = (fabs(u[e]) + sqrt(sc.g * he)) * dte / m.dc[e];
            numax = fmax(numax, nu);
        }
    }
    const DiagRec r = diag_block_reduce(DiagRec{mass, gam, hmin, numax});
    if (threadIdx.x == 0) {
        double *o = part + blockIdx.x * 6;
        o[0] = r.mass.hi, o[1] = r.mass.lo, o[2] = r.gam.hi, o[3] = r.gam.lo, o[4] = r.hmin, o[5] = r.numax;
    }
}

// Pass 2 (one block): thread t merges the partials of blocks t, t + TPB, ... in order, then a fixed
// tree over the threads.
__global__ void __launch_bounds__(TPB) k_diag_final(const double *__restrict__ part, int nb, double *__restrict__ out) {
    DD mass{0.0, 0.0}, gam{0.0, 0.0};
    double hmin = (double)INFINITY, numax = 0.0;
    for (int b = threadIdx.x; b < nb; b += TPB) {
        mass = dd_merge(mass, DD{part[b * 6 + 0], part[b * 6 + 1]});
        gam = dd_merge(gam, DD{part[b * 6 + 2], part[b * 6 + 3]});
        hmin = fmin(hmin, part[b * 6 + 4]);
        numax = fmax(numax, part[b * 6 + 5]);
    }
    // raw double-double parts: ranks are combined on the host in rank order
    const DiagRec r = diag_block_reduce(DiagRec{mass, gam, hmin, numax});
    if (threadIdx.x == 0) {
        out[0] = r.mass.hi, out[1] = r.mass.lo, out[2] = r.gam.hi, out[3] = r.gam.lo, out[4] = r.hmin, out[5] = r.numax;
    }
}

// ---------------------------------------------------------------- launchers
// G = row stride of ec = unrolled slot bound (6, 8 or 16 >= maxEdges).
#define FBLTS_DISPATCH_G(ecS, ...) \
    do {                           \
        if ((ecS) == 6) {          \
            constexpr int G = 6;   \
            __VA_ARGS__;           \
        } else if ((ecS) == 8) {   \
            constexpr int G = 8;   \
            __VA_ARGS__;           \
        } else {                   \
            constexpr int G = 16;  \
            __VA_ARGS__;           \
        }                          \
    } while (0)

// strides of one shared tile buffer (elements, 16-byte multiples) and the dynamic smem bytes
static void tile_strides(int hmax, int emax, int &CS2, int &ES2) {
    CS2 = (HALO0 + hmax + 3 + 1) & ~1;     // + alignment offsets and the ghost copy's slack, even
    ES2 = (emax + FGAP + 8 + 3) & ~3;       // + gap and slack; multiple of 4 (the uint32 pair array)
}
int stage_tiled_smem_bytes_host(int stage, int hmax, int emax, int nrec) {
    const int nca = stage == 4 ? 4 : (stage > 1 ? 3 : 1), nea = stage > 1 ? 4 : 2;
    int CS2, ES2;
    tile_strides(hmax, emax, CS2, ES2);
    (void)nrec;                                  // records live in a fixed 4-slot ring
    return 8 * (((NBUF + 1) & ~1) + NBUF * (nca * CS2 + nea * ES2 + ES2 / 2 + 2)) + 4 * TREC * 4;
}

#ifndef FBLTS_SUB_NTHR
#define FBLTS_SUB_NTHR 512
#endif
template <int G, bool VEL>
__global__ void __launch_bounds__(FBLTS_SUB_NTHR, 1) k_fine_sub(DevMesh m, int CS, int ES, int BUF, SubArgs a, DevError *err);

int stage_tiled_configure(const DevMesh &m) {
    cudaError_t e = cudaSuccess;
    auto set = [&](const void *f) {      // process-wide attributes: the limit, not one context's need
        if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE_SMEM_MAX);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    };
    FBLTS_DISPATCH_G(m.ecS, {
        set((const void *)k_stage_tiled<G, 1>);
        set((const void *)k_stage_tiled<G, 2>);
        set((const void *)k_stage_tiled<G, 3>);
        set((const void *)k_stage_tiled<G, 4>);
        set((const void *)k_fine_sub<G, false>);
        set((const void *)k_fine_sub<G, true>);
    });
    return (int)e;
}

void launch_stage_tiled(const DevMesh &m, int stage, int tile0, int tile1, int hmax, int emax, int nsm,
                        const StageArgs &a, DevError *err, cudaStream_t s) {
    if (tile1 <= tile0) return;
    int CS, ES;
    tile_strides(hmax, emax, CS, ES);
    FBLTS_DISPATCH_G(m.ecS, {
        const void *f = stage == 1   ? (const void *)k_stage_tiled<G, 1>
                        : stage == 2 ? (const void *)k_stage_tiled<G, 2>
                        : stage == 3 ? (const void *)k_stage_tiled<G, 3>
                                     : (const void *)k_stage_tiled<G, 4>;
        // grid = resident CTAs; each stages the records of its ceil(tiles / grid) tiles in shared memory,
        // which can lower the residency: settle both in at most three rounds
        int per = 1, grid = 1, smem = stage_tiled_smem_bytes_host(stage, hmax, emax, 0);
        for (int it = 0; it < 3; ++it) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, f, NTHR, smem);
            grid = std::max(1, std::min(tile1 - tile0, nsm * std::max(1, per)));
            const int want = stage_tiled_smem_bytes_host(stage, hmax, emax, (tile1 - tile0 + grid - 1) / grid);
            if (want == smem) break;
            smem = want;
        }
        {   // the launch must hold the records of ceil(tiles / grid) tiles per CTA
            const int need = stage_tiled_smem_bytes_host(stage, hmax, emax, (tile1 - tile0 + grid - 1) / grid);
            if (need > smem) smem = need;
        }
        static const bool verbose = std::getenv("FBLTS_VERBOSE") != nullptr;
        if (verbose)
            std::fprintf(stderr, "[fblts] stage_tiled s%d tiles [%d,%d) hmax %d emax %d smem %d B, %d CTA/SM, grid %d\n",
                         stage, tile0, tile1, hmax, emax, smem, per, grid);
        if (stage == 1) k_stage_tiled<G, 1><<<grid, NTHR, smem, s>>>(m, tile0, tile1, CS, ES, a, err);
        else if (stage == 2) k_stage_tiled<G, 2><<<grid, NTHR, smem, s>>>(m, tile0, tile1, CS, ES, a, err);
        else if (stage == 3) k_stage_tiled<G, 3><<<grid, NTHR, smem, s>>>(m, tile0, tile1, CS, ES, a, err);
        else k_stage_tiled<G, 4><<<grid, NTHR, smem, s>>>(m, tile0, tile1, CS, ES, a, err);
    });
}

// ====================================================================== fused fine subcycle
// A subcycle tile (fblts_internal.h SubTileMesh, a tile of F\F^5) goes through a whole fine
// subcycle of subeqn fine_fbrk32 inside one CTA: [velocity stage 3 of subcycle k-1 on
// the edges of rings 0-2 (VEL)], stage 1 on rings 0-2, stage 2 on rings 0-1, stage 3 on the tile,
// every stage value kept in shared memory; the rings are recomputed redundantly by the neighbouring
// tiles (same operands, same order: the same bits).  Per edge and stage the flux term
// T_e = l_e ((0.5 (H_c0 + H_c1)) u_bar_e) is computed once, then summed per cell in slot order, which
// is the staged kernels' (and the oracle's) arithmetic.  Every cell of a ring <= 3 is fine, so no
// region views are needed.
// Persistent CTAs (one per SM, SNT threads) walk the tiles with two shared buffers: while tile i is
// computed, tile i+1's contiguous ranges arrive by 1-D bulk copies (mbarrier) and its ring cells and
// foreign edges by cp.async gathers whose indices were fetched into registers before the compute.
constexpr int SNT = FBLTS_SUB_NTHR;
constexpr int SHPT = 1, SFPT = 3;          // ring-cell / foreign-edge indices prefetched per thread

static void sub_strides(int hmax, int emax, int rmax, int &CS, int &ES, int &RS, int &BUF) {
    CS = (HALO0 + hmax + 1 + 1) & ~1;
    ES = (emax + FGAP + 8 + 3) & ~3;
    RS = ((rmax + 7) / 8) * 2;             // doubles holding rmax uint16 (16-byte multiple)
    BUF = 5 * CS + 5 * ES + ES / 2 + RS;
}
int sub_smem_bytes_host(int hmax, int emax, int rmax) {
    int CS, ES, RS, BUF;
    sub_strides(hmax, emax, rmax, CS, ES, RS, BUF);
    return 8 * (2 + 2 * BUF);
}

struct SubRec {
    int c0, c1, h0, n1, n2, n3, eo0, eo1, f0, nF0, nF1, nF2, l0, s0, flags;
    __device__ __forceinline__ int nH() const { return n1 + n2 + n3; }
    __device__ __forceinline__ int nF() const { return nF0 + nF1 + nF2; }
};
__device__ __forceinline__ SubRec load_subrec(const SubTileMesh &t, int tile) {
    const int *p = t.info + (size_t)tile * FTINFO;
    return SubRec{p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7], p[8], p[9], p[10], p[11], p[12], p[13], p[14]};
}
struct SubBuf {                              // views of one buffer for tile r (local index 0 = first own cell / edge)
    double *hk, *hA, *hB, *zb, *A, *u, *S, *l, *d, *T;
    uint32_t *ecl;
    uint16_t *row;
    __device__ __forceinline__ SubBuf(double *B, int CS, int ES, const SubRec &r) {
        const int oc = r.c0 & 1, oe = r.eo0 & 1;
        hk = B + oc, hA = B + CS + oc, hB = B + 2 * CS + oc, zb = B + 3 * CS + oc, A = B + 4 * CS + oc;
        double *E = B + 5 * CS;
        u = E + oe, S = E + ES + oe, l = E + 2 * ES + oe, d = E + 3 * ES + oe, T = E + 4 * ES + oe;
        ecl = reinterpret_cast<uint32_t *>(E + 5 * ES) + (r.l0 & 3);
        row = reinterpret_cast<uint16_t *>(E + 5 * ES + ES / 2);
    }
};

template <bool VEL>
__device__ __forceinline__ void sub_issue_bulk(const DevMesh &m, const SubArgs &a, const SubRec &r, double *B, int CS,
                                               int ES, uint64_t *bar) {
    const int nLE = r.eo1 - r.eo0 + r.nF();
    const int ca = r.c0 & ~1, cb = (r.c1 + 1) & ~1, ea = r.eo0 & ~1, eb = (r.eo1 + 1) & ~1;
    const int la = r.l0 & ~3, lb = (r.l0 + nLE + 3) & ~3;
    const int nR2 = r.c1 - r.c0 + r.n1 + r.n2;
    const unsigned cbytes = 8u * (cb - ca), ebytes = 8u * (eb - ea), lbytes = 4u * (lb - la);
    const unsigned rbytes = 16u * ((m.maxE * nR2 + 7) / 8);   // rows are padded to 8 entries per tile
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    mbar_expect_tx(bar, (VEL ? 5u : 3u) * cbytes + (ebytes ? 4u * ebytes : 0u) + lbytes + rbytes);
    bulk_g2s(B, a.hk + ca, cbytes, bar);
    if (VEL) {
        bulk_g2s(B + CS, a.hm + ca, cbytes, bar);
        bulk_g2s(B + 2 * CS, a.h2 + ca, cbytes, bar);
    }
    bulk_g2s(B + 3 * CS, m.zb + ca, cbytes, bar);
    bulk_g2s(B + 4 * CS, m.areaCell + ca, cbytes, bar);
    double *E = B + 5 * CS;
    if (ebytes) {
        bulk_g2s(E, a.ubase + ea, ebytes, bar);
        bulk_g2s(E + ES, a.S + ea, ebytes, bar);
        bulk_g2s(E + 2 * ES, m.dv + ea, ebytes, bar);
        bulk_g2s(E + 3 * ES, m.dc + ea, ebytes, bar);
    }
    bulk_g2s(E + 5 * ES, m.st.ecl + la, lbytes, bar);
    bulk_g2s(E + 5 * ES + ES / 2, m.st.row + r.s0, rbytes, bar);
}

__device__ __forceinline__ void sub_load_idx(const SubTileMesh &t, const SubRec &r, int tid, int (&hx)[SHPT],
                                             int (&fx)[SFPT]) {
#pragma unroll
    for (int k = 0; k < SHPT; ++k) {
        const int q = k * SNT + tid;
        hx[k] = q < r.nH() ? t.halo[r.h0 + q] : 0;
    }
#pragma unroll
    for (int k = 0; k < SFPT; ++k) {
        const int q = k * SNT + tid;
        fx[k] = q < r.nF() ? t.fedge[r.f0 + q] : 0;
    }
}

template <bool VEL>
__device__ __forceinline__ void sub_issue_gather(const DevMesh &m, const SubArgs &a, const SubRec &r, const SubBuf &b,
                                                 int tid, const int (&hx)[SHPT], const int (&fx)[SFPT]) {
    const int nH = r.nH(), nF = r.nF(), n12 = r.n1 + r.n2, n01 = r.nF0 + r.nF1, nOE = r.eo1 - r.eo0;
    // ring cells: h^{n,k} on R1-R3; z_b on R1-R3 (VEL) or R1-R2; A on R1-R2; h^{n,k-1}, h2 on R1-R3 (VEL)
    auto cell = [&](int q, int x) {
        cp_async8(b.hk + HALO0 + q, a.hk + x);
        if (VEL) {
            cp_async8(b.hA + HALO0 + q, a.hm + x);
            cp_async8(b.hB + HALO0 + q, a.h2 + x);
        }
        if (VEL || q < n12) cp_async8(b.zb + HALO0 + q, m.zb + x);
        if (q < n12) cp_async8(b.A + HALO0 + q, m.areaCell + x);
    };
    // foreign edges: u, l on all; S, d where a velocity is formed (all with VEL, rings 0-1 without)
    auto edge = [&](int p, int e) {
        const int q = nOE + FGAP + p;
        cp_async8(b.u + q, a.ubase + e);
        cp_async8(b.l + q, m.dv + e);
        if (VEL || p < n01) {
            cp_async8(b.S + q, a.S + e);
            cp_async8(b.d + q, m.dc + e);
        }
    };
#pragma unroll
    for (int k = 0; k < SHPT; ++k)
        if (k * SNT + tid < nH) cell(k * SNT + tid, hx[k]);
    for (int q = SHPT * SNT + tid; q < nH; q += SNT) cell(q, m.st.halo[r.h0 + q]);
#pragma unroll
    for (int k = 0; k < SFPT; ++k)
        if (k * SNT + tid < nF) edge(k * SNT + tid, fx[k]);
    for (int p = SFPT * SNT + tid; p < nF; p += SNT) edge(p, m.st.fedge[r.f0 + p]);
}

template <int G, bool VEL>
__global__ void __launch_bounds__(SNT, 1) k_fine_sub(DevMesh m, int CS, int ES, int BUF, SubArgs a, DevError *err) {
    extern __shared__ __align__(16) double smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);   // 2 mbarriers
    double *buf0 = smem + 2;
    const SubTileMesh &t = m.st;
    const int tid = threadIdx.x, G0 = gridDim.x, nT = t.nTiles;
    int tile = blockIdx.x;
    if (tile >= nT) return;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    // the ring-cell / foreign-edge indices run one tile ahead of the copies: tile i+1's gathers are
    // issued as soon as tile i is staged (indices already in registers) and tile i+2's indices load
    // during tile i's compute
    int hx[SHPT], fx[SFPT];
    {
        const SubRec r0 = load_subrec(t, tile);
        if (tid == 0) sub_issue_bulk<VEL>(m, a, r0, buf0, CS, ES, &bar[0]);
        sub_load_idx(t, r0, tid, hx, fx);
        sub_issue_gather<VEL>(m, a, r0, SubBuf(buf0, CS, ES, r0), tid, hx, fx);
        cp_async_commit();
        if (tile + G0 < nT) sub_load_idx(t, load_subrec(t, tile + G0), tid, hx, fx);
    }
    unsigned phase = 0u;
    int buf = 0;
    for (; tile < nT; tile += G0, buf ^= 1) {
        const SubRec r = load_subrec(t, tile);
        const bool more = tile + G0 < nT;
        SubRec nx{};
        if (more) nx = load_subrec(t, tile + G0);
        mbar_wait(&bar[buf], (phase >> buf) & 1u);
        phase ^= 1u << buf;
        cp_async_wait_pending<0>();
        __syncthreads();                                  // tile r staged; the other buffer is free
        double *Bn = buf0 + (buf ^ 1) * BUF;
        if (more) {
            if (tid == 0) sub_issue_bulk<VEL>(m, a, nx, Bn, CS, ES, &bar[buf ^ 1]);
            sub_issue_gather<VEL>(m, a, nx, SubBuf(Bn, CS, ES, nx), tid, hx, fx);
            if (tile + 2 * G0 < nT) sub_load_idx(t, load_subrec(t, tile + 2 * G0), tid, hx, fx);
        }
        cp_async_commit();
        const SubBuf b(buf0 + buf * BUF, CS, ES, r);
        const int nOwn = r.c1 - r.c0, nOE = r.eo1 - r.eo0;
        const int nLE0 = nOE + r.nF0, nLE1 = nLE0 + r.nF1, nLE2 = nLE1 + r.nF2;
        const int nR1 = nOwn + r.n1, nR2 = nR1 + r.n2;
        // ---- edges of rings 0-2: u^{n,k} (VEL: velocity stage 3 of subcycle k-1) and the stage-1 flux
        for (int p = tid; p < nLE2; p += SNT) {
            const uint32_t pr = b.ecl[p];
            const int q = p < nOE ? p : p + FGAP;
            const int x0 = pr & 0xFFFF, x1 = pr >> 16;
            const double H0 = b.hk[x0], H1 = b.hk[x1];
            double ue = b.u[q];
            if (VEL) {
                const double HS0 = a.b3 * H0 + a.om2b3 * b.hB[x0] + a.b3 * b.hA[x0];
                const double HS1 = a.b3 * H1 + a.om2b3 * b.hB[x1] + a.b3 * b.hA[x1];
                const double phi = phi_fast(a.g, HS0, b.zb[x0], HS1, b.zb[x1], b.d[q]);
                ue = ue + a.c3f * (phi + b.S[q]);
                if (p < nOE) a.unew[r.eo0 + p] = ue;
                b.u[q] = ue;
            }
            const double Fe = (0.5 * (H0 + H1)) * ue;
            b.T[q] = b.l[q] * Fe;
        }
        __syncthreads();
        // cell-phase helper: -(sum of the signed flux terms of row rr in slot order) / A
        auto psi_row = [&](int rr, int x) {
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < G; ++j) {
                if (j < m.maxE) {
                    const uint16_t sl = b.row[j * nR2 + rr];
                    if (sl != TILE_SENT) {
                        const double tt = b.T[sl & 0x7FFF];
                        acc = acc + ((sl >> 15) ? -tt : tt);
                    }
                }
            }
            return -acc / b.A[x];
        };
        // ---- stage 1 on rows 0..nR2 (rings 0-2) -> hA
        for (int rr = tid; rr < nR2; rr += SNT) {
            const int x = rr < nOwn ? rr : HALO0 + rr - nOwn;
            const double v = b.hk[x] + a.c1f * psi_row(rr, x);
            b.hA[x] = v;
            if (rr < nOwn) {
                if (r.flags & 1) a.h1out[r.c0 + rr] = v;
                if (!(v > 0.0)) report(err, K_FINE_S1, a.k, r.c0 + rr, v);
            }
        }
        __syncthreads();
        // ---- stage-2 flux on the edges of rings 0-1: u_bar = u^{n,k} + dt/(3M) (Phi^fast(h*) + S)
        for (int p = tid; p < nLE1; p += SNT) {
            const uint32_t pr = b.ecl[p];
            const int q = p < nOE ? p : p + FGAP;
            const int x0 = pr & 0xFFFF, x1 = pr >> 16;
            const double H0 = b.hA[x0], H1 = b.hA[x1];
            const double HS0 = a.b1 * H0 + a.omb1 * b.hk[x0];
            const double HS1 = a.b1 * H1 + a.omb1 * b.hk[x1];
            const double phi = phi_fast(a.g, HS0, b.zb[x0], HS1, b.zb[x1], b.d[q]);
            const double ue = b.u[q] + a.c1f * (phi + b.S[q]);
            const double Fe = (0.5 * (H0 + H1)) * ue;
            b.T[q] = b.l[q] * Fe;
        }
        __syncthreads();
        // ---- stage 2 on rows 0..nR1 (rings 0-1) -> hB
        for (int rr = tid; rr < nR1; rr += SNT) {
            const int x = rr < nOwn ? rr : HALO0 + rr - nOwn;
            const double v = b.hk[x] + a.c2f * psi_row(rr, x);
            b.hB[x] = v;
            if (rr < nOwn) {
                a.h2out[r.c0 + rr] = v;
                if (!(v > 0.0)) report(err, K_FINE_S2, a.k, r.c0 + rr, v);
            }
        }
        __syncthreads();
        // ---- stage-3 flux on the tile's edges: u_bar = u^{n,k} + dt/(2M) (Phi^fast(h**) + S)
        for (int p = tid; p < nLE0; p += SNT) {
            const uint32_t pr = b.ecl[p];
            const int q = p < nOE ? p : p + FGAP;
            const int x0 = pr & 0xFFFF, x1 = pr >> 16;
            const double H0 = b.hB[x0], H1 = b.hB[x1];
            const double HS0 = a.b2 * H0 + a.omb2 * b.hk[x0];
            const double HS1 = a.b2 * H1 + a.omb2 * b.hk[x1];
            const double phi = phi_fast(a.g, HS0, b.zb[x0], HS1, b.zb[x1], b.d[q]);
            const double ue = b.u[q] + a.c2f * (phi + b.S[q]);
            const double Fe = (0.5 * (H0 + H1)) * ue;
            b.T[q] = b.l[q] * Fe;
        }
        __syncthreads();
        // ---- stage 3 on the tile -> h^{n,k+1}
        for (int rr = tid; rr < nOwn; rr += SNT) {
            const double v = b.hk[rr] + a.c3f * psi_row(rr, rr);
            a.out[r.c0 + rr] = v;
            if (!(v > 0.0)) report(err, K_FINE_S3, a.k, r.c0 + rr, v);
        }
    }
}

void launch_fine_sub(const DevMesh &m, bool vel, int nsm, const SubArgs &a, DevError *err, cudaStream_t s) {
    if (m.st.nTiles <= 0) return;
    int CS, ES, RS, BUF;
    sub_strides(m.st.hmax, m.st.emax, m.st.rmax, CS, ES, RS, BUF);
    const int smem = sub_smem_bytes_host(m.st.hmax, m.st.emax, m.st.rmax);
    const int grid = std::max(1, std::min(m.st.nTiles, nsm));
    FBLTS_DISPATCH_G(m.ecS, {
        if (vel) k_fine_sub<G, true><<<grid, SNT, smem, s>>>(m, CS, ES, BUF, a, err);
        else k_fine_sub<G, false><<<grid, SNT, smem, s>>>(m, CS, ES, BUF, a, err);
    });
}

// Views of the state at t^{n,k} for the slow-term refresh (reading DESIGN.md 3):
// cells: F -> h^{n,k}, IF-1 / IF-2 -> (k/M) h~^{n+1} + (1 - k/M) h^n (eq. pred_old), others h^n;
// edges: F_E -> u^{n,k}, IF-1_E -> (k/M) u~^{n+1} + (1 - k/M) u^n with u~^{n+1} recomputed as the
// coarse velocity stage 3 does, others u^n (fillers outside the stencil of F_E).
__global__ void __launch_bounds__(TPB) k_refresh_views(DevMesh m, FineArrays a, const double *__restrict__ uN,
                                                       const double *__restrict__ uk, const double *__restrict__ S,
                                                       double *__restrict__ hv, double *__restrict__ uv,
                                                       StepConst sc, PredConst p, unsigned nbC) {
    if (blockIdx.x < nbC) {
        const int i = blockIdx.x * TPB + threadIdx.x;
        if (i >= m.nOwnC) return;
        const int cl = ccls(m, i);
        const bool ifc = cl == 1 || (cl == 0 && i >= (i < m.nB ? m.cb.if2 : m.cbI.if2));
        hv[i] = cl == 2 ? a.hk[i] : (ifc ? pred_level(p, a, i) : a.hN[i]);
    } else {
        const int e = (blockIdx.x - nbC) * TPB + threadIdx.x;
        if (e >= m.nOwnE) return;
        const int ec = ecls(m.eb, e);
        if (ec == 3) {
            uv[e] = uk[e];
        } else if (ec == 2) {
            const int2 c = m.coe[e];
            const double phi3 = phi_fast(sc.g, hs3c(sc, a.h3, a.h2, a.hN, c.x), m.zb[c.x], hs3c(sc, a.h3, a.h2, a.hN, c.y),
                                         m.zb[c.y], m.dc[e]);
            const double u3 = uN[e] + sc.c3 * (phi3 + S[e]);
            uv[e] = p.a * u3 + p.oma * uN[e];
        } else {
            uv[e] = uN[e];
        }
    }
}


void launch_slow_pre_range(const DevMesh &m, const DevState &st, const double *h, const double *u, int v0, int c0,
                           int e0, cudaStream_t s, int v0vf) {
    // F_e in the vertex role: full sweeps, or a range sweep whose caller passes v0vf = the first vertex
    // that owns an edge >= e0 (<= v0; the extra vertices' q is recomputed, not used)
    const bool vf = m.vF && ((v0 == 0 && e0 == 0) || v0vf >= 0);
    if (vf && v0vf >= 0) v0 = std::min(v0, v0vf);
    const unsigned nbV = nblocks(std::max(0, m.nV - v0)), nbC = nblocks(std::max(0, m.nC - c0)),
                   nbE = vf ? 0u : nblocks(std::max(0, m.nE - e0));
    if (nbV + nbC + nbE == 0) return;
    FBLTS_DISPATCH_G(m.ecS, {
        if (vf) k_slow_pre<G, true><<<nbV + nbC + nbE, TPB, 0, s>>>(m, h, u, st.q, st.K, st.F, nbV, nbC, v0, c0, e0);
        else k_slow_pre<G, false><<<nbV + nbC + nbE, TPB, 0, s>>>(m, h, u, st.q, st.K, st.F, nbV, nbC, v0, c0, e0);
    });
}
void launch_slow_pre(const DevMesh &m, const DevState &st, const double *h, const double *u, cudaStream_t s) {
    launch_slow_pre_range(m, st, h, u, 0, 0, 0, s);
}
// q_hat_e = 0.5 (q_v0 + q_v1) on every local edge (energy-conserving PV flux only)
__global__ void __launch_bounds__(TPB) k_qhat(DevMesh m, const double *__restrict__ q, double *__restrict__ qe) {
    const int e = blockIdx.x * TPB + threadIdx.x;
    if (e >= m.nE) return;
    const int2 v = m.voe[e];
    qe[e] = 0.5 * (q[v.x] + q[v.y]);
}

void launch_slow_edge_range(const DevMesh &m, const DevState &st, const double *h, const double *u, double *out,
                            int e0, int e1, const StepConst &sc, cudaStream_t s, double *pvout, const VelFuse *vel) {
    if (e1 <= e0) return;
    const unsigned nb = nblocks(e1 - e0);
    if (sc.pve) k_qhat<<<nblocks(m.nE), TPB, 0, s>>>(m, st.q, st.qe);
    const VelFuse vf = vel ? *vel : VelFuse();
#define FBLTS_SLOW_EDGE4(ME2, HU, PV, VL)                                                                          \
    k_slow_edge<ME2, HU, PV, VL><<<nb, TPB, 0, s>>>(m, h, st.q, st.K, st.F, u, st.qe, out, pvout, sc.rho0, sc.cd,  \
                                                    sc.cw, e0, e1, vf, sc.g)
#define FBLTS_SLOW_EDGE3(ME2, HU, PV)                                                                              \
    do {                                                                                                         \
        if (vel) FBLTS_SLOW_EDGE4(ME2, HU, PV, true);                                                            \
        else FBLTS_SLOW_EDGE4(ME2, HU, PV, false);                                                               \
    } while (0)
#define FBLTS_SLOW_EDGE(ME2)                                                                                     \
    do {                                                                                                         \
        if (sc.pve) {                                                                                            \
            if (sc.hur) FBLTS_SLOW_EDGE3(ME2, true, true);                                                       \
            else FBLTS_SLOW_EDGE3(ME2, false, true);                                                             \
        } else {                                                                                                 \
            if (sc.hur) FBLTS_SLOW_EDGE3(ME2, true, false);                                                      \
            else FBLTS_SLOW_EDGE3(ME2, false, false);                                                            \
        }                                                                                                        \
    } while (0)
    if (m.maxE2 <= 10)
        FBLTS_SLOW_EDGE(10);
    else if (m.maxE2 <= 14)
        FBLTS_SLOW_EDGE(14);
    else
        FBLTS_SLOW_EDGE(30);
#undef FBLTS_SLOW_EDGE
#undef FBLTS_SLOW_EDGE3
#undef FBLTS_SLOW_EDGE4
}
void launch_slow_edge(const DevMesh &m, const DevState &st, const double *h, const double *u, const StepConst &sc,
                      cudaStream_t s) {
    launch_slow_edge_range(m, st, h, u, st.S, 0, m.nOwnE, sc, s);
}
void launch_coarse_s1(const DevMesh &m, const DevState &st, const double *hN, const double *uN,
                      const StepConst &sc, cudaStream_t s, const Bounds &b) {
    const int beg = b.begin, end = b.fl[5];
    if (end > beg)
        FBLTS_DISPATCH_G(m.ecS, k_coarse_stage<G, 1><<<nblocks(end - beg), TPB, 0, s>>>(m, hN, hN, uN, st.S, st.h1,
                                                                                         sc, beg, end, st.err));
}
void launch_coarse_s2(const DevMesh &m, const DevState &st, const double *hN, const double *uN,
                      const StepConst &sc, cudaStream_t s, const Bounds &b) {
    const int beg = b.begin, end = b.fl[3];
    if (end > beg)
        FBLTS_DISPATCH_G(m.ecS, k_coarse_stage<G, 2><<<nblocks(end - beg), TPB, 0, s>>>(m, hN, st.h1, uN, st.S, st.h2,
                                                                                         sc, beg, end, st.err));
}
void launch_coarse_s3(const DevMesh &m, const DevState &st, const double *hN, const double *uN, double *hNew,
                      const StepConst &sc, cudaStream_t s, const Bounds &b) {
    const int beg = b.begin, end = b.fl[1];
    if (end > beg)
        FBLTS_DISPATCH_G(m.ecS, k_coarse_stage<G, 3><<<nblocks(end - beg), TPB, 0, s>>>(m, hN, st.h2, uN, st.S, hNew,
                                                                                         sc, beg, end, st.err));
}
void launch_coarse_vel(const DevMesh &m, const DevState &st, const double *hN, const double *uN,
                       const double *hNew, double *uNew, const StepConst &sc, cudaStream_t s, bool if_edges) {
    const int end = m.eb.if2, fend = if_edges ? m.eb.f : end;
    if (fend > 0)
        k_coarse_vel<<<nblocks(fend), TPB, 0, s>>>(m, hN, st.h2, hNew, uN, st.S, uNew, sc, end, st.uIF2, st.uIF3,
                                                   m.eb.if1, fend);
}
static FineArrays fine_arrays(const DevState &st, const double *hN, const double *hNew, const double *hk) {
    FineArrays a;
    a.Sf = st.Sf;
    a.hN = hN;
    a.h1 = st.h1;
    a.h2 = st.h2;
    a.h3 = hNew;
    a.hk = hk;
    a.uIF2 = st.uIF2;
    a.uIF3 = st.uIF3;
    return a;
}

void launch_refresh_views(const DevMesh &m, const DevState &st, const double *hN, const double *hNew,
                          const double *hk, const double *uN, const double *uk, const StepConst &sc,
                          const PredConst &pc, cudaStream_t s) {
    const FineArrays a = fine_arrays(st, hN, hNew, hk);
    const unsigned nbC = nblocks(m.nOwnC), nbE = nblocks(m.nOwnE);
    k_refresh_views<<<nbC + nbE, TPB, 0, s>>>(m, a, uN, uk, st.S, st.hv, st.uv, sc, pc, nbC);
}
// Fine kernels: BAND instance over [b0, b1) (needs the region views), DEEP over [b1, end).
void launch_fine_s1(const DevMesh &m, const DevState &st, const double *hN, const double *hNew, const double *hk,
                    const double *uk, const StepConst &sc, const PredConst &pc, int k, cudaStream_t s,
                    const Bounds &b, bool deep) {
    const FineArrays a = fine_arrays(st, hN, hNew, hk);
    const int b0 = b.f, b1 = b.fl[1], end = b.end;
    FBLTS_DISPATCH_G(m.ecS, {
        if (b1 > b0) k_fine_s1<G, true><<<nblocks(b1 - b0), TPB, 0, s>>>(m, a, uk, st.h1, sc, pc, k, b0, b1, st.err);
        if (deep && end > b1) k_fine_s1<G, false><<<nblocks(end - b1), TPB, 0, s>>>(m, a, uk, st.h1, sc, pc, k, b1, end, st.err);
    });
}
void launch_fine_s2(const DevMesh &m, const DevState &st, const double *hN, const double *hNew, const double *hk,
                    const double *uk, const StepConst &sc, const PredConst &pc, int k, cudaStream_t s,
                    const Bounds &b, bool deep) {
    const FineArrays a = fine_arrays(st, hN, hNew, hk);
    const int b0 = b.f, b1 = b.fl[1], end = b.end;
    FBLTS_DISPATCH_G(m.ecS, {
        if (b1 > b0)
            k_fine_s2<G, true><<<nblocks(b1 - b0), TPB, 0, s>>>(m, a, uk, st.S, st.h2, sc, pc, k, b0, b1, st.err);
        if (deep && end > b1)
            k_fine_s2<G, false><<<nblocks(end - b1), TPB, 0, s>>>(m, a, uk, st.S, st.h2, sc, pc, k, b1, end, st.err);
    });
}
void launch_fine_s3(const DevMesh &m, const DevState &st, const double *hN, const double *uN, const double *hNew,
                    const double *hk, const double *uk, double *hnext, const StepConst &sc, const PredConst &pc,
                    int k, cudaStream_t s, const Bounds &b, bool deep) {
    const FineArrays a = fine_arrays(st, hN, hNew, hk);
    const int b0 = b.if2, b1 = b.fl[1], end = b.end;
    FBLTS_DISPATCH_G(m.ecS, {
        if (b1 > b0)
            k_fine_s3<G, true><<<nblocks(b1 - b0), TPB, 0, s>>>(m, a, uN, uk, st.S, hnext, st.accH, sc, pc, k, b0,
                                                                 b.f, b1, st.err);
        if (deep && end > b1)
            k_fine_s3<G, false><<<nblocks(end - b1), TPB, 0, s>>>(m, a, uN, uk, st.S, hnext, st.accH, sc, pc, k, b1,
                                                                   b1, end, st.err);
    });
}
void launch_fine_vel(const DevMesh &m, const DevState &st, const double *hN, const double *hNew, const double *hk,
                     const double *hnext, const double *uk, double *unext, const StepConst &sc,
                     const PredConst &pc, int k, cudaStream_t s, bool deep) {
    const FineArrays a = fine_arrays(st, hN, hNew, hk);
    const int b0 = m.eb.if2, b1 = m.eb.fl[1], end = m.eb.end;
    if (b1 > b0)
        k_fine_vel<true><<<nblocks(b1 - b0), TPB, 0, s>>>(m, a, hnext, uk, st.S, unext, st.accU, sc, pc, k, b0, b1);
    if (deep && end > b1)
        k_fine_vel<false><<<nblocks(end - b1), TPB, 0, s>>>(m, a, hnext, uk, st.S, unext, st.accU, sc, pc, k, b1, end);
}
void launch_correct(const DevMesh &m, const DevState &st, const double *hN, const double *uN, double *hNew,
                    double *uNew, const StepConst &sc, cudaStream_t s, const Bounds &b, bool edges) {
    const unsigned nbC = nblocks(b.f - b.if2), nbE = edges ? nblocks(m.eb.f - m.eb.if2) : 0u;
    if (nbC + nbE > 0)
        k_correct<<<nbC + nbE, TPB, 0, s>>>(m, hN, uN, st.accH, st.accU, hNew, uNew, sc, b.if2, b.f, nbC, st.err);
}
void launch_permute_in(const int32_t *old, const double *src, double *dst, int n, cudaStream_t s) {
    if (n > 0) k_permute_in<<<nblocks(n), TPB, 0, s>>>(old, src, dst, n);
}
void launch_validate(const double *v, int n, int positive, int *bad, cudaStream_t s) {
    if (n > 0) k_validate<<<nblocks(n), TPB, 0, s>>>(v, n, positive, bad);
}
void launch_permute_out(const int32_t *old, const double *src, double *dst, int n, cudaStream_t s) {
    if (n > 0) k_permute_out<<<nblocks(n), TPB, 0, s>>>(old, src, dst, n);
}
void launch_pack(const int32_t *idx, const double *a, double *buf, int n, cudaStream_t s) {
    if (n > 0) k_pack<<<nblocks(n), TPB, 0, s>>>(idx, a, buf, n);
}
void launch_unpack(const int32_t *idx, const double *buf, double *a, int n, cudaStream_t s) {
    if (n > 0) k_unpack<<<nblocks(n), TPB, 0, s>>>(idx, buf, a, n);
}
void launch_diagnostics(const DevMesh &m, const double *h, const double *u, const StepConst &sc, double *part,
                        double *out_dev, cudaStream_t s, bool cells_only, bool pv) {
    const int nb = cells_only ? DIAG_RB : DIAG_BLOCKS;     // role 0 (mass, min h) is blocks [0, DIAG_RB)
    k_diag_partial<<<nb, TPB, 0, s>>>(m, h, u, sc, part, pv ? 1 : 0);
    k_diag_final<<<1, TPB, 0, s>>>(part, nb, out_dev);
}

void launch_rk4_stage(const DevMesh &m, const DevState &st, int stage, const double *hN, const double *uN,
                      const double *hs, const double *us, double *hout, double *uout, double cnext, double dt6,
                      double g, cudaStream_t s) {
    const unsigned nbC = nblocks(m.nOwnC), nbE = nblocks(m.nOwnE);
    FBLTS_DISPATCH_G(m.ecS, k_rk4_stage<G><<<nbC + nbE, TPB, 0, s>>>(m, stage, hN, uN, hs, us, st.S, st.hT, st.rkAccU,
                                                                      hout, uout, cnext, dt6, g, nbC, st.err));
}


// ====================================================================== unsplit FB-LTS (N1)
// SURVEY 8(f) N1, P:L468-787 with the full Phi(U, HS) = Phi^fast(HS) + Phi^slow(U, HS) in every velocity
// update (reading Q16).  The stage velocities are stored (they need the slow terms at the stage), so
// every stage is: thickness sweep (stored U) -> FB-averaged thickness / views -> slow sweeps on the
// extent -> velocity sweep.  Same canonical arithmetic as the oracle (oracle/lts.py split=False).

// coarse thickness stage s on cells [0, end): out = hN + c Psi(U, H) and the FB average into hsv
// (s = 1: h* = b1 h1 + (1-b1) hN; 2: h** = b2 h2 + (1-b2) hN; 3: h*** = b3 h3 + (1-2b3) h2 + b3 hN)
template <int G, int STAGE>
__global__ void __launch_bounds__(TPB) k_un_cstage(DevMesh m, const double *__restrict__ hN,
                                                   const double *__restrict__ H, const double *__restrict__ U,
                                                   double *__restrict__ out, double *__restrict__ hsv,
                                                   StepConst sc, int end, DevError *err) {
    const int i = blockIdx.x * TPB + threadIdx.x;
    if (i >= end) return;
    int2 r[G];
    load_row<G>(m, i, r);
    const int n = m.nEoC[i];
    const double Hi = H[i];
    const double hn = hN[i];                          // before the division
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < G; ++j) {
        if (j < n) {
            bool pos;
            const int e = decode(r[j].x, pos);
            acc = acc + psi_term(pos, Hi, H[r[j].y], U[e], m.dv[e]);
        }
    }
    const double c = STAGE == 1 ? sc.c1 : (STAGE == 2 ? sc.c2 : sc.c3);
    const double psi = -acc / m.areaCell[i];
    const double v = hn + c * psi;
    out[i] = v;
    hsv[i] = STAGE == 1 ? sc.b1 * v + sc.omb1 * hn
                        : (STAGE == 2 ? sc.b2 * v + sc.omb2 * hn : sc.b3 * v + sc.om2b3 * Hi + sc.b3 * hn);
    if (!(v > 0.0)) report(err, STAGE == 1 ? K_COARSE_S1 : (STAGE == 2 ? K_COARSE_S2 : K_COARSE_S3), -1, i, v);
}

// velocity sweep on edges [e0, e1): out = base + c (Phi^fast(HS) + S); with acc != nullptr the edges
// [a0, a1) instead accumulate acc[e - a0] += Phi^fast(HS) + S (correction summand, k = 0 starts from 0)
__global__ void __launch_bounds__(TPB) k_un_vel(DevMesh m, const double *__restrict__ HS,
                                                const double *__restrict__ S, const double *__restrict__ base,
                                                double *__restrict__ out, double c, double g, int e0, int e1,
                                                double *__restrict__ acc, int a0, int a1, int first) {
    const int e = e0 + blockIdx.x * TPB + threadIdx.x;
    if (e >= e1) return;
    const int2 cc = m.coe[e];
    const bool ia = acc && e >= a0 && e < a1;
    const double b0 = ia ? (first ? 0.0 : acc[e - a0]) : base[e], se = S[e];   // loads before the division
    const double phi = phi_fast(g, HS[cc.x], m.zb[cc.x], HS[cc.y], m.zb[cc.y], m.dc[e]);
    if (ia) acc[e - a0] = b0 + (phi + se);
    else out[e] = b0 + c * (phi + se);
}

// fine-phase views of stage s (1..3) at subcycle k: HS view on every owned cell (view1/2/3: fine
// FB average, IF-1 predicted, IF-2/int coarse) and the stage's U view on every owned edge
// (U0 / U1 / U2: F_E fine, IF-1_E predicted from the stored coarse velocities, others coarse)
template <int S>
__global__ void __launch_bounds__(TPB) k_un_views(DevMesh m, FineArrays a, const double *__restrict__ hnext,
                                                  const double *__restrict__ uN, const double *__restrict__ ufine,
                                                  const double *__restrict__ u1c, const double *__restrict__ u2c,
                                                  const double *__restrict__ u3c, double *__restrict__ hsv,
                                                  double *__restrict__ uv, StepConst sc, PredConst p, unsigned nbC,
                                                  int c0, int e0) {
    if (blockIdx.x < nbC) {
        const int i = c0 + blockIdx.x * TPB + threadIdx.x;
        if (i >= m.nOwnC) return;
        double H, HS;
        if (S == 1) view1<true>(m, sc, p, a, i, H, HS);
        else if (S == 2) view2<true>(m, sc, p, a, i, H, HS);
        else HS = view3<true>(m, sc, p, a, hnext, i);
        hsv[i] = HS;
    } else {
        const int e = e0 + (blockIdx.x - nbC) * TPB + threadIdx.x;
        if (e >= m.nOwnE) return;
        const int ec = ecls(m.eb, e);
        double v;
        if (ec == 3) v = ufine[e];
        else if (ec == 2) v = S == 1 ? p.a * u3c[e] + p.oma * uN[e]
                                     : p.a * u3c[e] + p.b * (S == 2 ? u1c[e] : u2c[e]) + p.c * uN[e];
        else v = S == 1 ? uN[e] : (S == 2 ? u1c[e] : u2c[e]);
        uv[e] = v;
    }
}

// fine thickness stage 2 / 3 with stored velocities: cells [begin, end)
//   s = 2: F: hk2 = hk + dt/(2M) Psi(U1 = uk1 on F_E, H1 view)
//   s = 3: F: hkn = hk + dt/M Psi(U2 view, H2 view); IF-1 u IF-2: accH += Psi(U2, H2)
template <int G, int STAGE>
__global__ void __launch_bounds__(TPB) k_un_fstage(DevMesh m, FineArrays a, const double *__restrict__ U,
                                                   double *__restrict__ out, double *__restrict__ accH,
                                                   StepConst sc, PredConst p, int k, int begin, int end,
                                                   DevError *err) {
    const int i = begin + blockIdx.x * TPB + threadIdx.x;
    if (i >= end) return;
    int2 r[G];
    load_row<G>(m, i, r);
    const int n = m.nEoC[i];
    double Hi, HSi;
    if (STAGE == 2) view1<true>(m, sc, p, a, i, Hi, HSi);
    else view2<true>(m, sc, p, a, i, Hi, HSi);
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < G; ++j) {
        if (j < n) {
            bool pos;
            const int e = decode(r[j].x, pos);
            double Hn, HSn;
            if (STAGE == 2) view1<true>(m, sc, p, a, r[j].y, Hn, HSn);
            else view2<true>(m, sc, p, a, r[j].y, Hn, HSn);
            acc = acc + psi_term(pos, Hi, Hn, U[e], m.dv[e]);
        }
    }
    const bool fine = i >= m.cb.f;
    const double b0 = fine ? a.hk[i] : (k == 0 ? 0.0 : accH[i]);   // loaded before the division
    const double psi = -acc / m.areaCell[i];
    if (fine) {
        const double v = b0 + (STAGE == 2 ? sc.c2f : sc.c3f) * psi;
        out[i] = v;
        if (!(v > 0.0)) report(err, STAGE == 2 ? K_FINE_S2 : K_FINE_S3, k, i, v);
    } else {
        accH[i] = b0 + psi;
    }
}

void launch_un_cstage(const DevMesh &m, const DevState &st, int stage, const double *hN, const double *H,
                      const double *U, double *out, const StepConst &sc, int end, cudaStream_t s) {
    if (end <= 0) return;
    FBLTS_DISPATCH_G(m.ecS, {
        if (stage == 1) k_un_cstage<G, 1><<<nblocks(end), TPB, 0, s>>>(m, hN, H, U, out, st.hv, sc, end, st.err);
        else if (stage == 2) k_un_cstage<G, 2><<<nblocks(end), TPB, 0, s>>>(m, hN, H, U, out, st.hv, sc, end, st.err);
        else k_un_cstage<G, 3><<<nblocks(end), TPB, 0, s>>>(m, hN, H, U, out, st.hv, sc, end, st.err);
    });
}
void launch_un_vel(const DevMesh &m, const DevState &st, const double *base, double *out, double c, int e0, int e1,
                   double *acc, int a0, int a1, int first, const StepConst &sc, cudaStream_t s) {
    if (e1 > e0)
        k_un_vel<<<nblocks(e1 - e0), TPB, 0, s>>>(m, st.hv, st.Sk, base, out, c, sc.g, e0, e1, acc, a0, a1, first);
}
void launch_un_views(const DevMesh &m, const DevState &st, int stage, const double *hN, const double *hNew,
                     const double *hk, const double *hnext, const double *uN, const double *ufine,
                     const StepConst &sc, const PredConst &pc, cudaStream_t s, int c0, int e0) {
    const FineArrays a = fine_arrays(st, hN, hNew, hk);
    const unsigned nbC = c0 < m.nOwnC ? nblocks(m.nOwnC - c0) : 0u, nbE = e0 < m.nOwnE ? nblocks(m.nOwnE - e0) : 0u;
    if (nbC + nbE == 0) return;
#define FBLTS_UN_VIEWS(S)                                                                                         \
    k_un_views<S><<<nbC + nbE, TPB, 0, s>>>(m, a, hnext, uN, ufine, st.un[0], st.un[1], st.un[2], st.hv, st.uv, sc, \
                                            pc, nbC, c0, e0)
    if (stage == 1) FBLTS_UN_VIEWS(1);
    else if (stage == 2) FBLTS_UN_VIEWS(2);
    else FBLTS_UN_VIEWS(3);
#undef FBLTS_UN_VIEWS
}
void launch_un_fstage(const DevMesh &m, const DevState &st, int stage, const double *hN, const double *hNew,
                      const double *hk, const double *U, double *out, const StepConst &sc, const PredConst &pc,
                      int k, cudaStream_t s) {
    const FineArrays a = fine_arrays(st, hN, hNew, hk);
    const int b0 = stage == 2 ? m.cb.f : m.cb.if2, end = m.cb.end;
    if (end <= b0) return;
    FBLTS_DISPATCH_G(m.ecS, {
        if (stage == 2)
            k_un_fstage<G, 2><<<nblocks(end - b0), TPB, 0, s>>>(m, a, U, out, st.accH, sc, pc, k, b0, end, st.err);
        else
            k_un_fstage<G, 3><<<nblocks(end - b0), TPB, 0, s>>>(m, a, U, out, st.accH, sc, pc, k, b0, end, st.err);
    });
}

// ghost fill (staged stage sweeps): dst[k] = src[idx[k]] (0 for padding slots), k in [k0, k1)
__global__ void k_ghost_fill(const int32_t *__restrict__ idx, const double *__restrict__ src,
                             double *__restrict__ dst, int k0, int k1) {
    const int k = k0 + blockIdx.x * TPB + threadIdx.x;
    if (k >= k1) return;
    const int i = idx[k];
    dst[k] = i >= 0 ? src[i] : 0.0;
}
void launch_ghost_fill(const int32_t *idx, const double *src, double *dst, int k0, int k1, cudaStream_t s) {
    if (k1 > k0) k_ghost_fill<<<nblocks(k1 - k0), TPB, 0, s>>>(idx, src, dst, k0, k1);
}

// ---------------------------------------------------------------- prognostic absolute vorticity (N1)
// Theorem 2, SPEC step_prognostic_vorticity: the PV-flux term of every
// velocity update is integrated per edge exactly as the velocity integrates it (oracle lts.fblts_step
// eta=...): int_E dP = dt PV (coarse stage 3); F_E dP = sum_k dt/M PV^k (ascending k from +0.0);
// IF-1_E u IF-2_E dP = dt/M sum_k PV^k; then eta_v += (sum_j t_{e_j,v} d_{e_j} dP_{e_j}) / A_v.
__global__ void k_vort_int(double *__restrict__ dP, const double *__restrict__ P, double c3, int e1) {
    const int e = blockIdx.x * TPB + threadIdx.x;
    if (e < e1) dP[e] = c3 * P[e];
}
__global__ void k_vort_fine(double *__restrict__ dP, double *__restrict__ accP, const double *__restrict__ P,
                            double c3f, int if2, int f, int end, int first) {
    const int e = if2 + blockIdx.x * TPB + threadIdx.x;
    if (e >= end) return;
    if (e < f) accP[e - if2] = (first ? 0.0 : accP[e - if2]) + P[e];
    else dP[e] = (first ? 0.0 : dP[e]) + c3f * P[e];
}
__global__ void k_vort_close(double *__restrict__ dP, const double *__restrict__ accP, double c3f, int if2, int f) {
    const int e = if2 + blockIdx.x * TPB + threadIdx.x;
    if (e < f) dP[e] = c3f * accP[e - if2];
}
__global__ void k_vort_update(DevMesh m, double *__restrict__ eta, const double *__restrict__ dP) {
    const int v = blockIdx.x * TPB + threadIdx.x;
    if (v >= m.nV) return;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        bool pos;
        const int e = decode(m.eov[k * m.strideV + v], pos);
        const double t = m.dc[e] * dP[e];
        acc = acc + (pos ? t : -t);
    }
    eta[v] = eta[v] + acc / m.areaTri[v];
}
// split mode: the PV flux is frozen with S, so the per-edge integral is formed at the end of the step
// in the oracle's operation order (F_E: ascending k, dP + dt/M PV; IF edges: dt/M (sum_k PV))
__global__ void k_vort_split(double *__restrict__ dP, const double *__restrict__ P, double c3, double c3f, int M,
                             int if2, int f, int end) {
    const int e = blockIdx.x * TPB + threadIdx.x;
    if (e >= end) return;
    const double p = P[e];
    if (e < if2) {
        dP[e] = c3 * p;
    } else if (e < f) {
        double acc = 0.0;
        for (int k = 0; k < M; ++k) acc = acc + p;
        dP[e] = c3f * acc;
    } else {
        double acc = 0.0;
        for (int k = 0; k < M; ++k) acc = acc + c3f * p;
        dP[e] = acc;
    }
}
void launch_vort_split(const DevMesh &m, const DevState &st, const StepConst &sc, cudaStream_t s) {
    if (m.eb.end > 0)
        k_vort_split<<<nblocks(m.eb.end), TPB, 0, s>>>(st.dP, st.Pv, sc.c3, sc.c3f, sc.M, m.eb.if2, m.eb.f, m.eb.end);
}
void launch_vort_int(const DevState &st, double c3, int e1, cudaStream_t s) {
    if (e1 > 0) k_vort_int<<<nblocks(e1), TPB, 0, s>>>(st.dP, st.Pv, c3, e1);
}
void launch_vort_fine(const DevMesh &m, const DevState &st, double c3f, int first, cudaStream_t s) {
    if (m.eb.end > m.eb.if2)
        k_vort_fine<<<nblocks(m.eb.end - m.eb.if2), TPB, 0, s>>>(st.dP, st.accP, st.Pv, c3f, m.eb.if2, m.eb.f, m.eb.end, first);
}
void launch_vort_close(const DevMesh &m, const DevState &st, double c3f, cudaStream_t s) {
    if (m.eb.f > m.eb.if2) k_vort_close<<<nblocks(m.eb.f - m.eb.if2), TPB, 0, s>>>(st.dP, st.accP, c3f, m.eb.if2, m.eb.f);
}
void launch_vort_update(const DevMesh &m, const DevState &st, cudaStream_t s) {
    if (m.nV > 0) k_vort_update<<<nblocks(m.nV), TPB, 0, s>>>(m, st.eta, st.dP);
}
}  // namespace fblts

// Build configuration of this library (fblts_build_info, include/fblts.h): the compile-time
// knobs that change what the kernels do.  A development build (FBLTS_PROBE != 0 skips work,
// FBLTS_CHECK != 0 adds device bounds traps) must never produce a bench number.
#define FBLTS_STR2(x) #x
#define FBLTS_STR(x) FBLTS_STR2(x)
extern "C" const char *fblts_build_info(void) {
    return "probe=" FBLTS_STR(FBLTS_PROBE) " check=" FBLTS_STR(FBLTS_CHECK) " tile=" FBLTS_STR(FBLTS_TILE)
           " tile_minb=" FBLTS_STR(FBLTS_TILE_MINB) " tile_nbuf=" FBLTS_STR(FBLTS_TILE_NBUF)
           " tile_nthr=" FBLTS_STR(FBLTS_TILE_NTHR) " minb=" FBLTS_STR(FBLTS_MINB) " band_minb=" FBLTS_STR(FBLTS_BAND_MINB) 
#if defined(__CUDACC__)
           " fmad=off arch=sm_100a"
#endif
        ;
}
