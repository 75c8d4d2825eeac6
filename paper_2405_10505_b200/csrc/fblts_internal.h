// fblts_internal.h -- device-side data layout of libfblts (not part of the C ABI).
//
// Layout in HBM: every entity family is renumbered
// region-major then by space-filling curve, so each phase extent of FB-LTS is one
// contiguous index range:
//   cells : [ C^int | C^IF-2 | C^IF-1 | F^1 | F^2\F^1 | ... | F^5\F^4 | F\F^5 ]
//   edges : [ int_E | IF-2_E | IF-1_E | F^1_E | ... | F_E\F^5_E ]
//   vertices: SFC order.
// Cell kernels run one thread per cell and fetch the per-cell slot table
// ec[i*G + j] = (edge, neighbour) (row stride G = 6, 8 or 16 >= maxEdges, 16-byte
// aligned rows) with vector loads.  Per-edge tables read by one thread per edge
// over slots (edgesOnEdge, weightsOnEdge) and per-vertex tables are slot-major
// ([slot][stride]).  Edges are sign-encoded: e if the cell is cellsOnEdge[e][0]
// (n_{e,i} = +1), ~e otherwise; edgesOnVertex likewise: e if the vertex is
// verticesOnEdge[e][1] (t_{e,v} = +1).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fblts {

enum KernelKind {
    K_SLOW_PRE = 0, K_SLOW_EDGE, K_COARSE_S1, K_COARSE_S2, K_COARSE_S3, K_COARSE_VEL,
    K_FINE_S1, K_FINE_S2, K_FINE_S3, K_FINE_VEL, K_CORRECT, K_FINE_VS1, K_RK4_STAGE, K_SLOW_REFRESH, K_FINE_SUB,
    K_NUM
};

// Region boundaries of one region-major block: [begin,if2) int, [if2,if1) IF-2,
// [if1,f) IF-1, [f,end) fine; fl[l] = end of F^l (l = 1..5), fl[0] = f.
struct Bounds {
    int32_t begin, if2, if1, f, end;
    int32_t fl[6];
};

// Cell tiles for the staged stage kernels.  The owned cells are cut into
// tiles of at most TILE consecutive cells; tile boundaries include every region block boundary,
// so each stage extent is a whole number of tiles.  A tile's local cells are its own cells
// (local index i - c0) followed by its halo cells (neighbours outside the tile; local index
// HALO0 + position in its sorted halo list).  Its local edges (every edge of its cells) are the
// contiguous run [eo0, eo1) of edges it owns (local index e - eo0) followed by its "foreign"
// edges (sorted list; local index (eo1 - eo0) + FGAP + position).  The gaps keep the slack
// elements of the 16-byte aligned bulk copies of the contiguous ranges clear of the
// individually copied halo / foreign entries.  Per local edge (in list order, no gap),
//   ecl = (local cell of c1) << 16 | (local cell of c0),
// and per cell a slot-major 16-bit slot table  row[j * strideRow + i] = neg << 15 | local edge
// (TILE_SENT for j >= nEdgesOnCell).  info[t * TINFO + k], k = c0, h0, eo0, eo1, f0, l0, g0, ge0
// (offsets into the cell range, halo list, edge range, foreign list, ecl, cell ghosts, edge ghosts);
// record t + 1 gives the ends.
#ifndef FBLTS_TILE
#define FBLTS_TILE 256
#endif
constexpr int TILE = FBLTS_TILE;
constexpr int TINFO = 8;
constexpr int HALO0 = TILE + 2;
constexpr int FGAP = 2;
constexpr uint16_t TILE_SENT = 0xFFFFu;
constexpr int TILE_SMEM_MAX = 227 * 1024;     // opt-in dynamic shared memory per CTA (sm_100a)
struct TileMesh {
    int32_t nTiles;
    int32_t strideRow;                      // >= nOwnC
    int32_t hmax, emax;                     // largest halo / local-edge count of any tile
    const int32_t *__restrict__ info;       // [(nTiles + 1) * TINFO]
    const int32_t *__restrict__ halo;       // halo cells of all tiles
    const int32_t *__restrict__ fedge;      // foreign edges of all tiles
    const uint32_t *__restrict__ ecl;       // local-edge cell pairs of all tiles
    const uint16_t *__restrict__ row;       // [maxE][strideRow]
    // ghosts (round 2): the values a tile needs from its halo cells / foreign edges that do not change
    // during a step, stored per tile contiguously so that they arrive by bulk copies.  Tile t's halo cell
    // q at ghost index info[t*TINFO+6] + q (the range starts at the parity of the tile's first cell),
    // foreign edge q at info[t*TINFO+7] + q (parity of the owned run's end); gcidx / geidx give the
    // source of every ghost slot (-1: padding).  Gz, Gl, Gd are filled at bind; S's ghosts per step.
    const int32_t *__restrict__ gcidx;
    const int32_t *__restrict__ geidx;
    const double *__restrict__ Gz;
    const double *__restrict__ Gl;
    const double *__restrict__ Gd;
};

// Subcycle tiles (fused fine subcycle): the tiles of the deep fine region
// F\F^2 with their 3-ring neighbourhood, so that one CTA advances a tile through a whole fine
// subcycle (velocity stage 3 of subcycle k-1, thickness stages 1-3 of subcycle k) by recomputing
// the stage values on the rings it needs: stage 1 on rings 0-2, stage 2 on rings 0-1, stage 3 on
// the tile.  Local cells: own (i - c0), then the halo list R1 | R2 | R3 at HALO0 + position (each
// ring sorted).  Local edges (every edge of a ring-0..2 cell): the tile's owned run [eo0, eo1)
// (e - eo0), then FGAP, then the foreign edges sorted by (lowest ring of their two cells, index):
// nF0 | nF1 | nF2, so each stage's edge set is a prefix.  ecl as in TileMesh (per local edge, list
// order); rows: slot-major 16-bit slot tables of the rows own | R1 | R2 (row r -> local cell r or
// HALO0 + r - nOwn), each tile's table padded to 8 entries.  info[t * FTINFO + k], k = c0, c1, h0, n1, n2, n3, eo0, eo1, f0, nF0, nF1, nF2,
// l0, s0, flags (bit 0: a ring-1 cell lies outside the fused region, so stage 1 is written out).
constexpr int FTINFO = 16;
struct SubTileMesh {
    int32_t nTiles;
    int32_t hmax, emax;                     // largest R1+R2+R3 count / local-edge count of any tile
    int32_t rmax;                           // largest slot-table size (uint16 entries, padded to 8)
    const int32_t *__restrict__ info;
    const int32_t *__restrict__ halo;
    const int32_t *__restrict__ fedge;
    const uint32_t *__restrict__ ecl;
    const uint16_t *__restrict__ row;
};

struct DevMesh {
    int32_t nC, nE, nV;               // local entity counts (owned + halo)
    int32_t nOwnC, nOwnE;              // owned cells [0, nOwnC); edges touching owned cells [0, nOwnE)
    int32_t strideC, strideE, strideV; // padded slot strides
    int32_t maxE, maxE2;
    int32_t ecS;                       // row stride of ec (G: 6, 8 or 16 >= maxEdges)
    const int32_t *__restrict__ nEoC;  // [nC]
    const int2 *__restrict__ ec;       // [nC*maxE] (sign-encoded edge, neighbour cell), cell-major
    const double *__restrict__ areaCell;  // [nC]
    const double *__restrict__ zb;        // [nC]  z_b = -bottomDepth
    const int2 *__restrict__ coe;      // [nE] (c0, c1)
    const int2 *__restrict__ voe;      // [nE] (v0, v1)
    const double *__restrict__ dv;     // [nE] l_e
    const double *__restrict__ dc;     // [nE] d_e
    const int32_t *__restrict__ nEoE;  // [nE]
    const int32_t *__restrict__ eoe;   // [maxE2][strideE]
    const double *__restrict__ W;      // [maxE2][strideE]
    const double *__restrict__ tau;    // [nE] tau . n_e
    const double *__restrict__ uwn;    // [nE] wind u_W . n_e   (hurricane terms)
    const double *__restrict__ uwt;    // [nE] wind u_W . t_e
    const int32_t *__restrict__ eov;   // [3][strideV] sign-encoded
    const int32_t *__restrict__ cov;   // [3][strideV]
    const double *__restrict__ kite;   // [3][strideV]
    const double *__restrict__ areaTri; // [nV]
    const double *__restrict__ fV;     // [nV]
    const uint8_t *__restrict__ vOwn;  // [nV] 1 if this rank reports the vertex in the diagnostics
    const uint8_t *__restrict__ eOwn;  // [nE] 1 if this rank reports the edge in the diagnostics
    // Owned cells form two region-major blocks: the BOUNDARY block [0, nB) (cells some peer holds
    // in its ring-1 halo; all owned cells when there is one rank) and the INTERIOR block
    // [nB, nOwnC), so that a stage can compute the boundary block, hand it to the halo exchange
    // and compute the interior block while the exchange is in flight.
    int32_t nB;
    // 1: the edge e = eov[k][v] with v = voe[e][1] joins cov[k][v] and cov[(k+1)%3][v], for every local
    // edge exactly once -- the full slow_pre sweep then forms F_e in the vertex role (its h and u are
    // already loaded there) and runs no edge role
    int32_t vF;
    Bounds cb, cbI;                    // boundary / interior cell blocks (absolute indices)
    Bounds eb;                         // edges touching owned cells (eb.end = nOwnE)
    Bounds cbh;                        // halo cell block [nOwnC, nC), region-major, absolute indices
    TileMesh tm;                       // tiles of the owned cells
    SubTileMesh st;                    // subcycle tiles of F\F^2 (one rank; fused fine subcycle)
};

// blocks of the diagnostics reduction (fixed: the partial sums are merged in block order, so the
// result is a deterministic function of the state)
constexpr int DIAG_RB = 592;                  // blocks per role (cells, vertices, edges)
constexpr int DIAG_BLOCKS = 3 * DIAG_RB;

// Device error record (positivity / NaN), first failure wins.
struct DevError {
    int32_t flag;    // 0 = ok, 1 = positivity
    int32_t kind;    // KernelKind
    int32_t k;       // fine subcycle (or -1)
    int32_t index;   // local (permuted) cell index
    double value;
};

// Scalars of one coarse step, computed once on the host in double exactly as
// the oracle does (SURVEY c.1 canonical constants).
struct StepConst {
    double g, rho0;                 // g = gravity of the fast term, g (1 - beta_SAL)
    double b1, b2, b3, omb1, omb2, om2b3;
    double c1, c2, c3;        // dt/3, dt/2, dt
    double c1f, c2f, c3f;     // dt/(3M), dt/(2M), dt/M
    int32_t M;
    int32_t hur;              // hurricane drag / wind terms in the slow tendency (fblts_set_hurricane)
    int32_t pve;              // energy-conserving PV flux (fblts_config.pv_energy)
    double cd, cw;            // C_D, C_W
};

// Prediction coefficients for subcycle k (eq. preds): a = k/M, oma = 1 - a,
// a1 = (k+1)/M, oma1 = 1 - a1, b = 1/M, c = 1 - (k+1)/M.
struct PredConst {
    double a, oma, a1, oma1, b, c;
};

// Device pointers of the state and scratch arrays (all in the caller's workspace).
struct DevState {
    double *hN, *hNew, *h1, *h2, *hT;   // cells
    double *uN, *uNew, *uT, *S, *F;     // edges
    double *q;                          // vertices
    double *qe;                         // q_hat per edge (energy-conserving PV flux only)
    double *K;                          // cells
    double *accH, *accU;                // accH indexed by owned cell (IF cells used), accU by e - eb.if2 (IF edges)
    double *uIF2, *uIF3;                // coarse stage velocities u~^{n+1/2}, u~^{n+1} on IF-2_E u IF-1_E (by
                                        // e - eb.if2; u~^{n+1} on IF-1_E only), written by the coarse velocity
                                        // sweep, read by every fine stage-3 band sweep
    double *rkU[2], *rkAccU;            // RK4 scheme: stage velocities (ping-pong) and the velocity sum
    double *Sf;                         // slow tendency on F_E during the fine phase: S, or Sk (refresh)
    double *Sk, *hv, *uv;               // slow-term refresh: S^k on F_E and the t^{n,k} views;
                                        // unsplit: stage slow tendency, HS array / view, U view
    double *un[3];                      // unsplit: stored coarse stage velocities u~1, u~2, u~3
    double *unk[2];                     // unsplit: stored fine stage velocities uk1, uk2
    double *hT2;                        // fused subcycle: third fine level buffer (levels k-1, k, k+1 distinct)
    double *eta, *dP, *accP, *Pv;       // vorticity companion: eta per vertex, integrated PV flux per edge,
                                        // its IF-edge sum, the PV-flux part of the last slow sweep
    double *h2alt;                      // fused subcycle: stage-2 thickness of F\F^2 before it is published
    double *stage;                      // staging for set/get_state (max(nC, nE) doubles)
    int32_t *cellOld, *edgeOld;         // new -> old permutation (device)
    double *diag;                       // reduction scratch
    double *diagA;                      // reduction scratch of the asynchronous diagnostics
    double *sendbuf, *recvbuf;          // halo exchange buffers
    int32_t *xidx;                      // halo exchange index lists (all exchanges, send then recv)
    DevError *err;
    int32_t *vbad;                      // set_state check: first bad index of h, of u (INT_MAX-like if none)
};

// Staged stage sweep over the whole tiles [tile0, tile1) (kernels.cu): one thread per cell,
//   out_i = hbase_i + ch * Psi_i(u_bar, hprev),
//   u_bar_e = ubase_e                                   (STAGE 1)
//   u_bar_e = ubase_e + cu (Phi^fast_e(bb hprev + omb hbase) + S_e)   (STAGE 2, 3)
// which is the coarse stage s (hbase = h^n) and the fine stage s inside F (hbase = h^{n,k}).
// STAGE 4 fuses the deep fine velocity stage 3 of subcycle k-1 into stage 1 of subcycle k:
//   u^{n,k}_e = u^{n,k-1}_e + cu (Phi^fast_e(h***) + S_e),  h*** = bb h^{n,k} + omb h2 + bb h^{n,k-1}
//   (written to unew on the tile's owned edge run), then out_i = h^{n,k}_i + ch Psi_i(u^{n,k}, h^{n,k})
// with hprev = h^{n,k}, hbase = h^{n,k-1}, h2 = stage-2 thickness of subcycle k-1, ubase = u^{n,k-1}.
struct StageArgs {
    const double *hbase, *hprev, *ubase, *S;
    double *out;
    double cu, bb, omb, ch, g;
    int32_t kind, k;
    const double *h2 = nullptr;   // STAGE 4
    double *unew = nullptr;       // STAGE 4
    const double *gS = nullptr;   // ghosts of S (TileMesh), filled before the launch
};
// dst[k] = idx[k] >= 0 ? src[idx[k]] : 0 for k in [k0, k1) (ghost fill)
void launch_ghost_fill(const int32_t *idx, const double *src, double *dst, int k0, int k1, cudaStream_t s);
// Fused fine subcycle k on the subcycle tiles (kernels.cu k_fine_sub): with vel (k >= 1) first
//   u^{n,k}_e = u^{n,k-1}_e + dt/M (Phi^fast_e(h***) + S_e),  h*** = b3 h^{n,k} + (1-2b3) h2 + b3 h^{n,k-1}
// on the edges of rings 0-2 (written on the owned run), else u^{n,k} = ubase; then the three
// thickness stages of subeqn fine_fbrk32 with the stage velocities recomputed per edge.
struct SubArgs {
    const double *hk, *hm, *h2, *ubase, *S;   // h^{n,k}, h^{n,k-1}, stage-2 thickness of k-1, u^{n,k-1} (or u^{n,0})
    double *unew, *h1out, *h2out, *out;       // u^{n,k} (owned runs), stage 1 (border tiles), stage 2, h^{n,k+1}
    double g, b1, omb1, b2, omb2, b3, om2b3, c1f, c2f, c3f;
    int32_t k;
};
int sub_smem_bytes_host(int hmax, int emax, int rmax);
void launch_fine_sub(const DevMesh &m, bool vel, int nsm, const SubArgs &a, DevError *err, cudaStream_t s);

void launch_stage_tiled(const DevMesh &m, int stage, int tile0, int tile1, int hmax, int emax, int nsm,
                        const StageArgs &a, DevError *err, cudaStream_t s);
// bytes for tiles with <= hmax halo cells / emax local edges, and the records of nrec tiles per CTA
int stage_tiled_smem_bytes_host(int stage, int hmax, int emax, int nrec = 0);
int stage_tiled_configure(const DevMesh &m);      // sets the dynamic shared-memory limits (cudaError_t)

// Kernel launchers (kernels.cu).  All enqueue on `s`.
void launch_slow_pre(const DevMesh &m, const DevState &st, const double *h, const double *u, cudaStream_t s);
void launch_slow_edge(const DevMesh &m, const DevState &st, const double *h, const double *u, const StepConst &sc,
                      cudaStream_t s);
// restricted slow sweeps (vertices >= v0, cells >= c0, edges >= e0; S on edges [e0, e1) into out)
void launch_slow_pre_range(const DevMesh &m, const DevState &st, const double *h, const double *u, int v0, int c0,
                           int e0, cudaStream_t s,
                           int v0vf = -1);
// Unsplit velocity update fused into the slow edge sweep (k_slow_edge<..., VEL = true>): instead of
// writing S_e, out_e = base_e + c (Phi^fast_e(h) + S_e), or on edges [a0, a1) with acc != nullptr
// acc[e - a0] = (first ? 0 : acc[e - a0]) + (Phi^fast_e(h) + S_e) -- k_un_vel's arithmetic, same bits.
struct VelFuse {
    const double *base = nullptr;
    double *out = nullptr;
    double c = 0.0;
    double *acc = nullptr;
    int a0 = 0, a1 = 0, first = 0;
};
void launch_slow_edge_range(const DevMesh &m, const DevState &st, const double *h, const double *u, double *out,
                            int e0, int e1, const StepConst &sc, cudaStream_t s, double *pvout = nullptr,
                            const VelFuse *vel = nullptr);
// prognostic absolute vorticity companion (unsplit, config vorticity): kernels.cu
void launch_vort_int(const DevState &st, double c3, int e1, cudaStream_t s);
void launch_vort_fine(const DevMesh &m, const DevState &st, double c3f, int first, cudaStream_t s);
void launch_vort_close(const DevMesh &m, const DevState &st, double c3f, cudaStream_t s);
void launch_vort_update(const DevMesh &m, const DevState &st, cudaStream_t s);
void launch_vort_split(const DevMesh &m, const DevState &st, const StepConst &sc, cudaStream_t s);
// slow-term refresh views at t^{n,k} into st.hv (cells) and st.uv (edges)
void launch_refresh_views(const DevMesh &m, const DevState &st, const double *hN, const double *hNew,
                          const double *hk, const double *uN, const double *uk, const StepConst &sc,
                          const PredConst &pc, cudaStream_t s);
// cell launchers act on one owned cell block b (DevMesh::cb or DevMesh::cbI)
void launch_coarse_s1(const DevMesh &m, const DevState &st, const double *hN, const double *uN,
                      const StepConst &sc, cudaStream_t s, const Bounds &b);
void launch_coarse_s2(const DevMesh &m, const DevState &st, const double *hN, const double *uN,
                      const StepConst &sc, cudaStream_t s, const Bounds &b);
void launch_coarse_s3(const DevMesh &m, const DevState &st, const double *hN, const double *uN,
                      double *hNew, const StepConst &sc, cudaStream_t s, const Bounds &b);
// (if_edges: also u~^{n+1/2} and u~^{n+1} on the IF edges into st.uIF2 / st.uIF3, for the fine phase)
void launch_coarse_vel(const DevMesh &m, const DevState &st, const double *hN, const double *uN,
                       const double *hNew, double *uNew, const StepConst &sc, cudaStream_t s, bool if_edges = false);
void launch_fine_s1(const DevMesh &m, const DevState &st, const double *hN, const double *hNew,
                    const double *hk, const double *uk, const StepConst &sc, const PredConst &pc,
                    int k, cudaStream_t s, const Bounds &b, bool deep = true);
void launch_fine_s2(const DevMesh &m, const DevState &st, const double *hN, const double *hNew,
                    const double *hk, const double *uk, const StepConst &sc, const PredConst &pc,
                    int k, cudaStream_t s, const Bounds &b, bool deep = true);
void launch_fine_s3(const DevMesh &m, const DevState &st, const double *hN, const double *uN,
                    const double *hNew, const double *hk, const double *uk, double *hnext,
                    const StepConst &sc, const PredConst &pc, int k, cudaStream_t s, const Bounds &b,
                    bool deep = true);
void launch_fine_vel(const DevMesh &m, const DevState &st, const double *hN, const double *hNew,
                     const double *hk, const double *hnext, const double *uk, double *unext,
                     const StepConst &sc, const PredConst &pc, int k, cudaStream_t s, bool deep = true);
void launch_correct(const DevMesh &m, const DevState &st, const double *hN, const double *uN,
                    double *hNew, double *uNew, const StepConst &sc, cudaStream_t s, const Bounds &b, bool edges);
// Classical RK4 on the unsplit system (fbrk32.rk4_step), stage `stage` = 1..4 on every owned
// cell and edge: k = (Psi(us, hs), Phi^fast(hs) + S) with S = Phi^slow(us, hs) already in st.S;
// acc = k (stage 1), acc + 2 k (2, 3), acc + k (4); next stage (h^n, u^n) + cnext k, and after stage 4
// (h, u)^{n+1} = (h^n, u^n) + (dt/6) acc.
void launch_rk4_stage(const DevMesh &m, const DevState &st, int stage, const double *hN, const double *uN,
                      const double *hs, const double *us, double *hout, double *uout, double cnext,
                      double dt6, double g, cudaStream_t s);
// unsplit FB-LTS building blocks (kernels.cu, end)
void launch_un_cstage(const DevMesh &m, const DevState &st, int stage, const double *hN, const double *H,
                      const double *U, double *out, const StepConst &sc, int end, cudaStream_t s);
void launch_un_vel(const DevMesh &m, const DevState &st, const double *base, double *out, double c, int e0, int e1,
                   double *acc, int a0, int a1, int first, const StepConst &sc, cudaStream_t s);
void launch_un_views(const DevMesh &m, const DevState &st, int stage, const double *hN, const double *hNew,
                     const double *hk, const double *hnext, const double *uN, const double *ufine,
                     const StepConst &sc, const PredConst &pc, cudaStream_t s, int c0 = 0, int e0 = 0);
void launch_un_fstage(const DevMesh &m, const DevState &st, int stage, const double *hN, const double *hNew,
                      const double *hk, const double *U, double *out, const StepConst &sc, const PredConst &pc,
                      int k, cudaStream_t s);
void launch_permute_in(const int32_t *old_of_new, const double *src, double *dst, int n, cudaStream_t s);
void launch_permute_out(const int32_t *old_of_new, const double *src, double *dst, int n, cudaStream_t s);
// *bad = min(*bad, first index i < n with v[i] not finite, or not > 0 when positive)
void launch_validate(const double *v, int n, int positive, int *bad, cudaStream_t s);
// diagnostics: writes out[4] (device) = mass, Gamma, min h, max nu
// halo exchange: buf[k] = a[idx[k]] (pack), a[idx[k]] = buf[k] (unpack)
void launch_pack(const int32_t *idx, const double *a, double *buf, int n, cudaStream_t s);
void launch_unpack(const int32_t *idx, const double *buf, double *a, int n, cudaStream_t s);
// cells_only: the mass and min h partials alone (Gamma and max nu come back as 0)
// pv: the vertex role sums the PV volume integral A_v h_v q_v instead of Gamma (out[1])
void launch_diagnostics(const DevMesh &m, const double *h, const double *u, const StepConst &sc, double *part,
                        double *out_dev, cudaStream_t s, bool cells_only = false, bool pv = false);

}  // namespace fblts
