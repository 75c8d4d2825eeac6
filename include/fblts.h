/*
 * fblts.h -- C ABI of libfblts.so, the B200 (sm_100a) hot path of FB-LTS
 * (Lilly, Capodaglio, Engwirda, Higdon, Petersen, arXiv 2405.10505).
 *
 * What the library computes (PAPER.md line numbers, "P:Lnnn"):
 *   one FB-LTS coarse step in split mode = the slow tendency frozen at t^n
 *   (eq. splitting), Coarse Advancement on C u F^l,
 *   Interface Prediction on IF-1 (eq. preds), M fine FB-RK(3,2)
 *   subcycles on F (eq. fine_fbrk32) accumulating the interface
 *   summands, and the Interface Correction (eq. if_correction).
 *   The spatial operators are TRiSK on a Voronoi C-grid: Psi_i
 *   (eq. trisk_thickness), Phi^fast = -g grad(h + z_b)
 *   (eq. fast_terms), and the slow momentum terms
 *   q_hat F_perp - grad K (+ wind-stress forcing) (eq. nonlinear_swe P:L257-273,
 *   eq. trisk_vorticity).  FB weights default (0.531, 0.531, 0.313)
 *   (P:L327-328).  The readings of ambiguous passages are listed in DESIGN.md.
 *
 * Conventions
 *   - All indices are 0-based int32; all floating point is IEEE fp64.
 *   - Orientation: n_e points from cellsOnEdge[e][0] to cellsOnEdge[e][1];
 *     t_e = k x n_e; verticesOnEdge[e][1] lies on the +t_e side; edgesOnCell,
 *     cellsOnVertex are counter-clockwise (Fig. trisk).
 *   - Host arrays passed in are BORROWED for the duration of the call only; the
 *     library copies what it needs.  All state I/O is in the caller's ORIGINAL
 *     order; the library's region-major / space-filling-curve permutation is
 *     internal.
 *   - Device memory: the caller owns one workspace buffer (e.g. a torch uint8
 *     CUDA tensor) that must outlive the context.  The library owns its CUDA
 *     graphs, events, and (nranks > 1) its NCCL communicator, destroyed by
 *     fblts_destroy.
 *   - Streams: every enqueueing call works on cfg.stream (the caller's stream,
 *     e.g. torch.cuda.current_stream().cuda_stream; NULL = legacy default).
 *   - Errors: every int function returns 0 on success or a negative FBLTS_ERR_*
 *     code; fblts_last_error() returns a message naming the field/index/phase.
 *     fblts_step is asynchronous: device-side failures (h <= 0 or NaN) set a
 *     device flag that the next synchronising call (fblts_sync, fblts_get_state,
 *     fblts_diagnostics) reports as FBLTS_ERR_POSITIVITY.
 *   - Call order: create -> upload_mesh -> set_regions -> workspace_size ->
 *     bind_workspace -> set_state -> (set_forcing) -> step* -> get_state /
 *     diagnostics -> destroy.  Out-of-order calls return FBLTS_ERR_ORDER.
 *   - Determinism: identical inputs give bit-identical outputs.
 */
#ifndef FBLTS_H
#define FBLTS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FBLTS_OK               0
#define FBLTS_ERR_INVALID_ARG (-1)
#define FBLTS_ERR_MESH        (-2)
#define FBLTS_ERR_LABELS      (-3)
#define FBLTS_ERR_STATE       (-4)
#define FBLTS_ERR_CUDA        (-5)
#define FBLTS_ERR_NCCL        (-6)
#define FBLTS_ERR_POSITIVITY  (-7)
#define FBLTS_ERR_ORDER       (-8)

/* Region codes returned by fblts_get_labels (cells and edges):
 *   0 = C^int, 1 = C^IF-2, 2 = C^IF-1, 2+l (l = 1..5) = F^l \ F^(l-1), 8 = F \ F^5.
 * Cells: IF-1 = coarse cells 1..r hops from F, IF-2 = r+1..2r hops, int = farther;
 * F^l = fine cells within l*r hops of C.  Edges take the region
 * "closest to the fine region"; F^l_E = edges touching F^l. */
#define FBLTS_REGION_INT 0
#define FBLTS_REGION_IF2 1
#define FBLTS_REGION_IF1 2
#define FBLTS_REGION_F1  3
#define FBLTS_REGION_FDEEP 8

typedef struct fblts_ctx fblts_ctx;

/* TRiSK mesh, host arrays (MPAS field names). */
typedef struct {
    int32_t nCells, nEdges, nVertices;
    int32_t maxEdges;                 /* max edges per cell (row stride of edgesOnCell) */
    int32_t maxEdges2;                /* row stride of edgesOnEdge / weightsOnEdge */
    const int32_t *nEdgesOnCell;      /* [nCells] */
    const int32_t *edgesOnCell;       /* [nCells*maxEdges], CCW; unused slots ignored */
    const int32_t *cellsOnEdge;       /* [nEdges*2] (c0, c1): n_e points c0 -> c1 */
    const int32_t *verticesOnEdge;    /* [nEdges*2] (v0, v1): v1 on the +t_e side */
    const int32_t *nEdgesOnEdge;      /* [nEdges] */
    const int32_t *edgesOnEdge;       /* [nEdges*maxEdges2] */
    const double  *weightsOnEdge;     /* [nEdges*maxEdges2]: F_perp_e = sum_j W[e][j] F[eoe[e][j]] */
    const int32_t *edgesOnVertex;     /* [nVertices*3] */
    const int32_t *cellsOnVertex;     /* [nVertices*3], CCW */
    const double  *kiteAreasOnVertex; /* [nVertices*3], aligned with cellsOnVertex */
    const double  *areaCell;          /* [nCells]    A_i  (m^2) */
    const double  *areaTriangle;      /* [nVertices] A_v  (m^2) */
    const double  *dvEdge;            /* [nEdges]    l_e: primal edge length (m) */
    const double  *dcEdge;            /* [nEdges]    d_e: cell-centre distance (m) */
    const double  *fVertex;           /* [nVertices] Coriolis parameter (s^-1) */
    const double  *bottomDepth;       /* [nCells]    H > 0; z_b = -H (m) */
    const double  *xCell, *yCell, *zCell;  /* [nCells] positions, used only for the SFC order */
} fblts_mesh;

typedef struct {
    double  dt;          /* coarse step (s) */
    double  g;           /* gravity (m s^-2) */
    double  beta[3];     /* FB weights */
    double  rho0;        /* reference density for the wind-stress forcing (kg m^-3) */
    int32_t M;           /* fine subcycles per coarse step (>= 1) */
    int32_t r;           /* stencil radius for the region widths (2) */
    int32_t slow;        /* 1: slow terms on (split model); 0: gravity-wave model */
    int32_t device;      /* CUDA device ordinal */
    void   *stream;      /* cudaStream_t of the caller (NULL = legacy default stream) */
    int32_t rank;        /* this process's rank (0 for single GPU) */
    int32_t nranks;      /* number of ranks (1 for single GPU) */
    const void *nccl_id; /* 128-byte ncclUniqueId shared by all ranks; NULL if nranks == 1, or for
                            the members of a one-process loopback group (fblts_step_group) */
    int32_t scheme;      /* FBLTS_SCHEME_FBLTS (0): FB-LTS, split mode (global FB-RK(3,2) when there are
                            no fine cells or M = 1); FBLTS_SCHEME_RK4 (1): classical four-stage RK4 on
                            the unsplit system, global (M and the fine mask ignored), one
                            rank -- the paper's reference scheme, for speedup comparisons;
                            FBLTS_SCHEME_RK32 (2): RK(3,2) on the unsplit system, global, one rank */
    int32_t slow_refresh;/* 1: the paper's proposed variant: the slow tendency is
                            re-evaluated at every fine level t^{n,k} and used on the fine edges
                            (DESIGN.md 3 for the reading); FB-LTS scheme, one rank.  0: frozen S */
    double  sal_beta;    /* self-attraction-and-loading coefficient beta of the hurricane model's fast
                            term -g grad(xi - beta xi) (eq. hurricane_fast_terms),
                            0 <= beta < 1; the fast term uses g (1 - beta).  0: plain model */
    int32_t unsplit;     /* 1: unsplit FB-LTS: the full Phi(U, HS) =
                            Phi^fast + Phi^slow in every velocity update, stage velocities stored;
                            one rank, FB-LTS scheme, no slow refresh.  0: split mode (the paper's runs) */
    int32_t pv_energy;   /* 1: energy-conserving PV flux in the slow tendency (the variant
                            of reading Q2): q_hat_e F_perp_e is replaced by
                            sum_j W_{e,j} F_{e_j} (q_hat_e + q_hat_{e_j}) / 2, which does no work
                            (sum_e l_e d_e F_e PV_e = 0); one rank, no slow refresh.  0: centred q_hat */
    int32_t vorticity;   /* 1: advance the prognostic absolute vorticity companion eta_v with every step
                            (Theorem 2; SPEC step_prognostic_vorticity S:L472-480): the PV-flux
                            term q_hat_e F_perp_e of every velocity update, integrated per edge as the velocity
                            integrates it (int_E: dt PV of coarse stage 3; F_E: sum_k dt/M PV^k; IF edges:
                            dt/M sum_k PV^k), gives eta_v += (sum_j t_{e_j,v} d_{e_j} dP_{e_j}) / A_v; in split
                            mode PV is the frozen one inside S.  One rank, FB-LTS scheme, no slow refresh;
                            set / read with fblts_set_vorticity / fblts_get_vorticity */
} fblts_config;

#define FBLTS_SCHEME_FBLTS 0
#define FBLTS_SCHEME_RK4   1
#define FBLTS_SCHEME_RK32  2   /* RK(3,2) of Wicker & Skamarock on the unsplit system, global,
                                  one rank: the scheme FB-RK(3,2) extends (Table-1 analogue baseline) */

/* Create a context.  *out receives the handle (NULL on failure).
 * Errors: INVALID_ARG (M < 1, dt <= 0, r < 1, bad rank/nranks), CUDA, NCCL. */
int fblts_create(fblts_ctx **out, const fblts_config *cfg);

/* Copy and validate the mesh.  Checks index ranges, that every edge appears in
 * edgesOnCell of exactly its two cellsOnEdge entries, positive lengths/areas,
 * nEdgesOnCell <= maxEdges; message names field and index.  Errors: MESH, ORDER. */
int fblts_upload_mesh(fblts_ctx *ctx, const fblts_mesh *m);

/* Label the LTS regions from a fine-cell mask [nCells] (1 = fine), validate the
 * stencil assumption, build the region-major + SFC permutation and
 * (nranks > 1) the partition and halo lists.  Errors: LABELS, ORDER. */
int fblts_set_regions(fblts_ctx *ctx, const uint8_t *fine_mask);

/* Region codes in ORIGINAL order (see FBLTS_REGION_*); either pointer may be NULL. */
int fblts_get_labels(fblts_ctx *ctx, int8_t *cell_region, int8_t *edge_region);

/* Entity counts (out must hold 32 int64): out[0..2] = nCells, nEdges, nVertices; cells per
 * region code 0..8 at out[3..11], edges per code 0..8 at out[12..20]; out[21] = owned cells,
 * out[22] = owned edges (equal to nCells, nEdges for one rank); out[23] = kernel launches per
 * coarse step (nodes of the captured CUDA graph, 0 before the first fblts_step); out[24..27] =
 * cell tiles of the staged kernels: number of tiles, total halo cells, total local edges,
 * largest per-tile shared-memory footprint in bytes; out[28..31] = subcycle tiles of the fused
 * fine subcycle (0 when it is off): number of tiles, total ring-1..3 cells, total local edges,
 * shared-memory footprint in bytes. */
int fblts_get_counts(fblts_ctx *ctx, int64_t *out);

/* Halo exchange lists of this rank with `peer` (host logic, no device needed): which = 0 ring-1
 * cells (after every thickness stage), 1 = rings 1-2 cells (end of step), 2 = remote-owned edges
 * (end of step).  *n_send / *n_recv receive the counts; send_ids / recv_ids (may be NULL) receive
 * the GLOBAL ids in exchange order (ascending global id, identical on both sides); after
 * fblts_set_partition the whole-mesh ids (cells: gid; edges: (min gid << 32) | max gid). */
int fblts_get_halo(fblts_ctx *ctx, int32_t which, int32_t peer, int64_t *n_send, int64_t *n_recv,
                   int64_t *send_ids, int64_t *recv_ids);

/* Distributed set-up (optional; after upload_mesh, before set_regions): the uploaded mesh is this rank's
 * PIECE of a larger mesh -- the cells it owns plus a margin of cells owned by other ranks, closed (every
 * edge has two cells) -- and owner[i] / cell_gid[i] [nCells] give the owning rank and the id in the whole
 * mesh of piece cell i.  set_regions then labels the piece (exact for every cell whose
 * (2 + 5r)-ring neighbourhood lies in the piece -- keep the margin >= 2 + 5r + 2 rings wide), uses
 * `owner` instead of the dual-set partition, and orders every halo list by whole-mesh ids (cells: gid;
 * edges: (min gid << 32) | max gid of the edge's cells), so ranks that each hold only their piece agree
 * element by element.  Every rank's piece must contain fine cells if the whole mesh does.  State I/O
 * (set_state / get_state) is then in piece order.  Also valid with the whole mesh as the piece (an
 * externally chosen partition).  Errors: INVALID_ARG (owner outside [0, nranks), gid < 0 or >= 2^31 or
 * repeated, no owned cell), ORDER. */
int fblts_set_partition(fblts_ctx *ctx, const int32_t *owner, const int64_t *cell_gid);

/* 128-byte ncclUniqueId for a multi-rank context (call on rank 0, broadcast, pass as cfg.nccl_id). */
int fblts_nccl_unique_id(void *out128);

/* Bytes of device workspace needed after set_regions. */
int fblts_workspace_size(fblts_ctx *ctx, size_t *bytes);

/* Bind a caller-owned device buffer of >= workspace_size bytes (256-B aligned)
 * and upload the permuted mesh into it (synchronous on cfg.stream). */
int fblts_bind_workspace(fblts_ctx *ctx, void *device_ptr, size_t bytes);

/* Per-edge wind-stress projection tau . n_e [nEdges] (N m^-2), original order;
 * NULL = no forcing.  The slow term adds G_e = tau_n / (rho0 h_e^n) (reading Q19). */
int fblts_set_forcing(fblts_ctx *ctx, const double *tau_n);

/* Hurricane-model momentum terms in the slow tendency (eq. hurricane_model; SURVEY
 * 8(f) N4 with a synthetic wind): bottom drag -C_D |u|_e u_e / h_e and wind
 * +C_W |u_W - u|_e (u_W.n_e - u_e) / h_e, |u|_e from u_e and the tangential reconstruction
 * v_e = sum_j weightsOnEdge[e][j] u[edgesOnEdge[e][j]], h_e = (h_c0 + h_c1) / 2.  uw_n / uw_t: host
 * arrays [nEdges] (original order) of the wind's normal and tangential components, copied; both
 * NULL switches the terms off.  cd, cw: finite, >= 0.  Frozen with the rest of the slow tendency
 * (S at t^n).  Errors: INVALID_ARG (non-finite wind or coefficients), ORDER (before bind), CUDA. */
int fblts_set_hurricane(fblts_ctx *ctx, const double *uw_n, const double *uw_t, double cd, double cw);

/* Initial state, HOST arrays in original order: h [nCells] (m), u [nEdges] (m/s), t (s); copied
 * (synchronous; pinned host memory makes the copies DMA-speed).  The arrays are checked on the
 * device after the copy.  Errors: STATE (h <= 0 or non-finite, u non-finite; the message names the
 * smallest offending index; the context then holds no valid state until the next successful
 * set_state), ORDER, CUDA. */
int fblts_set_state(fblts_ctx *ctx, const double *h, const double *u, double t);

/* Prognostic absolute vorticity (cfg.vorticity = 1): eta [nVertices] in ORIGINAL vertex order, HOST
 * arrays, copied (synchronous).  set after fblts_set_state (e.g. the diagnostic curl u + f of the initial
 * state); get synchronises and reports device errors like fblts_get_state.  Errors: INVALID_ARG, ORDER
 * (no cfg.vorticity, or no state), STATE (non-finite eta), CUDA. */
int fblts_set_vorticity(fblts_ctx *ctx, const double *eta);
int fblts_get_vorticity(fblts_ctx *ctx, double *eta);

/* Enqueue n_coarse coarse steps on cfg.stream (asynchronous, CUDA-graph replay). */
int fblts_step(fblts_ctx *ctx, int32_t n_coarse);

/* Loopback group (testing the partitioned path on ONE device): the `n` contexts ctxs[r] (rank r of
 * n, same device and stream, all bound and with state set) advance n_coarse steps together; each
 * halo exchange is a device-to-device copy between their buffers.  No kernel waits on another. */
int fblts_step_group(fblts_ctx **ctxs, int32_t n, int32_t n_coarse);
int fblts_diagnostics_group(fblts_ctx **ctxs, int32_t n, double out[4]);

/* Synchronise cfg.stream and report asynchronous device errors (POSITIVITY, CUDA). */
int fblts_sync(fblts_ctx *ctx);

/* Read back the state into HOST arrays in original order (synchronises).  With nranks > 1 only
 * this rank's owned cells and the edges touching them are written; other entries are unchanged. */
int fblts_get_state(fblts_ctx *ctx, double *h, double *u, double *t);

/* out[4] = { total mass sum A_i h_i, total absolute vorticity sum_v (circulation_v + A_v f_v),
 *            min h, max Courant number (|u|+sqrt(g h_e)) dt_e / d_e } (Thms 1-2, eq. cfl).
 * Deterministic double-double reductions; with nranks > 1 the per-rank partials are all-gathered
 * (NCCL) and combined in rank order, so every rank returns the same bits (synchronises). */
int fblts_diagnostics(fblts_ctx *ctx, double out[4]);

/* out[2] = { total mass sum A_i h_i (Theorem 1), min h (positivity) } of the current
 * state: the cell part of fblts_diagnostics (same reduction, same bits), a cheap per-step monitor
 * (one pass over h and areaCell).  Synchronises;
 * several ranks: NCCL all-gather, combined in rank order.  Errors: ORDER, CUDA, NCCL, POSITIVITY. */
int fblts_diagnostics_mass(fblts_ctx *ctx, double out[2]);

/* *out = the volume integral of potential vorticity sum_v A_v h_v q_v (Remark rmk:volume_conservation_pv,
 * eq. vol_integral_pv), h_v = (sum_j kite_{v,j} h_{c_j}) / A_v, q_v = (zeta_v + f_v) / h_v:
 * equal to Gamma up to rounding, hence conserved wherever Theorem 2 holds.  Deterministic double-double
 * reduction (synchronises; several ranks: NCCL all-gather combined in rank order).  Errors: ORDER, CUDA. */
int fblts_diagnostics_pv(fblts_ctx *ctx, double *out);

/* The same four numbers as fblts_diagnostics (Thms 1-2, eq. cfl) for the state after the steps
 * enqueued so far, WITHOUT synchronising
 * (one rank): the reduction runs on a library stream that waits for the compute stream, its 48-byte
 * result is copied to pinned host memory and combined into out[4] by a host callback.  out must stay
 * valid until the next synchronising call (fblts_sync, fblts_get_state, fblts_diagnostics), after
 * which it holds the values.  Later steps that overwrite the state being reduced wait for the
 * reduction, so the numbers are those of the state at the call.  Errors: ORDER (no state, or
 * nranks > 1), CUDA. */
int fblts_diagnostics_async(fblts_ctx *ctx, double *out);

/* out[2] = { total mass, min h } of the state after the steps enqueued so far, WITHOUT synchronising: the
 * cell part of fblts_diagnostics_async (same reduction and bits as fblts_diagnostics_mass), a per-step
 * monitor that does not stall the step pipeline.  Same contract as fblts_diagnostics_async (one rank; out
 * valid after the next synchronising call).  Errors: ORDER, CUDA. */
int fblts_diagnostics_mass_async(fblts_ctx *ctx, double *out);

/* Instrumented replay for the roofline: runs n_coarse steps WITHOUT the graph, with
 * CUDA events around every launch on cfg.stream; ms[k] = total device ms of kernel
 * kind k, launches[k] = launch count, for k < FBLTS_NUM_KERNELS.  Advances the state. */
#define FBLTS_NUM_KERNELS 15
int fblts_profile(fblts_ctx *ctx, int32_t n_coarse, double *ms, int64_t *launches);
const char *fblts_kernel_name(int32_t kind);

/* Compile-time configuration of this library build, e.g. "probe=0 check=0 tile=256 ...": probe != 0
 * is a development build that skips work (never a measurement), check != 0 adds device-side bounds
 * traps.  Static string, no context needed. */
const char *fblts_build_info(void);

const char *fblts_last_error(const fblts_ctx *ctx);
void fblts_destroy(fblts_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* FBLTS_H */
