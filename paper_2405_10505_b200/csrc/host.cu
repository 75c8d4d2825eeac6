// host.cu -- C ABI of libfblts.so (include/fblts.h): context, mesh validation, LTS
// region labelling, region-major + space-filling-curve renumbering,
// partition into per-rank subdomains with halo lists, workspace carving, CUDA-graph step
// replay with NCCL halo exchanges, state I/O and diagnostics.
#include <algorithm>
#include <cmath>
#include <nvtx3/nvToolsExt.h>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <type_traits>
#include <string>
#include <vector>

#include <nccl.h>

#include "fblts.h"
#include "fblts_internal.h"

using namespace fblts;

namespace {

const char *kKernelNames[K_NUM] = {"slow_pre",  "slow_edge", "coarse_s1", "coarse_s2", "coarse_s3", "coarse_vel",
                                   "fine_s1",   "fine_s2",   "fine_s3",   "fine_vel",  "correct_if", "fine_vel_s1",
                                   "rk4_stage", "slow_refresh", "fine_sub"};

enum Phase { P_CREATED = 0, P_MESH, P_REGIONS, P_BOUND, P_STATE };

struct HostMesh {
    int nC = 0, nE = 0, nV = 0, maxE = 0, maxE2 = 0;
    std::vector<int32_t> nEoC, eoc, coe, voe, nEoE, eoe, eov, cov;
    std::vector<double> W, kite, areaCell, areaTri, dv, dc, fV, H, x, y, z;
};

struct Region {                 // global LTS labels (identical on every rank)
    std::vector<int8_t> cell, edge;
    int64_t ccount[9]{}, ecount[9]{};
};

// One halo exchange pattern: for each peer, the local indices this rank sends (its owned
// entries that the peer holds as halo) and receives (its halo entries owned by the peer),
// both in ascending global-id order so the two sides agree element by element.
struct Xchg {
    std::vector<int32_t> sendIdx, recvIdx;
    std::vector<int64_t> sendOff, recvOff;   // [nranks + 1]
    size_t sendAt = 0, recvAt = 0;           // offsets of the lists inside the device xidx table
};
enum { X_C1 = 0, X_C2 = 1, X_E = 2, X_NUM = 3 };

struct Local {                  // this rank's subdomain in local (device) numbering
    int nOwnC = 0, nC = 0, nOwnE = 0, nE = 0, nV = 0;
    int nB = 0;                                          // boundary block [0, nB) of the owned cells
    std::vector<int32_t> cellGlob, edgeGlob, vertGlob;   // local -> global
    Bounds cb{}, cbI{}, cbh{}, eb{};
    int64_t ocount[9]{}, oecount[9]{};                   // owned cells / edges touching owned, per code
    std::vector<uint8_t> vOwn, eOwn;
    Xchg x[X_NUM];
};

}  // namespace

struct fblts_ctx {
    fblts_config cfg{};
    cudaStream_t stream = nullptr;
    cudaStream_t cap = nullptr;
    cudaStream_t comm = nullptr;            // halo-exchange stream (nranks > 1)
    cudaEvent_t evFork = nullptr, evJoin = nullptr;
    // one rank, captured steps: the band (interface) thickness sweeps of fine stages 2 and 3 run on
    // `side`, concurrently with the staged deep sweep of the same stage (disjoint outputs, both read
    // only the previous stage); FBLTS_BAND_SIDE=0 serialises them (development comparisons)
    cudaStream_t side = nullptr;
    cudaEvent_t evSideF = nullptr, evSideJ = nullptr;
    bool band_side = true;
    std::string err;
    int phase = P_CREATED;
    // fblts_set_partition: the uploaded mesh is this rank's PIECE of a larger mesh (its owned cells plus
    // a margin), ext_part[i] = owning rank of piece cell i, gid[i] = its id in the whole mesh
    bool piece = false;
    std::vector<int32_t> ext_part;
    std::vector<int64_t> gid;
    HostMesh hm;
    Region rg;
    Local lo;
    StepConst sc{};
    // device
    char *ws = nullptr;
    size_t ws_bytes = 0;
    DevMesh dm{};
    DevState ds{};
    double *hbuf[2]{}, *ubuf[2]{};
    double *diag_out = nullptr;
    int parity = 0;  // state lives in hbuf[parity], ubuf[parity]
    double t = 0.0;
    bool have_fine = false;
    cudaGraphExec_t exec[2]{};
    size_t graph_nodes = 0;   // kernel launches per coarse step (nodes of the captured graph)
    void *nccl = nullptr;     // ncclComm_t (nranks > 1)
    // asynchronous diagnostics (fblts_diagnostics_async): side stream, per-state-buffer events that
    // the steps overwriting that buffer wait on, pinned result slots and host-callback payloads
    cudaStream_t dstream = nullptr;
    cudaEvent_t evHead = nullptr, evDiag[2]{};
    bool diagPending[2]{};
    double *dhost = nullptr;
    struct DiagJob {
        const double *slot;
        double *out;
        bool mass_only;            // out[2] = {mass, min h} instead of the four numbers
    } *djobs = nullptr;
    uint64_t ndiag = 0;
    unsigned char nccl_id[128]{};
    // host-side staging of the permuted device tables (filled at set_regions)
    std::vector<int32_t> d_nEoC, d_ec, d_nEoE, d_eoe, d_eov, d_cov, d_coe, d_voe, d_xidx;
    std::vector<double> d_area, d_zb, d_dv, d_dc, d_W, d_kite, d_areaTri, d_fV;
    int sE = 0, sV = 0, ecS = 6;
    size_t xmax = 1;           // largest send/recv buffer (doubles)
    // tiles of the owned cells (staged stage kernels)
    std::vector<int32_t> t_start, t_info, t_halo, t_fedge;
    std::vector<uint32_t> t_ecl;
    std::vector<uint16_t> t_row;
    int t_sRow = 32, t_hmax = 0, t_emax = 0;
    std::vector<int32_t> g_cidx, g_eidx;     // ghost slot sources (cells / edges), -1 = padding
    double *GS = nullptr;                    // ghosts of S (per step)
    int32_t *dGe = nullptr;                  // device copy of g_eidx
    struct GhostKey { const double *src = nullptr; int k0 = 0, k1 = 0; int64_t epoch = -1; };
    GhostKey gkS;                            // S ghost fill already enqueued in the current step
    int64_t step_epoch = 0;
    size_t t_nHalo = 0, t_nFedge = 0, t_nEcl = 0;
    bool deep_runs_ok = false;
    int vminF = 0;
    int vminF1 = -1;           // vF: first vertex owning an edge of IF-1_E .. F_E (-1: vF off)
    // unsplit fine views (enqueue_unsplit_step): first cell / edge the HS / U views of fine stages 1-2 are
    // read at (the F_E slow stencil), first edge the stage-3 thickness sweep reads U at (cells from IF-2)
    int un_c12 = 0, un_e12 = 0, un_e3 = 0;
    bool vF = false;           // DevMesh::vF (FBLTS_VF=0: off)
    bool un_fuse = true;       // unsplit: velocity update inside the slow edge sweep (FBLTS_UNFUSE=0: off)
    std::vector<int32_t> e_owner;          // local owner cell of every local edge (build_local)
    bool tiled = true;
    bool split = false;        // FBLTS_SPLIT=1: separate launches for the thin interface blocks
    bool fuse_vel = true;      // deep fine velocity stage fused into the next stage 1 (FBLTS_FUSE=0: off)
    // subcycle tiles of F\F^5 (fused fine subcycle; one rank, split FB-LTS).  Opt-in (FBLTS_SUB=1):
    // bitwise equal to the per-stage sweeps but measured slower on B200
    bool fuse_sub = false;
    int sub_level = 5;         // subcycle tiles cover F\F^sub_level (>= 2)
    std::vector<int32_t> s_info, s_halo, s_fedge;
    std::vector<uint32_t> s_ecl;
    std::vector<uint16_t> s_row;
    int s_nT = 0, s_hmax = 0, s_emax = 0, s_rmax = 0;
    size_t s_nHalo = 0, s_nFedge = 0, s_nEcl = 0, s_nRow = 0;
    int nsm = 148;         // FBLTS_TILED=0 selects the unstaged kernels (development comparisons)
};
namespace {

int fail(fblts_ctx *c, int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    return code;
}

#define CUDA_TRY(ctx, call)                                                                          \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess) return fail(ctx, FBLTS_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

int pad32(int n) { return (n + 31) / 32 * 32; }
void diag_wait(fblts_ctx *c, int b);

// ---------------------------------------------------------------- SFC keys
// 2-D Hilbert index (planar meshes) on a 2^16 x 2^16 grid over the bounding box.
uint64_t hilbert2(uint32_t x, uint32_t y, int order) {
    uint64_t d = 0;
    for (uint32_t s = 1u << (order - 1); s > 0; s >>= 1) {
        uint32_t rx = (x & s) ? 1 : 0, ry = (y & s) ? 1 : 0;
        d += (uint64_t)s * s * ((3 * rx) ^ ry);
        if (ry == 0) {
            if (rx == 1) {
                x = s - 1 - x;
                y = s - 1 - y;
            }
            std::swap(x, y);
        }
    }
    return d;
}
// 3-D Morton index (spherical meshes) on a 2^21 grid per axis.
uint64_t spread3(uint64_t v) {
    v &= 0x1fffff;
    v = (v | v << 32) & 0x1f00000000ffffULL;
    v = (v | v << 16) & 0x1f0000ff0000ffULL;
    v = (v | v << 8) & 0x100f00f00f00f00fULL;
    v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
    v = (v | v << 2) & 0x1249249249249249ULL;
    return v;
}

std::vector<uint64_t> sfc_keys(const HostMesh &m) {
    std::vector<uint64_t> key(m.nC);
    // spherical meshes: Hilbert per cube face (default; config 3 measured 2 % faster per step than 3-D
    // Morton, profiles/r2_sfc_config3.txt) or 3-D Morton (FBLTS_SFC=morton); the order changes only the
    // layout, never the arithmetic (every per-cell sum keeps its slot order)
    const char *sfc = std::getenv("FBLTS_SFC");
    const bool sphere_hilbert = !(sfc && std::string(sfc) == "morton");
    bool planar = true;
    for (int i = 0; i < m.nC && planar; ++i) planar = m.z[i] == 0.0;
    auto q = [](double v, double lo, double hi, double n) {
        double t = hi > lo ? (v - lo) / (hi - lo) : 0.0;
        t = std::min(std::max(t, 0.0), 1.0);
        return (uint32_t)std::min(n - 1.0, std::floor(t * n));
    };
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int i = 0; i < m.nC; ++i) {
        const double p[3] = {m.x[i], m.y[i], m.z[i]};
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], p[a]);
            hi[a] = std::max(hi[a], p[a]);
        }
    }
    for (int i = 0; i < m.nC; ++i) {
        if (planar) {
            key[i] = hilbert2(q(m.x[i], lo[0], hi[0], 65536.0), q(m.y[i], lo[1], hi[1], 65536.0), 16);
        } else if (sphere_hilbert) {
            // Hilbert curve per cube face: the face of the largest |coordinate|, the other two
            // coordinates projected gnomonically to [-1, 1], a 2^20-grid Hilbert index inside the face;
            // faces concatenated in the order +x, +y, -x, -y, +z, -z
            const double p[3] = {m.x[i], m.y[i], m.z[i]};
            int a = 0;
            for (int k = 1; k < 3; ++k)
                if (std::fabs(p[k]) > std::fabs(p[a])) a = k;
            const bool neg = p[a] < 0.0;
            const int face = a == 2 ? (neg ? 5 : 4) : (neg ? 2 + a : a);
            const double w = std::fabs(p[a]);
            const double pu = p[(a + 1) % 3] / w, pv = p[(a + 2) % 3] / w;
            key[i] = (uint64_t)face << 40 | hilbert2(q(pu, -1.0, 1.0, 1048576.0), q(pv, -1.0, 1.0, 1048576.0), 20);
        } else {
            key[i] = spread3(q(m.x[i], lo[0], hi[0], 2097152.0)) | spread3(q(m.y[i], lo[1], hi[1], 2097152.0)) << 1 |
                     spread3(q(m.z[i], lo[2], hi[2], 2097152.0)) << 2;
        }
    }
    return key;
}

// ---------------------------------------------------------------- labelling
// Multi-source BFS hop distance over cell neighbours (INT32_MAX when unreachable).
std::vector<int32_t> hops(const HostMesh &m, const std::vector<int32_t> &coc, const std::vector<uint8_t> &src) {
    std::vector<int32_t> d(m.nC, INT32_MAX), queue;
    queue.reserve(m.nC);
    for (int i = 0; i < m.nC; ++i)
        if (src[i]) {
            d[i] = 0;
            queue.push_back(i);
        }
    for (size_t h = 0; h < queue.size(); ++h) {
        const int i = queue[h];
        for (int j = 0; j < m.nEoC[i]; ++j) {
            const int nb = coc[(size_t)i * m.maxE + j];
            if (d[nb] == INT32_MAX) {
                d[nb] = d[i] + 1;
                queue.push_back(nb);
            }
        }
    }
    return d;
}

int region_class(int code) { return code < 3 ? code : 3; }


// ---------------------------------------------------------------- NCCL transport (nranks > 1)
int nccl_init(fblts_ctx *c) {
    ncclUniqueId id;
    std::memcpy(&id, c->cfg.nccl_id, sizeof id);
    ncclComm_t comm;
    const ncclResult_t r = ncclCommInitRank(&comm, c->cfg.nranks, id, c->cfg.rank);
    if (r != ncclSuccess) return fail(c, FBLTS_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    c->nccl = comm;
    return FBLTS_OK;
}

void nccl_destroy(fblts_ctx *c) {
    if (c->nccl) ncclCommDestroy((ncclComm_t)c->nccl);
    c->nccl = nullptr;
}

#define NCCL_TRY(ctx, call)                                                                            \
    do {                                                                                               \
        ncclResult_t r_ = (call);                                                                      \
        if (r_ != ncclSuccess) return fail(ctx, FBLTS_ERR_NCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
    } while (0)

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char *fblts_kernel_name(int32_t kind) { return (kind >= 0 && kind < K_NUM) ? kKernelNames[kind] : "?"; }

const char *fblts_last_error(const fblts_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int fblts_nccl_unique_id(void *out128) {
    if (!out128) return FBLTS_ERR_INVALID_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return FBLTS_ERR_NCCL;
    std::memcpy(out128, &id, sizeof id);
    return FBLTS_OK;
}

int fblts_create(fblts_ctx **out, const fblts_config *cfg) {
    if (!out || !cfg) return FBLTS_ERR_INVALID_ARG;
    *out = nullptr;
    if (!(cfg->dt > 0.0) || cfg->M < 1 || cfg->r < 1 || !(cfg->g > 0.0) || !(cfg->rho0 > 0.0))
        return FBLTS_ERR_INVALID_ARG;
    if (!(cfg->sal_beta >= 0.0 && cfg->sal_beta < 1.0)) return FBLTS_ERR_INVALID_ARG;
    if (cfg->nranks < 1 || cfg->nranks > 64 || cfg->rank < 0 || cfg->rank >= cfg->nranks) return FBLTS_ERR_INVALID_ARG;
    if (cfg->scheme != FBLTS_SCHEME_FBLTS && cfg->scheme != FBLTS_SCHEME_RK4 && cfg->scheme != FBLTS_SCHEME_RK32)
        return FBLTS_ERR_INVALID_ARG;
    if (cfg->scheme != FBLTS_SCHEME_FBLTS && cfg->nranks != 1) return FBLTS_ERR_INVALID_ARG;   // reference schemes: one rank
    if (cfg->slow_refresh && (cfg->nranks != 1 || cfg->scheme != FBLTS_SCHEME_FBLTS)) return FBLTS_ERR_INVALID_ARG;
    if (cfg->unsplit && (cfg->nranks != 1 || cfg->scheme != FBLTS_SCHEME_FBLTS || cfg->slow_refresh))
        return FBLTS_ERR_INVALID_ARG;
    if (cfg->pv_energy && (cfg->nranks != 1 || cfg->slow_refresh)) return FBLTS_ERR_INVALID_ARG;
    if (cfg->vorticity && (cfg->nranks != 1 || cfg->slow_refresh || cfg->scheme != FBLTS_SCHEME_FBLTS))
        return FBLTS_ERR_INVALID_ARG;
    // No CUDA call here: mesh upload, labelling and renumbering are host work, so a context
    // can be created (and its labels inspected) on a machine without a GPU.
    fblts_ctx *c = new fblts_ctx();
    c->cfg = *cfg;
    if (cfg->nccl_id) {                          // the caller's buffer is only borrowed
        std::memcpy(c->nccl_id, cfg->nccl_id, sizeof c->nccl_id);
        c->cfg.nccl_id = c->nccl_id;
    }
    c->stream = (cudaStream_t)cfg->stream;
    if (const char *ev = std::getenv("FBLTS_TILED")) c->tiled = std::atoi(ev) != 0;
    if (const char *ev = std::getenv("FBLTS_SPLIT")) c->split = std::atoi(ev) != 0;
    if (const char *ev = std::getenv("FBLTS_FUSE")) c->fuse_vel = std::atoi(ev) != 0;
    if (const char *ev = std::getenv("FBLTS_SUB")) c->fuse_sub = std::atoi(ev) != 0;
    if (const char *ev = std::getenv("FBLTS_BAND_SIDE")) c->band_side = std::atoi(ev) != 0;
    if (const char *ev = std::getenv("FBLTS_SUB_LEVEL")) c->sub_level = std::min(5, std::max(2, std::atoi(ev)));
    if (cfg->nranks != 1 || cfg->scheme != FBLTS_SCHEME_FBLTS || cfg->slow_refresh || cfg->unsplit) c->fuse_sub = false;
    // canonical constants (computed once in double, SURVEY c.1)
    StepConst &s = c->sc;
    const double dt = cfg->dt;
    const double M = (double)cfg->M;
    s.g = cfg->g * (1.0 - cfg->sal_beta);      // fast term -g grad(xi - beta xi)
    s.rho0 = cfg->rho0;
    s.pve = cfg->pv_energy ? 1 : 0;
    s.b1 = cfg->beta[0];
    s.b2 = cfg->beta[1];
    s.b3 = cfg->beta[2];
    s.omb1 = 1.0 - s.b1;
    s.omb2 = 1.0 - s.b2;
    s.om2b3 = 1.0 - 2.0 * s.b3;
    s.c1 = dt / 3.0;
    s.c2 = dt / 2.0;
    s.c3 = dt;
    s.c1f = dt / (3.0 * M);
    s.c2f = dt / (2.0 * M);
    s.c3f = dt / M;
    s.M = cfg->M;
    *out = c;
    return FBLTS_OK;
}

int fblts_upload_mesh(fblts_ctx *c, const fblts_mesh *m) {
    if (!c || !m) return FBLTS_ERR_INVALID_ARG;
    if (c->phase != P_CREATED) return fail(c, FBLTS_ERR_ORDER, "upload_mesh: mesh already uploaded");
    const int nC = m->nCells, nE = m->nEdges, nV = m->nVertices, mE = m->maxEdges, mE2 = m->maxEdges2;
    if (nC <= 0 || nE <= 0 || nV <= 0 || mE < 3 || mE > 16 || mE2 < 1 || mE2 > 30)
        return fail(c, FBLTS_ERR_MESH, "mesh counts: nCells=%d nEdges=%d nVertices=%d maxEdges=%d maxEdges2=%d", nC,
                    nE, nV, mE, mE2);
    if (!m->nEdgesOnCell || !m->edgesOnCell || !m->cellsOnEdge || !m->verticesOnEdge || !m->nEdgesOnEdge ||
        !m->edgesOnEdge || !m->weightsOnEdge || !m->edgesOnVertex || !m->cellsOnVertex || !m->kiteAreasOnVertex ||
        !m->areaCell || !m->areaTriangle || !m->dvEdge || !m->dcEdge || !m->fVertex || !m->bottomDepth ||
        !m->xCell || !m->yCell || !m->zCell)
        return fail(c, FBLTS_ERR_INVALID_ARG, "upload_mesh: a mesh array pointer is NULL");
    HostMesh &h = c->hm;
    h.nC = nC, h.nE = nE, h.nV = nV, h.maxE = mE, h.maxE2 = mE2;
    h.nEoC.assign(m->nEdgesOnCell, m->nEdgesOnCell + nC);
    h.eoc.assign(m->edgesOnCell, m->edgesOnCell + (size_t)nC * mE);
    h.coe.assign(m->cellsOnEdge, m->cellsOnEdge + (size_t)nE * 2);
    h.voe.assign(m->verticesOnEdge, m->verticesOnEdge + (size_t)nE * 2);
    h.nEoE.assign(m->nEdgesOnEdge, m->nEdgesOnEdge + nE);
    h.eoe.assign(m->edgesOnEdge, m->edgesOnEdge + (size_t)nE * mE2);
    h.W.assign(m->weightsOnEdge, m->weightsOnEdge + (size_t)nE * mE2);
    h.eov.assign(m->edgesOnVertex, m->edgesOnVertex + (size_t)nV * 3);
    h.cov.assign(m->cellsOnVertex, m->cellsOnVertex + (size_t)nV * 3);
    h.kite.assign(m->kiteAreasOnVertex, m->kiteAreasOnVertex + (size_t)nV * 3);
    h.areaCell.assign(m->areaCell, m->areaCell + nC);
    h.areaTri.assign(m->areaTriangle, m->areaTriangle + nV);
    h.dv.assign(m->dvEdge, m->dvEdge + nE);
    h.dc.assign(m->dcEdge, m->dcEdge + nE);
    h.fV.assign(m->fVertex, m->fVertex + nV);
    h.H.assign(m->bottomDepth, m->bottomDepth + nC);
    h.x.assign(m->xCell, m->xCell + nC);
    h.y.assign(m->yCell, m->yCell + nC);
    h.z.assign(m->zCell, m->zCell + nC);
    // ---- validation (structured errors name field and index)
    auto fin_pos = [](double v) { return std::isfinite(v) && v > 0.0; };
    for (int i = 0; i < nC; ++i) {
        if (h.nEoC[i] < 3 || h.nEoC[i] > mE) return fail(c, FBLTS_ERR_MESH, "nEdgesOnCell[%d]=%d", i, h.nEoC[i]);
        if (!fin_pos(h.areaCell[i])) return fail(c, FBLTS_ERR_MESH, "areaCell[%d]=%g", i, h.areaCell[i]);
        if (!fin_pos(h.H[i])) return fail(c, FBLTS_ERR_MESH, "bottomDepth[%d]=%g", i, h.H[i]);
    }
    for (int e = 0; e < nE; ++e) {
        const int a = h.coe[2 * e], b = h.coe[2 * e + 1];
        if (a < 0 || a >= nC || b < 0 || b >= nC || a == b)
            return fail(c, FBLTS_ERR_MESH, "cellsOnEdge[%d]=(%d,%d)", e, a, b);
        const int v0 = h.voe[2 * e], v1 = h.voe[2 * e + 1];
        if (v0 < 0 || v0 >= nV || v1 < 0 || v1 >= nV || v0 == v1)
            return fail(c, FBLTS_ERR_MESH, "verticesOnEdge[%d]=(%d,%d)", e, v0, v1);
        if (!fin_pos(h.dv[e])) return fail(c, FBLTS_ERR_MESH, "dvEdge[%d]=%g", e, h.dv[e]);
        if (!fin_pos(h.dc[e])) return fail(c, FBLTS_ERR_MESH, "dcEdge[%d]=%g", e, h.dc[e]);
        if (h.nEoE[e] < 0 || h.nEoE[e] > mE2) return fail(c, FBLTS_ERR_MESH, "nEdgesOnEdge[%d]=%d", e, h.nEoE[e]);
        for (int j = 0; j < h.nEoE[e]; ++j) {
            const int x = h.eoe[(size_t)e * mE2 + j];
            if (x < 0 || x >= nE) return fail(c, FBLTS_ERR_MESH, "edgesOnEdge[%d][%d]=%d", e, j, x);
            if (!std::isfinite(h.W[(size_t)e * mE2 + j]))
                return fail(c, FBLTS_ERR_MESH, "weightsOnEdge[%d][%d] not finite", e, j);
        }
    }
    std::vector<int8_t> seen(nE, 0);
    for (int i = 0; i < nC; ++i) {
        for (int j = 0; j < h.nEoC[i]; ++j) {
            const int e = h.eoc[(size_t)i * mE + j];
            if (e < 0 || e >= nE) return fail(c, FBLTS_ERR_MESH, "edgesOnCell[%d][%d]=%d", i, j, e);
            if (h.coe[2 * e] != i && h.coe[2 * e + 1] != i)
                return fail(c, FBLTS_ERR_MESH, "edgesOnCell[%d][%d]=%d but cellsOnEdge[%d]=(%d,%d)", i, j, e, e,
                            h.coe[2 * e], h.coe[2 * e + 1]);
            if (++seen[e] > 2) return fail(c, FBLTS_ERR_MESH, "edge %d listed by more than two cells", e);
        }
    }
    for (int e = 0; e < nE; ++e)
        if (seen[e] != 2) return fail(c, FBLTS_ERR_MESH, "edge %d appears in edgesOnCell %d times (need 2)", e, seen[e]);
    for (int v = 0; v < nV; ++v) {
        if (!fin_pos(h.areaTri[v])) return fail(c, FBLTS_ERR_MESH, "areaTriangle[%d]=%g", v, h.areaTri[v]);
        if (!std::isfinite(h.fV[v])) return fail(c, FBLTS_ERR_MESH, "fVertex[%d] not finite", v);
        for (int k = 0; k < 3; ++k) {
            const int e = h.eov[3 * v + k], ci = h.cov[3 * v + k];
            if (e < 0 || e >= nE || (h.voe[2 * e] != v && h.voe[2 * e + 1] != v))
                return fail(c, FBLTS_ERR_MESH, "edgesOnVertex[%d][%d]=%d", v, k, e);
            if (ci < 0 || ci >= nC) return fail(c, FBLTS_ERR_MESH, "cellsOnVertex[%d][%d]=%d", v, k, ci);
            if (!(h.kite[3 * v + k] >= 0.0)) return fail(c, FBLTS_ERR_MESH, "kiteAreasOnVertex[%d][%d]", v, k);
        }
    }
    c->phase = P_MESH;
    return FBLTS_OK;
}

}  // extern "C"

namespace {

// ---------------------------------------------------------------- partition + local subdomain
// Dual-set partition: the fine set and the coarse set (int + IF) are each sorted
// by space-filling-curve key and cut into nranks equal contiguous chunks; rank r owns chunk r of
// both, so the coarse phase and the fine phase are each balanced.
std::vector<int32_t> partition(const HostMesh &m, const Region &g, const std::vector<uint64_t> &key, int nranks) {
    std::vector<int32_t> part(m.nC, 0);
    if (nranks == 1) return part;
    for (int fineSet = 0; fineSet < 2; ++fineSet) {
        std::vector<int32_t> ids;
        for (int i = 0; i < m.nC; ++i)
            if ((g.cell[i] >= FBLTS_REGION_F1) == (fineSet == 1)) ids.push_back(i);
        std::stable_sort(ids.begin(), ids.end(), [&](int a, int b) { return key[a] < key[b]; });
        const size_t n = ids.size();
        for (int r = 0; r < nranks; ++r)
            for (size_t k = n * r / nranks; k < n * (r + 1) / nranks; ++k) part[ids[k]] = r;
    }
    return part;
}

// hop distance (0, 1, 2, 3 = farther) from the cells owned by rank p
std::vector<int8_t> dist_from(const HostMesh &m, const std::vector<int32_t> &coc, const std::vector<int32_t> &part,
                              int p) {
    std::vector<int8_t> d(m.nC, 3);
    for (int i = 0; i < m.nC; ++i)
        if (part[i] == p) d[i] = 0;
    for (int ring = 1; ring <= 2; ++ring)
        for (int i = 0; i < m.nC; ++i)
            if (d[i] == ring - 1)
                for (int j = 0; j < m.nEoC[i]; ++j) {
                    const int nb = coc[(size_t)i * m.maxE + j];
                    if (d[nb] == 3) d[nb] = (int8_t)ring;
                }
    return d;
}

Bounds bounds_from(const int64_t *cnt, int begin, int end) {
    Bounds b{};
    b.begin = begin;
    b.if2 = begin + (int)cnt[0];
    b.if1 = b.if2 + (int)cnt[1];
    b.f = b.if1 + (int)cnt[2];
    b.fl[0] = b.f;
    for (int l = 1; l <= 5; ++l) b.fl[l] = b.fl[l - 1] + (int)cnt[2 + l];
    b.end = end;
    return b;
}

// Tiles of the owned cells for the staged stage kernels (fblts_internal.h TileMesh): tile starts
// every TILE cells inside each region block, so every stage extent is a whole number of tiles.
int build_tiles(fblts_ctx *c) {
    const Local &L = c->lo;
    const int G = c->ecS, maxE = c->hm.maxE;
    std::vector<int32_t> bnd;
    for (const Bounds *b : {&L.cb, &L.cbI}) {
        bnd.insert(bnd.end(), {b->begin, b->if2, b->if1, b->f});
        for (int l = 1; l <= 5; ++l) bnd.push_back(b->fl[l]);
        bnd.push_back(b->end);
    }
    std::sort(bnd.begin(), bnd.end());
    bnd.erase(std::unique(bnd.begin(), bnd.end()), bnd.end());
    std::vector<int32_t> &ts = c->t_start;
    ts.clear();
    for (size_t k = 0; k + 1 < bnd.size(); ++k)
        for (int s = bnd[k]; s < bnd[k + 1]; s += TILE) ts.push_back(s);
    ts.push_back(L.nOwnC);
    const int nT = (int)ts.size() - 1;
    c->t_sRow = pad32(std::max(1, L.nOwnC));
    c->t_info.assign((size_t)(nT + 1) * TINFO, 0);
    c->t_halo.clear();
    c->t_fedge.clear();
    c->t_ecl.clear();
    c->t_row.assign((size_t)maxE * c->t_sRow, TILE_SENT);
    c->t_hmax = 0;
    c->t_emax = 0;
    std::vector<int32_t> hl, el, fl;
    for (int t = 0; t < nT; ++t) {
        const int c0 = ts[t], c1 = ts[t + 1];
        hl.clear();
        el.clear();
        fl.clear();
        for (int i = c0; i < c1; ++i)
            for (int j = 0; j < c->d_nEoC[i]; ++j) {
                const int es = c->d_ec[((size_t)i * G + j) * 2], nb = c->d_ec[((size_t)i * G + j) * 2 + 1];
                el.push_back(es >= 0 ? es : ~es);
                if (nb < c0 || nb >= c1) hl.push_back(nb);
            }
        std::sort(hl.begin(), hl.end());
        hl.erase(std::unique(hl.begin(), hl.end()), hl.end());
        std::sort(el.begin(), el.end());
        el.erase(std::unique(el.begin(), el.end()), el.end());
        // owned run: the longest run of consecutive indices among the edges whose owner cell is in
        // the tile (all of them with one rank); every other local edge is foreign
        size_t best = 0, bestLen = 0;
        auto owned = [&](size_t k) { return c->e_owner[el[k]] >= c0 && c->e_owner[el[k]] < c1; };
        for (size_t k = 0; k < el.size();) {
            if (!owned(k)) {
                ++k;
                continue;
            }
            size_t k2 = k + 1;
            while (k2 < el.size() && owned(k2) && el[k2] == el[k2 - 1] + 1) ++k2;
            if (k2 - k > bestLen) best = k, bestLen = k2 - k;
            k = k2;
        }
        const int eo0 = bestLen ? el[best] : 0, eo1 = eo0 + (int)bestLen;
        for (int e : el)
            if (e < eo0 || e >= eo1) fl.push_back(e);
        const int nLE = (int)el.size();
        if (nLE + FGAP >= 0x7FFF || HALO0 + (int)hl.size() > 0xFFFF)
            return fail(c, FBLTS_ERR_MESH, "tiles: tile %d has %d edges / %zu halo cells (too many)", t, nLE, hl.size());
        int32_t *rec = &c->t_info[(size_t)t * TINFO];
        rec[0] = c0, rec[1] = (int32_t)c->t_halo.size(), rec[2] = eo0, rec[3] = eo1;
        rec[4] = (int32_t)c->t_fedge.size(), rec[5] = (int32_t)c->t_ecl.size();
        auto lcell = [&](int x) {
            return (uint32_t)((x >= c0 && x < c1) ? x - c0
                                                  : HALO0 + (std::lower_bound(hl.begin(), hl.end(), x) - hl.begin()));
        };
        auto ledge = [&](int e) {
            return (uint32_t)((e >= eo0 && e < eo1) ? e - eo0
                                                    : (eo1 - eo0) + FGAP + (std::lower_bound(fl.begin(), fl.end(), e) - fl.begin()));
        };
        for (int i = c0; i < c1; ++i)
            for (int j = 0; j < c->d_nEoC[i]; ++j) {
                const int es = c->d_ec[((size_t)i * G + j) * 2];
                c->t_row[(size_t)j * c->t_sRow + i] = (uint16_t)((es < 0 ? 0x8000u : 0u) | ledge(es >= 0 ? es : ~es));
            }
        auto push_pair = [&](int e) {
            c->t_ecl.push_back(lcell(c->d_coe[2 * e + 1]) << 16 | lcell(c->d_coe[2 * e]));
        };
        for (int e = eo0; e < eo1; ++e) push_pair(e);
        for (int e : fl) push_pair(e);
        c->t_halo.insert(c->t_halo.end(), hl.begin(), hl.end());
        c->t_fedge.insert(c->t_fedge.end(), fl.begin(), fl.end());
        c->t_hmax = std::max(c->t_hmax, (int)hl.size());
        c->t_emax = std::max(c->t_emax, nLE);
    }
    int32_t *rec = &c->t_info[(size_t)nT * TINFO];
    rec[0] = L.nOwnC, rec[1] = (int32_t)c->t_halo.size(), rec[4] = (int32_t)c->t_fedge.size();
    rec[5] = (int32_t)c->t_ecl.size();
    // ghost layout: tile t's halo cells at [g0, g0 + nH) with g0 of the parity of its first cell, its
    // foreign edges at [ge0, ge0 + nF) with ge0 of the parity of its owned run's end (the bulk copies'
    // 16-byte alignment, kernels.cu issue_bulk); a padding slot may precede and follow each range
    {
        c->g_cidx.assign(1, -1);
        c->g_eidx.assign(1, -1);
        for (int t = 0; t < nT; ++t) {
            int32_t *r = &c->t_info[(size_t)t * TINFO];
            const int32_t *n = r + TINFO;
            const int oc = r[0] & 1, pe = r[3] & 1;
            if (((int)c->g_cidx.size() & 1) != oc) c->g_cidx.push_back(-1);
            r[6] = (int32_t)c->g_cidx.size();
            for (int q = r[1]; q < n[1]; ++q) c->g_cidx.push_back(c->t_halo[q]);
            if (((int)c->g_eidx.size() & 1) != pe) c->g_eidx.push_back(-1);
            r[7] = (int32_t)c->g_eidx.size();
            for (int q = r[4]; q < n[4]; ++q) c->g_eidx.push_back(c->t_fedge[q]);
        }
        rec[6] = (int32_t)c->g_cidx.size();
        rec[7] = (int32_t)c->g_eidx.size();
        for (int k = 0; k < 3; ++k) {            // slack of the last ranges' even-length copies
            c->g_cidx.push_back(-1);
            c->g_eidx.push_back(-1);
        }
    }
    // the fused deep velocity + stage-1 sweep writes each deep edge from the tile whose owned run
    // holds it: usable only if those runs tile [eb.fl[1], eb.end) exactly
    {
        std::vector<std::pair<int, int>> runs;
        for (int t = 0; t < nT; ++t) {
            const int c0 = ts[t];
            const bool deep = (c0 >= L.cb.fl[1] && c0 < L.cb.end) || (c0 >= L.cbI.fl[1] && c0 < L.cbI.end);
            const int32_t *rec = &c->t_info[(size_t)t * TINFO];
            if (deep && rec[3] > rec[2]) runs.push_back({rec[2], rec[3]});
        }
        std::sort(runs.begin(), runs.end());
        int at = L.eb.fl[1];
        bool ok = true;
        for (auto &r : runs) {
            if (r.first != at) ok = false;
            at = r.second;
        }
        c->deep_runs_ok = ok && at == L.eb.end;
    }
    c->t_nHalo = c->t_halo.size();
    c->t_nFedge = c->t_fedge.size();
    c->t_nEcl = c->t_ecl.size();
    if (c->t_halo.empty()) c->t_halo.push_back(0);
    if (c->t_fedge.empty()) c->t_fedge.push_back(0);
    if (c->t_ecl.empty()) c->t_ecl.push_back(0);
    return FBLTS_OK;
}

// Subcycle tiles (fblts_internal.h SubTileMesh): the tiles of build_tiles that lie in F\F^2 of the
// (single) owned block, each with its rings R1-R3, the edges of its rings 0-2 and their slot tables.
// A cell of F\F^2 is at least 5 hops from every coarse cell (r = 2), so its 3-ring neighbourhood is
// fine (a fine cell's value is its fine data in every view): the tile needs no region views, and
// the band kernels (cells of F^1 and coarser, at most 3 hops into F) never read its cells.
int build_subtiles(fblts_ctx *c) {
    c->s_nT = 0;
    c->s_info.assign(FTINFO, 0);
    c->s_halo.clear();
    c->s_fedge.clear();
    c->s_ecl.clear();
    c->s_row.clear();
    c->s_hmax = c->s_emax = c->s_rmax = 0;
    const Local &L = c->lo;
    if (!c->fuse_sub || L.cbI.end > L.cbI.begin || c->t_start.size() < 2) {
        c->fuse_sub = false;
        return FBLTS_OK;
    }
    // the bulk F\F^5 by default: the thin 2-hop bands F^3\F^2 .. F^5\F^4 cut into 256-cell tiles are
    // long strips whose 3-ring halos would triple the tile (FBLTS_SUB_LEVEL = 2..5 moves the start)
    const int G = c->ecS, maxE = c->hm.maxE, lo = L.cb.fl[c->sub_level], hi = L.cb.end;
    std::vector<int8_t> ring(L.nC, -1);
    std::vector<int32_t> lidx(L.nC, -1);
    std::vector<int32_t> R[4], el, fl[3];
    auto nbr = [&](int i, int j) { return c->d_ec[((size_t)i * G + j) * 2 + 1]; };
    auto edg = [&](int i, int j) {
        const int es = c->d_ec[((size_t)i * G + j) * 2];
        return es >= 0 ? es : ~es;
    };
    const int nT = (int)c->t_start.size() - 1;
    // each staged tile of the range becomes nsplit subcycle tiles; nsplit doubles (up to 4) while the
    // double-buffered footprint exceeds the shared memory (irregular tiles, e.g. on SCVT spheres)
    for (int nsplit = 1;; nsplit *= 2) {
    c->s_nT = 0;
    c->s_info.assign(FTINFO, 0);
    c->s_halo.clear();
    c->s_fedge.clear();
    c->s_ecl.clear();
    c->s_row.clear();
    c->s_hmax = c->s_emax = c->s_rmax = 0;
    for (int tt = 0; tt < nT * nsplit; ++tt) {
        const int t = tt / nsplit, part = tt % nsplit;
        const int T0 = c->t_start[t], T1 = c->t_start[t + 1];
        if (T0 < lo || T0 >= hi) continue;
        const int c0 = T0 + (int)((int64_t)(T1 - T0) * part / nsplit);
        const int c1 = T0 + (int)((int64_t)(T1 - T0) * (part + 1) / nsplit);
        if (c1 <= c0) continue;
        R[0].clear();
        for (int i = c0; i < c1; ++i) R[0].push_back(i), ring[i] = 0;
        for (int k = 1; k <= 3; ++k) {
            R[k].clear();
            for (int i : R[k - 1])
                for (int j = 0; j < c->d_nEoC[i]; ++j) {
                    const int nb = nbr(i, j);
                    if (nb < 0 || nb >= L.nOwnC) return fail(c, FBLTS_ERR_LABELS, "subtiles: tile %d reaches a halo cell", t);
                    if (ring[nb] < 0) ring[nb] = (int8_t)k, R[k].push_back(nb);
                }
            std::sort(R[k].begin(), R[k].end());
        }
        for (int k = 1; k <= 3; ++k)
            for (int x : R[k])
                if (x < L.cb.f)
                    return fail(c, FBLTS_ERR_LABELS, "subtiles: tile %d: ring-%d cell %d is not fine", t, k, x);
        const int nOwn = c1 - c0, n1 = (int)R[1].size(), n2 = (int)R[2].size(), n3 = (int)R[3].size();
        int q = 0;
        for (int i = c0; i < c1; ++i) lidx[i] = i - c0;
        for (int k = 1; k <= 3; ++k)
            for (int x : R[k]) lidx[x] = HALO0 + q++;
        bool border = false;
        for (int x : R[1]) border = border || x < lo;
        // local edges: every edge of a ring-0..2 cell; owned run of the staged tile, foreign by ring
        el.clear();
        for (int k = 0; k <= 2; ++k)
            for (int i : R[k])
                for (int j = 0; j < c->d_nEoC[i]; ++j) el.push_back(edg(i, j));
        std::sort(el.begin(), el.end());
        el.erase(std::unique(el.begin(), el.end()), el.end());
        const int32_t *trec = &c->t_info[(size_t)t * TINFO];
        int eo0 = trec[2], eo1 = trec[3];
        if (nsplit > 1) {           // the part's owned edges: the sub-run whose owner lies in [c0, c1)
            int a = eo0, b, cnt = 0;
            while (a < eo1 && c->e_owner[a] < c0) ++a;
            for (b = a; b < eo1 && c->e_owner[b] < c1; ++b) {}
            for (int e = trec[2]; e < trec[3]; ++e) cnt += c->e_owner[e] >= c0 && c->e_owner[e] < c1;
            if (cnt != b - a) {     // owners not monotone along the run: no split
                c->fuse_sub = false;
                return FBLTS_OK;
            }
            eo0 = a, eo1 = b;
        }
        const int nOE = eo1 - eo0;
        for (auto &f : fl) f.clear();
        for (int e : el) {
            const int r0 = ring[c->d_coe[2 * e]], r1 = ring[c->d_coe[2 * e + 1]];
            if (r0 < 0 || r1 < 0) return fail(c, FBLTS_ERR_LABELS, "subtiles: edge %d leaves the 3-ring set", e);
            const int mr = std::min(r0, r1);
            if (e >= eo0 && e < eo1) {
                if (mr != 0) return fail(c, FBLTS_ERR_LABELS, "subtiles: owned edge %d not on the tile", e);
                continue;
            }
            fl[mr].push_back(e);
        }
        const int nF = (int)(fl[0].size() + fl[1].size() + fl[2].size());
        if (nOE + FGAP + nF >= 0x7FFF || HALO0 + n1 + n2 + n3 > 0xFFFF)
            return fail(c, FBLTS_ERR_MESH, "subtiles: tile %d has %d edges / %d halo cells (too many)", t, nOE + nF,
                        n1 + n2 + n3);
        int32_t *rec = &c->s_info[(size_t)c->s_nT * FTINFO];
        rec[0] = c0, rec[1] = c1, rec[2] = (int32_t)c->s_halo.size(), rec[3] = n1, rec[4] = n2, rec[5] = n3;
        rec[6] = eo0, rec[7] = eo1, rec[8] = (int32_t)c->s_fedge.size();
        rec[9] = (int32_t)fl[0].size(), rec[10] = (int32_t)fl[1].size(), rec[11] = (int32_t)fl[2].size();
        rec[12] = (int32_t)c->s_ecl.size(), rec[13] = (int32_t)c->s_row.size(), rec[14] = border ? 1 : 0;
        for (int k = 1; k <= 3; ++k) c->s_halo.insert(c->s_halo.end(), R[k].begin(), R[k].end());
        // local edge index (q-space: owned run, FGAP, foreign list)
        std::vector<std::pair<int, int>> fpos;     // (edge, q) for the foreign edges
        int p = 0;
        for (auto &f : fl)
            for (int e : f) {
                c->s_fedge.push_back(e);
                fpos.push_back({e, nOE + FGAP + p++});
            }
        std::sort(fpos.begin(), fpos.end());
        auto ledge = [&](int e) {
            if (e >= eo0 && e < eo1) return e - eo0;
            return std::lower_bound(fpos.begin(), fpos.end(), std::make_pair(e, -1))->second;
        };
        auto pair = [&](int e) {
            return (uint32_t)lidx[c->d_coe[2 * e + 1]] << 16 | (uint32_t)lidx[c->d_coe[2 * e]];
        };
        for (int e = eo0; e < eo1; ++e) c->s_ecl.push_back(pair(e));
        for (auto &f : fl)
            for (int e : f) c->s_ecl.push_back(pair(e));
        const int nR2 = nOwn + n1 + n2;
        const size_t rb = c->s_row.size();
        c->s_row.resize(rb + (size_t)maxE * nR2, TILE_SENT);
        int r = 0;
        for (int k = 0; k <= 2; ++k)
            for (int i : R[k]) {
                for (int j = 0; j < c->d_nEoC[i]; ++j) {
                    const int es = c->d_ec[((size_t)i * G + j) * 2];
                    c->s_row[rb + (size_t)j * nR2 + r] = (uint16_t)((es < 0 ? 0x8000u : 0u) | ledge(es >= 0 ? es : ~es));
                }
                ++r;
            }
        c->s_row.resize((c->s_row.size() + 7) & ~(size_t)7, TILE_SENT);     // 16-byte aligned tables
        c->s_rmax = std::max(c->s_rmax, (int)(c->s_row.size() - rb));
        c->s_hmax = std::max(c->s_hmax, n1 + n2 + n3);
        c->s_emax = std::max(c->s_emax, nOE + FGAP + nF);
        for (int k = 0; k <= 3; ++k)
            for (int x : R[k]) ring[x] = -1, lidx[x] = -1;
        ++c->s_nT;
        c->s_info.resize((size_t)(c->s_nT + 1) * FTINFO, 0);
    }
    if (sub_smem_bytes_host(c->s_hmax, c->s_emax, c->s_rmax) <= TILE_SMEM_MAX || nsplit >= 4) break;
    }
    c->s_nHalo = c->s_halo.size(), c->s_nFedge = c->s_fedge.size(), c->s_nEcl = c->s_ecl.size();
    c->s_nRow = c->s_row.size();
    if (c->s_halo.empty()) c->s_halo.push_back(0);
    if (c->s_fedge.empty()) c->s_fedge.push_back(0);
    if (c->s_ecl.empty()) c->s_ecl.push_back(0);
    if (c->s_row.empty()) c->s_row.push_back(0);
    if (c->s_nT == 0 || sub_smem_bytes_host(c->s_hmax, c->s_emax, c->s_rmax) > TILE_SMEM_MAX) c->fuse_sub = false;
    return FBLTS_OK;
}


// first tile of the tile run starting at owned cell `cell` (a region block boundary)
int tile_at(const fblts_ctx *c, int cell) {
    return (int)(std::lower_bound(c->t_start.begin(), c->t_start.end(), cell) - c->t_start.begin());
}

int build_local(fblts_ctx *c, const std::vector<int32_t> &coc) {
    const HostMesh &m = c->hm;
    const Region &g = c->rg;
    Local &L = c->lo;
    const int R = c->cfg.nranks, me = c->cfg.rank;
    const std::vector<uint64_t> key = sfc_keys(m);
    const std::vector<int32_t> part = c->piece ? c->ext_part : partition(m, g, key, R);
    const std::vector<int8_t> dme = dist_from(m, coc, part, me);
    // ---- cells: owned (region-major, SFC) then halo rings 1-2 (region-major, ring, SFC)
    std::vector<int32_t> own, halo;
    for (int i = 0; i < m.nC; ++i) {
        if (dme[i] == 0) own.push_back(i);
        else if (dme[i] <= 2) halo.push_back(i);
    }
    // boundary block first (owned cells with a neighbour owned by another rank: what the peers'
    // ring-1 halos hold), then the interior block; each region-major, SFC inside a region.  With
    // one rank every owned cell is in the first block.
    std::vector<uint8_t> isB(m.nC, R == 1 ? 1 : 0);
    if (R > 1)
        for (int i : own)
            for (int j = 0; j < m.nEoC[i]; ++j)
                if (part[coc[(size_t)i * m.maxE + j]] != me) isB[i] = 1;
    std::stable_sort(own.begin(), own.end(), [&](int a, int b) {
        if (isB[a] != isB[b]) return isB[a] > isB[b];
        if (g.cell[a] != g.cell[b]) return g.cell[a] < g.cell[b];
        return key[a] < key[b];
    });
    std::stable_sort(halo.begin(), halo.end(), [&](int a, int b) {
        if (g.cell[a] != g.cell[b]) return g.cell[a] < g.cell[b];
        if (dme[a] != dme[b]) return dme[a] < dme[b];
        return key[a] < key[b];
    });
    L.nOwnC = (int)own.size();
    L.nB = 0;
    for (int i : own) L.nB += isB[i];
    L.cellGlob = own;
    L.cellGlob.insert(L.cellGlob.end(), halo.begin(), halo.end());
    L.nC = (int)L.cellGlob.size();
    std::vector<int32_t> cellLoc(m.nC, -1);
    for (int i = 0; i < L.nC; ++i) cellLoc[L.cellGlob[i]] = i;
    // ---- edges: touching owned cells (region-major, by owner), then the other edges of ring-1 cells
    std::vector<int32_t> eOwnL, eRest;
    std::vector<int8_t> emark(m.nE, 0);
    for (int k = 0; k < L.nC; ++k) {
        const int i = L.cellGlob[k];
        if (dme[i] > 1) continue;
        for (int j = 0; j < m.nEoC[i]; ++j) {
            const int e = m.eoc[(size_t)i * m.maxE + j];
            if (emark[e]) continue;
            emark[e] = 1;
            const bool touches = dme[m.coe[2 * e]] == 0 || dme[m.coe[2 * e + 1]] == 0;
            (touches ? eOwnL : eRest).push_back(e);
        }
    }
    // edge owner: the cell whose region code is the edge's (the smaller local index on a tie),
    // falling back to an owned cell; then edges sorted by (code, owner) are also contiguous per
    // owner-cell range, which gives every cell tile a contiguous range of its edges
    auto eowner = [&](int e) {
        const int a = m.coe[2 * e], b = m.coe[2 * e + 1];
        const int la = cellLoc[a], lb = cellLoc[b];
        const bool ma = g.cell[a] == g.edge[e] && la >= 0 && la < (int)own.size();
        const bool mb = g.cell[b] == g.edge[e] && lb >= 0 && lb < (int)own.size();
        if (ma && mb) return std::min(la, lb);
        if (ma) return la;
        if (mb) return lb;
        if (la >= 0 && lb >= 0) return std::min(la, lb);
        return la >= 0 ? la : lb;
    };
    std::stable_sort(eOwnL.begin(), eOwnL.end(), [&](int a, int b) {
        if (g.edge[a] != g.edge[b]) return g.edge[a] < g.edge[b];
        return eowner(a) < eowner(b);
    });
    std::stable_sort(eRest.begin(), eRest.end(), [&](int a, int b) { return eowner(a) < eowner(b); });
    c->e_owner.resize(eOwnL.size() + eRest.size());
    L.nOwnE = (int)eOwnL.size();
    L.edgeGlob = eOwnL;
    L.edgeGlob.insert(L.edgeGlob.end(), eRest.begin(), eRest.end());
    L.nE = (int)L.edgeGlob.size();
    std::vector<int32_t> edgeLoc(m.nE, -1);
    for (int e = 0; e < L.nE; ++e) edgeLoc[L.edgeGlob[e]] = e;
    for (int e = 0; e < L.nE; ++e) c->e_owner[e] = eowner(L.edgeGlob[e]);   // local owner cell (tiles)
    // ---- vertices: those of the edges touching owned cells, by owner cell
    std::vector<int32_t> verts;
    std::vector<int8_t> vmark(m.nV, 0);
    for (int k = 0; k < L.nOwnE; ++k) {
        const int e = L.edgeGlob[k];
        for (int s = 0; s < 2; ++s) {
            const int v = m.voe[2 * e + s];
            if (!vmark[v]) {
                vmark[v] = 1;
                verts.push_back(v);
            }
        }
    }
    auto vowner = [&](int v) {
        int o = INT32_MAX;
        for (int k = 0; k < 3; ++k) {
            const int l = cellLoc[m.cov[3 * v + k]];
            if (l >= 0) o = std::min(o, l);
        }
        return o;
    };
    std::stable_sort(verts.begin(), verts.end(), [&](int a, int b) { return vowner(a) < vowner(b); });
    L.vertGlob = verts;
    L.nV = (int)verts.size();
    std::vector<int32_t> vertLoc(m.nV, -1);
    for (int v = 0; v < L.nV; ++v) vertLoc[L.vertGlob[v]] = v;
    // ---- bounds (owned cells, halo cells, edges touching owned)
    std::fill(L.ocount, L.ocount + 9, 0);
    std::fill(L.oecount, L.oecount + 9, 0);
    int64_t hcount[9] = {0};
    int64_t bcount[9] = {0}, icount[9] = {0};
    for (int k = 0; k < L.nOwnC; ++k) {
        L.ocount[g.cell[L.cellGlob[k]]]++;
        (k < L.nB ? bcount : icount)[g.cell[L.cellGlob[k]]]++;
    }
    for (int k = L.nOwnC; k < L.nC; ++k) hcount[g.cell[L.cellGlob[k]]]++;
    for (int k = 0; k < L.nOwnE; ++k) L.oecount[g.edge[L.edgeGlob[k]]]++;
    L.cb = bounds_from(bcount, 0, L.nB);
    L.cbI = bounds_from(icount, L.nB, L.nOwnC);
    L.cbh = bounds_from(hcount, L.nOwnC, L.nC);
    L.eb = bounds_from(L.oecount, 0, L.nOwnE);
    // diagnostics ownership: the rank owning cellsOnVertex[v][0] / cellsOnEdge[e][0]
    L.vOwn.assign(L.nV, 0);
    for (int v = 0; v < L.nV; ++v) L.vOwn[v] = part[m.cov[3 * L.vertGlob[v]]] == me;
    L.eOwn.assign(L.nE, 0);
    for (int e = 0; e < L.nOwnE; ++e) L.eOwn[e] = part[m.coe[2 * L.edgeGlob[e]]] == me;
    c->vminF = L.nV;                          // first vertex of an F_E edge (slow-term refresh range)
    for (int e = L.eb.f; e < L.nOwnE; ++e)
        for (int k = 0; k < 2; ++k) c->vminF = std::min(c->vminF, vertLoc[m.voe[2 * L.edgeGlob[e] + k]]);
    c->have_fine = g.ccount[3] + g.ccount[4] + g.ccount[5] + g.ccount[6] + g.ccount[7] + g.ccount[8] > 0;   // global
    // ---- device tables in local numbering (dummy edge index nE for ring-2 slots outside the subdomain)
    c->sE = pad32(L.nE);
    c->sV = pad32(L.nV);
    const int sE = c->sE, sV = c->sV, G = c->ecS = m.maxE <= 6 ? 6 : (m.maxE <= 8 ? 8 : 16);
    // the kernels index the slot-major tables ([slot][stride]) and the cell rows in 32-bit int
    if ((int64_t)std::max(m.maxE2, 1) * sE > INT32_MAX || 3LL * sV > INT32_MAX || (int64_t)L.nC * G * 2 > INT32_MAX)
        return fail(c, FBLTS_ERR_MESH, "subdomain too large for 32-bit slot indices (nE=%d, maxEdges2=%d, nV=%d, "
                    "nC=%d): partition over more ranks", L.nE, m.maxE2, L.nV, L.nC);
    c->d_nEoC.assign(L.nC, 0);
    c->d_ec.assign((size_t)L.nC * G * 2, 0);
    c->d_area.assign(L.nC, 0.0);
    c->d_zb.assign(L.nC, 0.0);
    for (int i = 0; i < L.nC; ++i) {
        const int o = L.cellGlob[i];
        c->d_nEoC[i] = m.nEoC[o];
        c->d_area[i] = m.areaCell[o];
        c->d_zb[i] = -m.H[o];
        for (int j = 0; j < m.nEoC[o]; ++j) {
            const int e = m.eoc[(size_t)o * m.maxE + j];
            const int el = edgeLoc[e] >= 0 ? edgeLoc[e] : L.nE;
            const int nb = cellLoc[coc[(size_t)o * m.maxE + j]];
            c->d_ec[((size_t)i * G + j) * 2] = m.coe[2 * e] == o ? el : ~el;
            c->d_ec[((size_t)i * G + j) * 2 + 1] = nb >= 0 ? nb : 0;
        }
    }
    c->d_coe.assign((size_t)L.nE * 2, 0);
    c->d_voe.assign((size_t)L.nE * 2, 0);
    c->d_dv.assign(L.nE + 1, 0.0);
    c->d_dc.assign(L.nE + 1, 0.0);
    c->d_nEoE.assign(L.nE, 0);
    c->d_eoe.assign((size_t)m.maxE2 * sE, 0);
    c->d_W.assign((size_t)m.maxE2 * sE, 0.0);
    for (int e = 0; e < L.nE; ++e) {
        const int o = L.edgeGlob[e];
        c->d_coe[2 * e] = cellLoc[m.coe[2 * o]];
        c->d_coe[2 * e + 1] = cellLoc[m.coe[2 * o + 1]];
        c->d_dv[e] = m.dv[o];
        c->d_dc[e] = m.dc[o];
        if (e >= L.nOwnE) continue;           // slow_edge only runs on edges touching owned cells
        c->d_voe[2 * e] = vertLoc[m.voe[2 * o]];
        c->d_voe[2 * e + 1] = vertLoc[m.voe[2 * o + 1]];
        c->d_nEoE[e] = m.nEoE[o];
        for (int j = 0; j < m.nEoE[o]; ++j) {
            c->d_eoe[(size_t)j * sE + e] = edgeLoc[m.eoe[(size_t)o * m.maxE2 + j]];
            c->d_W[(size_t)j * sE + e] = m.W[(size_t)o * m.maxE2 + j];
        }
    }
    c->d_eov.assign((size_t)3 * sV, 0);
    c->d_cov.assign((size_t)3 * sV, 0);
    c->d_kite.assign((size_t)3 * sV, 0.0);
    c->d_areaTri.assign(L.nV, 0.0);
    c->d_fV.assign(L.nV, 0.0);
    for (int v = 0; v < L.nV; ++v) {
        const int o = L.vertGlob[v];
        c->d_areaTri[v] = m.areaTri[o];
        c->d_fV[v] = m.fV[o];
        for (int k = 0; k < 3; ++k) {
            const int e = m.eov[3 * o + k];
            const int en = edgeLoc[e];
            c->d_eov[(size_t)k * sV + v] = m.voe[2 * e + 1] == o ? en : ~en;
            c->d_cov[(size_t)k * sV + v] = cellLoc[m.cov[3 * o + k]];
            c->d_kite[(size_t)k * sV + v] = m.kite[3 * o + k];
        }
    }
    {   // F_e in slow_pre's vertex role: every local edge met exactly once as a positive eov slot whose
        // two kite cells (slots k, k+1) are the edge's cells
        const char *ev = getenv("FBLTS_VF");
        std::vector<uint8_t> seen(L.nE, 0);
        bool ok = !(ev && ev[0] == '0');
        for (int v = 0; ok && v < L.nV; ++v)
            for (int k = 0; k < 3; ++k) {
                const int es = c->d_eov[(size_t)k * sV + v];
                if (es < 0) continue;
                const int a = c->d_cov[(size_t)k * sV + v], b = c->d_cov[(size_t)((k + 1) % 3) * sV + v];
                if (es >= L.nE || seen[es] || a < 0 || b < 0 ||
                    !((c->d_coe[2 * es] == a && c->d_coe[2 * es + 1] == b) ||
                      (c->d_coe[2 * es] == b && c->d_coe[2 * es + 1] == a))) {
                    ok = false;
                    break;
                }
                seen[es] = 1;
            }
        for (int e = 0; ok && e < L.nE; ++e) ok = seen[e] != 0;
        c->vF = ok;
        c->vminF1 = -1;
        for (int v = 0; ok && v < L.nV && c->vminF1 < 0; ++v)
            for (int k = 0; k < 3; ++k)
                if (c->d_eov[(size_t)k * sV + v] >= L.eb.if1) {
                    c->vminF1 = v;
                    break;
                }
        if (ok && c->vminF1 < 0) c->vminF1 = L.nV;
    }
    c->un_c12 = L.nOwnC, c->un_e12 = L.nOwnE, c->un_e3 = L.nOwnE;
    {
        const char *uf = getenv("FBLTS_UNFUSE");
        c->un_fuse = !(uf && uf[0] == '0');
    }
    if (c->cfg.unsplit) {
        auto ce = [&](int e) {
            if (e >= 0) c->un_e12 = std::min(c->un_e12, e);
        };
        auto cc = [&](int i) {
            if (i >= 0) c->un_c12 = std::min(c->un_c12, i);
        };
        for (int v = c->vminF; v < L.nV; ++v)       // slow_pre vertex role: kite h, circulation u
            for (int k = 0; k < 3; ++k) {
                const int es = c->d_eov[(size_t)k * sV + v];
                cc(c->d_cov[(size_t)k * sV + v]);
                ce(es >= 0 ? es : ~es);
            }
        for (int i = L.cb.if1; i < L.nOwnC; ++i)   // cell role: u on the cell's edges
            for (int j = 0; j < c->d_nEoC[i]; ++j) {
                const int es = c->d_ec[((size_t)i * G + j) * 2];
                ce(es >= 0 ? es : ~es);
            }
        for (int e = L.eb.if1; e < L.nOwnE; ++e) {  // edge role (h, u) and slow_edge on F_E (h, u, eoe's u)
            ce(e);
            cc(c->d_coe[2 * e]);
            cc(c->d_coe[2 * e + 1]);
            if (e >= L.eb.f)
                for (int j = 0; j < c->d_nEoE[e]; ++j) ce(c->d_eoe[(size_t)j * sE + e]);
        }
        for (int i = L.cb.if2; i < L.nOwnC; ++i)
            for (int j = 0; j < c->d_nEoC[i]; ++j) {
                const int es = c->d_ec[((size_t)i * G + j) * 2];
                c->un_e3 = std::min(c->un_e3, es >= 0 ? es : ~es);
            }
    }
    // ---- halo exchanges (nranks > 1)
    for (int x = 0; x < X_NUM; ++x) {
        L.x[x] = Xchg();
        L.x[x].sendOff.assign(R + 1, 0);
        L.x[x].recvOff.assign(R + 1, 0);
    }
    c->xmax = 1;
    if (R > 1) {
        std::vector<std::vector<int32_t>> sendG[X_NUM], recvG[X_NUM];   // global ids per peer
        for (int x = 0; x < X_NUM; ++x) {
            sendG[x].assign(R, {});
            recvG[x].assign(R, {});
        }
        for (int k = L.nOwnC; k < L.nC; ++k) {
            const int i = L.cellGlob[k];
            if (dme[i] == 1) recvG[X_C1][part[i]].push_back(i);
            recvG[X_C2][part[i]].push_back(i);
        }
        for (int e = L.nOwnE; e < L.nE; ++e) {
            const int o = L.edgeGlob[e];
            recvG[X_E][part[m.coe[2 * o]]].push_back(o);
        }
        for (int p = 0; p < R; ++p) {
            if (p == me) continue;
            const std::vector<int8_t> dp = dist_from(m, coc, part, p);
            for (int k = 0; k < L.nOwnC; ++k) {
                const int i = L.cellGlob[k];
                if (dp[i] == 1) sendG[X_C1][p].push_back(i);
                if (dp[i] == 1 || dp[i] == 2) sendG[X_C2][p].push_back(i);
            }
            for (int k = 0; k < L.nOwnE; ++k) {
                const int o = L.edgeGlob[k];
                const int a = m.coe[2 * o], b = m.coe[2 * o + 1];
                if (part[a] != me) continue;                       // canonical sender: owner of c0
                if (dp[a] >= 1 && dp[b] >= 1 && std::min(dp[a], dp[b]) == 1) sendG[X_E][p].push_back(o);
            }
        }
        // both sides order a list by the entities' ids in the WHOLE mesh: the index itself for a global
        // upload; for pieces the cell's gid and, for an edge, the pair (min gid, max gid) of its cells
        // (two cells share at most one edge), so every rank derives the same order from its own piece
        auto ckey = [&](int i) -> int64_t { return c->piece ? c->gid[i] : (int64_t)i; };
        auto ekey = [&](int e) -> int64_t {
            if (!c->piece) return (int64_t)e;
            const int64_t a = c->gid[m.coe[2 * e]], b = c->gid[m.coe[2 * e + 1]];
            return (std::min(a, b) << 32) | std::max(a, b);
        };
        for (int x = 0; x < X_NUM; ++x) {
            const std::vector<int32_t> &loc = x == X_E ? edgeLoc : cellLoc;
            Xchg &X = L.x[x];
            for (int p = 0; p < R; ++p) {
                auto by = [&](int a, int b) { return x == X_E ? ekey(a) < ekey(b) : ckey(a) < ckey(b); };
                std::sort(sendG[x][p].begin(), sendG[x][p].end(), by);
                std::sort(recvG[x][p].begin(), recvG[x][p].end(), by);
                for (int gid : sendG[x][p]) X.sendIdx.push_back(loc[gid]);
                for (int gid : recvG[x][p]) X.recvIdx.push_back(loc[gid]);
                X.sendOff[p + 1] = (int64_t)X.sendIdx.size();
                X.recvOff[p + 1] = (int64_t)X.recvIdx.size();
            }
            c->xmax = std::max(c->xmax, std::max(X.sendIdx.size(), X.recvIdx.size()));
        }
    }
    c->d_xidx.clear();
    for (int x = 0; x < X_NUM; ++x) {
        L.x[x].sendAt = c->d_xidx.size();
        c->d_xidx.insert(c->d_xidx.end(), L.x[x].sendIdx.begin(), L.x[x].sendIdx.end());
        L.x[x].recvAt = c->d_xidx.size();
        c->d_xidx.insert(c->d_xidx.end(), L.x[x].recvIdx.begin(), L.x[x].recvIdx.end());
    }
    if (c->d_xidx.empty()) c->d_xidx.push_back(0);
    const int rc = build_tiles(c);
    if (rc) return rc;
    return build_subtiles(c);
}

}  // namespace

extern "C" {

int fblts_set_regions(fblts_ctx *c, const uint8_t *fine_mask) {
    if (!c || !fine_mask) return FBLTS_ERR_INVALID_ARG;
    if (c->phase != P_MESH) return fail(c, FBLTS_ERR_ORDER, "set_regions: needs exactly one prior upload_mesh");
    const HostMesh &m = c->hm;
    const int r = c->cfg.r;
    // cell neighbours across each edge slot
    std::vector<int32_t> coc((size_t)m.nC * m.maxE, -1);
    for (int i = 0; i < m.nC; ++i)
        for (int j = 0; j < m.nEoC[i]; ++j) {
            const int e = m.eoc[(size_t)i * m.maxE + j];
            coc[(size_t)i * m.maxE + j] = m.coe[2 * e] == i ? m.coe[2 * e + 1] : m.coe[2 * e];
        }
    std::vector<uint8_t> fine(m.nC), coarse(m.nC);
    for (int i = 0; i < m.nC; ++i) {
        fine[i] = fine_mask[i] ? 1 : 0;
        coarse[i] = !fine[i];
    }
    // LTS regions: hop distance to F for coarse cells, to C for fine cells
    const std::vector<int32_t> dF = hops(m, coc, fine), dC = hops(m, coc, coarse);
    Region &g = c->rg;
    g.cell.assign(m.nC, 0);
    for (int i = 0; i < m.nC; ++i) {
        if (fine[i]) {
            const int layer = dC[i] == INT32_MAX ? 6 : std::min(6, (dC[i] + r - 1) / r);
            g.cell[i] = (int8_t)(2 + layer);
        } else {
            g.cell[i] = dF[i] <= r ? FBLTS_REGION_IF1 : (dF[i] <= 2 * r ? FBLTS_REGION_IF2 : FBLTS_REGION_INT);
        }
    }
    g.edge.assign(m.nE, 0);
    for (int e = 0; e < m.nE; ++e) {
        const int a = g.cell[m.coe[2 * e]], b = g.cell[m.coe[2 * e + 1]];
        if (std::abs(region_class(a) - region_class(b)) > 1)
            return fail(c, FBLTS_ERR_LABELS, "labels: edge %d joins regions %d and %d (stencil assumption)", e, a, b);
        const bool fa = a >= 3, fb = b >= 3;
        g.edge[e] = (int8_t)(fa && fb ? std::min(a, b) : (fa ? a : (fb ? b : std::max(a, b))));
    }
    std::fill(g.ccount, g.ccount + 9, 0);
    std::fill(g.ecount, g.ecount + 9, 0);
    for (int i = 0; i < m.nC; ++i) g.ccount[g.cell[i]]++;
    for (int e = 0; e < m.nE; ++e) g.ecount[g.edge[e]]++;
    const int rc = build_local(c, coc);
    if (rc) return rc;
    c->phase = P_REGIONS;
    return FBLTS_OK;
}

int fblts_get_labels(fblts_ctx *c, int8_t *cell_region, int8_t *edge_region) {
    if (!c) return FBLTS_ERR_INVALID_ARG;
    if (c->phase < P_REGIONS) return fail(c, FBLTS_ERR_ORDER, "get_labels: call set_regions first");
    if (cell_region) std::copy(c->rg.cell.begin(), c->rg.cell.end(), cell_region);
    if (edge_region) std::copy(c->rg.edge.begin(), c->rg.edge.end(), edge_region);
    return FBLTS_OK;
}

int fblts_get_counts(fblts_ctx *c, int64_t *out) {
    if (!c || !out) return FBLTS_ERR_INVALID_ARG;
    if (c->phase < P_REGIONS) return fail(c, FBLTS_ERR_ORDER, "get_counts: call set_regions first");
    out[0] = c->hm.nC;
    out[1] = c->hm.nE;
    out[2] = c->hm.nV;
    for (int k = 0; k < 9; ++k) {
        out[3 + k] = c->lo.ocount[k];
        out[12 + k] = c->lo.oecount[k];
    }
    out[21] = c->lo.nOwnC;
    out[22] = c->lo.nOwnE;
    out[23] = (int64_t)c->graph_nodes;
    out[24] = (int64_t)c->t_start.size() - 1;
    out[25] = (int64_t)c->t_nHalo;
    out[26] = (int64_t)c->t_nEcl;
    out[27] = stage_tiled_smem_bytes_host(3, c->t_hmax, c->t_emax);
    out[28] = c->fuse_sub ? c->s_nT : 0;
    out[29] = c->fuse_sub ? (int64_t)c->s_nHalo : 0;
    out[30] = c->fuse_sub ? (int64_t)c->s_nFedge : 0;
    out[31] = c->fuse_sub ? sub_smem_bytes_host(c->s_hmax, c->s_emax, c->s_rmax) : 0;
    return FBLTS_OK;
}

int fblts_get_halo(fblts_ctx *c, int32_t which, int32_t peer, int64_t *n_send, int64_t *n_recv, int64_t *send_ids,
                   int64_t *recv_ids) {
    if (!c || which < 0 || which >= X_NUM || peer < 0 || peer >= c->cfg.nranks) return FBLTS_ERR_INVALID_ARG;
    if (c->phase < P_REGIONS) return fail(c, FBLTS_ERR_ORDER, "get_halo: call set_regions first");
    const Xchg &X = c->lo.x[which];
    const std::vector<int32_t> &glob = which == X_E ? c->lo.edgeGlob : c->lo.cellGlob;
    const int64_t s0 = X.sendOff[peer], s1 = X.sendOff[peer + 1], r0 = X.recvOff[peer], r1 = X.recvOff[peer + 1];
    if (n_send) *n_send = s1 - s0;
    if (n_recv) *n_recv = r1 - r0;
    // ids in the whole mesh: the uploaded index, or with fblts_set_partition the cell gid and for an
    // edge the key (min gid << 32) | max gid of its two cells
    auto id = [&](int32_t loc) -> int64_t {
        const int o = glob[loc];
        if (!c->piece) return o;
        if (which != X_E) return c->gid[o];
        const int64_t a = c->gid[c->hm.coe[2 * o]], b = c->gid[c->hm.coe[2 * o + 1]];
        return (std::min(a, b) << 32) | std::max(a, b);
    };
    if (send_ids)
        for (int64_t k = s0; k < s1; ++k) send_ids[k - s0] = id(X.sendIdx[k]);
    if (recv_ids)
        for (int64_t k = r0; k < r1; ++k) recv_ids[k - r0] = id(X.recvIdx[k]);
    return FBLTS_OK;
}

int fblts_set_partition(fblts_ctx *c, const int32_t *owner, const int64_t *cell_gid) {
    if (!c || !owner || !cell_gid) return FBLTS_ERR_INVALID_ARG;
    if (c->phase != P_MESH) return fail(c, FBLTS_ERR_ORDER, "set_partition: after upload_mesh, before set_regions");
    const int nC = c->hm.nC, R = c->cfg.nranks;
    std::vector<int32_t> part(owner, owner + nC);
    std::vector<int64_t> g(cell_gid, cell_gid + nC);
    int64_t mine = 0;
    for (int i = 0; i < nC; ++i) {
        if (part[i] < 0 || part[i] >= R) return fail(c, FBLTS_ERR_INVALID_ARG, "set_partition: owner[%d]=%d", i, part[i]);
        if (g[i] < 0 || g[i] >= ((int64_t)1 << 31)) return fail(c, FBLTS_ERR_INVALID_ARG, "set_partition: gid[%d] out of range", i);
        mine += part[i] == c->cfg.rank;
    }
    if (mine == 0) return fail(c, FBLTS_ERR_INVALID_ARG, "set_partition: rank %d owns no cell of its piece", c->cfg.rank);
    std::vector<int64_t> sorted(g);
    std::sort(sorted.begin(), sorted.end());
    for (int i = 1; i < nC; ++i)
        if (sorted[i] == sorted[i - 1]) return fail(c, FBLTS_ERR_INVALID_ARG, "set_partition: gid %lld repeated", (long long)sorted[i]);
    c->ext_part.swap(part);
    c->gid.swap(g);
    c->piece = true;
    return FBLTS_OK;
}

}  // extern "C"

namespace {
// workspace plan: the same sequence is used for sizing and for carving
struct Plan {
    size_t total = 0;
    size_t add(size_t bytes) {
        const size_t off = total;
        total += (bytes + 255) / 256 * 256;
        return off;
    }
};

size_t plan_workspace(fblts_ctx *c, char *base) {
    const HostMesh &m = c->hm;
    const Local &L = c->lo;
    Plan p;
    auto put = [&](auto *&ptr, size_t count) {
        using T = std::remove_pointer_t<std::remove_reference_t<decltype(ptr)>>;
        const size_t off = p.add(count * sizeof(T));
        if (base) ptr = reinterpret_cast<T *>(base + off);
    };
    DevMesh &d = c->dm;
    DevState &s = c->ds;
    int32_t *nEoC, *nEoE, *eoe, *eov, *cov;
    double *area, *zb, *W, *tau, *kite, *areaTri, *fV, *dv, *dc;
    int2 *coe, *voe, *ec;
    uint8_t *vOwn, *eOwn;
    const size_t nE1 = (size_t)L.nE + 1;               // + dummy edge
    put(nEoC, L.nC);
    put(ec, (size_t)L.nC * c->ecS);
    put(area, L.nC);
    put(zb, L.nC);
    put(coe, L.nE);
    put(voe, L.nE);
    put(dv, nE1);
    put(dc, nE1);
    put(tau, L.nE);
    double *uwn, *uwt;
    put(uwn, L.nE);
    put(uwt, L.nE);
    put(nEoE, L.nE);
    put(eoe, (size_t)m.maxE2 * c->sE);
    put(W, (size_t)m.maxE2 * c->sE);
    put(eov, (size_t)3 * c->sV);
    put(cov, (size_t)3 * c->sV);
    put(kite, (size_t)3 * c->sV);
    put(areaTri, L.nV);
    put(fV, L.nV);
    put(vOwn, L.nV);
    put(eOwn, L.nE);
    double *hA, *hB, *uA, *uB;
    put(hA, L.nC);
    put(hB, L.nC);
    put(s.h1, L.nC);
    put(s.h2, L.nC);
    put(s.hT, L.nC);
    put(s.K, L.nC);
    put(uA, nE1);
    put(uB, nE1);
    put(s.uT, nE1);
    put(s.S, L.nE);
    put(s.F, nE1);
    put(s.q, L.nV);
    put(s.qe, c->cfg.pv_energy ? (size_t)L.nE : 1);
    put(s.accH, std::max(1, L.nOwnC));
    put(s.accU, std::max(1, L.eb.f - L.eb.if2));
    put(s.uIF2, std::max(1, L.eb.f - L.eb.if2));
    put(s.uIF3, std::max(1, L.eb.f - L.eb.if2));
    const size_t nrk = c->cfg.scheme != FBLTS_SCHEME_FBLTS ? nE1 : 1;
    put(s.rkU[0], nrk);
    put(s.rkU[1], nrk);
    put(s.rkAccU, nrk);
    const bool rf = c->cfg.slow_refresh != 0 || c->cfg.unsplit != 0;
    put(s.Sk, rf ? nE1 : 1);
    put(s.uv, rf ? nE1 : 1);
    put(s.hv, rf ? (size_t)std::max(1, L.nC) : 1);
    const size_t nun = c->cfg.unsplit ? nE1 : 1;
    for (int q = 0; q < 3; ++q) put(s.un[q], nun);
    for (int q = 0; q < 2; ++q) put(s.unk[q], nun);
    const bool vt = c->cfg.vorticity != 0;
    put(s.eta, vt ? (size_t)std::max(1, L.nV) : 1);
    put(s.dP, vt ? nE1 : 1);
    put(s.accP, vt ? (size_t)std::max(1, L.eb.f - L.eb.if2) : 1);
    put(s.Pv, vt ? nE1 : 1);
    if (base && !vt) s.eta = s.dP = s.accP = s.Pv = nullptr;
    if (base) s.Sf = c->cfg.slow_refresh ? s.Sk : s.S;
    put(s.stage, std::max(m.nC, m.nE));
    put(s.cellOld, L.nC);
    put(s.edgeOld, L.nE);
    put(s.diag, DIAG_BLOCKS * 6 + 8 + 6 * 64);
    put(s.diagA, DIAG_BLOCKS * 6 + 8);
    put(s.err, 1);
    put(s.vbad, 2);
    put(s.sendbuf, c->xmax);
    put(s.recvbuf, c->xmax);
    put(s.xidx, c->d_xidx.size());
    TileMesh &tm = c->dm.tm;
    int32_t *tInfo, *tHalo, *tFedge;
    uint32_t *tEcl;
    uint16_t *tRow;
    put(tInfo, c->t_info.size());
    put(tHalo, std::max<size_t>(1, c->t_nHalo));
    put(tFedge, std::max<size_t>(1, c->t_nFedge));
    put(tEcl, std::max<size_t>(1, c->t_nEcl));
    put(tRow, (size_t)c->hm.maxE * c->t_sRow);
    // ghost slots of the staged sweeps: sources, static ghosts (z_b, l_e, d_e), S's ghosts
    const size_t nGc = std::max<size_t>(1, c->g_cidx.size()), nGe = std::max<size_t>(1, c->g_eidx.size());
    int32_t *gCi, *gEi;
    double *gz, *gl, *gd;
    put(gCi, nGc);
    put(gEi, nGe);
    put(gz, nGc);
    put(gl, nGe);
    put(gd, nGe);
    put(c->GS, nGe);
    const bool fs = c->fuse_sub;
    put(s.hT2, fs ? (size_t)L.nC : 1);
    put(s.h2alt, fs ? (size_t)L.nC : 1);
    SubTileMesh &sm = c->dm.st;
    int32_t *sInfo, *sHalo, *sFedge;
    uint32_t *sEcl;
    uint16_t *sRow;
    put(sInfo, fs ? c->s_info.size() : 1);
    put(sHalo, fs ? std::max<size_t>(1, c->s_nHalo) : 1);
    put(sFedge, fs ? std::max<size_t>(1, c->s_nFedge) : 1);
    put(sEcl, fs ? std::max<size_t>(1, c->s_nEcl) : 1);
    put(sRow, fs ? std::max<size_t>(1, c->s_nRow) : 1);
    if (base) {
        sm.nTiles = fs ? c->s_nT : 0;
        sm.hmax = c->s_hmax;
        sm.emax = c->s_emax;
        sm.rmax = c->s_rmax;
        sm.info = sInfo, sm.halo = sHalo, sm.fedge = sFedge, sm.ecl = sEcl, sm.row = sRow;
    }
    if (base) {
        tm.nTiles = (int32_t)c->t_start.size() - 1;
        tm.strideRow = c->t_sRow;
        tm.hmax = c->t_hmax;
        tm.emax = c->t_emax;
        tm.info = tInfo, tm.halo = tHalo, tm.fedge = tFedge, tm.ecl = tEcl, tm.row = tRow;
        tm.gcidx = gCi, tm.geidx = gEi, tm.Gz = gz, tm.Gl = gl, tm.Gd = gd;
        c->dGe = gEi;
    }
    if (base) {
        d.nC = L.nC, d.nE = L.nE, d.nV = L.nV, d.nOwnC = L.nOwnC, d.nOwnE = L.nOwnE;
        d.strideC = L.nC, d.strideE = c->sE, d.strideV = c->sV;
        d.maxE = m.maxE, d.maxE2 = m.maxE2, d.ecS = c->ecS;
        d.nEoC = nEoC, d.ec = ec, d.areaCell = area, d.zb = zb;
        d.coe = coe, d.voe = voe, d.dv = dv, d.dc = dc, d.nEoE = nEoE, d.eoe = eoe, d.W = W, d.tau = tau;
        d.uwn = uwn, d.uwt = uwt;
        d.eov = eov, d.cov = cov, d.kite = kite, d.areaTri = areaTri, d.fV = fV;
        d.vOwn = vOwn, d.eOwn = eOwn;
        d.nB = L.nB, d.cb = L.cb, d.cbI = L.cbI, d.eb = L.eb, d.cbh = L.cbh;
        d.vF = c->vF ? 1 : 0;
        c->hbuf[0] = hA, c->hbuf[1] = hB, c->ubuf[0] = uA, c->ubuf[1] = uB;
        s.hN = hA, s.hNew = hB, s.uN = uA, s.uNew = uB;
        c->diag_out = s.diag + DIAG_BLOCKS * 6;
    }
    return p.total;
}
}  // namespace

extern "C" {

int fblts_workspace_size(fblts_ctx *c, size_t *bytes) {
    if (!c || !bytes) return FBLTS_ERR_INVALID_ARG;
    if (c->phase < P_REGIONS) return fail(c, FBLTS_ERR_ORDER, "workspace_size: call set_regions first");
    *bytes = plan_workspace(c, nullptr);
    return FBLTS_OK;
}

int fblts_bind_workspace(fblts_ctx *c, void *ptr, size_t bytes) {
    if (!c || !ptr) return FBLTS_ERR_INVALID_ARG;
    if (c->phase != P_REGIONS) return fail(c, FBLTS_ERR_ORDER, "bind_workspace: call set_regions first (once)");
    const size_t need = plan_workspace(c, nullptr);
    if (bytes < need) return fail(c, FBLTS_ERR_INVALID_ARG, "bind_workspace: %zu bytes < %zu needed", bytes, need);
    if ((uintptr_t)ptr % 256) return fail(c, FBLTS_ERR_INVALID_ARG, "bind_workspace: pointer not 256-B aligned");
    CUDA_TRY(c, cudaSetDevice(c->cfg.device));
    if (!c->cap) CUDA_TRY(c, cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));
    if (c->cfg.nranks == 1 && !c->side) {
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->evSideF, cudaEventDisableTiming));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->evSideJ, cudaEventDisableTiming));
    }
    if (c->cfg.nranks > 1 && !c->comm) {
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->comm, cudaStreamNonBlocking));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->evFork, cudaEventDisableTiming));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->evJoin, cudaEventDisableTiming));
    }
    if (c->cfg.nranks > 1 && !c->nccl && c->cfg.nccl_id) {   // no id: loopback group member
        const int rc = nccl_init(c);
        if (rc) return rc;
    }
    c->ws = (char *)ptr;
    c->ws_bytes = bytes;
    CUDA_TRY(c, cudaMemsetAsync(ptr, 0, need, c->stream));
    plan_workspace(c, c->ws);
    cudaStream_t s = c->stream;
    DevMesh &d = c->dm;
    auto up = [&](const void *dst, const void *src, size_t n) {
        return cudaMemcpyAsync(const_cast<void *>(dst), src, n, cudaMemcpyHostToDevice, s);
    };
    const Local &L = c->lo;
    CUDA_TRY(c, up(d.nEoC, c->d_nEoC.data(), c->d_nEoC.size() * 4));
    CUDA_TRY(c, up(d.ec, c->d_ec.data(), c->d_ec.size() * 4));
    CUDA_TRY(c, up(d.areaCell, c->d_area.data(), (size_t)L.nC * 8));
    CUDA_TRY(c, up(d.zb, c->d_zb.data(), (size_t)L.nC * 8));
    CUDA_TRY(c, up(d.coe, c->d_coe.data(), (size_t)L.nE * 8));
    CUDA_TRY(c, up(d.voe, c->d_voe.data(), (size_t)L.nE * 8));
    CUDA_TRY(c, up(d.dv, c->d_dv.data(), c->d_dv.size() * 8));
    CUDA_TRY(c, up(d.dc, c->d_dc.data(), c->d_dc.size() * 8));
    CUDA_TRY(c, up(d.nEoE, c->d_nEoE.data(), (size_t)L.nE * 4));
    CUDA_TRY(c, up(d.eoe, c->d_eoe.data(), c->d_eoe.size() * 4));
    CUDA_TRY(c, up(d.W, c->d_W.data(), c->d_W.size() * 8));
    CUDA_TRY(c, up(d.eov, c->d_eov.data(), c->d_eov.size() * 4));
    CUDA_TRY(c, up(d.cov, c->d_cov.data(), c->d_cov.size() * 4));
    CUDA_TRY(c, up(d.kite, c->d_kite.data(), c->d_kite.size() * 8));
    CUDA_TRY(c, up(d.areaTri, c->d_areaTri.data(), (size_t)L.nV * 8));
    CUDA_TRY(c, up(d.fV, c->d_fV.data(), (size_t)L.nV * 8));
    CUDA_TRY(c, up(d.vOwn, L.vOwn.data(), (size_t)L.nV));
    CUDA_TRY(c, up(d.eOwn, L.eOwn.data(), (size_t)L.nE));
    CUDA_TRY(c, up(c->ds.cellOld, L.cellGlob.data(), (size_t)L.nC * 4));
    CUDA_TRY(c, up(c->ds.edgeOld, L.edgeGlob.data(), (size_t)L.nE * 4));
    CUDA_TRY(c, up(c->ds.xidx, c->d_xidx.data(), c->d_xidx.size() * 4));
    const TileMesh &tm = d.tm;
    CUDA_TRY(c, up(tm.info, c->t_info.data(), c->t_info.size() * 4));
    CUDA_TRY(c, up(tm.halo, c->t_halo.data(), c->t_halo.size() * 4));
    CUDA_TRY(c, up(tm.fedge, c->t_fedge.data(), c->t_fedge.size() * 4));
    CUDA_TRY(c, up(tm.ecl, c->t_ecl.data(), c->t_ecl.size() * 4));
    CUDA_TRY(c, up(tm.row, c->t_row.data(), c->t_row.size() * 2));
    CUDA_TRY(c, up(tm.gcidx, c->g_cidx.data(), c->g_cidx.size() * 4));
    CUDA_TRY(c, up(tm.geidx, c->g_eidx.data(), c->g_eidx.size() * 4));
    launch_ghost_fill(tm.gcidx, d.zb, const_cast<double *>(tm.Gz), 0, (int)c->g_cidx.size(), s);   // static ghosts
    launch_ghost_fill(tm.geidx, d.dv, const_cast<double *>(tm.Gl), 0, (int)c->g_eidx.size(), s);
    launch_ghost_fill(tm.geidx, d.dc, const_cast<double *>(tm.Gd), 0, (int)c->g_eidx.size(), s);
    CUDA_TRY(c, cudaGetLastError());
    if (c->fuse_sub) {
        const SubTileMesh &sm = d.st;
        CUDA_TRY(c, up(sm.info, c->s_info.data(), c->s_info.size() * 4));
        CUDA_TRY(c, up(sm.halo, c->s_halo.data(), c->s_halo.size() * 4));
        CUDA_TRY(c, up(sm.fedge, c->s_fedge.data(), c->s_fedge.size() * 4));
        CUDA_TRY(c, up(sm.ecl, c->s_ecl.data(), c->s_ecl.size() * 4));
        CUDA_TRY(c, up(sm.row, c->s_row.data(), c->s_row.size() * 2));
    }
    if (stage_tiled_smem_bytes_host(4, c->t_hmax, c->t_emax) > TILE_SMEM_MAX) c->split = true;    // size launches per block
    if (c->tiled) {   // stage_tiled_run halves a launch until it fits, down to one tile: every tile must fit alone
        for (size_t t = 0; t + 1 < c->t_start.size(); ++t) {
            const int32_t *r = &c->t_info[t * TINFO], *n = r + TINFO;
            if (stage_tiled_smem_bytes_host(4, n[1] - r[1], r[3] - r[2] + n[4] - r[4]) > TILE_SMEM_MAX) {
                c->tiled = false;        // untiled per-thread kernels instead (same arithmetic, same bits)
                break;
            }
        }
    }
    CUDA_TRY(c, cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, c->cfg.device));
    if (c->tiled) CUDA_TRY(c, (cudaError_t)stage_tiled_configure(d));
    CUDA_TRY(c, cudaStreamSynchronize(s));
    // host staging of the big device tables is no longer needed
    std::vector<int32_t>().swap(c->d_ec);
    std::vector<int32_t>().swap(c->d_eoe);
    std::vector<double>().swap(c->d_W);
    std::vector<int32_t>().swap(c->t_halo);
    std::vector<int32_t>().swap(c->t_fedge);
    std::vector<uint32_t>().swap(c->t_ecl);
    std::vector<uint16_t>().swap(c->t_row);
    std::vector<int32_t>().swap(c->s_halo);
    std::vector<int32_t>().swap(c->s_fedge);
    std::vector<uint32_t>().swap(c->s_ecl);
    std::vector<uint16_t>().swap(c->s_row);
    c->phase = P_BOUND;
    return FBLTS_OK;
}

int fblts_set_forcing(fblts_ctx *c, const double *tau_n) {
    if (!c) return FBLTS_ERR_INVALID_ARG;
    if (c->phase < P_BOUND) return fail(c, FBLTS_ERR_ORDER, "set_forcing: bind the workspace first");
    const Local &L = c->lo;
    std::vector<double> t(L.nE, 0.0);
    if (tau_n)
        for (int e = 0; e < L.nE; ++e) {
            const double v = tau_n[L.edgeGlob[e]];
            if (!std::isfinite(v)) return fail(c, FBLTS_ERR_INVALID_ARG, "forcing[%d] not finite", L.edgeGlob[e]);
            t[e] = v;
        }
    CUDA_TRY(c, cudaMemcpyAsync((void *)c->dm.tau, t.data(), (size_t)L.nE * 8, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return FBLTS_OK;
}

int fblts_set_hurricane(fblts_ctx *c, const double *uw_n, const double *uw_t, double cd, double cw) {
    if (!c) return FBLTS_ERR_INVALID_ARG;
    if (c->phase < P_BOUND) return fail(c, FBLTS_ERR_ORDER, "set_hurricane: bind the workspace first");
    if (!uw_n || !uw_t) {
        c->sc.hur = 0;
        c->sc.cd = c->sc.cw = 0.0;
    } else {
        if (!(std::isfinite(cd) && std::isfinite(cw) && cd >= 0.0 && cw >= 0.0))
            return fail(c, FBLTS_ERR_INVALID_ARG, "set_hurricane: C_D, C_W must be finite and >= 0");
        const Local &L = c->lo;
        std::vector<double> a(L.nE), b(L.nE);
        for (int e = 0; e < L.nE; ++e) {
            a[e] = uw_n[L.edgeGlob[e]];
            b[e] = uw_t[L.edgeGlob[e]];
            if (!std::isfinite(a[e]) || !std::isfinite(b[e]))
                return fail(c, FBLTS_ERR_INVALID_ARG, "set_hurricane: wind[%d] not finite", L.edgeGlob[e]);
        }
        CUDA_TRY(c, cudaMemcpyAsync((void *)c->dm.uwn, a.data(), (size_t)L.nE * 8, cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(c, cudaMemcpyAsync((void *)c->dm.uwt, b.data(), (size_t)L.nE * 8, cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        c->sc.hur = 1;
        c->sc.cd = cd;
        c->sc.cw = cw;
    }
    for (int p = 0; p < 2; ++p)               // the step graphs bake the constants: re-capture
        if (c->exec[p]) {
            cudaGraphExecDestroy(c->exec[p]);
            c->exec[p] = nullptr;
        }
    return FBLTS_OK;
}

int fblts_set_state(fblts_ctx *c, const double *h, const double *u, double t) {
    if (!c || !h || !u) return FBLTS_ERR_INVALID_ARG;
    if (c->phase < P_BOUND) return fail(c, FBLTS_ERR_ORDER, "set_state: bind the workspace first");
    cudaStream_t s = c->stream;
    const Local &L = c->lo;
    diag_wait(c, 0);
    diag_wait(c, 1);
    c->parity = 0;
    // the input check runs on the device, on the copied arrays (first offending index reported)
    int32_t bad[2] = {0, 0};
    CUDA_TRY(c, cudaMemsetAsync(c->ds.vbad, 0x7F, 2 * sizeof(int32_t), s));
    CUDA_TRY(c, cudaMemcpyAsync(c->ds.stage, h, (size_t)c->hm.nC * 8, cudaMemcpyHostToDevice, s));
    launch_validate(c->ds.stage, c->hm.nC, 1, c->ds.vbad, s);
    launch_permute_in(c->ds.cellOld, c->ds.stage, c->hbuf[0], L.nC, s);
    CUDA_TRY(c, cudaMemcpyAsync(c->ds.stage, u, (size_t)c->hm.nE * 8, cudaMemcpyHostToDevice, s));
    launch_validate(c->ds.stage, c->hm.nE, 0, c->ds.vbad + 1, s);
    launch_permute_in(c->ds.edgeOld, c->ds.stage, c->ubuf[0], L.nE, s);
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaMemsetAsync(c->ds.err, 0, sizeof(DevError), s));
    CUDA_TRY(c, cudaMemcpyAsync(bad, c->ds.vbad, sizeof bad, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaStreamSynchronize(s));
    constexpr int32_t none = 0x7F7F7F7F;
    if (bad[0] != none || bad[1] != none) {
        c->phase = P_BOUND;                  // the device state was overwritten: no valid state now
        if (bad[0] != none) return fail(c, FBLTS_ERR_STATE, "set_state: h[%d]=%g", bad[0], h[bad[0]]);
        return fail(c, FBLTS_ERR_STATE, "set_state: u[%d] not finite", bad[1]);
    }
    c->t = t;
    c->phase = P_STATE;
    return FBLTS_OK;
}

int fblts_set_vorticity(fblts_ctx *c, const double *eta) {
    if (!c || !eta) return FBLTS_ERR_INVALID_ARG;
    if (!c->cfg.vorticity) return fail(c, FBLTS_ERR_ORDER, "set_vorticity: context created without cfg.vorticity");
    if (c->phase != P_STATE) return fail(c, FBLTS_ERR_ORDER, "set_vorticity: set_state first");
    const Local &L = c->lo;
    std::vector<double> tmp(L.nV);
    for (int v = 0; v < L.nV; ++v) {
        tmp[v] = eta[L.vertGlob[v]];
        if (!std::isfinite(tmp[v])) return fail(c, FBLTS_ERR_STATE, "set_vorticity: eta[%d] not finite", L.vertGlob[v]);
    }
    CUDA_TRY(c, cudaMemcpyAsync(c->ds.eta, tmp.data(), (size_t)L.nV * 8, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return FBLTS_OK;
}


}  // extern "C"

namespace {

// Instrumented replay (fblts_profile): an event at every kernel-kind boundary, and an NVTX range per
// kernel kind (named as in fblts_kernel_name) around its enqueues, for nsys / ncu range filtering.
struct Recorder {
    std::vector<cudaEvent_t> ev;
    std::vector<int> kind;
    bool open = false;
    void mark(int k, cudaStream_t s) {
        cudaEvent_t a;
        cudaEventCreate(&a);
        cudaEventRecord(a, s);
        ev.push_back(a);
        kind.push_back(k);
        if (open) nvtxRangePop();
        open = k >= 0;
        if (open) nvtxRangePushA(kKernelNames[k]);
    }
    ~Recorder() {
        if (open) nvtxRangePop();
    }
};

// A phase is a run of kernels followed (except for a single rank) by one halo exchange of the
// array it produced: ring 1 after every thickness stage, rings 1-2 of h and the remote-owned
// edges of u at the end of the step.
struct PhaseX {
    int x;            // X_C1, X_C2 or -1
    double *a;        // array exchanged
    int x2;           // second exchange (X_E at the end of the step) or -1
    double *a2;
};

void stage_tiled_run(fblts_ctx *c, int stage, int cbegin, int cend, const StageArgs &a, cudaStream_t s) {
    if (cend <= cbegin) return;
    const int t0 = tile_at(c, cbegin), t1 = tile_at(c, cend);
    int hmax = 0, emax = 0;                  // shared memory sized for the tiles of this launch
    for (int t = t0; t < t1; ++t) {
        const int32_t *r = &c->t_info[(size_t)t * TINFO], *n = r + TINFO;
        hmax = std::max(hmax, n[1] - r[1]);
        emax = std::max(emax, r[3] - r[2] + n[4] - r[4]);
    }
    // records staged per CTA: at most ceil(tiles / nsm) (the grid is >= one CTA per SM, or one per tile)
    const int nrec = std::max(1, (t1 - t0 + c->nsm - 1) / std::max(1, c->nsm));
    if (stage_tiled_smem_bytes_host(stage, hmax, emax, nrec) > TILE_SMEM_MAX) {   // too large: halve the range
        if (t1 - t0 > 1) {
            const int mid = c->t_start[t0 + (t1 - t0) / 2];
            stage_tiled_run(c, stage, cbegin, mid, a, s);
            stage_tiled_run(c, stage, mid, cend, a, s);
            return;
        }
    }
    StageArgs g = a;
    g.gS = c->GS;
    if (stage > 1) {   // S's ghosts: the frozen S changes once per step, so they are refilled only for a new
                       // step or a launch range not yet covered (always for the refresh's S^k)
        const int32_t *r0 = &c->t_info[(size_t)t0 * TINFO], *r1 = &c->t_info[(size_t)t1 * TINFO];
        const int nGe = (int)c->g_eidx.size();
        const int ge0 = std::max(0, r0[7] - 1), ge1 = std::min(nGe, r1[7] + 2);
        fblts_ctx::GhostKey &k = c->gkS;
        const bool frozen = a.S == c->ds.S;
        if (!(frozen && k.src == a.S && k.epoch == c->step_epoch && k.k0 <= ge0 && ge1 <= k.k1)) {
            launch_ghost_fill(c->dGe, a.S, c->GS, ge0, ge1, s);
            k.src = frozen ? a.S : nullptr, k.epoch = c->step_epoch, k.k0 = ge0, k.k1 = ge1;
        }
    }
    launch_stage_tiled(c->dm, stage, t0, t1, hmax, emax, c->nsm, g, c->ds.err, s);
}
// The thin interface blocks [IF-2 .. F^5] have long, narrow tiles (more halo cells and edges per
// cell); with FBLTS_SPLIT=1 they get their own launch so that the bulk blocks (int, F\F^5) size
// shared memory for compact tiles.
void stage_tiled(fblts_ctx *c, int stage, const Bounds &B, int cbegin, int cend, const StageArgs &a, cudaStream_t s) {
    if (!c->split) return stage_tiled_run(c, stage, cbegin, cend, a, s);
    const int cuts[2] = {B.if2, B.fl[5]};
    int lo = cbegin;
    for (int k = 0; k < 2; ++k)
        if (cuts[k] > lo && cuts[k] < cend) {
            stage_tiled_run(c, stage, lo, cuts[k], a, s);
            lo = cuts[k];
        }
    stage_tiled_run(c, stage, lo, cend, a, s);
}

// Enqueue part `part` of phase `ph` of the step reading hbuf[par], ubuf[par]; returns false when
// past the end.  Part 0 = the phase's edge / slow kernels and its cell kernel on the BOUNDARY block
// (DevMesh::cb); part 1 = the cell kernel on the INTERIOR block (DevMesh::cbI).  The phase's halo
// exchange (PhaseX) reads only boundary-block cells, so with several ranks it runs between the
// two parts, overlapped with part 1.
bool enqueue_phase(fblts_ctx *c, int par, int ph, cudaStream_t s, Recorder *rec, PhaseX *px, int part) {
    if (ph == 0 && part == 0) c->step_epoch++;      // the S ghost cache is per enqueued step
    const DevMesh &m = c->dm;
    DevState st = c->ds;
    const StepConst &sc = c->sc;
    const double *hN = c->hbuf[par], *uN = c->ubuf[par];
    double *hNew = c->hbuf[1 - par], *uNew = c->ubuf[1 - par];
    const Bounds &B = part == 0 ? m.cb : m.cbI;
    const bool cells = B.end > B.begin;       // anything to do in this block
    auto mark = [&](int k) {
        if (rec) rec->mark(k, s);
    };
    const int M = sc.M;
    const bool T = c->tiled;
    // fused subcycle on F\F^2: the fine levels k-1, k, k+1 live in three distinct buffers (a tile
    // reads level k-1 on its rings while its neighbours write level k+1); level M lands in hNew
    const bool SUB = T && c->fuse_sub && m.st.nTiles > 0 && c->deep_runs_ok;
    double *hrot[3] = {hNew, st.hT, st.hT2};
    auto hb = [&](int k) { return SUB ? hrot[(M - 1 - k) % 3] : (((M - 1 - k) % 2 == 0) ? hNew : st.hT); };
    auto ub = [&](int k) { return ((M - 1 - k) % 2 == 0) ? uNew : st.uT; };
    auto pred = [&](int k) {
        PredConst pc;
        pc.a = (double)k / (double)M;
        pc.oma = 1.0 - pc.a;
        pc.a1 = (double)(k + 1) / (double)M;
        pc.oma1 = 1.0 - pc.a1;
        pc.b = 1.0 / (double)M;
        pc.c = 1.0 - (double)(k + 1) / (double)M;
        return pc;
    };
    // band sweep of fine stage 2 / 3 on the side stream (captured steps of one rank, staged path)
    // (measured: config 2 0.263 -> 0.224 ms per step, hex2048 2.440 -> 2.432, config 5 9.49 -> 9.54:
    // beside a long persistent deep sweep the band kernel only steals its SMs, so meshes of 8 M
    // owned cells and more keep one stream)
    const bool bandPar = !rec && T && c->side && c->band_side && c->cfg.nranks == 1 && m.nOwnC < (8 << 20);
    auto band_fork = [&]() -> cudaStream_t {
        if (!bandPar) return s;
        cudaEventRecord(c->evSideF, s);
        cudaStreamWaitEvent(c->side, c->evSideF, 0);
        return c->side;
    };
    auto band_join = [&](cudaStream_t sb) {
        if (sb == s) return;
        cudaEventRecord(c->evSideJ, sb);
        cudaStreamWaitEvent(s, c->evSideJ, 0);
    };
    const int subBegin = B.fl[c->sub_level];
    const int deepEnd = SUB ? subBegin : B.end;    // the staged deep kernels stop where the subcycle tiles start
    *px = PhaseX{-1, nullptr, -1, nullptr};
    const int nfine = c->have_fine ? 3 * M : 0;
    if (ph > 3 + nfine) return false;
    bool any = false;
    auto cell_mark = [&](int k) {      // part 1 adds time to the sweep part 0 counted (kind + 64)
        if (cells) {
            mark(part == 0 ? k : k + 64);
            any = true;
        }
    };
    if (ph == 0) {
        if (part == 0 && c->cfg.slow) {
            mark(K_SLOW_PRE);
            launch_slow_pre(m, st, hN, uN, s);
            mark(K_SLOW_EDGE);
            launch_slow_edge_range(m, st, hN, uN, st.S, 0, m.nOwnE, sc, s, c->cfg.vorticity ? st.Pv : nullptr);
            any = true;
        } else if (part == 0 && c->cfg.vorticity) {
            cudaMemsetAsync(st.Pv, 0, (size_t)std::max(1, m.nOwnE) * 8, s);   // gravity-wave model: no PV flux
        }
        cell_mark(K_COARSE_S1);
        if (T) stage_tiled(c, 1, B, B.begin, B.fl[5], StageArgs{hN, hN, uN, st.S, st.h1, 0, 0, 0, sc.c1, sc.g, K_COARSE_S1, -1}, s);
        else launch_coarse_s1(m, st, hN, uN, sc, s, B);
        *px = PhaseX{X_C1, st.h1, -1, nullptr};
    } else if (ph == 1) {
        cell_mark(K_COARSE_S2);
        if (T)
            stage_tiled(c, 2, B, B.begin, B.fl[3],
                        StageArgs{hN, st.h1, uN, st.S, st.h2, sc.c1, sc.b1, sc.omb1, sc.c2, sc.g, K_COARSE_S2, -1}, s);
        else launch_coarse_s2(m, st, hN, uN, sc, s, B);
        *px = PhaseX{X_C1, st.h2, -1, nullptr};
    } else if (ph == 2) {
        cell_mark(K_COARSE_S3);
        if (T)
            stage_tiled(c, 3, B, B.begin, B.fl[1],
                        StageArgs{hN, st.h2, uN, st.S, hNew, sc.c2, sc.b2, sc.omb2, sc.c3, sc.g, K_COARSE_S3, -1}, s);
        else launch_coarse_s3(m, st, hN, uN, hNew, sc, s, B);
        *px = PhaseX{X_C1, hNew, -1, nullptr};
    } else if (ph - 3 < nfine) {
        const int q = ph - 3, k = q / 3, stg = q % 3;
        const double *hk = k == 0 ? hN : hb(k - 1), *uk = k == 0 ? uN : ub(k - 1);
        if (stg == 0) {
            // k >= 1 with the fusion: the band velocity sweep runs alone and the deep velocity sweep
            // of subcycle k-1 is folded into the deep stage-1 sweep of subcycle k (STAGE 4)
            const bool fused = k > 0 && T && (c->fuse_vel || SUB) && c->deep_runs_ok;
            // stage 0 keeps the band sweeps on the compute stream: beside the persistent deep sweep the
            // coarse / band velocity sweeps measured slower on hex2048 (2.51 vs 2.43 ms per step)
            const bool par0 = false;
            const cudaStream_t sv = par0 ? band_fork() : s;
            if (part == 0) {
                if (k == 0) {
                    mark(K_COARSE_VEL);
                    launch_coarse_vel(m, st, hN, uN, hNew, uNew, sc, sv, true);
                } else {
                    mark(K_FINE_VEL);
                    launch_fine_vel(m, st, hN, hNew, k - 1 == 0 ? hN : hb(k - 2), hb(k - 1),
                                    k - 1 == 0 ? uN : ub(k - 2), ub(k - 1), sc, pred(k - 1), k - 1, sv, !fused);
                }
                any = true;
            }
            cell_mark(K_FINE_S1);
            if (!par0 || k == 0) launch_fine_s1(m, st, hN, hNew, hk, uk, sc, pred(k), k, sv, B, !T);
            if (fused) {
                cell_mark(K_FINE_VS1);
                StageArgs va{k - 1 == 0 ? hN : hb(k - 2), hk, k - 1 == 0 ? uN : ub(k - 2), st.Sf, st.h1,
                             sc.c3f, sc.b3, sc.om2b3, sc.c1f, sc.g, K_FINE_VS1, k};
                va.h2 = st.h2;
                va.unew = ub(k - 1);
                stage_tiled(c, 4, B, B.fl[1], deepEnd, va, s);
            } else if (T) {
                stage_tiled(c, 1, B, B.fl[1], deepEnd, StageArgs{hk, hk, uk, st.S, st.h1, 0, 0, 0, sc.c1f, sc.g, K_FINE_S1, k}, s);
            }
            if (par0) {
                band_join(sv);
                if (k > 0) launch_fine_s1(m, st, hN, hNew, hk, uk, sc, pred(k), k, s, B, !T);
            }
            if (SUB && part == 0) {
                // the whole subcycle k on F\F^2 (after the kernels above, which read level k-1 and
                // stage 2 of k-1 there; before the stage-2/3 sweeps, which read its stage 1 / 2)
                mark(K_FINE_SUB);
                SubArgs sa{hk, k == 0 ? hN : (k - 1 == 0 ? hN : hb(k - 2)), st.h2, k == 0 ? uN : (k - 1 == 0 ? uN : ub(k - 2)),
                           st.Sf, k == 0 ? nullptr : ub(k - 1), st.h1, k == 0 ? st.h2 : st.h2alt, hb(k),
                           sc.g, sc.b1, sc.omb1, sc.b2, sc.omb2, sc.b3, sc.om2b3, sc.c1f, sc.c2f, sc.c3f, k};
                launch_fine_sub(m, k > 0, c->nsm, sa, st.err, s);
                if (k > 0)        // publish stage 2 (the tiles read stage 2 of k-1 on their rings)
                    cudaMemcpyAsync(st.h2 + subBegin, st.h2alt + subBegin, (size_t)(B.end - subBegin) * 8,
                                    cudaMemcpyDeviceToDevice, s);
                any = true;
            }
            *px = PhaseX{X_C1, st.h1, -1, nullptr};
        } else if (stg == 1) {
            if (part == 0 && c->cfg.slow_refresh && c->cfg.slow) {
                // S^k on F_E from the state at t^{n,k}; S^0 = S (identical views)
                mark(K_SLOW_REFRESH);
                if (k == 0) {
                    if (m.eb.end > m.eb.f)
                        cudaMemcpyAsync(st.Sk + m.eb.f, st.S + m.eb.f, (size_t)(m.eb.end - m.eb.f) * 8,
                                        cudaMemcpyDeviceToDevice, s);
                } else {
                    launch_refresh_views(m, st, hN, hNew, hk, uN, uk, sc, pred(k), s);
                    launch_slow_pre_range(m, st, st.hv, st.uv, c->vminF, m.cb.if1, m.eb.if1, s, c->vminF1);
                    launch_slow_edge_range(m, st, st.hv, st.uv, st.Sk, m.eb.f, m.eb.end, sc, s);
                }
                any = true;
            }
            cell_mark(K_FINE_S2);
            cudaStream_t sb = band_fork();
            launch_fine_s2(m, st, hN, hNew, hk, uk, sc, pred(k), k, sb, B, !T);
            if (T)
                stage_tiled(c, 2, B, B.fl[1], deepEnd,
                            StageArgs{hk, st.h1, uk, st.Sf, st.h2, sc.c1f, sc.b1, sc.omb1, sc.c2f, sc.g, K_FINE_S2, k}, s);
            band_join(sb);
            *px = PhaseX{X_C1, st.h2, -1, nullptr};
        } else {
            cell_mark(K_FINE_S3);
            cudaStream_t sb = band_fork();
            launch_fine_s3(m, st, hN, uN, hNew, hk, uk, hb(k), sc, pred(k), k, sb, B, !T);
            if (T)
                stage_tiled(c, 3, B, B.fl[1], deepEnd,
                            StageArgs{hk, st.h2, uk, st.Sf, hb(k), sc.c2f, sc.b2, sc.omb2, sc.c3f, sc.g, K_FINE_S3, k}, s);
            band_join(sb);
            *px = PhaseX{X_C1, hb(k), -1, nullptr};
        }
    } else {                                     // ph == 3 + nfine: last velocity sweep, correction
        if (c->have_fine) {
            if (part == 0) {
                mark(K_FINE_VEL);
                launch_fine_vel(m, st, hN, hNew, M - 1 == 0 ? hN : hb(M - 2), hb(M - 1), M - 1 == 0 ? uN : ub(M - 2),
                                ub(M - 1), sc, pred(M - 1), M - 1, s);
                any = true;
            }
            if (cells || part == 0) {
                mark(part == 0 ? K_CORRECT : K_CORRECT + 64);
                any = true;
            }
            launch_correct(m, st, hN, uN, hNew, uNew, sc, s, B, part == 0);
        } else if (part == 0) {
            mark(K_COARSE_VEL);
            launch_coarse_vel(m, st, hN, uN, hNew, uNew, sc, s);
            any = true;
        }
        if (part == 0 && c->cfg.vorticity) {       // prognostic eta (Theorem 2), frozen PV flux
            launch_vort_split(m, st, sc, s);
            launch_vort_update(m, st, s);
        }
        *px = PhaseX{X_C2, hNew, X_E, uNew};
    }
    if (any) mark(-1);
    return true;
}

void pack(fblts_ctx *c, int x, const double *a, cudaStream_t s) {
    const Xchg &X = c->lo.x[x];
    launch_pack(c->ds.xidx + X.sendAt, a, c->ds.sendbuf, (int)X.sendIdx.size(), s);
}
void unpack(fblts_ctx *c, int x, double *a, cudaStream_t s) {
    const Xchg &X = c->lo.x[x];
    launch_unpack(c->ds.xidx + X.recvAt, c->ds.recvbuf, a, (int)X.recvIdx.size(), s);
}


// pack -> grouped ncclSend/ncclRecv with every peer sharing a halo -> unpack, all on stream s
int exchange_nccl(fblts_ctx *c, int x, double *a, cudaStream_t s) {
    if (x < 0) return FBLTS_OK;
    const Xchg &X = c->lo.x[x];
    pack(c, x, a, s);
    ncclComm_t comm = (ncclComm_t)c->nccl;
    NCCL_TRY(c, ncclGroupStart());
    for (int p = 0; p < c->cfg.nranks; ++p) {
        if (p == c->cfg.rank) continue;
        const size_t ns = X.sendOff[p + 1] - X.sendOff[p], nr = X.recvOff[p + 1] - X.recvOff[p];
        if (ns) NCCL_TRY(c, ncclSend(c->ds.sendbuf + X.sendOff[p], ns, ncclDouble, p, comm, s));
        if (nr) NCCL_TRY(c, ncclRecv(c->ds.recvbuf + X.recvOff[p], nr, ncclDouble, p, comm, s));
    }
    NCCL_TRY(c, ncclGroupEnd());
    unpack(c, x, a, s);
    return FBLTS_OK;
}

int allgather_nccl(fblts_ctx *c, const double *send6, double *recv) {
    (void)send6;   // the partial sums are already on the device at diag_out
    NCCL_TRY(c, ncclAllGather(c->diag_out, c->diag_out + 8, 6, ncclDouble, (ncclComm_t)c->nccl, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(recv, c->diag_out + 8, 6 * sizeof(double) * c->cfg.nranks, cudaMemcpyDeviceToHost,
                                c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return FBLTS_OK;
}

// One coarse step on one rank: every phase; with several ranks each stage's halo exchange runs on
// the communication stream, forked after the phase's boundary-block kernel and joined before the
// next phase, so it overlaps the interior-block kernel (the end-of-step exchange of rings 1-2 and
// of the remote-owned edges needs the interior values and runs after it).
// One classical RK4 step (FBLTS_SCHEME_RK4, one rank): per stage the slow terms at the stage state,
// then one launch for every cell and edge (stage tendency, running sum, next stage state).
int enqueue_rk4_step(fblts_ctx *c, int par, cudaStream_t s, Recorder *rec) {
    const DevMesh &m = c->dm;
    DevState st = c->ds;
    const double *hN = c->hbuf[par], *uN = c->ubuf[par];
    double *hNew = c->hbuf[1 - par], *uNew = c->ubuf[1 - par];
    const double dt = c->cfg.dt;
    const double cn[4] = {dt / 2, dt / 2, dt, 0.0};
    const double *hs = hN, *us = uN;
    double *hb[2] = {st.h1, st.h2};
    for (int stage = 1; stage <= 4; ++stage) {
        if (c->cfg.slow) {
            if (rec) rec->mark(K_SLOW_PRE, s);
            launch_slow_pre(m, st, hs, us, s);
            if (rec) rec->mark(K_SLOW_EDGE, s);
            launch_slow_edge(m, st, hs, us, c->sc, s);
        }
        double *ho = stage < 4 ? hb[stage % 2] : hNew;
        double *uo = stage < 4 ? st.rkU[stage % 2] : uNew;
        if (rec) rec->mark(K_RK4_STAGE, s);
        launch_rk4_stage(m, st, stage, hN, uN, hs, us, ho, uo, cn[stage - 1], dt / 6, c->sc.g, s);
        hs = ho;
        us = uo;
    }
    if (rec) rec->mark(-1, s);
    return FBLTS_OK;
}

// One RK(3,2) step (FBLTS_SCHEME_RK32, one rank; Wicker & Skamarock, the scheme FB-RK(3,2) extends,
// P:L283-285; oracle fbrk32.rk32_step): stage s = 1, 2, 3 evaluates the slow terms at the previous
// stage's (u, h), then one launch over every cell and edge writes (h, u)_s = (h, u)^n + c_s (Psi, Phi^fast
// + S) with c_s = dt/3, dt/2, dt (no running sum: launch_rk4_stage with stage 0).
int enqueue_rk32_step(fblts_ctx *c, int par, cudaStream_t s, Recorder *rec) {
    const DevMesh &m = c->dm;
    DevState st = c->ds;
    const double *hN = c->hbuf[par], *uN = c->ubuf[par];
    double *hNew = c->hbuf[1 - par], *uNew = c->ubuf[1 - par];
    const double dt = c->cfg.dt;
    const double cs[3] = {dt / 3.0, dt / 2.0, dt};
    const double *hs = hN, *us = uN;
    double *hb[2] = {st.h1, st.h2};
    for (int stage = 1; stage <= 3; ++stage) {
        if (c->cfg.slow) {
            if (rec) rec->mark(K_SLOW_PRE, s);
            launch_slow_pre(m, st, hs, us, s);
            if (rec) rec->mark(K_SLOW_EDGE, s);
            launch_slow_edge(m, st, hs, us, c->sc, s);
        }
        double *ho = stage < 3 ? hb[stage % 2] : hNew;
        double *uo = stage < 3 ? st.rkU[stage % 2] : uNew;
        if (rec) rec->mark(K_RK4_STAGE, s);
        launch_rk4_stage(m, st, 0, hN, uN, hs, us, ho, uo, cs[stage - 1], 0.0, c->sc.g, s);
        hs = ho;
        us = uo;
    }
    if (rec) rec->mark(-1, s);
    return FBLTS_OK;
}

// One unsplit FB-LTS coarse step (config unsplit, one rank): per stage a thickness
// sweep with the stored stage velocity, the FB-averaged thickness (coarse) or the stage's HS and U
// views (fine), the slow sweeps on the stage's extent and the velocity sweep (oracle lts.py split=False).
int enqueue_unsplit_step(fblts_ctx *c, int par, cudaStream_t s, Recorder *rec) {
    const DevMesh &m = c->dm;
    DevState st = c->ds;
    const StepConst &sc = c->sc;
    const double *hN = c->hbuf[par], *uN = c->ubuf[par];
    double *hNew = c->hbuf[1 - par], *uNew = c->ubuf[1 - par];
    const int M = sc.M;
    auto mark = [&](int k) {
        if (rec) rec->mark(k, s);
    };
    auto hb = [&](int k) { return ((M - 1 - k) % 2 == 0) ? hNew : st.hT; };
    auto ub = [&](int k) { return ((M - 1 - k) % 2 == 0) ? uNew : st.uT; };
    auto pred = [&](int k) {
        PredConst pc;
        pc.a = (double)k / (double)M;
        pc.oma = 1.0 - pc.a;
        pc.a1 = (double)(k + 1) / (double)M;
        pc.oma1 = 1.0 - pc.a1;
        pc.b = 1.0 / (double)M;
        pc.c = 1.0 - (double)(k + 1) / (double)M;
        return pc;
    };
    const bool vort = c->cfg.vorticity != 0;
    // slow sweeps + velocity update on [e0, e1): with the slow terms on, the update runs inside the
    // slow edge sweep (VelFuse: no S store, no separate velocity sweep; the same bits as k_un_vel)
    auto slow_vel = [&](const double *U, int e0, int e1, double *pvout, int vkind, const double *base, double *out,
                        double cc, double *acc, int a0, int a1, int first) {
        if (!c->cfg.slow) {                                 // S = 0 (and the PV flux part)
            if (e1 > e0) cudaMemsetAsync(st.Sk + e0, 0, (size_t)(e1 - e0) * 8, s);
            if (pvout && e1 > e0) cudaMemsetAsync(pvout + e0, 0, (size_t)(e1 - e0) * 8, s);
            mark(vkind);
            launch_un_vel(m, st, base, out, cc, e0, e1, acc, a0, a1, first, sc, s);
            return;
        }
        mark(K_SLOW_PRE);
        // S on F_E needs q, K, F only on its stencil (vertices of F_E edges, cells from IF-1, edges
        // from IF-1_E; the slow-term refresh's range); wider extents and the energy-conserving PV
        // flux (q_hat on the edges of the cells of F_E edges: one more vertex ring) take the whole mesh
        if (e0 >= m.eb.f && !sc.pve) launch_slow_pre_range(m, st, st.hv, U, c->vminF, m.cb.if1, m.eb.if1, s, c->vminF1);
        else launch_slow_pre_range(m, st, st.hv, U, 0, 0, 0, s);
        mark(K_SLOW_EDGE);
        if (!c->un_fuse) {                                  // FBLTS_UNFUSE=0: S stored, separate velocity sweep
            launch_slow_edge_range(m, st, st.hv, U, st.Sk, e0, e1, sc, s, pvout);
            mark(vkind);
            launch_un_vel(m, st, base, out, cc, e0, e1, acc, a0, a1, first, sc, s);
            return;
        }
        VelFuse vf;
        vf.base = base;
        vf.out = out;
        vf.c = cc;
        vf.acc = acc;
        vf.a0 = a0;
        vf.a1 = a1;
        vf.first = first;
        launch_slow_edge_range(m, st, st.hv, U, nullptr, e0, e1, sc, s, pvout, &vf);
    };
    // fine views of stages 1-2 on the F_E slow stencil only (the energy-conserving PV flux reads the whole mesh)
    const int v12c = sc.pve ? 0 : c->un_c12, v12e = sc.pve ? 0 : c->un_e12;
    // ---- coarse phase: extents X1 = C u F^5, Y1 = C_E u F^4_E, X2 = C u F^3, Y2 = C_E u F^2_E,
    //      X3 = C u F^1, Y3 = IF-1_E u int_E (IF-2_E computed as scratch)
    const double *Hs[3] = {hN, st.h1, st.h2};
    const double *Us[3] = {uN, st.un[0], st.un[1]};
    double *Hout[3] = {st.h1, st.h2, hNew};
    const int Xend[3] = {m.cb.fl[5], m.cb.fl[3], m.cb.fl[1]}, Yend[3] = {m.eb.fl[4], m.eb.fl[2], m.eb.f};
    const double cs[3] = {sc.c1, sc.c2, sc.c3};
    const int kinds[3] = {K_COARSE_S1, K_COARSE_S2, K_COARSE_S3};
    for (int q = 0; q < 3; ++q) {
        mark(kinds[q]);
        launch_un_cstage(m, st, q + 1, hN, Hs[q], Us[q], Hout[q], sc, Xend[q], s);
        slow_vel(Us[q], 0, Yend[q], vort && q == 2 ? st.Pv : nullptr, K_COARSE_VEL, uN, st.un[q], cs[q], nullptr, 0, 0,
                 0);
        if (vort && q == 2) launch_vort_int(st, sc.c3, m.eb.if2, s);     // eta companion: int_E, dt PV
    }
    if (m.eb.if2 > 0) CUDA_TRY(c, cudaMemcpyAsync(uNew, st.un[2], (size_t)m.eb.if2 * 8, cudaMemcpyDeviceToDevice, s));
    // ---- fine phase
    if (c->have_fine) {
        for (int k = 0; k < M; ++k) {
            const double *hk = k == 0 ? hN : hb(k - 1), *uk = k == 0 ? uN : ub(k - 1);
            const PredConst pc = pred(k);
            mark(K_FINE_S1);                                         // stage 1: thickness (U0 = u^{n,k} on F_E)
            launch_fine_s1(m, st, hN, hNew, hk, uk, sc, pc, k, s, m.cb, true);
            launch_un_views(m, st, 1, hN, hNew, hk, nullptr, uN, uk, sc, pc, s, v12c, v12e);
            slow_vel(st.uv, m.eb.f, m.eb.end, nullptr, K_FINE_VEL, uk, st.unk[0], sc.c1f, nullptr, 0, 0, 0);
            mark(K_FINE_S2);                                         // stage 2
            launch_un_fstage(m, st, 2, hN, hNew, hk, st.unk[0], st.h2, sc, pc, k, s);
            launch_un_views(m, st, 2, hN, hNew, hk, nullptr, uN, st.unk[0], sc, pc, s, v12c, v12e);
            slow_vel(st.uv, m.eb.f, m.eb.end, nullptr, K_FINE_VEL, uk, st.unk[1], sc.c2f, nullptr, 0, 0, 0);
            mark(K_FINE_S3);                                         // stage 3 + correction summands
            launch_un_views(m, st, 3, hN, hNew, hk, hk, uN, st.unk[1], sc, pc, s, m.nOwnC, c->un_e3);   // U2 view for the sweep
            launch_un_fstage(m, st, 3, hN, hNew, hk, st.uv, hb(k), sc, pc, k, s);
            launch_un_views(m, st, 3, hN, hNew, hk, hb(k), uN, st.unk[1], sc, pc, s, 0, 0);
            slow_vel(st.uv, m.eb.if2, m.eb.end, vort ? st.Pv : nullptr, K_FINE_VEL, uk, ub(k), sc.c3f, st.accU, m.eb.if2,
                     m.eb.f, k == 0);
            if (vort) launch_vort_fine(m, st, sc.c3f, k == 0, s);   // F_E: += dt/M PV^k; IF edges: sum_k PV^k
        }
        mark(K_CORRECT);
        launch_correct(m, st, hN, uN, hNew, uNew, sc, s, m.cb, true);
        if (vort) launch_vort_close(m, st, sc.c3f, s);             // IF edges: dt/M sum_k PV^k
    }
    if (vort) launch_vort_update(m, st, s);                        // eta_v += (sum t d dP) / A_v
    mark(-1);
    return FBLTS_OK;
}

int enqueue_step(fblts_ctx *c, int par, cudaStream_t s, Recorder *rec) {
    if (c->cfg.scheme == FBLTS_SCHEME_RK4) return enqueue_rk4_step(c, par, s, rec);
    if (c->cfg.scheme == FBLTS_SCHEME_RK32) return enqueue_rk32_step(c, par, s, rec);
    if (c->cfg.unsplit) return enqueue_unsplit_step(c, par, s, rec);
    const bool multi = c->cfg.nranks > 1;
    PhaseX px, px1;
    for (int ph = 0; enqueue_phase(c, par, ph, s, rec, &px, 0); ++ph) {
        const bool overlap = multi && px.x >= 0 && px.x2 < 0;
        if (overlap) {
            CUDA_TRY(c, cudaEventRecord(c->evFork, s));
            CUDA_TRY(c, cudaStreamWaitEvent(c->comm, c->evFork, 0));
            const int rc = exchange_nccl(c, px.x, px.a, c->comm);
            if (rc) return rc;
            CUDA_TRY(c, cudaEventRecord(c->evJoin, c->comm));
        }
        enqueue_phase(c, par, ph, s, rec, &px1, 1);
        if (overlap) {
            CUDA_TRY(c, cudaStreamWaitEvent(s, c->evJoin, 0));
        } else if (multi) {
            int rc = exchange_nccl(c, px.x, px.a, s);
            if (!rc && px.x2 >= 0) rc = exchange_nccl(c, px.x2, px.a2, s);
            if (rc) return rc;
        }
    }
    return FBLTS_OK;
}

int capture(fblts_ctx *c, int par) {
    cudaGraph_t g;
    CUDA_TRY(c, cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
    const int rc = enqueue_step(c, par, c->cap, nullptr);
    cudaError_t e = cudaStreamEndCapture(c->cap, &g);
    if (rc) return rc;
    CUDA_TRY(c, e);
    size_t nodes = 0;
    CUDA_TRY(c, cudaGraphGetNodes(g, nullptr, &nodes));
    c->graph_nodes = nodes;
    CUDA_TRY(c, cudaGraphInstantiate(&c->exec[par], g, 0));
    CUDA_TRY(c, cudaGraphDestroy(g));
    return FBLTS_OK;
}

int check_device_error(fblts_ctx *c) {
    DevError e{};
    CUDA_TRY(c, cudaMemcpy(&e, c->ds.err, sizeof e, cudaMemcpyDeviceToHost));
    if (e.flag) {
        const int idx = e.index >= 0 && e.index < c->lo.nC ? c->lo.cellGlob[e.index] : -1;
        return fail(c, FBLTS_ERR_POSITIVITY, "positivity: h=%g in %s (subcycle k=%d) at cell %d (region %d)", e.value,
                    fblts_kernel_name(e.kind), e.k, idx, idx >= 0 ? (int)c->rg.cell[idx] : -1);
    }
    return FBLTS_OK;
}

// host double-double merge, identical to the device one
void dd_merge_host(double &ah, double &al, double bh, double bl) {
    const double s = ah + bh;
    const double bb = s - ah;
    const double err = (ah - (s - bb)) + (bh - bb) + (al + bl);
    const double hi = s + err;
    al = err - (hi - s);
    ah = hi;
}

int diag_partial(fblts_ctx *c, double out6[6], bool cells_only = false, bool pv = false) {
    launch_diagnostics(c->dm, c->hbuf[c->parity], c->ubuf[c->parity], c->sc, c->ds.diag, c->diag_out, c->stream,
                       cells_only, pv);
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaMemcpyAsync(out6, c->diag_out, 6 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return FBLTS_OK;
}

// asynchronous diagnostics: the compute stream waits for the last asynchronous reduction that
// reads state buffer b before anything overwrites b
constexpr int DIAG_RING = 1024;
void diag_wait(fblts_ctx *c, int b) {
    if (c->diagPending[b]) {
        cudaStreamWaitEvent(c->stream, c->evDiag[b], 0);
        c->diagPending[b] = false;
    }
}
void diag_combine(const double *parts, int n, double out[4]);
void CUDART_CB diag_host_fn(void *p) {
    const fblts_ctx::DiagJob *j = static_cast<const fblts_ctx::DiagJob *>(p);
    if (j->mass_only) {
        double four[4];
        diag_combine(j->slot, 1, four);
        j->out[0] = four[0];
        j->out[1] = four[2];
    } else {
        diag_combine(j->slot, 1, j->out);
    }
}

void diag_combine(const double *parts, int n, double out[4]) {
    double mh = 0.0, ml = 0.0, gh = 0.0, gl = 0.0, hmin = INFINITY, numax = 0.0;
    for (int r = 0; r < n; ++r) {
        dd_merge_host(mh, ml, parts[6 * r + 0], parts[6 * r + 1]);
        dd_merge_host(gh, gl, parts[6 * r + 2], parts[6 * r + 3]);
        hmin = std::min(hmin, parts[6 * r + 4]);
        numax = std::max(numax, parts[6 * r + 5]);
    }
    out[0] = mh + ml;
    out[1] = gh + gl;
    out[2] = hmin;
    out[3] = numax;
}


}  // namespace

extern "C" {

int fblts_step(fblts_ctx *c, int32_t n) {
    if (!c || n < 0) return FBLTS_ERR_INVALID_ARG;
    if (c->phase != P_STATE) return fail(c, FBLTS_ERR_ORDER, "step: call set_state first");
    if (c->cfg.nranks > 1 && !c->nccl) return fail(c, FBLTS_ERR_ORDER, "step: loopback contexts use fblts_step_group");
    CUDA_TRY(c, cudaSetDevice(c->cfg.device));
    for (int p = 0; p < 2; ++p)
        if (!c->exec[p]) {
            const int rc = capture(c, p);
            if (rc) return rc;
        }
    nvtxRangePushA("fblts_step");           // one NVTX range per call (n graph replays, one per coarse step)
    for (int i = 0; i < n; ++i) {
        diag_wait(c, 1 - c->parity);
        const cudaError_t e = cudaGraphLaunch(c->exec[c->parity], c->stream);
        if (e != cudaSuccess) {
            nvtxRangePop();
            return fail(c, FBLTS_ERR_CUDA, "cudaGraphLaunch: %s", cudaGetErrorString(e));
        }
        c->parity ^= 1;
        c->t += c->cfg.dt;
    }
    nvtxRangePop();
    return FBLTS_OK;
}

// Loopback group step: the nranks contexts of ONE process (all on one device and one stream)
// advance together phase by phase; a halo exchange is a device-to-device copy from the peer's
// send buffer.  No kernel waits on another; used to test the partitioned path on one GPU.
int fblts_step_group(fblts_ctx **cs, int32_t n, int32_t n_coarse) {
    if (!cs || n < 1 || n_coarse < 0) return FBLTS_ERR_INVALID_ARG;
    for (int r = 0; r < n; ++r) {
        if (!cs[r] || cs[r]->cfg.rank != r || cs[r]->cfg.nranks != n) return FBLTS_ERR_INVALID_ARG;
        if (cs[r]->phase != P_STATE) return fail(cs[r], FBLTS_ERR_ORDER, "step_group: call set_state first");
        if (cs[r]->stream != cs[0]->stream) return fail(cs[r], FBLTS_ERR_INVALID_ARG, "step_group: one stream");
    }
    cudaStream_t s = cs[0]->stream;
    for (int it = 0; it < n_coarse; ++it) {
        std::vector<PhaseX> px(n), px1(n);
        for (int ph = 0;; ++ph) {
            bool any = false;
            for (int r = 0; r < n; ++r) any = enqueue_phase(cs[r], cs[r]->parity, ph, s, nullptr, &px[r], 0) || any;
            if (!any) break;
            // stage exchanges depend on the boundary blocks only (as in the overlapped NCCL path);
            // the end-of-step exchange follows the interior blocks
            const bool stage_x = px[0].x2 < 0;
            if (!stage_x)
                for (int r = 0; r < n; ++r) enqueue_phase(cs[r], cs[r]->parity, ph, s, nullptr, &px1[r], 1);
            for (int pass = 0; pass < 2; ++pass) {
                for (int r = 0; r < n; ++r) {
                    const int x = pass == 0 ? px[r].x : px[r].x2;
                    if (x >= 0) pack(cs[r], x, pass == 0 ? px[r].a : px[r].a2, s);
                }
                for (int r = 0; r < n; ++r) {
                    const int x = pass == 0 ? px[r].x : px[r].x2;
                    if (x < 0) continue;
                    const Xchg &X = cs[r]->lo.x[x];
                    for (int p = 0; p < n; ++p) {
                        const int64_t cnt = X.recvOff[p + 1] - X.recvOff[p];
                        if (!cnt) continue;
                        const Xchg &Y = cs[p]->lo.x[x];
                        if (Y.sendOff[r + 1] - Y.sendOff[r] != cnt)
                            return fail(cs[r], FBLTS_ERR_INVALID_ARG, "step_group: halo size mismatch with rank %d", p);
                        CUDA_TRY(cs[r], cudaMemcpyAsync(cs[r]->ds.recvbuf + X.recvOff[p], cs[p]->ds.sendbuf + Y.sendOff[r],
                                                        cnt * 8, cudaMemcpyDeviceToDevice, s));
                    }
                }
                for (int r = 0; r < n; ++r) {
                    const int x = pass == 0 ? px[r].x : px[r].x2;
                    if (x >= 0) unpack(cs[r], x, pass == 0 ? px[r].a : px[r].a2, s);
                }
            }
            if (stage_x)
                for (int r = 0; r < n; ++r) enqueue_phase(cs[r], cs[r]->parity, ph, s, nullptr, &px1[r], 1);
        }
        for (int r = 0; r < n; ++r) {
            cs[r]->parity ^= 1;
            cs[r]->t += cs[r]->cfg.dt;
        }
    }
    CUDA_TRY(cs[0], cudaGetLastError());
    return FBLTS_OK;
}

int fblts_sync(fblts_ctx *c) {
    if (!c) return FBLTS_ERR_INVALID_ARG;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->dstream) CUDA_TRY(c, cudaStreamSynchronize(c->dstream));
    if (c->phase >= P_BOUND) return check_device_error(c);
    return FBLTS_OK;
}

int fblts_get_state(fblts_ctx *c, double *h, double *u, double *t) {
    if (!c) return FBLTS_ERR_INVALID_ARG;
    if (c->phase != P_STATE) return fail(c, FBLTS_ERR_ORDER, "get_state: no state set");
    cudaStream_t s = c->stream;
    const Local &L = c->lo;
    // owned entries only (all entries for one rank); other entries of h, u are left untouched
    if (h) {
        if (c->cfg.nranks > 1) CUDA_TRY(c, cudaMemcpyAsync(c->ds.stage, h, (size_t)c->hm.nC * 8, cudaMemcpyHostToDevice, s));
        launch_permute_out(c->ds.cellOld, c->hbuf[c->parity], c->ds.stage, L.nOwnC, s);
        CUDA_TRY(c, cudaMemcpyAsync(h, c->ds.stage, (size_t)c->hm.nC * 8, cudaMemcpyDeviceToHost, s));
    }
    if (u) {
        CUDA_TRY(c, cudaStreamSynchronize(s));
        if (c->cfg.nranks > 1) CUDA_TRY(c, cudaMemcpyAsync(c->ds.stage, u, (size_t)c->hm.nE * 8, cudaMemcpyHostToDevice, s));
        launch_permute_out(c->ds.edgeOld, c->ubuf[c->parity], c->ds.stage, L.nOwnE, s);
        CUDA_TRY(c, cudaMemcpyAsync(u, c->ds.stage, (size_t)c->hm.nE * 8, cudaMemcpyDeviceToHost, s));
    }
    CUDA_TRY(c, cudaStreamSynchronize(s));
    if (c->dstream) CUDA_TRY(c, cudaStreamSynchronize(c->dstream));   // outstanding async diagnostics
    CUDA_TRY(c, cudaGetLastError());
    if (t) *t = c->t;
    return check_device_error(c);
}

int fblts_get_vorticity(fblts_ctx *c, double *eta) {
    if (!c || !eta) return FBLTS_ERR_INVALID_ARG;
    if (!c->cfg.vorticity) return fail(c, FBLTS_ERR_ORDER, "get_vorticity: context created without cfg.vorticity");
    if (c->phase != P_STATE) return fail(c, FBLTS_ERR_ORDER, "get_vorticity: no state set");
    const Local &L = c->lo;
    std::vector<double> tmp(L.nV);
    CUDA_TRY(c, cudaMemcpyAsync(tmp.data(), c->ds.eta, (size_t)L.nV * 8, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    for (int v = 0; v < L.nV; ++v) eta[L.vertGlob[v]] = tmp[v];
    return check_device_error(c);
}

static int diagnostics_async(fblts_ctx *c, double *out, bool mass_only);
int fblts_diagnostics_async(fblts_ctx *c, double *out) { return diagnostics_async(c, out, false); }
int fblts_diagnostics_mass_async(fblts_ctx *c, double *out) { return diagnostics_async(c, out, true); }
static int diagnostics_async(fblts_ctx *c, double *out, bool mass_only) {
    if (!c || !out) return FBLTS_ERR_INVALID_ARG;
    if (c->phase != P_STATE) return fail(c, FBLTS_ERR_ORDER, "diagnostics_async: no state set");
    if (c->cfg.nranks > 1) return fail(c, FBLTS_ERR_ORDER, "diagnostics_async: one rank (use fblts_diagnostics)");
    CUDA_TRY(c, cudaSetDevice(c->cfg.device));
    if (!c->dstream) {
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->dstream, cudaStreamNonBlocking));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->evHead, cudaEventDisableTiming));
        for (auto &e : c->evDiag) CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CUDA_TRY(c, cudaHostAlloc((void **)&c->dhost, sizeof(double) * 6 * DIAG_RING, cudaHostAllocDefault));
        c->djobs = new fblts_ctx::DiagJob[DIAG_RING];
    }
    const uint64_t k = c->ndiag++;
    if (k > 0 && k % DIAG_RING == 0) CUDA_TRY(c, cudaStreamSynchronize(c->dstream));   // ring slots reusable
    const int slot = (int)(k % DIAG_RING), b = c->parity;
    CUDA_TRY(c, cudaEventRecord(c->evHead, c->stream));                // the state the caller sees now
    CUDA_TRY(c, cudaStreamWaitEvent(c->dstream, c->evHead, 0));
    double *dout = c->ds.diagA + DIAG_BLOCKS * 6;
    launch_diagnostics(c->dm, c->hbuf[b], c->ubuf[b], c->sc, c->ds.diagA, dout, c->dstream, mass_only);
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaEventRecord(c->evDiag[b], c->dstream));
    c->diagPending[b] = true;
    double *hs = c->dhost + 6 * (size_t)slot;
    CUDA_TRY(c, cudaMemcpyAsync(hs, dout, 6 * sizeof(double), cudaMemcpyDeviceToHost, c->dstream));
    c->djobs[slot] = fblts_ctx::DiagJob{hs, out, mass_only};
    CUDA_TRY(c, cudaLaunchHostFunc(c->dstream, diag_host_fn, &c->djobs[slot]));
    return FBLTS_OK;
}

int fblts_diagnostics(fblts_ctx *c, double out[4]) {
    if (!c || !out) return FBLTS_ERR_INVALID_ARG;
    if (c->phase != P_STATE) return fail(c, FBLTS_ERR_ORDER, "diagnostics: no state set");
    if (c->cfg.nranks > 1 && !c->nccl)
        return fail(c, FBLTS_ERR_ORDER, "diagnostics: loopback contexts use fblts_diagnostics_group");
    if (c->dstream) CUDA_TRY(c, cudaStreamSynchronize(c->dstream));   // completes outstanding async results
    double part[6];
    int rc = diag_partial(c, part);
    if (rc) return rc;
    if (c->cfg.nranks == 1) {
        diag_combine(part, 1, out);
    } else {
        std::vector<double> all(6 * (size_t)c->cfg.nranks);
        rc = allgather_nccl(c, part, all.data());
        if (rc) return rc;
        diag_combine(all.data(), c->cfg.nranks, out);
    }
    return check_device_error(c);
}

// PV volume integral sum_v A_v h_v q_v (Remark rmk:volume_conservation_pv, eq. vol_integral_pv).
int fblts_diagnostics_pv(fblts_ctx *c, double *out) {
    if (!c || !out) return FBLTS_ERR_INVALID_ARG;
    if (c->phase != P_STATE) return fail(c, FBLTS_ERR_ORDER, "diagnostics_pv: no state set");
    if (c->cfg.nranks > 1 && !c->nccl)
        return fail(c, FBLTS_ERR_ORDER, "diagnostics_pv: loopback contexts are not supported");
    if (c->dstream) CUDA_TRY(c, cudaStreamSynchronize(c->dstream));
    double part[6], four[4];
    int rc = diag_partial(c, part, false, true);
    if (rc) return rc;
    if (c->cfg.nranks == 1) {
        diag_combine(part, 1, four);
    } else {
        std::vector<double> all(6 * (size_t)c->cfg.nranks);
        rc = allgather_nccl(c, part, all.data());
        if (rc) return rc;
        diag_combine(all.data(), c->cfg.nranks, four);
    }
    *out = four[1];
    return check_device_error(c);
}

// Mass and min h only (the cell part of fblts_diagnostics): a cheap per-step monitor.
int fblts_diagnostics_mass(fblts_ctx *c, double out[2]) {
    if (!c || !out) return FBLTS_ERR_INVALID_ARG;
    if (c->phase != P_STATE) return fail(c, FBLTS_ERR_ORDER, "diagnostics_mass: no state set");
    if (c->cfg.nranks > 1 && !c->nccl)
        return fail(c, FBLTS_ERR_ORDER, "diagnostics_mass: loopback contexts use fblts_diagnostics_group");
    if (c->dstream) CUDA_TRY(c, cudaStreamSynchronize(c->dstream));
    double part[6], four[4];
    int rc = diag_partial(c, part, true);
    if (rc) return rc;
    if (c->cfg.nranks == 1) {
        diag_combine(part, 1, four);
    } else {
        std::vector<double> all(6 * (size_t)c->cfg.nranks);
        rc = allgather_nccl(c, part, all.data());
        if (rc) return rc;
        diag_combine(all.data(), c->cfg.nranks, four);
    }
    out[0] = four[0];
    out[1] = four[2];
    return check_device_error(c);
}

// Diagnostics of a loopback group (partial sums combined in rank order, as over NCCL).
int fblts_diagnostics_group(fblts_ctx **cs, int32_t n, double out[4]) {
    if (!cs || n < 1 || !out) return FBLTS_ERR_INVALID_ARG;
    std::vector<double> all(6 * (size_t)n);
    for (int r = 0; r < n; ++r) {
        if (cs[r]->phase != P_STATE) return fail(cs[r], FBLTS_ERR_ORDER, "diagnostics_group: no state set");
        const int rc = diag_partial(cs[r], &all[6 * (size_t)r]);
        if (rc) return rc;
    }
    diag_combine(all.data(), n, out);
    for (int r = 0; r < n; ++r) {
        const int rc = check_device_error(cs[r]);
        if (rc) return rc;
    }
    return FBLTS_OK;
}

int fblts_profile(fblts_ctx *c, int32_t n, double *ms, int64_t *launches) {
    if (!c || !ms || !launches || n < 0) return FBLTS_ERR_INVALID_ARG;
    if (c->phase != P_STATE) return fail(c, FBLTS_ERR_ORDER, "profile: call set_state first");
    if (c->cfg.nranks > 1 && !c->nccl) return fail(c, FBLTS_ERR_ORDER, "profile: not for loopback contexts");
    for (int k = 0; k < K_NUM; ++k) {
        ms[k] = 0.0;
        launches[k] = 0;
    }
    for (int i = 0; i < n; ++i) {
        Recorder rec;
        diag_wait(c, 1 - c->parity);
        const int rc = enqueue_step(c, c->parity, c->stream, &rec);
        if (rc) return rc;
        CUDA_TRY(c, cudaGetLastError());
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        for (size_t j = 0; j + 1 < rec.ev.size(); ++j) {
            float t = 0.f;
            cudaEventElapsedTime(&t, rec.ev[j], rec.ev[j + 1]);
            if (rec.kind[j] >= 0) {
                ms[rec.kind[j] & 63] += t;
                if (rec.kind[j] < 64) launches[rec.kind[j]] += 1;
            }
        }
        for (auto e : rec.ev) cudaEventDestroy(e);
        c->parity ^= 1;
        c->t += c->cfg.dt;
    }
    return check_device_error(c);
}

void fblts_destroy(fblts_ctx *c) {
    if (!c) return;
    for (auto &e : c->exec)
        if (e) cudaGraphExecDestroy(e);
    if (c->cap) cudaStreamDestroy(c->cap);
    if (c->comm) cudaStreamDestroy(c->comm);
    if (c->evFork) cudaEventDestroy(c->evFork);
    if (c->evJoin) cudaEventDestroy(c->evJoin);
    if (c->side) {
        cudaStreamDestroy(c->side);
        cudaEventDestroy(c->evSideF);
        cudaEventDestroy(c->evSideJ);
    }
    if (c->dstream) {
        cudaStreamSynchronize(c->dstream);
        cudaStreamDestroy(c->dstream);
        cudaEventDestroy(c->evHead);
        for (auto e : c->evDiag) cudaEventDestroy(e);
        cudaFreeHost(c->dhost);
        delete[] c->djobs;
    }
    nccl_destroy(c);
    delete c;
}

}  // extern "C"
