// host.cu -- C ABI of libfblts.so (include/fblts.h): context, mesh validation, LTS
// region labelling, region-major + space-filling-curve renumbering,
// workspace carving, CUDA-graph step replay, state I/O and diagnostics.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <type_traits>
#include <string>
#include <vector>

#include "fblts.h"
#include "fblts_internal.h"

using namespace fblts;

namespace {

const char *kKernelNames[K_NUM] = {"slow_pre",  "slow_edge", "coarse_s1", "coarse_s2", "coarse_s3", "coarse_vel",
                                   "fine_s1",   "fine_s2",   "fine_s3",   "fine_vel",  "correct_if"};

enum Phase { P_CREATED = 0, P_MESH, P_REGIONS, P_BOUND, P_STATE };

struct HostMesh {
    int nC = 0, nE = 0, nV = 0, maxE = 0, maxE2 = 0;
    std::vector<int32_t> nEoC, eoc, coe, voe, nEoE, eoe, eov, cov;
    std::vector<double> W, kite, areaCell, areaTri, dv, dc, fV, H, x, y, z;
};

struct Region {
    std::vector<int8_t> cell, edge;
    std::vector<int32_t> cellOld, cellNew, edgeOld, edgeNew, vertOld, vertNew;
    Bounds cb{}, eb{};
    int64_t ccount[9]{}, ecount[9]{};
};

struct Buf {
    size_t off, bytes;
};

}  // namespace

struct fblts_ctx {
    fblts_config cfg{};
    cudaStream_t stream = nullptr;
    cudaStream_t cap = nullptr;
    std::string err;
    int phase = P_CREATED;
    HostMesh hm;
    Region rg;
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
    // host-side staging of the permuted device tables (filled at set_regions)
    std::vector<int32_t> d_nEoC, d_ec, d_nEoE, d_eoe, d_eov, d_cov, d_coe, d_voe;
    std::vector<double> d_area, d_zb, d_dv, d_dc, d_W, d_kite, d_areaTri, d_fV, d_tau;
    int sC = 0, sE = 0, sV = 0, ecS = 6;
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

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char *fblts_kernel_name(int32_t kind) { return (kind >= 0 && kind < K_NUM) ? kKernelNames[kind] : "?"; }

const char *fblts_last_error(const fblts_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int fblts_create(fblts_ctx **out, const fblts_config *cfg) {
    if (!out || !cfg) return FBLTS_ERR_INVALID_ARG;
    *out = nullptr;
    if (!(cfg->dt > 0.0) || cfg->M < 1 || cfg->r < 1 || !(cfg->g > 0.0) || !(cfg->rho0 > 0.0))
        return FBLTS_ERR_INVALID_ARG;
    if (cfg->nranks != 1 || cfg->rank != 0) return FBLTS_ERR_INVALID_ARG;  // multi-rank: see DESIGN.md
    // No CUDA call here: mesh upload, labelling and renumbering are host work, so a context
    // can be created (and its labels inspected) on a machine without a GPU.
    fblts_ctx *c = new fblts_ctx();
    c->cfg = *cfg;
    c->stream = (cudaStream_t)cfg->stream;
    // canonical constants (computed once in double, SURVEY c.1)
    StepConst &s = c->sc;
    const double dt = cfg->dt;
    const double M = (double)cfg->M;
    s.g = cfg->g;
    s.rho0 = cfg->rho0;
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
    // ---- renumbering: region-major, SFC within a region (cells), owner order (edges, vertices)
    const std::vector<uint64_t> key = sfc_keys(m);
    g.cellOld.resize(m.nC);
    std::iota(g.cellOld.begin(), g.cellOld.end(), 0);
    std::stable_sort(g.cellOld.begin(), g.cellOld.end(), [&](int a, int b) {
        if (g.cell[a] != g.cell[b]) return g.cell[a] < g.cell[b];
        return key[a] < key[b];
    });
    g.cellNew.resize(m.nC);
    for (int i = 0; i < m.nC; ++i) g.cellNew[g.cellOld[i]] = i;
    std::vector<int32_t> eown(m.nE);
    for (int e = 0; e < m.nE; ++e) eown[e] = std::min(g.cellNew[m.coe[2 * e]], g.cellNew[m.coe[2 * e + 1]]);
    g.edgeOld.resize(m.nE);
    std::iota(g.edgeOld.begin(), g.edgeOld.end(), 0);
    std::stable_sort(g.edgeOld.begin(), g.edgeOld.end(), [&](int a, int b) {
        if (g.edge[a] != g.edge[b]) return g.edge[a] < g.edge[b];
        return eown[a] < eown[b];
    });
    g.edgeNew.resize(m.nE);
    for (int e = 0; e < m.nE; ++e) g.edgeNew[g.edgeOld[e]] = e;
    std::vector<int32_t> vown(m.nV);
    for (int v = 0; v < m.nV; ++v)
        vown[v] = std::min(g.cellNew[m.cov[3 * v]], std::min(g.cellNew[m.cov[3 * v + 1]], g.cellNew[m.cov[3 * v + 2]]));
    g.vertOld.resize(m.nV);
    std::iota(g.vertOld.begin(), g.vertOld.end(), 0);
    std::stable_sort(g.vertOld.begin(), g.vertOld.end(), [&](int a, int b) { return vown[a] < vown[b]; });
    g.vertNew.resize(m.nV);
    for (int v = 0; v < m.nV; ++v) g.vertNew[g.vertOld[v]] = v;
    // ---- region bounds
    std::fill(g.ccount, g.ccount + 9, 0);
    std::fill(g.ecount, g.ecount + 9, 0);
    for (int i = 0; i < m.nC; ++i) g.ccount[g.cell[i]]++;
    for (int e = 0; e < m.nE; ++e) g.ecount[g.edge[e]]++;
    auto bounds = [](const int64_t *cnt, int n) {
        Bounds b{};
        b.if2 = (int)cnt[0];
        b.if1 = b.if2 + (int)cnt[1];
        b.f = b.if1 + (int)cnt[2];
        b.fl[0] = b.f;
        for (int l = 1; l <= 5; ++l) b.fl[l] = b.fl[l - 1] + (int)cnt[2 + l];
        b.end = n;
        return b;
    };
    g.cb = bounds(g.ccount, m.nC);
    g.eb = bounds(g.ecount, m.nE);
    c->have_fine = g.cb.f < m.nC;
    // ---- permuted device tables (host staging; uploaded at bind_workspace)
    c->sC = pad32(m.nC);
    c->sE = pad32(m.nE);
    c->sV = pad32(m.nV);
    const int sE = c->sE, sV = c->sV;
    c->d_nEoC.assign(m.nC, 0);
    c->ecS = m.maxE <= 6 ? 6 : (m.maxE <= 8 ? 8 : 16);
    c->d_ec.assign((size_t)m.nC * c->ecS * 2, 0);
    c->d_area.assign(m.nC, 0.0);
    c->d_zb.assign(m.nC, 0.0);
    for (int i = 0; i < m.nC; ++i) {
        const int o = g.cellOld[i];
        c->d_nEoC[i] = m.nEoC[o];
        c->d_area[i] = m.areaCell[o];
        c->d_zb[i] = -m.H[o];
        for (int j = 0; j < m.nEoC[o]; ++j) {
            const int e = m.eoc[(size_t)o * m.maxE + j];
            const int en = g.edgeNew[e];
            c->d_ec[((size_t)i * c->ecS + j) * 2] = m.coe[2 * e] == o ? en : ~en;
            c->d_ec[((size_t)i * c->ecS + j) * 2 + 1] = g.cellNew[coc[(size_t)o * m.maxE + j]];
        }
    }
    c->d_coe.assign((size_t)m.nE * 2, 0);
    c->d_voe.assign((size_t)m.nE * 2, 0);
    c->d_dv.assign(m.nE, 0.0);
    c->d_dc.assign(m.nE, 0.0);
    c->d_tau.assign(m.nE, 0.0);
    c->d_nEoE.assign(m.nE, 0);
    c->d_eoe.assign((size_t)m.maxE2 * sE, 0);
    c->d_W.assign((size_t)m.maxE2 * sE, 0.0);
    for (int e = 0; e < m.nE; ++e) {
        const int o = g.edgeOld[e];
        c->d_coe[2 * e] = g.cellNew[m.coe[2 * o]];
        c->d_coe[2 * e + 1] = g.cellNew[m.coe[2 * o + 1]];
        c->d_voe[2 * e] = g.vertNew[m.voe[2 * o]];
        c->d_voe[2 * e + 1] = g.vertNew[m.voe[2 * o + 1]];
        c->d_dv[e] = m.dv[o];
        c->d_dc[e] = m.dc[o];
        c->d_nEoE[e] = m.nEoE[o];
        for (int j = 0; j < m.nEoE[o]; ++j) {
            c->d_eoe[(size_t)j * sE + e] = g.edgeNew[m.eoe[(size_t)o * m.maxE2 + j]];
            c->d_W[(size_t)j * sE + e] = m.W[(size_t)o * m.maxE2 + j];
        }
    }
    c->d_eov.assign((size_t)3 * sV, 0);
    c->d_cov.assign((size_t)3 * sV, 0);
    c->d_kite.assign((size_t)3 * sV, 0.0);
    c->d_areaTri.assign(m.nV, 0.0);
    c->d_fV.assign(m.nV, 0.0);
    for (int v = 0; v < m.nV; ++v) {
        const int o = g.vertOld[v];
        c->d_areaTri[v] = m.areaTri[o];
        c->d_fV[v] = m.fV[o];
        for (int k = 0; k < 3; ++k) {
            const int e = m.eov[3 * o + k];
            const int en = g.edgeNew[e];
            c->d_eov[(size_t)k * sV + v] = m.voe[2 * e + 1] == o ? en : ~en;
            c->d_cov[(size_t)k * sV + v] = g.cellNew[m.cov[3 * o + k]];
            c->d_kite[(size_t)k * sV + v] = m.kite[3 * o + k];
        }
    }
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
        out[3 + k] = c->rg.ccount[k];
        out[12 + k] = c->rg.ecount[k];
    }
    out[21] = c->hm.nC;
    out[22] = c->hm.nE;
    out[23] = (int64_t)c->graph_nodes;
    return FBLTS_OK;
}

namespace {
// workspace plan: the same sequence is used for sizing and for carving
struct Plan {
    std::vector<size_t> sizes;
    size_t total = 0;
    size_t add(size_t bytes) {
        const size_t off = total;
        total += (bytes + 255) / 256 * 256;
        sizes.push_back(bytes);
        return off;
    }
};

size_t plan_workspace(fblts_ctx *c, char *base) {
    const HostMesh &m = c->hm;
    const Region &g = c->rg;
    Plan p;
    auto put = [&](auto *&ptr, size_t count) {
        using T = std::remove_pointer_t<std::remove_reference_t<decltype(ptr)>>;
        const size_t off = p.add(count * sizeof(T));
        if (base) ptr = reinterpret_cast<T *>(base + off);
    };
    DevMesh &d = c->dm;
    DevState &s = c->ds;
    int32_t *nEoC, *nEoE, *eoe, *eov, *cov;
    double *area, *zb, *W, *tau, *kite, *areaTri, *fV;
    int2 *coe, *voe, *ec;
    double *dv, *dc;
    put(nEoC, m.nC);
    put(ec, (size_t)m.nC * c->ecS);
    put(area, m.nC);
    put(zb, m.nC);
    put(coe, m.nE);
    put(voe, m.nE);
    put(dv, m.nE);
    put(dc, m.nE);
    put(tau, m.nE);
    put(nEoE, m.nE);
    put(eoe, (size_t)m.maxE2 * c->sE);
    put(W, (size_t)m.maxE2 * c->sE);
    put(eov, (size_t)3 * c->sV);
    put(cov, (size_t)3 * c->sV);
    put(kite, (size_t)3 * c->sV);
    put(areaTri, m.nV);
    put(fV, m.nV);
    double *hA, *hB, *uA, *uB;
    put(hA, m.nC);
    put(hB, m.nC);
    put(s.h1, m.nC);
    put(s.h2, m.nC);
    put(s.hT, m.nC);
    put(s.K, m.nC);
    put(uA, m.nE);
    put(uB, m.nE);
    put(s.uT, m.nE);
    put(s.S, m.nE);
    put(s.F, m.nE);
    put(s.q, m.nV);
    put(s.accH, std::max(1, g.cb.f - g.cb.if2));
    put(s.accU, std::max(1, g.eb.f - g.eb.if2));
    put(s.stage, std::max(m.nC, m.nE));
    put(s.cellOld, m.nC);
    put(s.edgeOld, m.nE);
    put(s.diag, 296 * 6 + 8);
    put(s.err, 1);
    if (base) {
        d.nC = m.nC, d.nE = m.nE, d.nV = m.nV;
        d.strideC = c->sC, d.strideE = c->sE, d.strideV = c->sV;
        d.maxE = m.maxE, d.maxE2 = m.maxE2, d.ecS = c->ecS;
        d.nEoC = nEoC, d.ec = ec, d.areaCell = area, d.zb = zb;
        d.coe = coe, d.voe = voe, d.dv = dv, d.dc = dc, d.nEoE = nEoE, d.eoe = eoe, d.W = W, d.tau = tau;
        d.eov = eov, d.cov = cov, d.kite = kite, d.areaTri = areaTri, d.fV = fV;
        d.cb = g.cb, d.eb = g.eb;
        c->hbuf[0] = hA, c->hbuf[1] = hB, c->ubuf[0] = uA, c->ubuf[1] = uB;
        s.hN = hA, s.hNew = hB, s.uN = uA, s.uNew = uB;
        c->diag_out = s.diag + 296 * 6;
    }
    return p.total;
}
}  // namespace

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
    c->ws = (char *)ptr;
    c->ws_bytes = bytes;
    plan_workspace(c, c->ws);
    cudaStream_t s = c->stream;
    DevMesh &d = c->dm;
    auto up = [&](const void *dst, const void *src, size_t n) {
        return cudaMemcpyAsync(const_cast<void *>(dst), src, n, cudaMemcpyHostToDevice, s);
    };
    const HostMesh &m = c->hm;
    CUDA_TRY(c, up(d.nEoC, c->d_nEoC.data(), c->d_nEoC.size() * 4));
    CUDA_TRY(c, up(d.ec, c->d_ec.data(), c->d_ec.size() * 4));
    CUDA_TRY(c, up(d.areaCell, c->d_area.data(), m.nC * 8));
    CUDA_TRY(c, up(d.zb, c->d_zb.data(), m.nC * 8));
    CUDA_TRY(c, up(d.coe, c->d_coe.data(), (size_t)m.nE * 8));
    CUDA_TRY(c, up(d.voe, c->d_voe.data(), (size_t)m.nE * 8));
    CUDA_TRY(c, up(d.dv, c->d_dv.data(), (size_t)m.nE * 8));
    CUDA_TRY(c, up(d.dc, c->d_dc.data(), (size_t)m.nE * 8));
    CUDA_TRY(c, up(d.tau, c->d_tau.data(), (size_t)m.nE * 8));
    CUDA_TRY(c, up(d.nEoE, c->d_nEoE.data(), (size_t)m.nE * 4));
    CUDA_TRY(c, up(d.eoe, c->d_eoe.data(), c->d_eoe.size() * 4));
    CUDA_TRY(c, up(d.W, c->d_W.data(), c->d_W.size() * 8));
    CUDA_TRY(c, up(d.eov, c->d_eov.data(), c->d_eov.size() * 4));
    CUDA_TRY(c, up(d.cov, c->d_cov.data(), c->d_cov.size() * 4));
    CUDA_TRY(c, up(d.kite, c->d_kite.data(), c->d_kite.size() * 8));
    CUDA_TRY(c, up(d.areaTri, c->d_areaTri.data(), (size_t)m.nV * 8));
    CUDA_TRY(c, up(d.fV, c->d_fV.data(), (size_t)m.nV * 8));
    CUDA_TRY(c, up(c->ds.cellOld, c->rg.cellOld.data(), (size_t)m.nC * 4));
    CUDA_TRY(c, up(c->ds.edgeOld, c->rg.edgeOld.data(), (size_t)m.nE * 4));
    CUDA_TRY(c, cudaMemsetAsync(c->ds.S, 0, (size_t)m.nE * 8, s));
    CUDA_TRY(c, cudaMemsetAsync(c->ds.err, 0, sizeof(DevError), s));
    CUDA_TRY(c, cudaStreamSynchronize(s));
    // host staging of the device tables is no longer needed
    std::vector<int32_t>().swap(c->d_ec);

    std::vector<int32_t>().swap(c->d_eoe);
    std::vector<double>().swap(c->d_W);
    c->phase = P_BOUND;
    return FBLTS_OK;
}

int fblts_set_forcing(fblts_ctx *c, const double *tau_n) {
    if (!c) return FBLTS_ERR_INVALID_ARG;
    if (c->phase < P_BOUND) return fail(c, FBLTS_ERR_ORDER, "set_forcing: bind the workspace first");
    const int nE = c->hm.nE;
    std::vector<double> t(nE, 0.0);
    if (tau_n)
        for (int e = 0; e < nE; ++e) {
            if (!std::isfinite(tau_n[e])) return fail(c, FBLTS_ERR_INVALID_ARG, "forcing[%d] not finite", e);
            t[e] = tau_n[c->rg.edgeOld[e]];
        }
    CUDA_TRY(c, cudaMemcpyAsync((void *)c->dm.tau, t.data(), (size_t)nE * 8, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return FBLTS_OK;
}

int fblts_set_state(fblts_ctx *c, const double *h, const double *u, double t) {
    if (!c || !h || !u) return FBLTS_ERR_INVALID_ARG;
    if (c->phase < P_BOUND) return fail(c, FBLTS_ERR_ORDER, "set_state: bind the workspace first");
    for (int i = 0; i < c->hm.nC; ++i)
        if (!(std::isfinite(h[i]) && h[i] > 0.0)) return fail(c, FBLTS_ERR_STATE, "set_state: h[%d]=%g", i, h[i]);
    for (int e = 0; e < c->hm.nE; ++e)
        if (!std::isfinite(u[e])) return fail(c, FBLTS_ERR_STATE, "set_state: u[%d] not finite", e);
    cudaStream_t s = c->stream;
    const int nC = c->hm.nC, nE = c->hm.nE;
    c->parity = 0;
    CUDA_TRY(c, cudaMemcpyAsync(c->ds.stage, h, (size_t)nC * 8, cudaMemcpyHostToDevice, s));
    launch_permute_in(c->ds.cellOld, c->ds.stage, c->hbuf[0], nC, s);
    CUDA_TRY(c, cudaMemcpyAsync(c->ds.stage, u, (size_t)nE * 8, cudaMemcpyHostToDevice, s));
    launch_permute_in(c->ds.edgeOld, c->ds.stage, c->ubuf[0], nE, s);
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaMemsetAsync(c->ds.err, 0, sizeof(DevError), s));
    CUDA_TRY(c, cudaStreamSynchronize(s));
    c->t = t;
    c->phase = P_STATE;
    return FBLTS_OK;
}

}  // extern "C"

namespace {

struct Recorder {
    std::vector<cudaEvent_t> ev;
    std::vector<int> kind;
    void mark(int k, cudaStream_t s) {
        cudaEvent_t a;
        cudaEventCreate(&a);
        cudaEventRecord(a, s);
        ev.push_back(a);
        kind.push_back(k);
    }
};

// Enqueue one coarse step reading hbuf[par], ubuf[par] and writing hbuf[1-par], ubuf[1-par].
void enqueue_step(fblts_ctx *c, int par, cudaStream_t s, Recorder *rec) {
    const DevMesh &m = c->dm;
    DevState st = c->ds;
    const StepConst &sc = c->sc;
    const double *hN = c->hbuf[par], *uN = c->ubuf[par];
    double *hNew = c->hbuf[1 - par], *uNew = c->ubuf[1 - par];
    auto mark = [&](int k) {
        if (rec) rec->mark(k, s);
    };
    if (c->cfg.slow) {
        mark(K_SLOW_PRE);
        launch_slow_pre(m, st, hN, uN, s);
        mark(K_SLOW_EDGE);
        launch_slow_edge(m, st, hN, sc, s);
    }
    mark(K_COARSE_S1);
    launch_coarse_s1(m, st, hN, uN, sc, s);
    mark(K_COARSE_S2);
    launch_coarse_s2(m, st, hN, uN, sc, s);
    mark(K_COARSE_S3);
    launch_coarse_s3(m, st, hN, uN, hNew, sc, s);
    mark(K_COARSE_VEL);
    launch_coarse_vel(m, st, hN, uN, hNew, uNew, sc, s);
    if (c->have_fine) {
        const int M = sc.M;
        auto hb = [&](int k) { return ((M - 1 - k) % 2 == 0) ? hNew : st.hT; };
        auto ub = [&](int k) { return ((M - 1 - k) % 2 == 0) ? uNew : st.uT; };
        for (int k = 0; k < M; ++k) {
            PredConst pc;
            pc.a = (double)k / (double)M;
            pc.oma = 1.0 - pc.a;
            pc.a1 = (double)(k + 1) / (double)M;
            pc.oma1 = 1.0 - pc.a1;
            pc.b = 1.0 / (double)M;
            pc.c = 1.0 - (double)(k + 1) / (double)M;
            const double *hk = k == 0 ? hN : hb(k - 1);
            const double *uk = k == 0 ? uN : ub(k - 1);
            double *hnext = hb(k), *unext = ub(k);
            mark(K_FINE_S1);
            launch_fine_s1(m, st, hN, hNew, hk, uk, sc, pc, k, s);
            mark(K_FINE_S2);
            launch_fine_s2(m, st, hN, hNew, hk, uk, sc, pc, k, s);
            mark(K_FINE_S3);
            launch_fine_s3(m, st, hN, uN, hNew, hk, uk, hnext, sc, pc, k, s);
            mark(K_FINE_VEL);
            launch_fine_vel(m, st, hN, hNew, hk, hnext, uk, unext, sc, pc, k, s);
        }
        mark(K_CORRECT);
        launch_correct(m, st, hN, uN, hNew, uNew, sc, s);
    }
    mark(-1);
}

int capture(fblts_ctx *c, int par) {
    cudaGraph_t g;
    CUDA_TRY(c, cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
    enqueue_step(c, par, c->cap, nullptr);
    CUDA_TRY(c, cudaStreamEndCapture(c->cap, &g));
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
        const int idx = e.index >= 0 && e.index < c->hm.nC ? c->rg.cellOld[e.index] : -1;
        return fail(c, FBLTS_ERR_POSITIVITY, "positivity: h=%g in %s (subcycle k=%d) at cell %d (region %d)", e.value,
                    fblts_kernel_name(e.kind), e.k, idx, idx >= 0 ? (int)c->rg.cell[idx] : -1);
    }
    return FBLTS_OK;
}

}  // namespace

extern "C" {

int fblts_step(fblts_ctx *c, int32_t n) {
    if (!c || n < 0) return FBLTS_ERR_INVALID_ARG;
    if (c->phase != P_STATE) return fail(c, FBLTS_ERR_ORDER, "step: call set_state first");
    CUDA_TRY(c, cudaSetDevice(c->cfg.device));
    for (int p = 0; p < 2; ++p)
        if (!c->exec[p]) {
            const int rc = capture(c, p);
            if (rc) return rc;
        }
    for (int i = 0; i < n; ++i) {
        CUDA_TRY(c, cudaGraphLaunch(c->exec[c->parity], c->stream));
        c->parity ^= 1;
        c->t += c->cfg.dt;
    }
    return FBLTS_OK;
}

int fblts_sync(fblts_ctx *c) {
    if (!c) return FBLTS_ERR_INVALID_ARG;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->phase >= P_BOUND) return check_device_error(c);
    return FBLTS_OK;
}

int fblts_get_state(fblts_ctx *c, double *h, double *u, double *t) {
    if (!c) return FBLTS_ERR_INVALID_ARG;
    if (c->phase != P_STATE) return fail(c, FBLTS_ERR_ORDER, "get_state: no state set");
    cudaStream_t s = c->stream;
    const int nC = c->hm.nC, nE = c->hm.nE;
    if (h) {
        launch_permute_out(c->ds.cellOld, c->hbuf[c->parity], c->ds.stage, nC, s);
        CUDA_TRY(c, cudaMemcpyAsync(h, c->ds.stage, (size_t)nC * 8, cudaMemcpyDeviceToHost, s));
    }
    if (u) {
        launch_permute_out(c->ds.edgeOld, c->ubuf[c->parity], c->ds.stage, nE, s);
        CUDA_TRY(c, cudaMemcpyAsync(u, c->ds.stage, (size_t)nE * 8, cudaMemcpyDeviceToHost, s));
    }
    CUDA_TRY(c, cudaStreamSynchronize(s));
    CUDA_TRY(c, cudaGetLastError());
    if (t) *t = c->t;
    return check_device_error(c);
}

int fblts_diagnostics(fblts_ctx *c, double out[4]) {
    if (!c || !out) return FBLTS_ERR_INVALID_ARG;
    if (c->phase != P_STATE) return fail(c, FBLTS_ERR_ORDER, "diagnostics: no state set");
    launch_diagnostics(c->dm, c->ds, c->hbuf[c->parity], c->ubuf[c->parity], c->sc, c->diag_out, c->stream);
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaMemcpyAsync(out, c->diag_out, 4 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return check_device_error(c);
}

int fblts_profile(fblts_ctx *c, int32_t n, double *ms, int64_t *launches) {
    if (!c || !ms || !launches || n < 0) return FBLTS_ERR_INVALID_ARG;
    if (c->phase != P_STATE) return fail(c, FBLTS_ERR_ORDER, "profile: call set_state first");
    for (int k = 0; k < K_NUM; ++k) {
        ms[k] = 0.0;
        launches[k] = 0;
    }
    for (int i = 0; i < n; ++i) {
        Recorder rec;
        enqueue_step(c, c->parity, c->stream, &rec);
        CUDA_TRY(c, cudaGetLastError());
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        for (size_t j = 0; j + 1 < rec.ev.size(); ++j) {
            float t = 0.f;
            cudaEventElapsedTime(&t, rec.ev[j], rec.ev[j + 1]);
            if (rec.kind[j] >= 0) {
                ms[rec.kind[j]] += t;
                launches[rec.kind[j]] += 1;
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
    delete c;
}

}  // extern "C"
