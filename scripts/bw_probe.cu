// bw_probe.cu -- development microbenchmark (not part of the library): how fast can a persistent,
// double-buffered 1-D bulk-copy (TMA) pipeline stream K separate fp64 arrays through shared memory,
// compared with plain coalesced loads?  Mirrors the staged tile kernel's access pattern (K arrays,
// T elements of each per tile) without its arithmetic.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o bw_probe scripts/bw_probe.cu && ./bw_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
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
                     : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

constexpr int KMAX = 12;
struct Arrs { const double *a[KMAX]; };

// persistent: CTA walks tiles blockIdx.x + k*gridDim.x; NB buffers; thread 0 issues K bulk copies per tile
template <int NB>
__global__ void k_tma(Arrs A, int K, long n, int T, double *out) {
    extern __shared__ __align__(16) double sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm);
    double *buf = sm + 8;
    const long ntiles = n / T;
    long tile = blockIdx.x;
    if (threadIdx.x == 0) { for (int b = 0; b < NB; ++b) mbar_init(&bar[b], 1); asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
    __syncthreads();
    auto issue = [&](long t, int b) {
        if (threadIdx.x == 0 && t < ntiles) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_expect_tx(&bar[b], (unsigned)(K * T * 8));
            for (int k = 0; k < K; ++k) bulk_g2s(buf + ((size_t)b * K + k) * T, A.a[k] + t * T, T * 8, &bar[b]);
        }
    };
    for (int b = 0; b < NB - 1; ++b) issue(tile + b * gridDim.x, b);
    unsigned phase = 0;
    int b = 0;
    for (; tile < ntiles; tile += gridDim.x, b = (b + 1) % NB) {
        issue(tile + (NB - 1) * gridDim.x, (b + NB - 1) % NB);
        mbar_wait(&bar[b], (phase >> b) & 1u);
        phase ^= 1u << b;
        for (int i = threadIdx.x; i < T; i += blockDim.x) {
            double s = 0.0;
            for (int k = 0; k < K; ++k) s += buf[((size_t)b * K + k) * T + i];
            out[tile * T + i] = s;
        }
        __syncthreads();
    }
}

// the stage tile's shape: 3 cell arrays of TC doubles, 4 edge arrays of TE doubles, one uint32 pair array of TE
// (as TE/2 doubles); GATH scattered 8-byte cp.async gathers per tile (halo cells / foreign edges)
template <int NB>
__global__ void k_tile(Arrs A, long n, int TC, int TE, int GATH, const int *gidx, double *out) {
    extern __shared__ __align__(16) double sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm);
    double *buf = sm + 8;
    const int BUFD = 3 * TC + 4 * TE + TE / 2 + GATH;
    const long ntiles = n / TE;
    long tile = blockIdx.x;
    if (threadIdx.x == 0) { for (int b = 0; b < NB; ++b) mbar_init(&bar[b], 1); asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
    __syncthreads();
    auto issue = [&](long t, int b) {
        if (t >= ntiles) return;
        double *B = buf + (size_t)b * BUFD;
        if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_expect_tx(&bar[b], (unsigned)((3 * TC + 4 * TE + TE / 2) * 8));
            for (int k = 0; k < 3; ++k) bulk_g2s(B + k * TC, A.a[k] + t * TC, TC * 8, &bar[b]);
            for (int k = 0; k < 4; ++k) bulk_g2s(B + 3 * TC + k * TE, A.a[3 + k] + t * TE, TE * 8, &bar[b]);
            bulk_g2s(B + 3 * TC + 4 * TE, A.a[7] + t * (TE / 2), TE * 4, &bar[b]);
        }
        for (int q = threadIdx.x; q < GATH; q += blockDim.x) {
            const long src = gidx[(t * GATH + q) % (1 << 20)];
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(B + 3 * TC + 4 * TE + TE / 2 + q)), "l"(A.a[8] + src) : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    for (int b = 0; b < NB - 1; ++b) issue(tile + b * gridDim.x, b);
    unsigned phase = 0;
    int b = 0;
    for (; tile < ntiles; tile += gridDim.x, b = (b + 1) % NB) {
        mbar_wait(&bar[b], (phase >> b) & 1u);
        phase ^= 1u << b;
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        issue(tile + (NB - 1) * gridDim.x, (b + NB - 1) % NB);
        const double *B = buf + (size_t)b * BUFD;
        for (int i = threadIdx.x; i < TC; i += blockDim.x) {
            double s = B[i] + B[TC + i] + B[2 * TC + i];
            out[tile * TC + i] = s;
        }
        __syncthreads();
    }
}

__global__ void k_ldg(Arrs A, int K, long n, double *out) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < KMAX; ++k) if (k < K) s += A.a[k][i];
        out[i] = s;
    }
}

int main() {
    const long n = 1L << 25;          // 32 M doubles per array (256 MB)
    int nsm;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    Arrs A;
    for (int k = 0; k < KMAX; ++k) { double *p; CK(cudaMalloc(&p, n * 8)); CK(cudaMemset(p, 0, n * 8)); A.a[k] = p; }
    double *out; CK(cudaMalloc(&out, n * 8));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto report = [&](const char *what, float ms, int K) {
        printf("%-40s %8.3f ms  %7.1f GB/s\n", what, ms, (K + 1) * n * 8.0 / (ms * 1e-3) / 1e9);
    };
    {   // the stage tile's shape, with and without the scattered gathers
        int *gidx; CK(cudaMalloc(&gidx, (1 << 20) * 4));
        {
            int *h = new int[1 << 20];
            unsigned x = 12345;
            for (int i = 0; i < (1 << 20); ++i) { x = x * 1664525u + 1013904223u; h[i] = (int)(x % (unsigned)(n - 1)); }
            CK(cudaMemcpy(gidx, h, (1 << 20) * 4, cudaMemcpyHostToDevice));
            delete[] h;
        }
        const int TC = 256, TE = 870 & ~7;
        for (int gath : {0, 250, 700}) {
            for (int per : {2, 3}) {
                const size_t smem = 64 + (size_t)2 * (3 * TC + 4 * TE + TE / 2 + gath) * 8;
                if (smem * per > 225 * 1024) continue;
                CK(cudaFuncSetAttribute(k_tile<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                float ms = 0;
                for (int r = 0; r < 2; ++r) {
                    cudaEventRecord(e0);
                    k_tile<2><<<nsm * per, 256, smem>>>(A, n, TC, TE, gath, gidx, out);
                    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
                }
                CK(cudaGetLastError());
                cudaEventElapsedTime(&ms, e0, e1);
                const long ntiles = n / TE;
                const double bytes = (double)ntiles * ((3 * TC + 4 * TE + TE / 2 + gath) * 8.0 + TC * 8.0);
                printf("tile TC=%d TE=%d gathers=%d cta/sm=%d (%zu KB)  %8.3f ms  %7.1f GB/s\n", TC, TE, gath, per,
                       smem / 1024, ms, bytes / (ms * 1e-3) / 1e9);
            }
        }
    }
    for (int K : {1, 4, 9}) {
        for (int it = 0; it < 2; ++it) {
            cudaEventRecord(e0);
            k_ldg<<<nsm * 8, 256>>>(A, K, n, out);
            cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        }
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        char lab[64]; snprintf(lab, 64, "ldg K=%d", K); report(lab, ms, K);
        for (int T : {256, 512, 1024, 2048}) {
            for (int per : {1, 2, 3, 4}) {
                const size_t smem = 64 + (size_t)2 * K * T * 8;
                if (smem * per > 220 * 1024) continue;
                CK(cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                for (int r = 0; r < 2; ++r) {
                    cudaEventRecord(e0);
                    k_tma<2><<<nsm * per, 256, smem>>>(A, K, n, T, out);
                    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
                }
                CK(cudaGetLastError());
                cudaEventElapsedTime(&ms, e0, e1);
                snprintf(lab, 64, "tma2 K=%d T=%d cta/sm=%d (%zu KB)", K, T, per, smem / 1024);
                report(lab, ms, K);
            }
        }
        for (int T : {256, 512}) {
            const size_t smem = 64 + (size_t)4 * K * T * 8;
            if (smem > 220 * 1024) continue;
            CK(cudaFuncSetAttribute(k_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            for (int per : {1, 2}) {
                if (smem * per > 220 * 1024) continue;
                for (int r = 0; r < 2; ++r) {
                    cudaEventRecord(e0);
                    k_tma<4><<<nsm * per, 256, smem>>>(A, K, n, T, out);
                    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
                }
                cudaEventElapsedTime(&ms, e0, e1);
                snprintf(lab, 64, "tma4 K=%d T=%d cta/sm=%d (%zu KB)", K, T, per, smem / 1024);
                report(lab, ms, K);
            }
        }
    }
    return 0;
}
