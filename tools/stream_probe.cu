// Memory-system probe for the stage-kernel access pattern (development aid):
// 16 planes x N cells of fp64, read once.  Compares plain LDG streaming with
// the TMA bulk ring (cp.async.bulk + mbarrier) used by k_stage.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kPlanes = 16;

template <int CPT>
__global__ void ldg_stream(const double* __restrict__ p, size_t np, int ncell, double* out) {
    double s = 0.0;
    const int stride = gridDim.x * blockDim.x;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += stride * CPT) {
        double v[CPT][kPlanes];
#pragma unroll
        for (int u = 0; u < CPT; ++u)
#pragma unroll
            for (int k = 0; k < kPlanes; ++k) v[u][k] = (c + u * stride < ncell) ? __ldcs(p + k * np + c + u * stride) : 0.0;
#pragma unroll
        for (int u = 0; u < CPT; ++u)
#pragma unroll
            for (int k = 0; k < kPlanes; ++k) s += v[u][k];
    }
    if (s == 1.2345) out[0] = s;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NS, int TILE>
__global__ void tma_stream(const double* __restrict__ p, size_t np, int ncell, int chunk, double* out, int rev = 0) {
    extern __shared__ __align__(128) double tiles[];
    __shared__ __align__(8) uint64_t bars[NS];
    const int c0 = blockIdx.x * chunk, c1 = min(c0 + chunk, ncell);
    const int ntiles = c1 > c0 ? (c1 - c0 + TILE - 1) / TILE : 0;
    auto issue = [&](int t, int slot) {
        if (rev) t = ntiles - 1 - t;
        const int start = c0 + t * TILE;
        const int n = min(TILE, c1 - start);
        const uint32_t bytes = ((n + 1) & ~1) * 8;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[slot])),
                     "r"(bytes * kPlanes) : "memory");
        for (int k = 0; k < kPlanes; ++k)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             smem_u32(tiles + ((size_t)slot * kPlanes + k) * TILE)),
                         "l"(p + k * np + start), "r"(bytes), "r"(smem_u32(&bars[slot])) : "memory");
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int s = 0; s < NS && s < ntiles; ++s) issue(s, s);
    }
    __syncthreads();
    double s = 0.0;
    for (int t = 0; t < ntiles; ++t) {
        const int slot = t % NS;
        asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}\n" ::"r"(
                         smem_u32(&bars[slot])),
                     "r"((uint32_t)((t / NS) & 1)) : "memory");
        for (int i = threadIdx.x; i < TILE; i += blockDim.x)
#pragma unroll
            for (int k = 0; k < kPlanes; ++k) s += tiles[((size_t)slot * kPlanes + k) * TILE + i];
        __syncthreads();
        if (threadIdx.x == 0 && t + NS < ntiles) issue(t + NS, slot);
    }
    if (s == 1.2345) out[0] = s;
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int ncell = 1 << 20;
    const size_t np = ncell;
    double *p, *o;
    cudaMalloc(&p, np * kPlanes * 8);
    cudaMemset(p, 0, np * kPlanes * 8);
    cudaMalloc(&o, 8);
    double* flush;
    cudaMalloc(&flush, 256 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double bytes = (double)np * kPlanes * 8;
    auto timeit = [&](const char* name, auto launch) {
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaMemset(flush, r, 256 << 20);
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%-28s %7.1f us  %6.0f GB/s  (%s)\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int bps : {2, 4, 8})
        for (int cpt : {1, 2}) {
            char nm[64];
            snprintf(nm, 64, "ldg cpt%d blocks/SM %d", cpt, bps);
            if (cpt == 1) timeit(nm, [&] { ldg_stream<1><<<nsm * bps, 256>>>(p, np, ncell, o); });
            else timeit(nm, [&] { ldg_stream<2><<<nsm * bps, 256>>>(p, np, ncell, o); });
        }
    for (int bps : {1, 2, 3}) {
        const int nb = nsm * bps;
        int chunk = (ncell + nb - 1) / nb;
        chunk = (chunk + 31) / 32 * 32;
        char nm[64];
        {
            auto k = tma_stream<2, 256>;
            size_t sm = 2 * kPlanes * 256 * 8;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
            snprintf(nm, 64, "tma ns2 tile256 b/SM %d", bps);
            timeit(nm, [&] { k<<<nb, 256, sm>>>(p, np, ncell, chunk, o, 0); });
        }
        {
            auto k = tma_stream<4, 128>;
            size_t sm = 4 * kPlanes * 128 * 8;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
            snprintf(nm, 64, "tma ns4 tile128 b/SM %d", bps);
            timeit(nm, [&] { k<<<nb, 256, sm>>>(p, np, ncell, chunk, o, 0); });
        }
        {
            auto k = tma_stream<3, 256>;
            size_t sm = 3 * kPlanes * 256 * 8;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
            snprintf(nm, 64, "tma ns3 tile256 b/SM %d", bps);
            timeit(nm, [&] { k<<<nb, 256, sm>>>(p, np, ncell, chunk, o, 0); });
        }
    }
    // L2 re-read: forward pass then reverse pass, set sizes around the L2
    for (int ncell2 : {1 << 19, 3 << 18, 1 << 20}) {
        const int nb = nsm * 2;
        int chunk = (ncell2 + nb - 1) / nb;
        chunk = (chunk + 31) / 32 * 32;
        auto k = tma_stream<3, 256>;
        size_t sm = 3 * kPlanes * 256 * 8;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        float t1 = 1e9, t2 = 1e9;
        for (int r = 0; r < 3; ++r) {
            cudaMemset(flush, r, 256 << 20);
            cudaEventRecord(a);
            k<<<nb, 256, sm>>>(p, ncell2, ncell2, chunk, o, 0);
            cudaEvent_t m;
            cudaEventCreate(&m);
            cudaEventRecord(m);
            k<<<nb, 256, sm>>>(p, ncell2, ncell2, chunk, o, 1);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float x, y;
            cudaEventElapsedTime(&x, a, m);
            cudaEventElapsedTime(&y, m, b);
            t1 = x < t1 ? x : t1;
            t2 = y < t2 ? y : t2;
        }
        const double by = (double)ncell2 * kPlanes * 8;
        printf("tma set %4.0f MB: cold %6.1f us %5.0f GB/s, reverse re-read %6.1f us %5.0f GB/s\n", by / 1e6,
               t1 * 1e3, by / (t1 * 1e-3) / 1e9, t2 * 1e3, by / (t2 * 1e-3) / 1e9);
    }
    return 0;
}
