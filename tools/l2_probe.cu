// L2 reuse probe: stream a state set forward, then immediately again in the
// reverse order, for set sizes below / around the 126 MB L2 (development aid).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double ld_pol(const double* p, unsigned long long pol) {
    double v;
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}

__global__ void pass(const double* __restrict__ p, size_t n, int reverse, int hint, double* out) {
    unsigned long long pol;
    if (hint) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    double s = 0.0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const size_t nit = (n + stride - 1) / stride;
    for (size_t it = 0; it < nit; ++it) {
        const size_t i0 = (reverse ? (nit - 1 - it) : it) * stride + blockIdx.x * blockDim.x + threadIdx.x;
        if (i0 < n) s += ld_pol(p + i0, pol);
    }
    if (s == 1.2345) out[0] = s;
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int l2;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
    int maxp;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
    printf("L2 %d MB, max persisting %d MB\n", l2 >> 20, maxp >> 20);
    double *p, *o, *flush;
    const size_t maxn = (size_t)160 << 17;  // 160 MB of doubles
    cudaMalloc(&p, maxn * 8);
    cudaMemset(p, 0, maxn * 8);
    cudaMalloc(&o, 8);
    cudaMalloc(&flush, 512 << 20);
    cudaEvent_t e[3];
    for (auto& x : e) cudaEventCreate(&x);
    for (int mb : {32, 64, 96, 112, 134, 160})
        for (int hint : {0, 1}) {
            const size_t n = (size_t)mb << 17;
            float t1 = 1e9, t2 = 1e9;
            for (int r = 0; r < 3; ++r) {
                cudaMemset(flush, r, 512 << 20);
                cudaEventRecord(e[0]);
                pass<<<nsm * 8, 256>>>(p, n, 0, hint, o);
                cudaEventRecord(e[1]);
                pass<<<nsm * 8, 256>>>(p, n, 1, hint, o);
                cudaEventRecord(e[2]);
                cudaEventSynchronize(e[2]);
                float a, b;
                cudaEventElapsedTime(&a, e[0], e[1]);
                cudaEventElapsedTime(&b, e[1], e[2]);
                t1 = a < t1 ? a : t1;
                t2 = b < t2 ? b : t2;
            }
            printf("%4d MB hint %d: cold %6.1f us (%5.0f GB/s)  reverse-reread %6.1f us (%5.0f GB/s)\n", mb, hint,
                   t1 * 1e3, n * 8 / (t1 * 1e-3) / 1e9, t2 * 1e3, n * 8 / (t2 * 1e-3) / 1e9);
        }
    return 0;
}
