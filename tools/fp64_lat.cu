// FP64 pipe microbenchmark: dependent-chain latency and throughput vs ILP and
// warps per SM (development aid for the stage-kernel schedule).
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void chain(double* out, int iters, double y, double z, long long* cyc) {
    double x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x * 1e-9 + k;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], y, z);
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += x[k];
    if (s == 1.2345) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int ILP>
void run(int blocks_per_sm, int threads, int nsm, double* d, long long* dc) {
    const int iters = 2048;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    chain<ILP><<<nsm * blocks_per_sm, threads>>>(d, 64, 0.9999999, 1e-9, dc);
    cudaEventRecord(a);
    chain<ILP><<<nsm * blocks_per_sm, threads>>>(d, iters, 0.9999999, 1e-9, dc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long cyc;
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    const double ops = (double)nsm * blocks_per_sm * threads * iters * ILP;
    const int warps_per_smsp = blocks_per_sm * threads / 32 / 4;
    printf("ILP %d warps/SMSP %2d: %.2f Tdfma/s  cycles per dependent step %.1f\n", ILP, warps_per_smsp,
           ops / (ms * 1e-3) / 1e12, (double)cyc / iters);
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    long long* dc;
    cudaMalloc(&d, 8);
    cudaMalloc(&dc, 8);
    for (int wps : {1, 2, 4, 8, 16}) {
        const int threads = wps * 4 * 32 <= 1024 ? wps * 4 * 32 : 1024;
        const int bps = wps * 4 * 32 / threads;
        run<1>(bps, threads, nsm, d, dc);
        run<2>(bps, threads, nsm, d, dc);
        run<4>(bps, threads, nsm, d, dc);
        run<8>(bps, threads, nsm, d, dc);
    }
    return 0;
}
