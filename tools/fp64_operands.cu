// FP64 pipe microbenchmark, part 2: DFMA throughput by operand pattern
// (development aid: what fraction of the DFMA-chain peak can code with
// distinct register operands reach at the stage kernels' occupancy?).
//   A: x = fma(x, y, z)        y, z shared by all chains (operand reuse)
//   B: x = fma(x, y_k, z_k)    per-chain registers (3 distinct sources)
//   C: x = fma(x, y_k, c)      one source a compile-time constant
//   D: Horner step  p = fma(p, r_k, c_j)  over 4 chains with different c_j (constant bank)
//   E: B with an integer instruction (IADD) between the DFMAs (issue-slot sharing)
#include <cstdio>
#include <cuda_runtime.h>

__constant__ double kc[8] = {0.11, 0.22, 0.33, 0.44, 0.55, 0.66, 0.77, 0.88};

template <int ILP, int MODE>
__global__ void __launch_bounds__(128) probe(double* out, const double* in, int iters) {
    double x[ILP], y[ILP], z[ILP];
    int n[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
        x[k] = in[threadIdx.x + 32 * k];
        y[k] = in[threadIdx.x + 32 * k + 1] * 1e-3 + 0.999;
        z[k] = in[threadIdx.x + 32 * k + 2] * 1e-9;
        n[k] = threadIdx.x + k;
    }
    const double ys = y[0], zs = z[0];
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            if (MODE == 0) x[k] = fma(x[k], ys, zs);
            if (MODE == 1) x[k] = fma(x[k], y[k], z[k]);
            if (MODE == 2) x[k] = fma(x[k], y[k], 1e-9);
            if (MODE == 3) x[k] = fma(x[k], y[k], kc[(i + k) & 7]);
            if (MODE == 4) {
                x[k] = fma(x[k], y[k], z[k]);
                n[k] = n[k] * 3 + i;
            }
        }
    }
    double s = 0;
    int m = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
        s += x[k];
        m += n[k];
    }
    if (s == 1.2345 || m == 77) out[0] = s + m;
}

template <int ILP, int MODE>
void run(int wps, int nsm, double* d, double* in) {
    const int iters = 4096;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = nsm * wps;  // 128 threads = 1 warp per SMSP per block
    probe<ILP, MODE><<<blocks, 128>>>(d, in, 64);
    cudaEventRecord(a);
    probe<ILP, MODE><<<blocks, 128>>>(d, in, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = (double)blocks * 128 * iters * ILP;
    printf("mode %c ILP %d warps/SMSP %2d: %.2f Tdfma/s\n", "ABCDE"[MODE], ILP, wps, ops / (ms * 1e-3) / 1e12);
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double *d, *in;
    cudaMalloc(&d, 8);
    cudaMalloc(&in, 8 * 4096);
    cudaMemset(in, 0, 8 * 4096);
    for (int wps : {2, 4, 8}) {
        run<2, 0>(wps, nsm, d, in); run<2, 1>(wps, nsm, d, in); run<2, 2>(wps, nsm, d, in); run<2, 3>(wps, nsm, d, in); run<2, 4>(wps, nsm, d, in);
        run<4, 0>(wps, nsm, d, in); run<4, 1>(wps, nsm, d, in); run<4, 2>(wps, nsm, d, in); run<4, 3>(wps, nsm, d, in); run<4, 4>(wps, nsm, d, in);
        run<8, 0>(wps, nsm, d, in); run<8, 1>(wps, nsm, d, in); run<8, 2>(wps, nsm, d, in); run<8, 3>(wps, nsm, d, in); run<8, 4>(wps, nsm, d, in);
    }
    return 0;
}
