// Grid all-reduce latency probe (resident kernel's stage boundary): one
// block per SM, N all-reduces of NV doubles; variants of the arrival/wait.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../paper_1907_05560_b200/csrc/resident_kernels.cuh"
using namespace oscb200;

template <int NV, int VAR>
__global__ void __launch_bounds__(kBlock, 1) k_probe(int n, double* part, unsigned* bar, double* out) {
    __shared__ ResShared S;
    extern __shared__ double scratch[];
    unsigned phase = 0;
    double acc = threadIdx.x * 1e-3;
    for (int i = 0; i < n; ++i) {
        double v[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) v[k] = acc + k;
        if (VAR == 0) {
            if (!res_allreduce<NV>(v, acc, part, bar, phase, S, S.fin, scratch)) break;
        } else if (VAR == 2) {  // write partial + barrier, no read
            block_reduce<NV>(v, acc, S.red);
            double* slot = part + (size_t)(phase & 1) * gridDim.x * kSlotDoubles;
            if (threadIdx.x == 0) {
                double* p = slot + (size_t)blockIdx.x * kSlotDoubles;
                for (int k = 0; k < NV; ++k) p[k] = v[k];
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
                res_wait(bar, (phase + 1) * gridDim.x);
            }
            ++phase;
            __syncthreads();
        } else if (VAR == 3) {  // barrier + read partials + reduce, no write
            __syncthreads();
            if (threadIdx.x == 0) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
                res_wait(bar, (phase + 1) * gridDim.x);
            }
            double* slot = part + (size_t)(phase & 1) * gridDim.x * kSlotDoubles;
            ++phase;
            __syncthreads();
            double fv[NV];
            double fm = 0.0;
            for (int k = 0; k < NV; ++k) fv[k] = 0.0;
            for (int b = threadIdx.x; b < (int)gridDim.x; b += kBlock) {
                const double* p = slot + (size_t)b * kSlotDoubles;
                for (int k = 0; k < NV; ++k) fv[k] += __ldcg(p + k);
                fm = fmax(fm, __ldcg(p + NV));
            }
            block_reduce<NV>(fv, fm, S.red);
            if (threadIdx.x == 0) S.fin[0] = fv[0];
            __syncthreads();
        } else {  // counter only (no partial exchange): pure barrier cost
            __syncthreads();
            if (threadIdx.x == 0) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
                res_wait(bar, (phase + 1) * gridDim.x);
            }
            ++phase;
            __syncthreads();
        }
        acc += S.fin[0] * 1e-9;
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

// Cluster-hierarchical all-reduce: block partial -> DSMEM slot of cluster
// rank 0 -> cluster barrier -> rank 0 sums CL partials, stores the cluster
// partial, arrives on the global counter -> every block waits on the counter
// and reads the G = grid/CL cluster partials.
template <int NV, int CL>
__global__ void __launch_bounds__(kBlock, 1) k_probe_cl(int n, double* part, unsigned* bar, double* out) {
    __shared__ ResShared S;
    __shared__ double cslot[CL][NV + 1];
    unsigned phase = 0;
    double acc = threadIdx.x * 1e-3;
    unsigned crank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    const int ncl = gridDim.x / CL, cid = blockIdx.x / CL;
    for (int i = 0; i < n; ++i) {
        double v[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) v[k] = acc + k;
        block_reduce<NV>(v, acc, S.red);
        if (threadIdx.x <= NV) {
            // write this block's partial into rank 0's cslot[crank]
            double x = threadIdx.x < NV ? v[0] * 0 + S.red[threadIdx.x] : acc;
            (void)x;
            unsigned local = (unsigned)__cvta_generic_to_shared(&cslot[crank][threadIdx.x]);
            unsigned remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(local));
            const double val = threadIdx.x < NV ? v[threadIdx.x % NV] : acc;
            asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(remote), "d"(val) : "memory");
        }
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        double* slot = part + (size_t)(phase & 1) * gridDim.x * kSlotDoubles;
        if (crank == 0 && threadIdx.x <= NV) {
            double t = 0.0;
            for (int q = 0; q < CL; ++q) t = threadIdx.x < NV ? t + cslot[q][threadIdx.x] : fmax(t, cslot[q][threadIdx.x]);
            slot[(size_t)threadIdx.x * ncl + cid] = t;
        }
        if (crank == 0) {
            __syncthreads();
            if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        }
        if (threadIdx.x == 0) res_wait(bar, (phase + 1) * ncl);
        ++phase;
        __syncthreads();
        double fv[NV];
        double fm = 0.0;
        for (int k = 0; k < NV; ++k) fv[k] = 0.0;
        for (int b = threadIdx.x; b < ncl; b += kBlock) {
            for (int k = 0; k < NV; ++k) fv[k] += __ldcg(slot + (size_t)k * ncl + b);
            fm = fmax(fm, __ldcg(slot + (size_t)NV * ncl + b));
        }
        block_reduce<NV>(fv, fm, S.red);
        if (threadIdx.x == 0) S.fin[0] = fv[0];
        __syncthreads();
        // cslot reuse next iteration: every rank must be done reading... (rank 0 read above before the barrier)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        acc += S.fin[0] * 1e-9;
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

template <int NV, int CL>
void run_cl(int nsm, const char* name) {
    double *part, *out;
    unsigned* bar;
    cudaMalloc(&part, 2 * nsm * kSlotDoubles * sizeof(double));
    cudaMalloc(&out, 8);
    cudaMalloc(&bar, 4);
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.blockDim = dim3(kBlock);
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int ncl = 0;
    cfg.gridDim = dim3(nsm / CL * CL);
    cudaOccupancyMaxActiveClusters(&ncl, (void*)k_probe_cl<NV, CL>, &cfg);
    const int grid = std::min(nsm / CL, ncl) * CL;
    cfg.gridDim = dim3(grid);
    cfg.numAttrs = 2;
    const int n = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(bar, 0, 4);
        cudaEventRecord(e0);
        cudaError_t le = cudaLaunchKernelEx(&cfg, k_probe_cl<NV, CL>, n, part, bar, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) printf("%-28s NV=%2d CL=%d grid=%d (max clusters %d) %.3f us per all-reduce (%s / %s)\n", name, NV, CL, grid, ncl,
                             ms * 1e3 / n, cudaGetErrorString(le), cudaGetErrorString(cudaGetLastError()));
    }
}

template <int NV, int VAR>
void run(int nsm, const char* name) {
    double *part, *out;
    unsigned* bar;
    cudaMalloc(&part, 2 * nsm * kSlotDoubles * sizeof(double));
    cudaMalloc(&out, 8);
    cudaMalloc(&bar, 4);
    const int n = 2000;
    void* args[4];
    int nn = n;
    args[0] = &nn; args[1] = &part; args[2] = &bar; args[3] = &out;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(bar, 0, 4);
        cudaEventRecord(e0);
        const size_t sm = (size_t)kResScratch * sizeof(double);
        cudaFuncSetAttribute(k_probe<NV, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        cudaLaunchCooperativeKernel((void*)k_probe<NV, VAR>, nsm, kBlock, args, sm, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) printf("%-28s NV=%2d  %.3f us per all-reduce (%s)\n", name, NV, ms * 1e3 / n,
                             cudaGetErrorString(cudaGetLastError()));
    }
}

int main(int argc, char** argv) {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    if (argc > 1) nsm = std::atoi(argv[1]);  // grid size (blocks, one per SM)
    printf("grid %d\n", nsm);
    run<12, 1>(nsm, "counter barrier only");
    run<12, 2>(nsm, "block reduce+write+barrier");
    run<12, 3>(nsm, "barrier+read+reduce");
    run<24, 2>(nsm, "block reduce+write+barrier");
    run<24, 3>(nsm, "barrier+read+reduce");
    run<6, 0>(nsm, "allreduce");
    run<12, 0>(nsm, "allreduce");
    run<24, 0>(nsm, "allreduce");
    run_cl<12, 2>(nsm, "cluster allreduce");
    run_cl<12, 4>(nsm, "cluster allreduce");
    run_cl<12, 8>(nsm, "cluster allreduce");
    run_cl<24, 4>(nsm, "cluster allreduce");
    return 0;
}
