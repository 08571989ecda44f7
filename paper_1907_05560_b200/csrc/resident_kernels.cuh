// Resident multi-step kernel for small 2-flavour problems (configs[0]):
// the whole local state lives in shared memory for the duration of a batch
// of steps, one block per SM, and the stage boundaries of do_step
// (solver.cpp:343-412) become grid-wide all-reductions instead of kernel
// launches.  Same arithmetic per cell as the stage kernels (step_kernels.cuh);
// what changes:
//   * psi0, the candidate result and the S3 -> S4 propagator stash are
//     shared-memory arrays of the block's chunk (no HBM traffic between
//     steps, no TMA ring, no prologue per stage: the trajectory records of a
//     step are built once);
//   * after each stage every block publishes its partial moments, arrives on
//     a monotonic counter (release), waits for all blocks (acquire) and then
//     reduces all partials itself in a fixed order — identical totals in
//     every block, no "last block" round trip;
//   * every block runs the lane_body control update (ctl_advance) on its own
//     shared copy of Ctl; the inputs are identical, so are the decisions, and
//     all blocks leave the step loop together (terminate, failure, or a due
//     snapshot).  Block 0 publishes Ctl and every block writes its psi0 back
//     to the global buffer Ctl::cur names.
#pragma once

#include "oscflat_b200.h"
#include "step_kernels.cuh"

namespace oscb200 {

constexpr int kResMaxNV = 2 * 12 + 1;  // S2: two moment sets + the max slot

struct ResShared {
    Ctl c;                    // this block's copy of the control block
    double tot0[12];          // sums0: moments of psi0 at r
    double tot1[24];          // sums1 | sums2 (S2)
    double tot3[12];          // sums3 (S3)
    double totn[13];          // S4: next-step sums0 + max error
    double red[kWarps * (kResMaxNV)];
    double fin[kResMaxNV];
    int accept;
    int stop;
};

// Bounded spin on the arrival counter (acquire).  Returns false after ~1 s
// so a protocol fault cannot wedge the GPU.
__device__ __forceinline__ bool res_wait(const unsigned* bar, unsigned target) {
    for (long long i = 0; i < (1ll << 25); ++i) {
        unsigned v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        if ((int)(v - target) >= 0) return true;
        __nanosleep(32);
    }
    return false;
}

// Grid all-reduce of NV sums + 1 max, in two halves so independent work can
// run while the other blocks arrive.  res_arrive: block partial (fixed tree)
// -> part[phase & 1][value][block] -> release arrival.  res_finish: acquire
// wait -> every block sums all partials in the same fixed order ->
// out[0..NV] = totals, max.
// Block partial (block_cols_store, step_kernels.cuh) into
// part[phase & 1][value][block], then the release arrival.
template <int NV>
__device__ __forceinline__ void res_arrive(double (&v)[NV], double mx, double* part, unsigned* bar,
                                           unsigned phase, ResShared& S, double* scratch) {
    block_cols_store<NV>(v, mx, scratch, part + (size_t)(phase & 1) * gridDim.x * kSlotDoubles + blockIdx.x,
                         gridDim.x);
    // (the barrier ending block_cols_store orders every column's store before
    // thread 0's release: the cooperative-groups grid sync pattern)
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    (void)S;
}

template <int NV>
__device__ __forceinline__ bool res_finish(double* part, unsigned* bar, unsigned& phase, ResShared& S,
                                           double* out) {
    const int tid = threadIdx.x;
    if (tid == 0) S.stop = res_wait(bar, (phase + 1) * gridDim.x) ? 0 : 1;
    const double* slot = part + (size_t)(phase & 1) * gridDim.x * kSlotDoubles;
    ++phase;
    __syncthreads();
    if (S.stop) return false;
    cols_reduce<NV>(slot, (int)gridDim.x, out);
    return true;
}
template <int NV>
__device__ __forceinline__ bool res_allreduce(double (&v)[NV], double mx, double* part, unsigned* bar,
                                              unsigned& phase, ResShared& S, double* out, double* scratch) {
    res_arrive<NV>(v, mx, part, bar, phase, S, scratch);
    return res_finish<NV>(part, bar, phase, S, out);
}

// Per-cell propagators carried between the stages of a step ([24][ch]):
// Um (S2 -> S3), Uf then Q = (Uf + U2)/2 (S2 -> S4), P (S3 -> S4).
constexpr int kResProps = 24;

// Shared-memory bytes of the resident kernel for a chunk of `ch` cells.
constexpr int kResScratch = kResMaxNV * kBlock;  // all-reduce transposition scratch (doubles)
inline size_t resident_smem_bytes(int ch, int ntr_max, int E) {
    return (size_t)(2 * kPlanes + kResProps) * ch * sizeof(double) + (size_t)ntr_max * sizeof(TrajRec) +
           (size_t)6 * E * sizeof(double) + (size_t)kResScratch * sizeof(double);
}

// nsteps evolution steps with the state resident in shared memory.
// ch: cells per block; ntr_cap: trajectory records per block;
// part: [2][gridDim.x][kSlotDoubles]; bar: arrival counter, zero at launch.
template <int MODEL>
__global__ void __launch_bounds__(kBlock, 1)
    k_resident(const __grid_constant__ StepArgs a, int nsteps, int ch, int ntr_cap, double* part, unsigned* bar) {
    constexpr int NM = MODEL == 0 ? 3 : (MODEL == 1 ? 6 : 12);
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ ResShared S;
    const int tid = threadIdx.x;
    const int c0 = blockIdx.x * ch;
    const int c1 = min(c0 + ch, a.ncell);
    const int n = c1 > c0 ? c1 - c0 : 0;
    const size_t np = a.npad;
    double* buf[2] = {reinterpret_cast<double*>(dsm), reinterpret_cast<double*>(dsm) + (size_t)kPlanes * ch};
    double* pst = buf[1] + (size_t)kPlanes * ch;
    TrajRec* rec = reinterpret_cast<TrajRec*>(pst + (size_t)kResProps * ch);
    // pst rows: 0-7 Um, 8-15 Uf -> Q, 16-23 P (class c at 4 c + {c, a, b, d})
    auto put = [&](int row, int k, const Prop (&u)[2]) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            pst[(size_t)(row + 4 * c + 0) * ch + k] = u[c].c;
            pst[(size_t)(row + 4 * c + 1) * ch + k] = u[c].a;
            pst[(size_t)(row + 4 * c + 2) * ch + k] = u[c].b;
            pst[(size_t)(row + 4 * c + 3) * ch + k] = u[c].d;
        }
    };
    auto get = [&](int row, int k, Prop (&u)[2]) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
            u[c] = Prop{pst[(size_t)(row + 4 * c + 0) * ch + k], pst[(size_t)(row + 4 * c + 1) * ch + k],
                        pst[(size_t)(row + 4 * c + 2) * ch + k], pst[(size_t)(row + 4 * c + 3) * ch + k]};
    };
    double* ktab = reinterpret_cast<double*>(rec + ntr_cap);
    double* scratch = ktab + 6 * a.E;  // [kResMaxNV][kBlock] (res_arrive)

    grid_dependency_wait();
    if (tid == 0) {
        const volatile Ctl* gc = a.ctl;
        unsigned char* dst = reinterpret_cast<unsigned char*>(&S.c);
        const volatile unsigned char* src = reinterpret_cast<const volatile unsigned char*>(gc);
        for (int i = 0; i < (int)sizeof(Ctl); ++i) dst[i] = src[i];
    }
    if (tid < NM) S.tot0[tid] = __ldcg(a.xbuf + tid);  // sums0 from S1 (osc_begin)
    __syncthreads();
    int lb = 0;  // local buffer holding psi0
    {
        const double* g = a.psi0_buf[S.c.cur];
        for (int i = tid; i < kPlanes * n; i += kBlock) {
            const int p = i / n, k = i - p * n;
            buf[0][(size_t)p * ch + k] = __ldcg(g + psi_off(a, p, (size_t)c0 + k));
        }
        for (int i = tid; i < 6 * a.E; i += kBlock) {
            const int row = i / a.E, e = i - row * a.E;
            ktab[i] = row == 0 ? __ldg(a.vac11 + e)
                               : (row == 1 ? __ldg(a.vac12 + e) : __ldg(a.g + (size_t)(row - 2) * a.E + e));
        }
    }
    const int tr0 = n ? (int)div_e(c0, a.e_magic, a.e_shift) : 0;
    const int ntr = n ? (int)div_e(c1 - 1, a.e_magic, a.e_shift) - tr0 + 1 : 0;
    unsigned phase = 0;
    // sums0 of the loaded psi0 at r (S1), formed as S4 below forms the
    // next-step moments and reduced by the same all-reduce: a restored state
    // (set_state / resume_from) starts from the bits an uninterrupted run has
    for (int i = tid; i < ntr; i += kBlock) {
        const int traj = tr0 + i;
        const Geo G = traj_geom<MODEL>(a, a.t_lo + traj / a.P, traj % a.P, S.c.r);
#pragma unroll
        for (int j = 0; j < 4; ++j) rec[i].fold[0][j] = G.f[j];
    }
    __syncthreads();
    bool started = true;
    {
        double acc[NM];
#pragma unroll
        for (int k = 0; k < NM; ++k) acc[k] = 0.0;
        for (int k = tid; k < n; k += kBlock) {
            const int cell = c0 + k;
            const int traj = (int)div_e(cell, a.e_magic, a.e_shift);
            const int e = cell - traj * a.E;
            CellK K;
            K.v11 = ktab[e];
            K.v12 = ktab[a.E + e];
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                K.g[s] = ktab[(2 + s) * a.E + e];
                K.g2[s] = K.g[s] + K.g[s];
            }
            double x[4][4];
#pragma unroll
            for (int s = 0; s < 4; ++s)
#pragma unroll
                for (int c = 0; c < 4; ++c) x[s][c] = buf[0][(size_t)(s * 4 + c) * ch + k];
            double B[2][3], Rr[3];
            class_bloch(x, K, B);
            bloch_sum(B, Rr);
            fold_acc<NM>(acc, Rr, rec[traj - tr0].fold[0]);
        }
        if (nsteps > 0) {
            started = res_allreduce<NM>(acc, 0.0, part, bar, phase, S, S.fin, scratch);
            if (started && tid < NM) S.tot0[tid] = S.fin[tid];
            __syncthreads();
        }
    }

    // The geometric part of a step's trajectory records (dl slots, direction
    // factors, fold coefficients at r+dr (fold[0]) and r+dr/2 (fold[1]);
    // geometry.cpp:66-216): a function of (r, dr) only, so the next step's is
    // built while S4's all-reduce completes, for the outcome "accepted, next
    // step at the capped size", and kept if the control then decides exactly
    // that (every fixed-step run; same operations, same bits).
    auto geometry = [&](double r, double dr) {
        const double rk[3] = {r, r + 0.5 * dr, r + dr};
        for (int i = tid; i < ntr; i += kBlock) {
            const int traj = tr0 + i;
            const int th = a.t_lo + traj / a.P, ph = traj % a.P;
            Geo G[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) G[q] = traj_geom<MODEL>(a, th, ph, rk[q]);
            TrajRec& R = rec[i];
            R.dl[0] = (0.5 * dr) / (0.5 * (G[0].cdl + G[1].cdl));
            R.dl[1] = (0.5 * dr) / (0.5 * (G[1].cdl + G[2].cdl));
            R.dl[2] = dr / (0.5 * (G[0].cdl + G[2].cdl));
#pragma unroll
            for (int q = 0; q < 3; ++q)
#pragma unroll
                for (int j = 0; j < 3; ++j) R.n[q][j] = G[q].n[j];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                R.fold[0][j] = G[2].f[j];
                R.fold[1][j] = G[1].f[j];
            }
        }
    };
    double r_sp = 0.0, dr_sp = 0.0;  // the (r, dr) the records' geometry was built for ahead of time
    bool have_sp = false;

    for (int step = 0; started && step < nsteps; ++step) {
        if (S.c.terminate | S.c.status | S.c.pause) break;
        const double r = S.c.r, dr = S.c.dr;
        const double rk[3] = {r, r + 0.5 * dr, r + dr};
        const double Am[3] = {S.c.A[0], S.c.A[1], S.c.A[2]};
        const double* x0 = buf[lb];
        double* xr = buf[lb ^ 1];

        // trajectory records of the step: the geometry (unless built ahead),
        // then H0 from the moments of psi0
        if (!(have_sp && r == r_sp && dr == dr_sp)) geometry(r, dr);
        for (int i = tid; i < ntr; i += kBlock) {  // (each thread reads the direction factors it wrote)
            TrajRec& R = rec[i];
            double hv[3];
            assemble<MODEL>(S.tot0, rk[0], a.Rnu, R.n[0], hv);
            R.hb[0][0] = hv[0] + 0.5 * Am[0];
            R.hb[0][1] = hv[1];
            R.hb[0][2] = hv[2];
        }
        __syncthreads();

        auto load_cell = [&](int k, CellK& K, double (&x)[4][4], const TrajRec*& R) {
            const int cell = c0 + k;
            const int traj = (int)div_e(cell, a.e_magic, a.e_shift);
            const int e = cell - traj * a.E;
            R = &rec[traj - tr0];
            K.v11 = ktab[e];
            K.v12 = ktab[a.E + e];
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                K.g[s] = ktab[(2 + s) * a.E + e];
                K.g2[s] = K.g[s] + K.g[s];
            }
#pragma unroll
            for (int s = 0; s < 4; ++s)
#pragma unroll
                for (int c = 0; c < 4; ++c) x[s][c] = x0[(size_t)(s * 4 + c) * ch + k];
        };

        // ---- S2: mid and full1 moments (sums2 at r+dr/2, sums1 at r+dr)
        {
            double acc[2 * NM];
#pragma unroll
            for (int k = 0; k < 2 * NM; ++k) acc[k] = 0.0;
            for (int k = tid; k < n; k += kBlock) {
                CellK K;
                double x[4][4];
                const TrajRec* R;
                load_cell(k, K, x, R);
                Prop um[2], uf[2];
                const PropReq rq[2] = {{R->hb[0], R->dl[0], false, um}, {R->hb[0], R->dl[2], false, uf}};
                make_props_n(K, rq);
                double B[2][3], Rr[3];
                class_bloch(x, K, B);
                bloch_rho(um, B, Rr);
                fold_acc<NM>(acc + NM, Rr, R->fold[1]);
                bloch_rho(uf, B, Rr);
                fold_acc<NM>(acc, Rr, R->fold[0]);
                put(0, k, um);
                put(8, k, uf);
            }
            if (!res_allreduce<2 * NM>(acc, 0.0, part, bar, phase, S, S.fin, scratch)) break;
            if (tid < 2 * NM) S.tot1[tid] = S.fin[tid];
        }
        // H1 (sums1, r+dr) and H2 (sums2, r+dr/2)
        for (int i = tid; i < 2 * ntr; i += kBlock) {
            TrajRec& R = rec[i >> 1];
            const int h = (i & 1) ? 2 : 1, q = (i & 1) ? 1 : 2;
            double hv[3];
            assemble<MODEL>(S.tot1 + (h == 1 ? 0 : NM), rk[q], a.Rnu, R.n[q], hv);
            R.hb[h][0] = hv[0] + 0.5 * Am[q];
            R.hb[h][1] = hv[1];
            R.hb[h][2] = hv[2];
        }
        __syncthreads();

        // ---- S3: half2 = P psi0 with P = Uh(H2) Um(H0); sums3 at r+dr.  While
        // the other blocks arrive: U2(H1) and Q = (Uf + U2)/2 for S4.
        {
            double acc[NM];
#pragma unroll
            for (int k = 0; k < NM; ++k) acc[k] = 0.0;
            for (int k = tid; k < n; k += kBlock) {
                CellK K;
                double x[4][4];
                const TrajRec* R;
                load_cell(k, K, x, R);
                Prop uh[2], um[2], P[2];
                {
                    const PropReq rq[1] = {{R->hb[2], R->dl[1], false, uh}};
                    make_props_n(K, rq);
                }
                get(0, k, um);
                P[0] = prop_mul(uh[0], um[0]);
                P[1] = prop_mul(uh[1], um[1]);
                double B[2][3], Rr[3];
                class_bloch(x, K, B);
                bloch_rho(P, B, Rr);
                fold_acc<NM>(acc, Rr, R->fold[0]);
                put(16, k, P);
            }
            res_arrive<NM>(acc, 0.0, part, bar, phase, S, scratch);
            for (int k = tid; k < n; k += kBlock) {
                CellK K;
                double x[4][4];
                const TrajRec* R;
                load_cell(k, K, x, R);
                Prop u2[2], uf[2], Q[2];
                {
                    const PropReq rq[1] = {{R->hb[1], R->dl[2], true, u2}};
                    make_props_n(K, rq);
                }
                get(8, k, uf);
#pragma unroll
                for (int c = 0; c < 2; ++c)
                    Q[c] = Prop{fma(uf[c].c, 0.5, u2[c].c), fma(uf[c].a, 0.5, u2[c].a), fma(uf[c].b, 0.5, u2[c].b),
                                fma(uf[c].d, 0.5, u2[c].d)};
                put(8, k, Q);
            }
            if (!res_finish<NM>(part, bar, phase, S, S.fin)) break;
            if (tid < NM) S.tot3[tid] = S.fin[tid];
        }
        // H3 (sums3, r+dr)
        for (int i = tid; i < ntr; i += kBlock) {
            TrajRec& R = rec[i];
            double hv[3];
            assemble<MODEL>(S.tot3, rk[2], a.Rnu, R.n[2], hv);
            R.hb[3][0] = hv[0] + 0.5 * Am[2];
            R.hb[3][1] = hv[1];
            R.hb[3][2] = hv[2];
        }
        __syncthreads();

        // ---- S4: result = Rm psi0, err = max |(Q - Rm) psi0|, next sums0
        {
            double acc[NM];
#pragma unroll
            for (int k = 0; k < NM; ++k) acc[k] = 0.0;
            double emax = 0.0;
            for (int k = tid; k < n; k += kBlock) {
                CellK K;
                double x[4][4];
                const TrajRec* R;
                load_cell(k, K, x, R);
                Prop u3[2], P[2], Q[2];
                {
                    const PropReq rq3[1] = {{R->hb[3], R->dl[2], true, u3}};
                    make_props_n(K, rq3);
                }
                get(16, k, P);
                get(8, k, Q);
                Prop Rm[2], Dm[2];
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    Rm[c] = Prop{fma(P[c].c, 0.5, u3[c].c), fma(P[c].a, 0.5, u3[c].a), fma(P[c].b, 0.5, u3[c].b),
                                 fma(P[c].d, 0.5, u3[c].d)};
                    Dm[c] = Prop{Q[c].c - Rm[c].c, Q[c].a - Rm[c].a, Q[c].b - Rm[c].b, Q[c].d - Rm[c].d};
                }
                // moments of the candidate through its class Bloch vectors, as
                // the stage kernels' S1 and S4 form them (same bits)
                double B[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}}, Rr[3];
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    double out[4], d[4];
                    apply(Rm[s & 1], x[s], out);
                    apply(Dm[s & 1], x[s], d);
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        xr[(size_t)(s * 4 + c) * ch + k] = out[c];
                        emax = max_abs(emax, d[c]);
                    }
                    bloch_add(out, K, s, B);
                }
                bloch_sum(B, Rr);
                fold_acc<NM>(acc, Rr, R->fold[0]);
            }
            res_arrive<NM>(acc, emax, part, bar, phase, S, scratch);
            // while the other blocks arrive: the next step's geometry (the
            // records are free: every thread has passed the barrier in
            // res_arrive), predicted as ctl_advance computes it for an
            // accepted step whose next size hits dr_max
            r_sp = r + dr;
            dr_sp = S.c.dr_max;
            if (r_sp + dr_sp > S.c.Rn) dr_sp = S.c.Rn - r_sp;
            geometry(r_sp, dr_sp);
            have_sp = true;
            if (!res_finish<NM>(part, bar, phase, S, S.fin)) break;
            if (tid <= NM) S.totn[tid] = S.fin[tid];
        }

        // ---- lane_body control, redundantly and identically in every block
        if (tid == 0) {
            bool ok = true;
            for (int k = 0; k < NM; ++k) ok = ok && isfinite(S.tot0[k]) && isfinite(S.tot3[k]);
            for (int k = 0; k < 2 * NM; ++k) ok = ok && isfinite(S.tot1[k]);
            S.accept = ctl_advance(&S.c, a, S.totn[NM], ok);
        }
        __syncthreads();
        if (S.accept) {
            lb ^= 1;
            if (tid < NM) S.tot0[tid] = S.totn[tid];
        }
        __syncthreads();
    }

    // publish: psi0 to the global buffer Ctl::cur names, Ctl and sums0 (block 0)
    {
        double* g = a.psi0_buf[S.c.cur];
        for (int i = tid; i < kPlanes * n; i += kBlock) {
            const int p = i / n, k = i - p * n;
            g[psi_off(a, p, (size_t)c0 + k)] = buf[lb][(size_t)p * ch + k];
        }
    }
    if (blockIdx.x == 0) {
        if (tid < NM) a.xbuf[tid] = S.tot0[tid];
        if (tid == 0) {
            if (S.stop) {  // barrier timeout: report instead of hanging
                S.c.status = OSC_ERR_PARALLEL;
                S.c.reason = 4;
                S.c.terminate = 4;
            }
            *a.ctl = S.c;
        }
    }
}

}  // namespace oscb200
