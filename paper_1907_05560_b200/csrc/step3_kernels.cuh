// 3-flavour stage kernels (BASELINE configs[1]; not in the reference, which
// accepts Flvs = 2 only — DESIGN.md §9).  Same S1-S4 schedule, moments,
// reductions and device control as the 2-flavour kernels (step_kernels.cuh);
// what changes:
//   * psi in C^3: species s = 2 f + pc (f = e, mu, tau; pc = particle class),
//     6 components (re/im of e, mu, tau), state planes (s*6 + c);
//   * work item = (particle class, cell): the three species of a class share
//     the beam Hamiltonian, so one 3x3 propagator (su3_exp.cuh) per evolve
//     serves three 3x3 complex mat-vecs;
//   * rho = psi psi^dagger (9 reals); moments: 9 per geometric moment
//     (single angle 9, bulb 18);
//   * H_nu = H_vac(E) + diag(A,0,0) + H_nunu,
//     H_nubar = conj(H_vac) - diag(A,0,0) - conj(H_nunu).
#pragma once

#include "step_kernels.cuh"
#include "su3_exp.cuh"

namespace oscb200 {

constexpr int kNM3Max = 18;  // 9 x (a, b): single-angle and bulb geometries
// stash planes (schedule 1): [0, 36) mid (S2) -> half2 (S3, in place) in the
// state plane order, [36, 72) Uf = exp(-i H0 dl2) of each class (S2 -> S4,
// 3x3 complex row-major, re/im)
constexpr int kSt3Uf = 36;
constexpr int kSt3Planes = 72;

#ifndef OSC3_MIN_BLOCKS
#define OSC3_MIN_BLOCKS 1  // resident 3-flavour blocks per SM the register budget targets
#endif
#ifndef OSC3_BLOCK
#define OSC3_BLOCK 256
#endif
// Threads per 3-flavour block (one block per SM).  The 3-flavour kernels are
// latency-bound, so a block's time is its rounds of (class, cell) items per
// thread times the latency of one item: configs[1] (2 x 65536 items over 148
// SMs, 3.46 per thread at 256 threads) takes 4 rounds with 256 threads, 3 with
// 320 (200 registers instead of 255).
constexpr int kBlock3 = OSC3_BLOCK;
constexpr int kWarps3 = kBlock3 / 32;

struct TrajRec3 {
    double hb[4][9];   // beam part (H_nunu + matter) for H0..H3, particle convention
    double dl[3];
    double fold[2][2]; // (w, w n1)
    double n1[3];      // cos theta' at r, r+dr/2, r+dr
    double pad_;
};

// packed Hermitian helpers: index 0-2 diagonal, (3,4) 01, (5,6) 02, (7,8) 12
__device__ __forceinline__ Herm3 herm_of(const double* v, const double* b, int pc) {
    // particle: v + b ; antiparticle: conj(v) - conj(b)
    // real parts v +- b; imaginary parts v_im + b_im (particle) or
    // -v_im + b_im (antiparticle: conj(v) - conj(b))
    Herm3 h;
    const double sg = pc ? -1.0 : 1.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) h.d[k] = v[k] + sg * b[k];
    h.o01 = Cx{v[3] + sg * b[3], sg * v[4] + b[4]};
    h.o02 = Cx{v[5] + sg * b[5], sg * v[6] + b[6]};
    h.o12 = Cx{v[7] + sg * b[7], sg * v[8] + b[8]};
    return h;
}

__device__ __forceinline__ void apply3(const Mat3& U, const double (&x)[6], double (&y)[6]) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        double re = 0.0, im = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const Cx u = U.m[i][j];
            re = fma(u.re, x[2 * j], fma(-u.im, x[2 * j + 1], re));
            im = fma(u.re, x[2 * j + 1], fma(u.im, x[2 * j], im));
        }
        y[2 * i] = re;
        y[2 * i + 1] = im;
    }
}

// weighted rho = psi psi^dagger of the 3 species of a class, summed; for
// antiparticles the row enters minus-conjugated (combine_species,
// geometry.cpp:119-136) — folded into the signed weight g and an imaginary
// sign flip.
__device__ __forceinline__ void weighted_rho3(const double (&y)[3][6], const double (&g)[3], int pc,
                                              double (&R)[9]) {
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = 0.0;
#pragma unroll
    for (int f = 0; f < 3; ++f) {
        const double ar = y[f][0], ai = y[f][1], br = y[f][2], bi = y[f][3], cr = y[f][4], ci = y[f][5];
        const double gi = pc ? -g[f] : g[f];
        R[0] += g[f] * (ar * ar + ai * ai);
        R[1] += g[f] * (br * br + bi * bi);
        R[2] += g[f] * (cr * cr + ci * ci);
        R[3] += g[f] * (ar * br + ai * bi);  // a conj(b)
        R[4] += gi * (ai * br - ar * bi);
        R[5] += g[f] * (ar * cr + ai * ci);  // a conj(c)
        R[6] += gi * (ai * cr - ar * ci);
        R[7] += g[f] * (br * cr + bi * ci);  // b conj(c)
        R[8] += gi * (bi * cr - br * ci);
    }
}

// Single GPU (a.cr3): lane_body's control for the previous step's S4 at the
// start of S2 (and in k_finalize3), as cr_control does for 2 flavours: every
// block reduces S4's block partials, decides on a shared copy of the control
// block, block 0 stores it with the promoted sums0 and slot 3.  tot0: the
// step's sums0 (NM values).
template <int NM>
__device__ __forceinline__ void cr_control3(const StepArgs& a, StageShared& S, bool finalize, double* tot0) {
    const int tid = threadIdx.x;
    for (int i = tid; i < kCtlWords; i += blockDim.x)
        reinterpret_cast<unsigned long long*>(&S.cs)[i] = __ldcg(reinterpret_cast<const unsigned long long*>(a.ctl) + i);
    const double x0 = tid < NM ? __ldcg(a.xbuf + tid) : 0.0;
    cr_reduce<NM, kBlock3>(a.cpart[3], a.nblocks, S.red, S.fin);
    Ctl& c = S.cs;
    if (tid == 0) {
        S.accept = c.pend ? ctl_advance(&c, a, S.fin[NM], c.bad_sums == 0) : -1;
        S.r = c.r;
        S.dr = c.dr;
        S.A[0] = c.A[0];
        S.A[1] = c.A[1];
        S.A[2] = c.A[2];
        S.iter = c.iter;
        S.cur = c.cur;
        S.stop = c.terminate | c.status | c.pause;
        c.pend = (finalize || S.stop) ? 0 : 1;
    }
    __syncthreads();
    if (tid < NM) {
        const double v = S.accept == 1 ? S.fin[tid] : x0;
        if (tot0) tot0[tid] = v;
        if (blockIdx.x == 0) {
            if (S.accept == 1) a.xbuf[tid] = v;
            if (S.accept >= 0) {
                a.xbuf[3 * kSlotDoubles + tid] = S.fin[tid];
                if (tid == 0) a.xbuf[3 * kSlotDoubles + 36] = S.fin[NM];
            }
        }
    }
    // the advanced copy goes to the other control buffer (see StepArgs::ctl_out)
    if (blockIdx.x == 0) store_ctl(a.ctl_out, c);
    __syncthreads();
}

#ifndef OSC3_S4_OOL
#define OSC3_S4_OOL 0  // (S4 evaluates two exponentials since U1 and half2 come from the stash)
#endif
__host__ __device__ constexpr int stage3_pf_planes(int stage) { return stage == 4 ? 36 : 18; }
__host__ __device__ constexpr size_t stage3_rec_bytes(int ntr_max) { return ((size_t)ntr_max * sizeof(TrajRec3) + 15) & ~(size_t)15; }
__device__ __forceinline__ void cp_async16_cg(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// Pair plane q (the (re, im) pair of one amplitude or matrix entry) of a cell
// in a buffer of planes of pairs.
__device__ __forceinline__ double2* pair_at(double* base, int q, size_t np, size_t cell) {
    return reinterpret_cast<double2*>(base + 2 * ((size_t)q * np + cell));
}
__device__ __forceinline__ const double2* pair_at(const double* base, int q, size_t np, size_t cell) {
    return reinterpret_cast<const double2*>(base + 2 * ((size_t)q * np + cell));
}
__device__ __noinline__ Mat3 exp_herm3_ool(const Herm3& H, double tau) { return exp_herm3(H, tau); }

template <int MODEL, int STAGE>
__global__ void __launch_bounds__(kBlock3, OSC3_MIN_BLOCKS) k_stage3(StepArgs a) {
    using Tr = StageTraits<STAGE>;
    constexpr int NG = MODEL == 0 ? 1 : 2;  // geometric moments (a | a, b)
    constexpr int NM = 9 * NG;
    constexpr int NV = NM * Tr::nsets;
    extern __shared__ __align__(128) unsigned char dsm3[];
    __shared__ double tot[4][kNM3Max];
    __shared__ double red[kWarps3 * (2 * kNM3Max + 1)];
    __shared__ int is_last;

    const Ctl* ctl = a.ctl;
    grid_dependency_wait();
    // S2 (single GPU): the previous step's control first (cr_control3)
    __shared__ StageShared CS;
    const bool ctl2 = STAGE == 2 && a.cr3;
    if (ctl2) {
        cr_control3<NM>(a, CS, false, &tot[0][0]);
        if (CS.stop) return;
    } else if (STAGE != 0 && (ctl->terminate || ctl->status || ctl->pause)) {
        return;
    }
    const int tid = threadIdx.x;
    const int nb_half = gridDim.x / 2;
    const int pc = blockIdx.x >= nb_half;
    const int hb_ = blockIdx.x - pc * nb_half;
    const int c0 = hb_ * a.chunk;
    const int c1 = min(c0 + a.chunk, a.ncell);
    const double r = ctl2 ? CS.r : ctl->r, dr = ctl2 ? CS.dr : ctl->dr;
    const double rk[3] = {r, r + 0.5 * dr, r + dr};
    const int cur = ctl2 ? CS.cur : ctl->cur;
    const double* __restrict__ psi0 = a.psi0_buf[cur];
    double* __restrict__ res = a.psi0_buf[cur ^ 1];
    const size_t np = a.npad;
    TrajRec3* rec = reinterpret_cast<TrajRec3*>(dsm3);

    if (a.cr3 && (STAGE == 3 || STAGE == 4)) {
        // single GPU: S2's / S3's block partials reduced here (the same tree
        // their last block applied; cr_reduce, step_kernels.cuh), sums0 and
        // (S4) sums1 | sums2 as S3's block 0 stored them
        const double x0 = tid < NM ? __ldcg(a.xbuf + tid) : 0.0;
        const double x1 = (STAGE == 4 && tid < 2 * NM)
                              ? __ldcg(a.xbuf + kSlotDoubles + (tid < NM ? tid : 36 + tid - NM))
                              : 0.0;
        __shared__ double cfin[2 * kNM3Max + 1];
        if (STAGE == 3)
            cr_reduce<2 * NM, kBlock3>(a.cpart[1], (int)gridDim.x, red, cfin);
        else
            cr_reduce<NM, kBlock3>(a.cpart[2], (int)gridDim.x, red, cfin);
        if (tid < NM) tot[0][tid] = x0;
        if (STAGE == 4 && tid < 2 * NM) tot[1 + tid / NM][tid % NM] = x1;
        if (tid < (STAGE == 3 ? 2 * NM : NM)) {
            const int set = tid / NM, j = tid % NM;
            const double v = cfin[set * NM + j];
            tot[STAGE == 3 ? 1 + set : 3][j] = v;
            if (blockIdx.x == 0) {
                // slot layout: 36 doubles per set (S2: sums1 | sums2)
                a.xbuf[(STAGE == 3 ? 1 : 2) * kSlotDoubles + set * 36 + j] = v;
                if (!isfinite(v)) atomicOr(&a.ctl->bad_sums, 1);  // check_sums_finite
            }
        }
    } else if (tid < 4 * NM && !ctl2) {
        const int h = tid / NM, k = tid % NM;
        if (Tr::hmask & (1 << h)) {
            const int slot = h == 0 ? 0 : (h == 3 ? 2 : 1);
            const int off = h == 2 ? 36 : 0;

            // slot layout per set: 9 x geometric moment (a at 0..8, b at 9..17)
            tot[h][k] = slot_total(a, slot, off + k);
            if (a.p2p && !isfinite(tot[h][k])) atomicOr(&a.ctl->bad_sums, 1);
        }
    }
    if (STAGE == 0 && blockIdx.x == 0 && tid == 0) {
        a.ctl->A[0] = matter_potential(a, rk[0]);
        a.ctl->A[1] = matter_potential(a, rk[1]);
        a.ctl->A[2] = matter_potential(a, rk[2]);
    }
    __syncthreads();
    const double Am[3] = {ctl2 ? CS.A[0] : (STAGE ? ctl->A[0] : 0.0), ctl2 ? CS.A[1] : (STAGE ? ctl->A[1] : 0.0),
                          ctl2 ? CS.A[2] : (STAGE ? ctl->A[2] : 0.0)};
    const int tr0 = c1 > c0 ? (int)div_e(c0, a.e_magic, a.e_shift) : 0;
    const int ntr = c1 > c0 ? (int)div_e(c1 - 1, a.e_magic, a.e_shift) - tr0 + 1 : 0;
    for (int i = tid; i < ntr; i += kBlock3) {
        const int traj = tr0 + i;
        const int th = a.t_lo + traj / a.P;
        Geo G[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) G[q] = traj_geom<MODEL>(a, th, 0, rk[q]);
        TrajRec3& R = rec[i];
        R.dl[0] = (0.5 * dr) / (0.5 * (G[0].cdl + G[1].cdl));
        R.dl[1] = (0.5 * dr) / (0.5 * (G[1].cdl + G[2].cdl));
        R.dl[2] = dr / (0.5 * (G[0].cdl + G[2].cdl));
#pragma unroll
        for (int q = 0; q < 3; ++q) R.n1[q] = G[q].n[0];
        const int fq[2] = {Tr::fold0, Tr::fold1};
#pragma unroll
        for (int f = 0; f < Tr::nsets; ++f) {
            R.fold[f][0] = G[fq[f]].f[0];
            R.fold[f][1] = G[fq[f]].f[1];
        }
        constexpr int hr[4] = {0, 2, 1, 2};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            if (!(Tr::hmask & (1 << h))) continue;
            const int q = hr[h];
            double D = 1.0;
            if (MODEL == 0) {
                const double ra = a.Rnu / rk[q], t = 1.0 - sqrt(1.0 - ra * ra);
                D = 0.5 * t * t;
            }
#pragma unroll
            for (int k = 0; k < 9; ++k)
                R.hb[h][k] = MODEL == 0 ? tot[h][k] * D : tot[h][k] + tot[h][9 + k] * (-R.n1[q]);
            R.hb[h][0] += Am[q];  // matter diag(A, 0, 0)
        }
    }
    __syncthreads();

    double acc[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] = 0.0;
    double emax = 0.0;
    const bool stash = a.schedule == 1;

    // Streamed operands of the next cell are copied into this thread's
    // shared-memory column while the current cell's exponentials run
    // (cp.async, double-buffered): one block of 8 warps per SM (255
    // registers) cannot hide their latency otherwise, and in registers they
    // would spill.  Slots [0, 18): psi0 of the class (S3 with the stash: mid
    // = Um psi0 from S2), [18, 36) (S4 with the stash): half2 from S3.
    constexpr int PF = stage3_pf_planes(STAGE);
    double* pf = reinterpret_cast<double*>(dsm3 + stage3_rec_bytes(a.ntr_max));
    double2* pf2 = reinterpret_cast<double2*>(pf);           // the same columns as (re, im) pairs: [2][PF / 2][kBlock3]
    double2* ufc = pf2 + (size_t)PF * kBlock3;               // S4, a.uf_cols: [9][kBlock3]
    const double* src0 = (STAGE == 3 && stash) ? a.stash : psi0;
    auto issue = [&](int cl, int buf) {
        if (cl < c1) {
#pragma unroll
            for (int j = 0; j < PF / 2; ++j) {  // pair j % 9 = 3 f + amplitude of species 2 f + pc
                if (j >= 9 && !stash) break;
                cp_async16_cg(pf2 + ((size_t)buf * (PF / 2) + j) * kBlock3 + tid,
                              pair_at(j < 9 ? src0 : a.stash, (2 * ((j % 9) / 3) + pc) * 3 + j % 3, np, cl));
            }
        }
        cp_async_commit();
    };
    issue(c0 + tid, 0);
    int it = 0;
    for (int cell = c0 + tid; cell < c1; cell += kBlock3, ++it) {
        const int traj = (int)div_e(cell, a.e_magic, a.e_shift);
        const int e = cell - traj * a.E;
        const TrajRec3& R = rec[traj - tr0];
        cp_async_wait_all();  // this thread's copies of this cell
        issue(cell + kBlock3, (it + 1) & 1);
        if (STAGE == 4 && stash && a.uf_cols) {
            // U1 (full1's propagator, stashed by S2) is needed at the end of
            // the cell: copied into this thread's column now, so its L2
            // latency hides behind the exponentials (read straight from
            // global it stalled S4 ~20 % of the time)
#pragma unroll
            for (int j = 0; j < 9; ++j)
                cp_async16_cg(ufc + (size_t)j * kBlock3 + tid, pair_at(a.stash, kSt3Uf / 2 + pc * 9 + j, np, cell));
            cp_async_commit();
        }
        const double2* cur_pf = pf2 + (size_t)(it & 1) * (PF / 2) * kBlock3 + tid;
        double x[3][6];
#pragma unroll
        for (int j = 0; j < 9; ++j) {
            const double2 v = cur_pf[(size_t)j * kBlock3];
            x[j / 3][2 * (j % 3)] = v.x;
            x[j / 3][2 * (j % 3) + 1] = v.y;
        }
        double g[3];
#pragma unroll
        for (int f = 0; f < 3; ++f) g[f] = __ldg(a.g + (size_t)(2 * f + pc) * a.E + e);
        double v[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) v[k] = __ldg(a.vac3 + (size_t)e * 9 + k);
        double Rr[9];
        // S4 evaluates the exponential five times: one out-of-line copy there
        // (inlined, the stage misses the instruction cache a third of the time)
        auto prop = [&](int h, int slot) {
            return (STAGE == 4 && OSC3_S4_OOL) ? exp_herm3_ool(herm_of(v, R.hb[h], pc), R.dl[slot])
                                               : exp_herm3(herm_of(v, R.hb[h], pc), R.dl[slot]);
        };

        if (STAGE == 0) {
            weighted_rho3(x, g, pc, Rr);
#pragma unroll
            for (int j = 0; j < NG; ++j)
#pragma unroll
                for (int k = 0; k < 9; ++k) acc[9 * j + k] += R.fold[0][j] * Rr[k];
        } else if (STAGE == 2) {
            // mid and full1 share H0: one eigendecomposition, two exponentials
            const Eig3 e0 = eig_herm3(herm_of(v, R.hb[0], pc));
            const Mat3 um = exp_from_eig(e0, R.dl[0]), uf = exp_from_eig(e0, R.dl[2]);
            double y[3][6];
#pragma unroll
            for (int f = 0; f < 3; ++f) apply3(um, x[f], y[f]);
            weighted_rho3(y, g, pc, Rr);
#pragma unroll
            for (int j = 0; j < NG; ++j)
#pragma unroll
                for (int k = 0; k < 9; ++k) acc[NM + 9 * j + k] += R.fold[1][j] * Rr[k];
            if (stash) {
                // S3 continues from mid, S4 averages with full1's propagator:
                // neither recomputes an exponential of H0
#pragma unroll
                for (int f = 0; f < 3; ++f)
#pragma unroll
                    for (int h = 0; h < 3; ++h)
                        __stcg(pair_at(a.stash, (2 * f + pc) * 3 + h, np, cell), make_double2(y[f][2 * h], y[f][2 * h + 1]));
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                        __stcg(pair_at(a.stash, kSt3Uf / 2 + pc * 9 + i * 3 + j, np, cell),
                               make_double2(uf.m[i][j].re, uf.m[i][j].im));
            }
#pragma unroll
            for (int f = 0; f < 3; ++f) apply3(uf, x[f], y[f]);
            weighted_rho3(y, g, pc, Rr);
#pragma unroll
            for (int j = 0; j < NG; ++j)
#pragma unroll
                for (int k = 0; k < 9; ++k) acc[9 * j + k] += R.fold[0][j] * Rr[k];
        } else if (STAGE == 3) {
            const Mat3 uh = prop(2, 1);
            Mat3 um;
            if (!stash) um = prop(0, 0);
            double hh[3][6];
#pragma unroll
            for (int f = 0; f < 3; ++f) {
                double mid[6];
                if (stash) {  // mid = Um psi0 from S2 (prefetched); half2 replaces it in place
#pragma unroll
                    for (int c = 0; c < 6; ++c) mid[c] = x[f][c];
                } else {
                    apply3(um, x[f], mid);
                }
                apply3(uh, mid, hh[f]);
                if (stash)
#pragma unroll
                    for (int h = 0; h < 3; ++h)
                        __stcg(pair_at(a.stash, (2 * f + pc) * 3 + h, np, cell), make_double2(hh[f][2 * h], hh[f][2 * h + 1]));
            }
            weighted_rho3(hh, g, pc, Rr);
#pragma unroll
            for (int j = 0; j < NG; ++j)
#pragma unroll
                for (int k = 0; k < 9; ++k) acc[9 * j + k] += R.fold[0][j] * Rr[k];
        } else {
            // (the exponentials first: with the out-of-line copy everything
            // live across a call goes to the stack)
            const Mat3 u3 = prop(3, 2);
            double out[3][6];
            {
                double h2[3][6];
                if (stash) {  // (prefetched)
#pragma unroll
                    for (int j = 0; j < 9; ++j) {
                        const double2 v = cur_pf[(size_t)(9 + j) * kBlock3];
                        h2[j / 3][2 * (j % 3)] = v.x;
                        h2[j / 3][2 * (j % 3) + 1] = v.y;
                    }
                } else {
                    const Mat3 um = prop(0, 0), uh = prop(2, 1);
#pragma unroll
                    for (int f = 0; f < 3; ++f) {
                        double mid[6];
                        apply3(um, x[f], mid);
                        apply3(uh, mid, h2[f]);
                    }
                }
#pragma unroll
                for (int f = 0; f < 3; ++f) {
                    double f3[6];
                    apply3(u3, x[f], f3);
#pragma unroll
                    for (int c = 0; c < 6; ++c) out[f][c] = (h2[f][c] + f3[c]) * 0.5;  // evolve_avg, beam.cpp:188-218
#pragma unroll
                    for (int h = 0; h < 3; ++h)
                        *pair_at(res, (2 * f + pc) * 3 + h, np, cell) = make_double2(out[f][2 * h], out[f][2 * h + 1]);
                }
            }
            weighted_rho3(out, g, pc, Rr);
#pragma unroll
            for (int j = 0; j < NG; ++j)
#pragma unroll
                for (int k = 0; k < 9; ++k) acc[9 * j + k] += R.fold[0][j] * Rr[k];
            // avgA = (full1 + full2)/2 = Q psi0 with Q = (U1 + U2)/2: one
            // 3x3 apply per species for the error instead of two; U1 comes
            // from S2 (stash) or is recomputed
            const Mat3 u2 = prop(1, 2);
            Mat3 Q;
            if (stash && a.uf_cols) {
                cp_async_wait_all();  // (the column copy above; the next cell's operands have landed long since)
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                    {
                        const double2 v = ufc[(size_t)(i * 3 + j) * kBlock3 + tid];
                        Q.m[i][j] = Cx{v.x, v.y};
                    }
            } else if (stash) {
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                    {
                        const double2 v = __ldcg(pair_at(a.stash, kSt3Uf / 2 + pc * 9 + i * 3 + j, np, cell));
                        Q.m[i][j] = Cx{v.x, v.y};
                    }
            } else {
                Q = prop(0, 2);
            }
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    Q.m[i][j] = Cx{(Q.m[i][j].re + u2.m[i][j].re) * 0.5, (Q.m[i][j].im + u2.m[i][j].im) * 0.5};
#pragma unroll
            for (int f = 0; f < 3; ++f) {
                double av[6];
                apply3(Q, x[f], av);
#pragma unroll
                for (int c = 0; c < 6; ++c) emax = max_abs(emax, av[c] - out[f][c]);
            }
        }
    }
    grid_launch_dependents();

    // block partial by transposition through the prefetch columns (free
    // now; sized for NV + 1 columns), stored [value][block] (a reducer's
    // loads of one value across blocks coalesce)
    const bool cr_out = a.cr3 && (STAGE == 2 || STAGE == 3 || STAGE == 4);  // reduced by every block of S3 / S4 / next S2
    block_cols_store<NV, kBlock3>(acc, emax, pf, (cr_out ? a.cpart[Tr::slot] : a.partials) + blockIdx.x, gridDim.x);
    if (cr_out) return;
    if (tid == 0) {
        __threadfence();
        const unsigned ticket = atomicAdd(&a.ctl->counter[Tr::slot], 1u);
        is_last = ticket == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    __shared__ double fin[2 * kNM3Max + 1];
    __shared__ double pub[kSlotDoubles];
    cols_reduce<NV, kBlock3>(a.partials, (int)gridDim.x, fin);
    if (tid < kSlotDoubles) {
        // slot layout: per set 36 doubles (9 x up to 4 geometric moments),
        // S2 = sums1 | sums2, S4 error at index 36
        const int k = tid;
        double v = 0.0;
        if (STAGE == 2) {
            if (k < 72) {
                const int set = k / 36, j = k % 36;
                v = j < NM ? fin[set * NM + j] : 0.0;
            }
        } else if (k < 36) {
            v = k < NM ? fin[k] : 0.0;
        } else if (k == 36) {
            v = fin[NV];
        }
        if (!a.p2p) a.xsend[(size_t)Tr::slot * kSlotDoubles + k] = v;
        if (!a.p2p && STAGE != 4 && !isfinite(v)) atomicOr(&a.ctl->bad_sums, 1);
        pub[k] = v;
    }
    if (a.p2p) {
        __syncthreads();
        p2p_publish(a, Tr::slot, tid < kSlotDoubles ? pub[tid] : 0.0);
    }
    if (tid == 0) a.ctl->counter[Tr::slot] = 0;
    if (STAGE == 4 && (a.fuse_ctl || a.p2p)) {
        __threadfence();
        __syncthreads();
        control_update(a, true);
    }
}

// Dynamic shared memory of a 3-flavour stage: trajectory records, then the
// double-buffered per-thread prefetch columns.
inline size_t stage3_smem_bytes(int ntr_max, int stage, int uf_cols = 0) {
    // (the columns double as the block-partial scratch: 2 x 18 moments + max in S2;
    // S4 with uf_cols: 18 more single-buffered columns for U1)
    const int cols = std::max(2 * stage3_pf_planes(stage) + ((stage == 4 && uf_cols) ? 18 : 0), 2 * kNM3Max + 1);
    return stage3_rec_bytes(ntr_max) + (size_t)cols * kBlock3 * sizeof(double);
}

// Single GPU: the control update of a batch's last step (one block).
template <int MODEL>
__global__ void __launch_bounds__(kBlock3, 1) k_finalize3(StepArgs a) {
    __shared__ StageShared S;
    grid_dependency_wait();
    cr_control3<MODEL == 0 ? 9 : 18>(a, S, true, nullptr);
}

// 3-flavour init: pure flavour f = s / 2 plus eps noise on the other two
// flavours, splitmix64-seeded by the global beam index j*6 + s (generalises
// beam.cpp:41-57).
__global__ void k_init3(StepArgs a, double eps) {
    const int cell = blockIdx.x * blockDim.x + threadIdx.x;
    if (cell >= a.ncell) return;
    double* psi = a.psi0_buf[a.ctl->cur];
    const int traj = cell / a.E, e = cell - traj * a.E;
    const uint64_t j = (uint64_t)(a.t_lo * a.P + traj);
    const size_t np = a.npad;
    for (int s = 0; s < 6; ++s) {
        const int f = s / 2;
        double c[6] = {0, 0, 0, 0, 0, 0};
        c[2 * f] = 1.0;
        if (eps != 0.0) {
            const uint64_t seed = j * 6 + s;
            const int o1 = (f + 1) % 3, o2 = (f + 2) % 3;
            const double u1 = eps * unit_noise(seed, e, 0), v1 = eps * unit_noise(seed, e, 1);
            const double u2 = eps * unit_noise(seed, e, 2), v2 = eps * unit_noise(seed, e, 3);
            const double q = __dsub_rn(__dsub_rn(__dsub_rn(__dsub_rn(1.0, __dmul_rn(u1, u1)), __dmul_rn(v1, v1)),
                                                 __dmul_rn(u2, u2)),
                                       __dmul_rn(v2, v2));
            c[2 * f] = sqrt(fmax(0.0, q));
            c[2 * o1] = u1;
            c[2 * o1 + 1] = v1;
            c[2 * o2] = u2;
            c[2 * o2 + 1] = v2;
        }
        for (int k = 0; k < 6; ++k) psi[psi_off(a, s * 6 + k, cell)] = c[k];
    }
}

}  // namespace oscb200
