// Host side of the drop-in: the OscCtx behind the C-ABI in
// include/oscflat_b200.h.  Replaces solver::Engine::Impl
// (reference solver.cpp:198-456): owns the device state, launches the fused
// stage kernels, exchanges moment partials between GPUs (NCCL all-gather,
// fixed rank-order combine), and runs the step loop with the control state
// resident on the device so that batches of steps are replayed as one CUDA
// graph without host round trips.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "oscflat_b200.h"
#include "status.hpp"
#include "step3_kernels.cuh"
#include "resident_kernels.cuh"
#include "step_kernels.cuh"

namespace oscb200 {

thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }

#define CUDA_OK(x)                                                                              \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess)                                                                  \
            throw Error(OSC_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));        \
    } while (0)

// ---------------------------------------------------------------- NCCL (dlopen)
// NCCL is resolved at run time so a single-GPU context never needs it and the
// process uses whichever libnccl.so.2 is already loaded (e.g. torch's).
namespace nccl {
typedef struct ncclComm* Comm;
struct UniqueId {
    char internal[128];
};
typedef int (*GetUniqueIdFn)(UniqueId*);
typedef int (*CommInitRankFn)(Comm*, int, UniqueId, int);
typedef int (*AllGatherFn)(const void*, void*, size_t, int, Comm, cudaStream_t);
typedef int (*CommDestroyFn)(Comm);
typedef const char* (*GetErrorStringFn)(int);
constexpr int kFloat64 = 8;  // ncclFloat64 (nccl.h)

struct Api {
    void* h = nullptr;
    GetUniqueIdFn get_unique_id = nullptr;
    CommInitRankFn comm_init_rank = nullptr;
    AllGatherFn all_gather = nullptr;
    CommDestroyFn comm_destroy = nullptr;
    GetErrorStringFn error_string = nullptr;
};

Api& api() {
    static Api a;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (a.h) break;
        }
        if (!a.h) return;
        a.get_unique_id = (GetUniqueIdFn)dlsym(a.h, "ncclGetUniqueId");
        a.comm_init_rank = (CommInitRankFn)dlsym(a.h, "ncclCommInitRank");
        a.all_gather = (AllGatherFn)dlsym(a.h, "ncclAllGather");
        a.comm_destroy = (CommDestroyFn)dlsym(a.h, "ncclCommDestroy");
        a.error_string = (GetErrorStringFn)dlsym(a.h, "ncclGetErrorString");
    });
    if (!a.h || !a.get_unique_id || !a.comm_init_rank || !a.all_gather)
        throw Error(OSC_ERR_PARALLEL, "NCCL (libnccl.so.2) is not loadable");
    return a;
}

void check(int rc, const char* what) {
    if (rc != 0)
        throw Error(OSC_ERR_PARALLEL, std::string(what) + ": " +
                                          (api().error_string ? api().error_string(rc) : "nccl error"));
}
}  // namespace nccl

// ------------------------------------------------------------------ kernels
using StageFn = void (*)(StepArgs);

template <int MODEL>
StageFn stage_fn(int stage, int schedule) {
    switch (stage) {
        case 0: return k_stage<MODEL, 0>;
        case 2: return k_stage<MODEL, 2>;
        case 3: return k_stage<MODEL, 3>;
        default: return schedule == 1 ? k_stage<MODEL, 4, 1> : k_stage<MODEL, 4, 0>;
    }
}
template <int MODEL>
StageFn stage3_fn(int stage) {
    switch (stage) {
        case 0: return k_stage3<MODEL, 0>;
        case 2: return k_stage3<MODEL, 2>;
        case 3: return k_stage3<MODEL, 3>;
        default: return k_stage3<MODEL, 4>;
    }
}
StageFn finalize_fn(int model) {
    switch (model) {
        case 0: return k_finalize<0>;
        case 1: return k_finalize<1>;
        case 2: return k_finalize<2>;
        case 3: return k_finalize<3>;
        default: return k_finalize<4>;
    }
}
using ResidentFn = void (*)(StepArgs, int, int, int, double*, unsigned*);
ResidentFn resident_kernel(int model) {
    switch (model) {
        case 0: return k_resident<0>;
        case 1: return k_resident<1>;
        case 2: return k_resident<2>;
        case 3: return k_resident<3>;
        default: return k_resident<4>;
    }
}

StageFn stage_kernel(int nflav, int model, int stage, int schedule = 1) {
    if (nflav == 3) return model == 0 ? stage3_fn<0>(stage) : stage3_fn<1>(stage);
    switch (model) {
        case 0: return stage_fn<0>(stage, schedule);
        case 1: return stage_fn<1>(stage, schedule);
        case 2: return stage_fn<2>(stage, schedule);
        case 3: return stage_fn<3>(stage, schedule);
        default: return stage_fn<4>(stage, schedule);
    }
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { free(); }
    void alloc(size_t count) {
        free();
        if (count == 0) count = 1;
        CUDA_OK(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void free() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

}  // namespace oscb200

using namespace oscb200;

// The dynamic shared-memory limit is a per-kernel, process-wide attribute:
// always set it to the most the kernel can take (the opt-in maximum less its
// static shared memory), so a smaller context created later can never lower
// it under a larger one's launches.
template <class F>
void set_max_dynamic_smem(F* fn, int device) {
    int optin = 0;
    CUDA_OK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    cudaFuncAttributes fa{};
    CUDA_OK(cudaFuncGetAttributes(&fa, fn));
    CUDA_OK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes));
}

#ifndef OSC_CR
#define OSC_CR 1  // single GPU: consumer-side reduction of the stage partials (k_finalize per batch)
#endif
#ifndef OSC_EARLY_PDL
#define OSC_EARLY_PDL 1  // one-wave grids release the next stage at their main loop's start
#endif
#ifndef OSC_GRID_WAVES
#define OSC_GRID_WAVES 1  // waves of stage-kernel blocks (2: half-size chunks, SMs that finish early take more)
#endif
#ifndef OSC_GRAPH_STEPS
#define OSC_GRAPH_STEPS 8  // steps per captured CUDA graph (stage kernels)
#endif

struct OscCtx {
    OscDesc desc{};
    int rank = 0, nranks = 1, device = 0;
    bool coll = false;  // multi-rank exchange path (nranks > 1, or forced for testing)
    DevBuf<unsigned long long> xll;    // device-initiated exchange receive buffer [4][kMaxRanks][kLLWords]
    std::vector<void*> ipc_opened;     // peer mappings to close
    int t_lo = 0, t_hi = 0;
    int T = 0, P = 0, E = 0;
    int ntraj = 0, ncell = 0, npad = 0;
    int nsm = 0, nblocks = 0, chunk = 0, ntr_max = 0;
    int nblocks23 = 0, chunk23 = 0;  // S2/S3 grid (2 flavours)
    int one_wave = 0;                // all stage grids resident at once (early programmatic launch)
    int rec_stride = 0;              // trajectory record stride (0: compact)
    uint32_t e_magic = 0, e_shift = 0;
    int schedule = 1;  // 1: S3 stashes propagators for S4 (default), 0: S4 recomputes them
    int nflav = 2;
    int nplanes = 16;  // state planes per buffer
    DevBuf<double> vac3;
    int use_pdl = 1;
    int resident_ok = 0;  // the whole state fits in shared memory (k_resident)
    int launch_mode = 0;  // 0 stage kernels + graphs, 2 resident
    int rch = 0, rntr = 0;
    size_t rsmem = 0;
    DevBuf<double> rpart;
    DevBuf<unsigned> rbar;
    unsigned long long nlaunch = 0;  // kernels this context launched
    bool capturing = false;
    int graph_kernels = 0;
    void count(int k = 1) {
        if (capturing) graph_kernels += k;
        else nlaunch += k;
    }
    cudaStream_t stream = nullptr;
    nccl::Comm comm = nullptr;
    // In-process group (osc_create_group: Engine lanes mapped onto GPUs, one
    // context per rank, one host thread): a group handle owns its ranks in
    // `kids`; `ordered` selects the stream-ordered exchange (rank slots copied
    // between the ranks' exchange buffers behind cross-stream events: any
    // device placement, several ranks per GPU included) instead of the
    // device-initiated one over peer pointers (distinct GPUs).
    std::vector<OscCtx*> kids;
    int ordered = 0;
    bool in_group = false;  // (a rank of a group: the group drives its exchange)
    std::vector<cudaEvent_t> gev;
    std::vector<cudaEvent_t> xev;  // chunked host transfers (set/get_state)

    DevBuf<double> cos2, sin0, cphi, sphi, vac11, vac12, g, ktab_g;
    DevBuf<double> cpart[4];  // single GPU: block partials of S2, S3, S4 (consumer-side reduction)
    DevBuf<double> psi[2], bloch[2], stash, ustash, xbuf, xsend, partials, staging;
    // snapshot I/O: spectrum weights [nsp][E] (mode 2), mode-2 output, the
    // second packing buffer and pinned host buffers of the async dumps
    DevBuf<double> fw, mode2buf, staging2;
    cudaStream_t copy_stream = nullptr;
    double* pinned[2] = {nullptr, nullptr};
    size_t pinned_n = 0;
    // control block pair (StepArgs::ctl_out): `par` names the current one;
    // single-GPU stage kernels flip it at every S2
    DevBuf<Ctl> ctl;
    int par = 0;
    Ctl* ctl_cur() const { return ctl.p + par; }
    bool flips() const { return args.cr || args.cr3; }
    DevBuf<unsigned long long> scratch;
    Ctl* h_ctl = nullptr;  // pinned mirror
    // the class Bloch planes of psi0 no longer match it (set_state, a
    // resident batch): the stage kernels rerun S1 before their next step
    bool bloch_stale = false;

    StepArgs args{};
    cudaGraphExec_t graph[2] = {nullptr, nullptr};  // by the control parity at launch
    int graph_steps = 0;
    void drop_graphs() {
        for (auto& g : graph)
            if (g) {
                cudaGraphExecDestroy(g);
                g = nullptr;
            }
    }

    ~OscCtx() {
        for (OscCtx* k : kids) delete k;
        for (cudaEvent_t e : gev) cudaEventDestroy(e);
        for (double*& p : pinned)
            if (p) cudaFreeHost(p);
        if (!kids.empty()) return;  // (a group handle owns no device buffers)
        cudaSetDevice(device);  // (a group's ranks live on several devices)
        for (cudaEvent_t e : xev) cudaEventDestroy(e);
        drop_graphs();
        if (comm) {
            try {
                nccl::api().comm_destroy(comm);
            } catch (...) {
            }
        }
        for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
        if (h_ctl) cudaFreeHost(h_ctl);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (stream) cudaStreamDestroy(stream);
    }

    // Stage kernels are launched with programmatic dependent launch so each
    // one is scheduled while its predecessor drains (griddepcontrol in the
    // kernels orders the dependent reads).
    void launch_stage(int stage) {
        const StageFn fn = stage_kernel(nflav, desc.model, stage, schedule);
        StepArgs la = args;  // (args.ctl == args.ctl_out == the current control block)
        if (stage == 2 && flips()) {
            // S2 reads the current control block and writes the advanced one
            // into the other buffer, which becomes current
            la.ctl_out = ctl.p + (par ^ 1);
            set_par(par ^ 1);
        }
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((nflav == 2 && (stage == 2 || stage == 3)) ? nblocks23 : nblocks);
        cfg.blockDim = dim3(nflav == 3 ? kBlock3 : kBlock);
        cfg.dynamicSmemBytes = nflav == 3 ? stage3_smem_bytes(ntr_max, stage, args.uf_cols) : stage_smem_bytes(stage, schedule, ntr_max, E, rec_stride);
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = use_pdl ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CUDA_OK(cudaLaunchKernelEx(&cfg, fn, la));
        count();
    }

    // Single GPU: the control update of the last step of a batch (its S4
    // partials are otherwise consumed by the next step's S2).
    void finalize() {
        if (!args.cr && !args.cr3) return;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(1);
        cfg.blockDim = dim3(args.cr3 ? kBlock3 : kBlock);
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = use_pdl ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CUDA_OK(cudaLaunchKernelEx(&cfg, args.cr3 ? (desc.model == 0 ? k_finalize3<0> : k_finalize3<1>)
                                                   : finalize_fn(desc.model),
                                   args));
        count();
    }

    void exchange(int slot) {
        if (!coll || args.p2p || in_group) return;
        nccl::check(nccl::api().all_gather(xsend.p + (size_t)slot * kSlotDoubles,
                                           xbuf.p + (size_t)slot * nranks * kSlotDoubles, kSlotDoubles,
                                           nccl::kFloat64, comm, stream),
                    "ncclAllGather");
    }

    // One evolution step = S2, S3, S4 (+ exchange after each; control fused
    // into S4's last block on a single GPU).
    void enqueue_step() {
        launch_stage(2);
        exchange(1);
        launch_stage(3);
        exchange(2);
        launch_stage(4);
        exchange(3);
        if (coll && !args.p2p) {  // (device-initiated exchange: fused into S4)
            k_control<<<1, 128, 0, stream>>>(args);
            count();
            CUDA_OK(cudaGetLastError());
        }
    }

    void enqueue_moments0() {
        launch_stage(0);
        exchange(0);
    }

    // A graph of `steps` (even) steps for the current control parity,
    // instantiated and uploaded (so its first launch costs no setup).
    cudaGraphExec_t get_graph(int steps) {
        cudaGraphExec_t& gx = graph[par];
        if (gx) return gx;
        const int par0 = par;
        cudaGraph_t g_ = nullptr;
        CUDA_OK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
        capturing = true;
        graph_kernels = 0;
        for (int i = 0; i < steps; ++i) enqueue_step();
        capturing = false;
        CUDA_OK(cudaStreamEndCapture(stream, &g_));
        if (par != par0) throw Error(OSC_ERR_CUDA, "graph: odd number of control flips");
        CUDA_OK(cudaGraphInstantiate(&gx, g_, 0));
        cudaGraphDestroy(g_);
        CUDA_OK(cudaGraphUpload(gx, stream));
        graph_steps = steps;
        return gx;
    }
    // Build (and upload) the step graphs of both parities now, outside any
    // timed region.
    void prepare_graphs() {
        if (launch_mode != 0) return;
        get_graph(OSC_GRAPH_STEPS);
        if (!flips()) return;
        set_par(par ^ 1);  // (host side only: nothing is launched)
        get_graph(OSC_GRAPH_STEPS);
        set_par(par ^ 1);
    }
    void set_par(int p) {
        par = p;
        args.ctl = args.ctl_out = ctl_cur();
    }

    // n steps in one cooperative launch with the state resident in shared
    // memory (single GPU, small problems).
    void launch_resident(int n) {
        CUDA_OK(cudaMemsetAsync(rbar.p, 0, sizeof(unsigned), stream));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(nsm);
        cfg.blockDim = dim3(kBlock);
        cfg.dynamicSmemBytes = rsmem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CUDA_OK(cudaLaunchKernelEx(&cfg, resident_kernel(desc.model), args, n, rch, rntr, rpart.p, rbar.p));
        count();
    }

    void enqueue_steps(int n) {
        if (n <= 0) return;
        if (launch_mode == 2) {
            launch_resident(n);
            bloch_stale = true;  // (the resident kernel keeps no Bloch planes)
            return;
        }
        if (bloch_stale) {  // S1 rebuilds the Bloch planes (and sums0) of psi0
            enqueue_moments0();
            bloch_stale = false;
        }
        if (n >= OSC_GRAPH_STEPS) {
            cudaGraphExec_t gx = get_graph(OSC_GRAPH_STEPS);
            for (; n >= OSC_GRAPH_STEPS; n -= OSC_GRAPH_STEPS) {
                CUDA_OK(cudaGraphLaunch(gx, stream));
                nlaunch += graph_kernels;
            }
        }
        for (; n > 0; --n) enqueue_step();
        finalize();
    }

    void download_ctl() {
        CUDA_OK(cudaMemcpyAsync(h_ctl, ctl_cur(), sizeof(Ctl), cudaMemcpyDeviceToHost, stream));
        CUDA_OK(cudaStreamSynchronize(stream));
    }
    void upload_ctl() {
        CUDA_OK(cudaMemcpyAsync(ctl_cur(), h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, stream));
        CUDA_OK(cudaStreamSynchronize(stream));
    }

    void raise_device_status() {
        if (!h_ctl->status) return;
        const std::string where = " at r = " + std::to_string(h_ctl->r) + " km, iteration " +
                                  std::to_string(h_ctl->iter);
        switch (h_ctl->reason) {
            case 1: throw Error(OSC_ERR_NUMERIC, "non-finite amplitudes" + where);
            case 2: throw Error(OSC_ERR_NUMERIC, "non-finite Hamiltonian sum" + where);
            case 3: throw Error(OSC_ERR_NUMERIC, "step collapse: rejected step would need dr < min_dr" + where);
            default: throw Error(OSC_ERR_NUMERIC, "device numeric failure" + where);
        }
    }

    void check_radius(double r) const {
        if (desc.model != OSC_MODEL_SINGLE_ANGLE && desc.model != OSC_MODEL_PLANE && r < desc.Rnu)
            throw Error(OSC_ERR_NUMERIC, "fill_cache: r below the neutrino sphere");
        if (desc.matter_profile != OSC_MATTER_OFF && r < desc.Rnu)
            throw Error(OSC_ERR_NUMERIC, "baryon_density: r below the neutrino sphere");
    }

    // Arm the device control block like Engine::run's first packet
    // (solver.cpp:492-500).
    void begin(const OscStepControl& c, int commit) {
        begin_ctl(c, commit);
        if (!h_ctl->terminate) {
            check_radius(c.r);
            enqueue_moments0();
            bloch_stale = false;
        }
    }
    // The control block part of begin (no launches).
    void begin_ctl(const OscStepControl& c, int commit) {
        download_ctl();
        Ctl& h = *h_ctl;
        h.r = c.r;
        h.dr = commit ? std::min(c.dr, std::max(0.0, c.Rn - c.r)) : c.dr;
        h.iter = c.iter;
        h.accepted = h.rejected = 0;
        h.err = 0.0;
        h.status = h.reason = 0;
        h.bad_sums = 0;
        h.pend = 0;
        h.dump_mask = 0;  // snapshot gates are armed by osc_run_dumps only
        h.pause = 0;
        h.nstep += 1;  // (exchange tags never repeat across runs)
        h.commit = commit;
        h.dr_max = c.dr_max;
        h.dr_min = c.dr_min;
        h.eps0 = c.eps0;
        h.kappa = c.kappa;
        h.Rn = c.Rn;
        h.Ts = commit ? c.Ts : 0;
        std::memset(h.counter, 0, sizeof h.counter);
        const double r_eps = 1e-12 * std::max(1.0, std::fabs(c.Rn));
        h.terminate = 0;
        if (commit) {
            if (c.r >= c.Rn - r_eps) h.terminate = 1;
            if (c.Ts > 0 && c.iter >= c.Ts) h.terminate = 2;
        }
        upload_ctl();
    }
};

static void enable_mr_cr(OscCtx* c);

namespace {

// DFMA-chain microkernel for the FP64 roofline denominator: 8 independent
// dependency chains per thread keep the FP64 pipe saturated.
__global__ void k_dfma_peak(double* out, int iters, double y, double z) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-7 + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], y, z);
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) out[0] = s;  // keep the chains live
}

// flavor::evolve_bin (beam.hpp:105-121) through the production propagator
// code: path 0 = make_props_n (branch-free chain, one fallback branch that
// redoes the cell with the libdevice paths), 1 = the safe path only.  One
// beam Hamiltonian per item: class 0 of CellK{v11 = v12 = 0} with hb = h.
__global__ void k_debug_evolve(int n, const double* h, const double* dl, const double* psi, double* out, int path) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    CellK K{};
    const double hb[3] = {h[3 * i], h[3 * i + 1], h[3 * i + 2]};
    Prop u[2];
    if (path == 0) {
        const PropReq rq[1] = {{hb, dl[i], false, u}};
        make_props_n(K, rq);
    } else {
        make_props_safe(K, hb, dl[i], false, u[0], u[1]);
    }
    const double x[4] = {psi[4 * i], psi[4 * i + 1], psi[4 * i + 2], psi[4 * i + 3]};
    double y[4];
    apply(u[0], x, y);
    for (int k = 0; k < 4; ++k) out[4 * i + k] = y[k];
}

// exp(-i H tau) of 3x3 Hermitian matrices through the device code of the
// 3-flavour stages (su3_exp.cuh): path 0 = exp_herm3, 1 = eig_herm3 +
// exp_from_eig (S2's shared decomposition).  H [n][9] packed (d0 d1 d2, re/im
// of h01, h02, h12), U [n][18] row-major re/im.
__global__ void k_debug_exp3(int n, const double* H, const double* tau, double* U, int path) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Herm3 h;
    for (int k = 0; k < 3; ++k) h.d[k] = H[9 * i + k];
    h.o01 = Cx{H[9 * i + 3], H[9 * i + 4]};
    h.o02 = Cx{H[9 * i + 5], H[9 * i + 6]};
    h.o12 = Cx{H[9 * i + 7], H[9 * i + 8]};
    const Mat3 u = path == 0 ? exp_herm3(h, tau[i]) : exp_from_eig(eig_herm3(h), tau[i]);
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            U[18 * i + (r * 3 + c) * 2] = u.m[r][c].re;
            U[18 * i + (r * 3 + c) * 2 + 1] = u.m[r][c].im;
        }
}

void validate(const OscDesc* d) {
    if (!d) throw Error(OSC_ERR_CONFIG, "osc_create: null desc");
    if (d->model < 0 || d->model > 4) throw Error(OSC_ERR_CONFIG, "osc_create: bad model");
    if (d->abins < 1 || d->pbins < 1 || d->ebins < 1)
        throw Error(OSC_ERR_CONFIG, "osc_create: Abins, Pbins, Ebins must be >= 1");
    if (d->model == OSC_MODEL_SINGLE_ANGLE && (d->abins != 1 || d->pbins != 1))
        throw Error(OSC_ERR_CONFIG, "single-angle model needs abins = pbins = 1");
    if (d->model == OSC_MODEL_BULB && d->pbins != 1)
        throw Error(OSC_ERR_CONFIG, "bulb model needs pbins = 1");
    if (d->nflav != 0 && d->nflav != 2 && d->nflav != 3)
        throw Error(OSC_ERR_CONFIG, "osc_create: only 2 or 3 flavours are supported");
    if (d->nflav == 3 && (d->model > OSC_MODEL_BULB || !d->vac3 || !d->fw6))
        throw Error(OSC_ERR_CONFIG, "3 flavours: single-angle / bulb models with vac3 and fw6 tables");
    if (!d->cos2_theta0 || !d->sin_theta0 || !d->cos_phi || !d->sin_phi || !d->vac_h11 ||
        !d->vac_h12 || !d->fw)
        throw Error(OSC_ERR_CONFIG, "osc_create: null table");
    if (d->matter_profile < 0 || d->matter_profile > 3)
        throw Error(OSC_ERR_CONFIG, "osc_create: bad matter profile");
}

template <class T>
void upload(DevBuf<T>& b, const T* src, size_t n) {
    b.alloc(n);
    CUDA_OK(cudaMemcpy(b.p, src, n * sizeof(T), cudaMemcpyHostToDevice));
}

}  // namespace

extern "C" {

const char* osc_last_error(void) { return g_last_error.c_str(); }
int osc_version(void) { return 1; }

int osc_comm_unique_id(void* out128) {
    return guarded([&] {
        nccl::UniqueId id;
        nccl::check(nccl::api().get_unique_id(&id), "ncclGetUniqueId");
        std::memcpy(out128, &id, sizeof id);
    });
}

int osc_create(const OscDesc* desc, const OscComm* comm, OscCtx** out) {
    return guarded([&] {
        validate(desc);
        if (!out) throw Error(OSC_ERR_CONFIG, "osc_create: null out");
        auto c = std::make_unique<OscCtx>();
        c->desc = *desc;
        c->rank = comm ? comm->rank : 0;
        c->nranks = comm ? comm->nranks : 1;
        c->coll = c->nranks > 1 || (comm && (comm->flags & OSC_COMM_FORCE_COLLECTIVES));
        c->device = comm ? comm->device : 0;
        if (c->nranks < 1 || c->nranks > kMaxRanks || c->rank < 0 || c->rank >= c->nranks)
            throw Error(OSC_ERR_CONFIG, "osc_create: bad rank / nranks");
        if (desc->model == OSC_MODEL_SINGLE_ANGLE && c->nranks != 1)
            throw Error(OSC_ERR_CONFIG, "single-angle model does not support multiple workers");
        if (c->nranks > desc->abins) throw Error(OSC_ERR_CONFIG, "Engine: more lanes than theta bins");
        CUDA_OK(cudaSetDevice(c->device));
        int major = 0;
        CUDA_OK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, c->device));
        if (major < 10) throw Error(OSC_ERR_CUDA, "oscflat_b200 needs an sm_100 (Blackwell) GPU");
        CUDA_OK(cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, c->device));
        CUDA_OK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));

        // theta partition: make_partitions (parallel.cpp:11-24)
        const int base = desc->abins / c->nranks, extra = desc->abins % c->nranks;
        c->t_lo = c->rank * base + std::min(c->rank, extra);
        c->t_hi = c->t_lo + base + (c->rank < extra ? 1 : 0);
        c->T = desc->abins;
        c->P = desc->pbins;
        c->E = desc->ebins;
        c->ntraj = (c->t_hi - c->t_lo) * c->P;
        c->ncell = c->ntraj * c->E;
        c->npad = (c->ncell + 31) / 32 * 32;

        upload(c->cos2, desc->cos2_theta0, c->T);
        upload(c->sin0, desc->sin_theta0, c->T);
        upload(c->cphi, desc->cos_phi, c->P);
        upload(c->sphi, desc->sin_phi, c->P);
        upload(c->vac11, desc->vac_h11, c->E);
        upload(c->vac12, desc->vac_h12, c->E);
        c->nflav = desc->nflav == 3 ? 3 : 2;
        c->nplanes = c->nflav == 3 ? 36 : 16;
        const int nsp = c->nflav == 3 ? 6 : 4;
        const double* fw = c->nflav == 3 ? desc->fw6 : desc->fw;
        const double* cpl = c->nflav == 3 ? desc->couplings6 : desc->couplings;
        std::vector<double> g(nsp * static_cast<size_t>(c->E));
        for (int s = 0; s < nsp; ++s)
            for (int e = 0; e < c->E; ++e)
                g[(size_t)s * c->E + e] = ((s & 1) ? -1.0 : 1.0) * cpl[s] * fw[(size_t)s * c->E + e];
        upload(c->g, g.data(), g.size());
        if (c->nflav == 2) {  // contiguous per-energy table for the stage kernels' bulk copy
            std::vector<double> kt((size_t)((6 * c->E + 1) & ~1), 0.0);
            for (int e = 0; e < c->E; ++e) {  // [E][6]: v11, v12, g0..g3 (three 16-byte loads per cell)
                kt[6 * (size_t)e] = desc->vac_h11[e];
                kt[6 * (size_t)e + 1] = desc->vac_h12[e];
                for (int s = 0; s < 4; ++s) kt[6 * (size_t)e + 2 + s] = g[(size_t)s * c->E + e];
            }
            upload(c->ktab_g, kt.data(), kt.size());
        }
        upload(c->fw, fw, (size_t)nsp * c->E);
        if (c->nflav == 3) upload(c->vac3, desc->vac3, 9 * (size_t)c->E);
        const size_t plane = (size_t)c->npad * c->nplanes;
        c->psi[0].alloc(plane);
        c->psi[1].alloc(plane);
        CUDA_OK(cudaMemset(c->psi[0].p, 0, plane * sizeof(double)));
        CUDA_OK(cudaMemset(c->psi[1].p, 0, plane * sizeof(double)));
        if (c->nflav == 2)
            for (auto& b : c->bloch) {
                b.alloc((size_t)c->npad * kBlochPlanes);
                CUDA_OK(cudaMemset(b.p, 0, b.n * sizeof(double)));
            }
        c->xbuf.alloc((size_t)4 * c->nranks * kSlotDoubles);
        CUDA_OK(cudaMemset(c->xbuf.p, 0, c->xbuf.n * sizeof(double)));
        c->xll.alloc((size_t)4 * kMaxRanks * kLLWords);
        CUDA_OK(cudaMemset(c->xll.p, 0, c->xll.n * sizeof(unsigned long long)));
        if (c->coll) {
            c->xsend.alloc((size_t)4 * kSlotDoubles);
            CUDA_OK(cudaMemset(c->xsend.p, 0, c->xsend.n * sizeof(double)));
        }
        c->ctl.alloc(2);
        CUDA_OK(cudaMemset(c->ctl.p, 0, 2 * sizeof(Ctl)));
        c->scratch.alloc(4);
        CUDA_OK(cudaMallocHost(&c->h_ctl, sizeof(Ctl)));
        std::memset(c->h_ctl, 0, sizeof(Ctl));

        // Launch geometry: one resident wave of blocks (2 per SM, the
        // __launch_bounds__ target), half of them per particle class; each
        // block owns a contiguous, warp-aligned chunk of cells.  When the
        // per-trajectory records of a chunk would push a block's shared
        // memory past what two resident blocks per SM allow (few energy bins
        // per trajectory: the cylinder model), the grid doubles (two waves of
        // half-size chunks) instead of running at half occupancy.
        {
            const int occ = desc->nflav == 3 ? OSC3_MIN_BLOCKS : OSC_MIN_BLOCKS;
            int waves = OSC_GRID_WAVES;  // env OSC_GRID_WAVES overrides (tests: multi-wave grids)
            if (const char* env = std::getenv("OSC_GRID_WAVES")) waves = std::max(1, std::atoi(env));
            int nb = std::max(1, c->nsm * occ * (desc->nflav == 3 ? 1 : waves));
            for (int tries = 0;; ++tries) {
                // 3 flavours: blocks split in halves by particle class
                const int per = c->nflav == 3 ? nb / 2 : nb;
                int chunk = (c->ncell + per - 1) / per;
                chunk = std::max(32, (chunk + 31) / 32 * 32);
                c->nblocks = c->nflav == 3 ? 2 * per : nb;
                c->chunk = chunk;
                c->ntr_max = chunk / c->E + 2;
                size_t smax = 0;
                if (c->nflav == 3) {
                    smax = stage3_smem_bytes(c->ntr_max, 4);
                } else {
                    // padded record stride where two blocks per SM still fit, else compact
                    // (env OSC_REC_COMPACT=1 forces the compact stride: tests).  Models
                    // 2-4 (four geometric moments) spill a few registers at the two-
                    // blocks-per-SM budget: the compact stride leaves L1 more room for
                    // them (configs[3]: 129.9 -> 125.4 us/step; configs[2], model 1,
                    // no spills: padded 118.0 vs compact 118.9)
                    const char* rc_env = std::getenv("OSC_REC_COMPACT");
                    const bool force_compact = (rc_env && std::atoi(rc_env) == 1) || desc->model >= OSC_MODEL_EXT_BULB;
                    for (int stride : {kRecStridePadded, 0}) {
                        if (force_compact && stride) continue;
                        smax = 0;
                        for (int st : {0, 2, 3, 4})
                            for (int sch : {0, 1})
                                smax = std::max(smax, stage_smem_bytes(st, sch, c->ntr_max, c->E, stride));
                        c->rec_stride = stride;
                        int per_sm = 0;
                        set_max_dynamic_smem(stage_kernel(2, desc->model, 4, 1), c->device);
                        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                            &per_sm, stage_kernel(2, desc->model, 4, 1), kBlock, std::min<size_t>(smax, 227 * 1024)));
                        if (per_sm >= occ) break;
                    }
                }
                if (smax > 200 * 1024)
                    throw Error(OSC_ERR_CONFIG, "osc_create: trajectory records exceed shared memory");
                for (int st : {0, 2, 3, 4})
                    for (int sch : {0, 1}) set_max_dynamic_smem(stage_kernel(c->nflav, desc->model, st, sch), c->device);
                if (c->nflav == 3 || tries >= 3 || chunk <= 32 * 32) break;
                int per_sm = 0;
                CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stage_kernel(2, desc->model, 4, 1),
                                                                      kBlock, smax));
                if (per_sm >= occ) break;
                nb *= 2;
            }
            // magic numbers for the division by E inside the kernels
            uint32_t l = 0;
            while ((1u << l) < (uint32_t)c->E) ++l;
            c->e_shift = l;
            c->e_magic = (uint32_t)((((uint64_t)1 << 32) * (((uint64_t)1 << l) - (uint64_t)c->E)) / (uint64_t)c->E + 1);
        }
        // S2/S3 (2 flavours): their own occupancy target, in proportion to
        // the grid above (cells per block shrink; the records still fit)
        c->nblocks23 = c->nblocks;
        c->chunk23 = c->chunk;
        if (c->nflav == 2 && OSC_MIN_BLOCKS_S23 != OSC_MIN_BLOCKS) {
            const int nb23 = c->nblocks / OSC_MIN_BLOCKS * OSC_MIN_BLOCKS_S23;
            int ch = (c->ncell + nb23 - 1) / nb23;
            c->chunk23 = std::max(32, (ch + 31) / 32 * 32);
            c->nblocks23 = nb23;
        }
        c->partials.alloc((size_t)std::max(c->nblocks, c->nblocks23) * kSlotDoubles);
        // early dependent launch needs every stage grid resident at once
        if (c->nflav == 2 && OSC_EARLY_PDL) {
            int ok = 1;
            for (int st : {0, 2, 3, 4})
                for (int sch : {0, 1}) {
                    int per = 0;
                    const size_t sm = stage_smem_bytes(st, sch, c->ntr_max, c->E, c->rec_stride);
                    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, stage_kernel(2, desc->model, st, sch),
                                                                          kBlock, sm));
                    const int nb = (st == 2 || st == 3) ? c->nblocks23 : c->nblocks;
                    if ((long long)per * c->nsm < nb) ok = 0;
                }
            c->one_wave = ok;
        }
        if (!c->coll && c->nflav == 3 && OSC_CR)
            for (int k = 1; k < 4; ++k) {
                c->cpart[k].alloc((size_t)c->nblocks * (2 * kNM3Max + 1));
                CUDA_OK(cudaMemset(c->cpart[k].p, 0, c->cpart[k].n * sizeof(double)));
            }
        if (c->nflav == 2)  // (multi-rank contexts reduce consumer-side once the peers are connected)
            for (int k = 1; k < 4; ++k) {
                c->cpart[k].alloc((size_t)std::max(c->nblocks, c->nblocks23) * (2 * 12 + 1));
                CUDA_OK(cudaMemset(c->cpart[k].p, 0, c->cpart[k].n * sizeof(double)));
            }

        // resident kernel: single GPU, 2 flavours
        if (!c->coll && c->nflav == 2) {
            // resident: the local state, the result and the stash of a chunk
            // per SM in shared memory
            c->rch = (c->ncell + c->nsm - 1) / c->nsm;
            c->rntr = c->rch / c->E + 2;
            c->rsmem = resident_smem_bytes(c->rch, c->rntr, c->E);
            if (c->rsmem <= 200 * 1024) {
                const ResidentFn rf = resident_kernel(desc->model);
                set_max_dynamic_smem(rf, c->device);
                int rper = 0;
                CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rper, rf, kBlock, c->rsmem));
                if (rper >= 1) {
                    c->resident_ok = 1;
                    c->rpart.alloc((size_t)2 * c->nsm * kSlotDoubles);
                    c->rbar.alloc(1);
                }
            }
            // default: resident where the state fits, else the PDL-pipelined
            // stage kernels; env OSC_LAUNCH=0/2 overrides
            c->launch_mode = c->resident_ok ? 2 : 0;
            if (const char* env = std::getenv("OSC_LAUNCH")) {
                const int m = std::atoi(env);
                if (m == 0 || (m == 2 && c->resident_ok)) c->launch_mode = m;
            }
        }

        if (c->coll && !(comm->flags & OSC_COMM_GROUP)) {
            nccl::UniqueId id;
            if (comm->nccl_unique_id) {
                std::memcpy(&id, comm->nccl_unique_id, sizeof id);
            } else {
                if (c->nranks > 1) throw Error(OSC_ERR_PARALLEL, "osc_create: missing NCCL unique id");
                nccl::check(nccl::api().get_unique_id(&id), "ncclGetUniqueId");
            }
            nccl::check(nccl::api().comm_init_rank(&c->comm, c->nranks, id, c->rank), "ncclCommInitRank");
        }

        StepArgs& a = c->args;
        a.model = desc->model;
        a.P = c->P;
        a.E = c->E;
        a.t_lo = c->t_lo;
        a.T_loc = c->t_hi - c->t_lo;
        a.T_glob = c->T;
        a.ntraj = c->ntraj;
        a.ncell = c->ncell;
        a.npad = c->npad;
        a.chunk = c->chunk;
        a.chunk23 = c->chunk23;
        a.ntr_max = c->ntr_max;
        a.nranks = c->nranks;
        a.fuse_ctl = !c->coll;
        a.cr = (!c->coll && c->nflav == 2 && OSC_CR) ? 1 : 0;
        a.cr3 = (!c->coll && c->nflav == 3 && OSC_CR) ? 1 : 0;
        a.nblocks = c->nblocks;
        a.nblocks23 = c->nblocks23;
        a.one_wave = c->one_wave;
        a.rec_stride = c->rec_stride;
        for (int k = 0; k < 4; ++k) a.cpart[k] = c->cpart[k].p;
        a.e_magic = c->e_magic;
        a.e_shift = c->e_shift;
        a.schedule = c->schedule;
        // 3 flavours: S4's U1 columns where the block's shared memory still holds them
        a.uf_cols = c->nflav == 3 && stage3_smem_bytes(c->ntr_max, 4, 1) <= 200 * 1024;
        c->stash.alloc((size_t)c->npad * (c->nflav == 3 ? kSt3Planes : c->nplanes));
        if (c->nflav == 2) c->ustash.alloc((size_t)c->npad * kUPlanes);
        a.Rnu = desc->Rnu;
        a.dcos2 = 1.0 / c->T;
        a.phi_measure = desc->model >= OSC_MODEL_EXT_BULB ? 1.0 / c->P : 1.0;
        // plane: w = dcos / P;  cylinder: w = (R/rho)(cos a0/cos a) (da0 / pi) / P
        a.wscale = desc->model == OSC_MODEL_PLANE ? 1.0 / ((double)c->T * c->P)
                   : desc->model == OSC_MODEL_CYLINDER ? 1.0 / ((double)c->T * c->P)
                                                        : 0.0;
        a.cos2 = c->cos2.p;
        a.sin0 = c->sin0.p;
        a.cphi = c->cphi.p;
        a.sphi = c->sphi.p;
        a.vac11 = c->vac11.p;
        a.vac12 = c->vac12.p;
        a.g = c->g.p;
        a.ktab = c->ktab_g.p;
        a.vac3 = c->vac3.p;
        a.nmom = c->nflav == 3 ? 36 : 12;
        a.nplanes = c->nplanes;
        a.matter_profile = desc->matter_profile;
        a.Ye = desc->Ye;
        a.nb0 = desc->nb0;
        a.hNS = desc->hNS;
        a.Mns = desc->Mns;
        a.gs = desc->gs;
        a.S = desc->S;
        a.psi0_buf[0] = c->psi[0].p;
        a.psi0_buf[1] = c->psi[1].p;
        a.bloch_buf[0] = c->bloch[0].p;
        a.bloch_buf[1] = c->bloch[1].p;
        a.stash = c->stash.p;
        a.ustash = c->ustash.p;
        a.xbuf = c->xbuf.p;
        a.xsend = c->coll ? c->xsend.p : c->xbuf.p;
        a.p2p = 0;
        a.rank = c->rank;
        a.xll = c->xll.p;
        a.partials = c->partials.p;
        a.ctl = a.ctl_out = c->ctl_cur();
        a.ll_timeout_ns = 10000000000ll;  // 10 s
        if (const char* env = std::getenv("OSC_LL_TIMEOUT_S")) a.ll_timeout_ns = (long long)(std::atof(env) * 1e9);
        CUDA_OK(cudaDeviceSynchronize());
        *out = c.release();
    });
}

}  // extern "C"

// ------------------------------------------------------------------ groups
// Every entry point below accepts either one context or a group handle
// (osc_create_group); `ranks_of` lists the contexts that hold state.
namespace {

std::vector<OscCtx*> ranks_of(OscCtx* c) { return c->kids.empty() ? std::vector<OscCtx*>{c} : c->kids; }
std::vector<const OscCtx*> ranks_of(const OscCtx* c) {
    if (c->kids.empty()) return {c};
    return std::vector<const OscCtx*>(c->kids.begin(), c->kids.end());
}
void use(const OscCtx* c) { CUDA_OK(cudaSetDevice(c->device)); }
size_t local_doubles(const OscCtx* c) { return (size_t)c->ncell * c->nplanes; }
size_t total_doubles(const OscCtx* c) {
    size_t n = 0;
    for (const OscCtx* k : ranks_of(c)) n += local_doubles(k);
    return n;
}
size_t mode2_local(const OscCtx* c) { return (size_t)c->ntraj * (c->nflav == 3 ? 6 : 4); }
size_t mode2_total(const OscCtx* c) {
    size_t n = 0;
    for (const OscCtx* k : ranks_of(c)) n += mode2_local(k);
    return n;
}
// rank 0's control block (every rank holds the same decisions)
Ctl& hctl(OscCtx* c) { return *ranks_of(c)[0]->h_ctl; }

// Stream-ordered exchange of slot `slot` (the group's replacement of the
// NCCL all-gather): every rank's rank slot (xsend, written by its stage's
// last block) is copied into every rank's exchange buffer at [slot][q],
// behind an event of the producing rank's stream.
void ordered_exchange(OscCtx* g, int slot) {
    const int n = (int)g->kids.size();
    for (int q = 0; q < n; ++q) {
        use(g->kids[q]);
        CUDA_OK(cudaEventRecord(g->gev[q], g->kids[q]->stream));
    }
    for (int r = 0; r < n; ++r) {
        OscCtx* k = g->kids[r];
        use(k);
        for (int q = 0; q < n; ++q) {
            OscCtx* src = g->kids[q];
            if (q != r) CUDA_OK(cudaStreamWaitEvent(k->stream, g->gev[q], 0));
            CUDA_OK(cudaMemcpyPeerAsync(k->xbuf.p + ((size_t)slot * n + q) * kSlotDoubles, k->device,
                                        src->xsend.p + (size_t)slot * kSlotDoubles, src->device,
                                        kSlotDoubles * sizeof(double), k->stream));
        }
    }
}

// S1 on every rank + the slot-0 exchange.
void g_moments0(OscCtx* g) {
    if (g->kids.empty()) {
        g->enqueue_moments0();
        g->bloch_stale = false;
        return;
    }
    if (g->ordered) {
        for (OscCtx* k : g->kids) {
            use(k);
            k->launch_stage(0);
        }
        ordered_exchange(g, 0);
    } else {
        for (OscCtx* k : g->kids) {
            use(k);
            k->enqueue_moments0();
        }
    }
    for (OscCtx* k : g->kids) k->bloch_stale = false;
}

// Engine::run's first packet on every rank (+ S1 unless already terminated).
void g_begin(OscCtx* g, const OscStepControl& c, int commit) {
    if (g->kids.empty()) {
        g->begin(c, commit);
        return;
    }
    for (OscCtx* k : g->kids) {
        use(k);
        k->begin_ctl(c, commit);
    }
    if (hctl(g).terminate) return;
    g->kids[0]->check_radius(c.r);
    g_moments0(g);
}

// n steps on every rank.  Device-initiated exchange: each rank enqueues its
// own graphs (the ranks meet inside the kernels).  Stream-ordered exchange:
// stage by stage across the ranks with the exchange between stages and the
// per-rank control kernel after S4.
void g_enqueue_steps(OscCtx* g, int n) {
    if (g->kids.empty()) {
        g->enqueue_steps(n);
        return;
    }
    if (!g->ordered) {
        for (OscCtx* k : g->kids) {
            use(k);
            k->enqueue_steps(n);
        }
        return;
    }
    bool stale = false;
    for (OscCtx* k : g->kids) stale = stale || k->bloch_stale;
    if (stale && n > 0) g_moments0(g);
    for (int i = 0; i < n; ++i) {
        for (int st = 2; st <= 4; ++st) {
            for (OscCtx* k : g->kids) {
                use(k);
                k->launch_stage(st);
            }
            ordered_exchange(g, st - 1);
        }
        for (OscCtx* k : g->kids) {
            use(k);
            k_control<<<1, 128, 0, k->stream>>>(k->args);
            k->count();
            CUDA_OK(cudaGetLastError());
        }
    }
}

void g_prepare_graphs(OscCtx* g) {
    if (g->ordered) return;
    for (OscCtx* k : ranks_of(g)) {
        use(k);
        k->prepare_graphs();
    }
}

// Control blocks of every rank to the host; the first device-detected
// failure (in rank order) is raised.  Returns rank 0's copy.
Ctl& g_download(OscCtx* g) {
    for (OscCtx* k : ranks_of(g)) {
        use(k);
        k->download_ctl();
    }
    for (OscCtx* k : ranks_of(g)) k->raise_device_status();
    return hctl(g);
}

void g_sync(OscCtx* g) {
    for (OscCtx* k : ranks_of(g)) {
        use(k);
        CUDA_OK(cudaStreamSynchronize(k->stream));
    }
}

// Host transfers of the mode-1 payload in chunks of whole trajectories on the
// copy stream, each chunk's (un)packing on the compute stream overlapping
// the next chunk's copy (cross-stream events); the compute stream ends
// ordered after the last copy.
constexpr int kXferChunks = 8;
void ensure_xfer(OscCtx* c) {
    if (!c->copy_stream) CUDA_OK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    while ((int)c->xev.size() < kXferChunks + 1) {
        cudaEvent_t e;
        CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->xev.push_back(e);
    }
}
// element range of chunk k (whole trajectories)
void xfer_chunk(const OscCtx* c, int k, size_t& i0, size_t& i1) {
    const size_t per_traj = (size_t)c->E * c->nplanes;
    const size_t tpc = ((size_t)c->ntraj + kXferChunks - 1) / kXferChunks;
    i0 = std::min((size_t)c->ntraj, tpc * k) * per_traj;
    i1 = std::min((size_t)c->ntraj, tpc * (k + 1)) * per_traj;
}
bool chunked(const OscCtx* c, cudaMemcpyKind kind) {
    return kind != cudaMemcpyDeviceToDevice && kind != cudaMemcpyDefault && local_doubles(c) >= ((size_t)1 << 20) &&
           c->ntraj >= kXferChunks;
}

void set_state_local(OscCtx* c, const double* src, cudaMemcpyKind kind) {
    const size_t want = local_doubles(c);
    use(c);
    if (c->staging.n < want) c->staging.alloc(want);
    if (chunked(c, kind)) {
        ensure_xfer(c);
        CUDA_OK(cudaEventRecord(c->xev[kXferChunks], c->stream));  // staging free
        CUDA_OK(cudaStreamWaitEvent(c->copy_stream, c->xev[kXferChunks], 0));
        for (int k = 0; k < kXferChunks; ++k) {
            size_t i0, i1;
            xfer_chunk(c, k, i0, i1);
            if (i1 <= i0) continue;
            CUDA_OK(cudaMemcpyAsync(c->staging.p + i0, src + i0, (i1 - i0) * sizeof(double), kind, c->copy_stream));
            CUDA_OK(cudaEventRecord(c->xev[k], c->copy_stream));
            CUDA_OK(cudaStreamWaitEvent(c->stream, c->xev[k], 0));
            k_unpack<<<c->nsm * 8, 256, 0, c->stream>>>(c->args, c->staging.p, i0, i1);
            c->count();
        }
    } else {
        CUDA_OK(cudaMemcpyAsync(c->staging.p, src, want * sizeof(double), kind, c->stream));
        k_unpack<<<c->nsm * 8, 256, 0, c->stream>>>(c->args, c->staging.p, 0, want);
        c->count();
    }
    CUDA_OK(cudaGetLastError());
    c->bloch_stale = true;
}

void get_state_local(OscCtx* c, double* dst, cudaMemcpyKind kind) {
    const size_t want = local_doubles(c);
    use(c);
    if (c->staging.n < want) c->staging.alloc(want);
    if (chunked(c, kind)) {
        ensure_xfer(c);
        for (int k = 0; k < kXferChunks; ++k) {
            size_t i0, i1;
            xfer_chunk(c, k, i0, i1);
            if (i1 <= i0) continue;
            k_pack<<<c->nsm * 8, 256, 0, c->stream>>>(c->args, c->staging.p, i0, i1);
            c->count();
            CUDA_OK(cudaEventRecord(c->xev[k], c->stream));
            CUDA_OK(cudaStreamWaitEvent(c->copy_stream, c->xev[k], 0));
            CUDA_OK(cudaMemcpyAsync(dst + i0, c->staging.p + i0, (i1 - i0) * sizeof(double), kind, c->copy_stream));
        }
        CUDA_OK(cudaEventRecord(c->xev[kXferChunks], c->copy_stream));
        CUDA_OK(cudaStreamWaitEvent(c->stream, c->xev[kXferChunks], 0));
    } else {
        k_pack<<<c->nsm * 8, 256, 0, c->stream>>>(c->args, c->staging.p, 0, want);
        c->count();
        CUDA_OK(cudaGetLastError());
        CUDA_OK(cudaMemcpyAsync(dst, c->staging.p, want * sizeof(double), kind, c->stream));
    }
    CUDA_OK(cudaGetLastError());
}

// Whole payloads: the ranks' theta blocks are contiguous and in rank order,
// so the mode-1 payload ([traj][species][comp][ebin]) is their concatenation.
void set_state_impl(OscCtx* g, const double* src, size_t n, cudaMemcpyKind kind) {
    if (n != total_doubles(g)) throw Error(OSC_ERR_IO, "fill_mode1: payload size does not match the configured problem");
    size_t off = 0;
    for (OscCtx* k : ranks_of(g)) {
        set_state_local(k, src + off, kind);
        off += local_doubles(k);
    }
    g_sync(g);
}

void get_state_impl(OscCtx* g, double* dst, size_t n, cudaMemcpyKind kind) {
    if (n != total_doubles(g)) throw Error(OSC_ERR_IO, "extract_mode1: payload size mismatch");
    size_t off = 0;
    for (OscCtx* k : ranks_of(g)) {
        get_state_local(k, dst + off, kind);
        off += local_doubles(k);
    }
    g_sync(g);
}

}  // namespace

extern "C" {

int osc_device_count(int* n) {
    return guarded([&] {
        int c = 0;
        if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
        *n = c;
    });
}

int osc_create_group(const OscDesc* desc, int nranks, const int* devices, int flags, OscCtx** out) {
    return guarded([&] {
        validate(desc);
        if (!out) throw Error(OSC_ERR_CONFIG, "osc_create_group: null out");
        if (nranks < 1 || nranks > kMaxRanks) throw Error(OSC_ERR_CONFIG, "osc_create_group: bad rank count");
        int ndev = 0;
        CUDA_OK(cudaGetDeviceCount(&ndev));
        std::vector<int> dev(nranks);
        for (int q = 0; q < nranks; ++q) {
            dev[q] = devices ? devices[q] : q % std::max(1, ndev);
            if (dev[q] < 0 || dev[q] >= ndev) throw Error(OSC_ERR_CONFIG, "osc_create_group: bad device index");
        }
        if (nranks == 1) {
            const OscComm one{0, 1, dev[0], nullptr, 0};
            const int rc = osc_create(desc, &one, out);
            if (rc != OSC_OK) throw Error(rc, g_last_error);
            return;
        }
        auto g = std::make_unique<OscCtx>();
        g->desc = *desc;
        g->nranks = nranks;
        g->coll = true;
        g->device = dev[0];
        g->T = desc->abins;
        g->P = desc->pbins;
        g->E = desc->ebins;
        g->t_lo = 0;
        g->t_hi = desc->abins;
        g->nflav = desc->nflav == 3 ? 3 : 2;
        g->nplanes = g->nflav == 3 ? 36 : 16;
        // device-initiated exchange on request, with one rank per GPU and
        // peer access between every pair; otherwise the ordered exchange
        bool ordered = !(flags & OSC_GROUP_PEER) || (flags & OSC_GROUP_ORDERED);
        for (int a = 0; a < nranks && !ordered; ++a)
            for (int b = 0; b < nranks && !ordered; ++b) {
                if (a == b) continue;
                if (dev[a] == dev[b]) {
                    ordered = true;
                    break;
                }
                int can = 0;
                CUDA_OK(cudaDeviceCanAccessPeer(&can, dev[a], dev[b]));
                if (!can) ordered = true;
            }
        g->ordered = ordered ? 1 : 0;
        for (int q = 0; q < nranks; ++q) {
            const OscComm cm{q, nranks, dev[q], nullptr, OSC_COMM_GROUP};
            OscCtx* k = nullptr;
            const int rc = osc_create(desc, &cm, &k);
            if (rc != OSC_OK) throw Error(rc, g_last_error);
            k->in_group = true;
            g->kids.push_back(k);
            g->ntraj += k->ntraj;
            g->ncell += k->ncell;
        }
        g->gev.resize(nranks);
        for (int q = 0; q < nranks; ++q) {
            use(g->kids[q]);
            CUDA_OK(cudaEventCreateWithFlags(&g->gev[q], cudaEventDisableTiming));
        }
        if (!ordered) {
            for (int a = 0; a < nranks; ++a) {
                use(g->kids[a]);
                for (int b = 0; b < nranks; ++b) {
                    if (a == b) continue;
                    const cudaError_t e = cudaDeviceEnablePeerAccess(dev[b], 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) {
                        cudaGetLastError();
                    } else {
                        CUDA_OK(e);
                    }
                }
            }
            for (OscCtx* k : g->kids) {
                for (int q = 0; q < nranks; ++q) k->args.peer_xll[q] = g->kids[q]->xll.p;
                k->args.p2p = 1;
                enable_mr_cr(k);
                k->drop_graphs();
            }
        }
        *out = g.release();
    });
}

int osc_group_info(const OscCtx* c, int* nranks, int* ordered) {
    return guarded([&] {
        if (!c) throw Error(OSC_ERR_CONFIG, "null context");
        if (nranks) *nranks = c->kids.empty() ? 1 : (int)c->kids.size();
        if (ordered) *ordered = c->ordered;
    });
}

int osc_destroy(OscCtx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        for (OscCtx* k : ranks_of(ctx)) {
            cudaSetDevice(k->device);
            cudaStreamSynchronize(k->stream);
        }
        delete ctx;
    });
}

int osc_local_range(const OscCtx* c, int* t_lo, int* t_hi, size_t* n) {
    return guarded([&] {
        if (!c) throw Error(OSC_ERR_CONFIG, "null context");
        if (t_lo) *t_lo = c->t_lo;
        if (t_hi) *t_hi = c->t_hi;
        if (n) *n = total_doubles(c);
    });
}

int osc_init_states(OscCtx* g) {
    return guarded([&] {
        for (OscCtx* c : ranks_of(g)) {
            use(c);
            if (c->nflav == 3)
                k_init3<<<(c->ncell + 255) / 256, 256, 0, c->stream>>>(c->args, c->desc.perturb);
            else
                k_init<<<(c->ncell + 255) / 256, 256, 0, c->stream>>>(c->args, c->desc.perturb);
            c->count();
            CUDA_OK(cudaGetLastError());
        }
        g_sync(g);
    });
}

int osc_set_state(OscCtx* c, const double* m, size_t n) {
    return guarded([&] { set_state_impl(c, m, n, cudaMemcpyHostToDevice); });
}
int osc_get_state(OscCtx* c, double* m, size_t n) {
    return guarded([&] { get_state_impl(c, m, n, cudaMemcpyDeviceToHost); });
}
int osc_set_state_device(OscCtx* c, const double* m, size_t n) {
    return guarded([&] { set_state_impl(c, m, n, cudaMemcpyDefault); });
}
int osc_get_state_device(OscCtx* c, double* m, size_t n) {
    return guarded([&] { get_state_impl(c, m, n, cudaMemcpyDefault); });
}

int osc_trial_step_error(OscCtx* c, double r, double dr, double* err) {
    return guarded([&] {
        // (a multi-process rank cannot take a trial step alone; a group can)
        if (c->kids.empty() && c->nranks != 1)
            throw Error(OSC_ERR_CONFIG, "trial_step_error: single-lane engines only");
        OscStepControl s{};
        s.r = r;
        s.dr = dr;
        s.dr_max = dr;
        s.dr_min = 0.0;
        s.eps0 = 1e300;
        s.kappa = 1.0;
        s.Rn = r + dr;
        if (c->kids.empty()) {
            use(c);
            c->begin(s, /*commit=*/0);
            c->enqueue_step();
            c->finalize();
        } else {
            g_begin(c, s, 0);
            if (c->ordered) {
                g_enqueue_steps(c, 1);
            } else {
                for (OscCtx* k : c->kids) {
                    use(k);
                    k->enqueue_step();
                    k->finalize();
                }
            }
        }
        *err = g_download(c).err;
    });
}

int osc_begin(OscCtx* c, const OscStepControl* ctl) {
    return guarded([&] {
        g_begin(c, *ctl, 1);
        g_prepare_graphs(c);
    });
}

int osc_enqueue_steps(OscCtx* c, int n) {
    return guarded([&] { g_enqueue_steps(c, n); });
}

int osc_query(OscCtx* c, double* r, double* dr, uint64_t* iter, uint64_t* acc, uint64_t* rej, double* err,
              int* status, int* term) {
    return guarded([&] {
        for (OscCtx* k : ranks_of(c)) {
            use(k);
            k->download_ctl();
        }
        const Ctl& h = hctl(c);
        if (r) *r = h.r;
        if (dr) *dr = h.dr;
        if (iter) *iter = h.iter;
        if (acc) *acc = h.accepted;
        if (rej) *rej = h.rejected;
        if (err) *err = h.err;
        int st = 0;
        for (OscCtx* k : ranks_of(c)) st = st ? st : k->h_ctl->status;
        if (status) *status = st;
        if (term) *term = h.terminate;
    });
}

int osc_synchronize(OscCtx* c) {
    return guarded([&] { g_sync(c); });
}

void* osc_stream(OscCtx* c) { return c ? (void*)ranks_of(c)[0]->stream : nullptr; }

int osc_launches_per_step(const OscCtx* c) {
    if (!c) return 0;
    const OscCtx* k = ranks_of(c)[0];
    return k->coll && !k->args.p2p ? 4 : 3;
}

int osc_debug_sums(OscCtx* g, double* out) {
    return guarded([&] {
        OscCtx* c = ranks_of(g)[0];
        CUDA_OK(cudaSetDevice(c->device));
        std::vector<double> x(c->xbuf.n);
        CUDA_OK(cudaStreamSynchronize(c->stream));
        CUDA_OK(cudaMemcpy(x.data(), c->xbuf.p, x.size() * sizeof(double), cudaMemcpyDeviceToHost));
        // totals per slot in rank order: sums0 | sums1 | sums2 | sums3 | next
        auto total = [&](int slot, int k) {
            double t = 0.0;
            for (int q = 0; q < c->nranks; ++q) t += x[((size_t)slot * c->nranks + q) * kSlotDoubles + k];
            return t;
        };
        for (int k = 0; k < 12; ++k) {
            out[k] = total(0, k);
            out[12 + k] = total(1, k);
            out[24 + k] = total(1, 12 + k);
            out[36 + k] = total(2, k);
            out[48 + k] = total(3, k);
        }
    });
}

int osc_set_schedule(OscCtx* g, int schedule) {
    return guarded([&] {
        if (schedule != 0 && schedule != 1) throw Error(OSC_ERR_CONFIG, "schedule must be 0 or 1");
        for (OscCtx* c : ranks_of(g)) {
            use(c);
            if (schedule == 1 && !c->stash.p) c->stash.alloc((size_t)c->npad * (c->nflav == 3 ? kSt3Planes : c->nplanes));
            c->schedule = schedule;
            c->args.schedule = schedule;
            c->args.stash = c->stash.p;
            c->drop_graphs();
        }
    });
}

int osc_set_launch_mode(OscCtx* c, int mode) {
    return guarded([&] {
        if (mode != 0 && mode != 2) throw Error(OSC_ERR_CONFIG, "launch mode must be 0 or 2");
        if (mode == 2 && !c->resident_ok)
            throw Error(OSC_ERR_CONFIG, "resident kernel unavailable (multi-rank, 3 flavours or state too large)");
        c->launch_mode = mode;
    });
}

int osc_get_launch_mode(OscCtx* c) { return c ? c->launch_mode : 0; }

unsigned long long osc_launch_count(const OscCtx* c) {
    unsigned long long n = 0;
    if (c)
        for (const OscCtx* k : ranks_of(c)) n += k->nlaunch;
    return n;
}

int osc_comm_export(OscCtx* c, void* out128) {
    return guarded([&] {
        if (!c->kids.empty()) throw Error(OSC_ERR_CONFIG, "osc_comm_export: group contexts exchange in-process");
        if (!out128) throw Error(OSC_ERR_CONFIG, "osc_comm_export: null out");
        CUDA_OK(cudaSetDevice(c->device));
        cudaIpcMemHandle_t h[2];
        std::memset(h, 0, sizeof h);
        CUDA_OK(cudaIpcGetMemHandle(&h[0], c->xll.p));  // (second handle reserved)
        static_assert(sizeof h == 128, "IPC handle size");
        std::memcpy(out128, h, sizeof h);
    });
}

}  // extern "C"

// Device-initiated exchange connected: 2-flavour contexts switch to the
// consumer-side reduction with the S2-side control (as on one GPU; the rank
// totals travel tagged 4 nstep + slot, step_kernels.cuh mr_totals).  Env
// OSC_MR_CR=0 keeps the last-block publish per stage and the control fused
// into S4's last block.
static void enable_mr_cr(OscCtx* c) {
    const char* env = std::getenv("OSC_MR_CR");
    c->args.cr = (c->nflav == 2 && OSC_CR && !(env && std::atoi(env) == 0)) ? 1 : 0;
}

extern "C" {

int osc_comm_connect(OscCtx* c, const void* handles) {
    return guarded([&] {
        if (!c->coll) throw Error(OSC_ERR_CONFIG, "osc_comm_connect: not a multi-rank context");
        if (!handles) throw Error(OSC_ERR_CONFIG, "osc_comm_connect: null handles");
        CUDA_OK(cudaSetDevice(c->device));
        CUDA_OK(cudaStreamSynchronize(c->stream));
        StepArgs& a = c->args;
        for (int q = 0; q < c->nranks; ++q) {
            if (q == c->rank) {
                a.peer_xll[q] = c->xll.p;
                continue;
            }
            cudaIpcMemHandle_t h[2];
            std::memcpy(h, static_cast<const char*>(handles) + (size_t)q * sizeof h, sizeof h);
            void* pb = nullptr;
            CUDA_OK(cudaIpcOpenMemHandle(&pb, h[0], cudaIpcMemLazyEnablePeerAccess));
            c->ipc_opened.push_back(pb);
            a.peer_xll[q] = static_cast<unsigned long long*>(pb);
        }
        a.p2p = 1;
        enable_mr_cr(c);
        c->drop_graphs();  // kernel arguments changed
    });
}

int osc_fp64_peak(int device, double* dfma_per_s, double* ms_out) {
    return guarded([&] {
        CUDA_OK(cudaSetDevice(device));
        int nsm = 0;
        CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
        double* d = nullptr;
        CUDA_OK(cudaMalloc(&d, sizeof(double)));
        cudaEvent_t e0, e1;
        CUDA_OK(cudaEventCreate(&e0));
        CUDA_OK(cudaEventCreate(&e1));
        const int blocks = nsm * 8, threads = 256, iters = 4096;
        k_dfma_peak<<<blocks, threads>>>(d, 64, 0.999999, 1e-9);  // warm-up
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            CUDA_OK(cudaEventRecord(e0));
            k_dfma_peak<<<blocks, threads>>>(d, iters, 0.999999, 1e-9);
            CUDA_OK(cudaEventRecord(e1));
            CUDA_OK(cudaEventSynchronize(e1));
            float ms = 0.f;
            CUDA_OK(cudaEventElapsedTime(&ms, e0, e1));
            best = std::min(best, ms);
        }
        CUDA_OK(cudaGetLastError());
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(d);
        *dfma_per_s = (double)blocks * threads * 8.0 * iters / (best * 1e-3);
        if (ms_out) *ms_out = best;
    });
}

int osc_debug_evolve_bin(int device, size_t n, const double* h, const double* dl, const double* psi,
                         double* out, int path) {
    return guarded([&] {
        if (n == 0) return;
        if (!h || !dl || !psi || !out) throw Error(OSC_ERR_CONFIG, "osc_debug_evolve_bin: null argument");
        CUDA_OK(cudaSetDevice(device));
        double* d = nullptr;
        CUDA_OK(cudaMalloc(&d, n * 12 * sizeof(double)));
        std::unique_ptr<double, decltype(&cudaFree)> hold(d, &cudaFree);
        CUDA_OK(cudaMemcpy(d, h, n * 3 * sizeof(double), cudaMemcpyHostToDevice));
        CUDA_OK(cudaMemcpy(d + 3 * n, dl, n * sizeof(double), cudaMemcpyHostToDevice));
        CUDA_OK(cudaMemcpy(d + 4 * n, psi, n * 4 * sizeof(double), cudaMemcpyHostToDevice));
        k_debug_evolve<<<(unsigned)((n + 127) / 128), 128>>>((int)n, d, d + 3 * n, d + 4 * n, d + 8 * n, path);
        CUDA_OK(cudaGetLastError());
        CUDA_OK(cudaMemcpy(out, d + 8 * n, n * 4 * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

int osc_debug_exp3(int device, size_t n, const double* H, const double* tau, double* U, int path) {
    return guarded([&] {
        if (n == 0) return;
        if (!H || !tau || !U) throw Error(OSC_ERR_CONFIG, "osc_debug_exp3: null argument");
        CUDA_OK(cudaSetDevice(device));
        double* d = nullptr;
        CUDA_OK(cudaMalloc(&d, n * 28 * sizeof(double)));
        std::unique_ptr<double, decltype(&cudaFree)> hold(d, &cudaFree);
        CUDA_OK(cudaMemcpy(d, H, n * 9 * sizeof(double), cudaMemcpyHostToDevice));
        CUDA_OK(cudaMemcpy(d + 9 * n, tau, n * sizeof(double), cudaMemcpyHostToDevice));
        k_debug_exp3<<<(unsigned)((n + 127) / 128), 128>>>((int)n, d, d + 9 * n, d + 10 * n, path);
        CUDA_OK(cudaGetLastError());
        CUDA_OK(cudaMemcpy(U, d + 10 * n, n * 18 * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

int osc_profile_stages(OscCtx* c, int nsteps, float* ms_out) {
    return guarded([&] {
        if (!c->kids.empty()) throw Error(OSC_ERR_CONFIG, "osc_profile_stages: single-GPU contexts only");
        CUDA_OK(cudaSetDevice(c->device));
        if (c->nranks != 1) throw Error(OSC_ERR_CONFIG, "osc_profile_stages: single-GPU contexts only");
        cudaEvent_t ev[4];
        for (auto& e : ev) CUDA_OK(cudaEventCreate(&e));
        double acc[3] = {0, 0, 0};
        for (int i = 0; i < nsteps; ++i) {
            CUDA_OK(cudaEventRecord(ev[0], c->stream));
            c->launch_stage(2);
            CUDA_OK(cudaEventRecord(ev[1], c->stream));
            c->launch_stage(3);
            CUDA_OK(cudaEventRecord(ev[2], c->stream));
            c->launch_stage(4);
            CUDA_OK(cudaEventRecord(ev[3], c->stream));
            CUDA_OK(cudaEventSynchronize(ev[3]));
            for (int k = 0; k < 3; ++k) {
                float ms = 0.f;
                CUDA_OK(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
                acc[k] += ms;
            }
        }
        c->finalize();
        CUDA_OK(cudaStreamSynchronize(c->stream));
        for (auto& e : ev) cudaEventDestroy(e);
        for (int k = 0; k < 3; ++k) ms_out[k] = (float)(acc[k] / std::max(1, nsteps));
    });
}

int osc_debug_trace(unsigned long long* out, size_t n) {
    return guarded([&] {
#if OSC_TRACE
        const size_t have = (size_t)kTraceLaunches * kTraceBlocks * kTracePts;
        CUDA_OK(cudaDeviceSynchronize());
        CUDA_OK(cudaMemcpyFromSymbol(out, g_trace, std::min(n, have) * sizeof(unsigned long long)));
#else
        (void)out;
        (void)n;
        throw Error(OSC_ERR_CONFIG, "osc_debug_trace: library built without -DOSC_TRACE");
#endif
    });
}

int osc_max_norm_dev(OscCtx* g, double* out) {
    return guarded([&] {
        double worst = 0.0;
        for (OscCtx* c : ranks_of(g)) {
            use(c);
            CUDA_OK(cudaMemsetAsync(c->scratch.p, 0, sizeof(unsigned long long), c->stream));
            k_norm_dev<<<c->nsm * 4, 256, 0, c->stream>>>(c->args, c->scratch.p);
            c->count();
            CUDA_OK(cudaGetLastError());
            unsigned long long bits = 0;
            CUDA_OK(cudaMemcpyAsync(&bits, c->scratch.p, sizeof bits, cudaMemcpyDeviceToHost, c->stream));
            CUDA_OK(cudaStreamSynchronize(c->stream));
            double v;
            std::memcpy(&v, &bits, sizeof v);
            worst = std::max(worst, v);
        }
        *out = worst;
    });
}

}  // extern "C"

namespace {

// Enqueue the mode-2 extraction of one rank into its mode2buf (its stream).
void enqueue_mode2(OscCtx* c) {
    const size_t n = mode2_local(c);
    if (c->mode2buf.n < n) c->mode2buf.alloc(n);
    k_mode2<<<(int)std::min<size_t>((n + 255) / 256, (size_t)c->nsm * 8), 256, 0, c->stream>>>(c->args, c->fw.p,
                                                                                             c->mode2buf.p);
    c->count();
    CUDA_OK(cudaGetLastError());
}

// Steps per host round trip of Engine::run: graph batches of up to 64 steps,
// never past Ts, and — with a wall-time limit Tn — sized from the measured
// step time so that the last batches before Tn shrink to single steps (the
// reference checks Tn after every step, solver.cpp:453).
struct Batcher {
    const OscStepControl* ctl;
    double step_s = -1.0;  // measured seconds per step (-1: unknown)
    int last = 0;
    int next(uint64_t iter, double elapsed) const {
        int b = 64;
        if (ctl->Ts > 0) {
            const uint64_t left = ctl->Ts - std::min<uint64_t>(ctl->Ts, iter);
            b = (int)std::max<uint64_t>(1, std::min<uint64_t>(left, 64));
        }
        if (ctl->Tn > 0.0) {
            const int cap = step_s < 0.0 ? std::max(1, 2 * last)
                                         : (int)std::max(1.0, std::min(64.0, 0.5 * (ctl->Tn - elapsed) / step_s));
            b = std::min(b, std::max(1, cap));
        }
        return b;
    }
    void measured(int steps, double secs) {
        if (steps > 0 && secs > 0.0) step_s = step_s < 0.0 ? secs / steps : std::min(step_s, secs / steps);
    }
};

void fill_summary(OscCtx* g, const OscStepControl* ctl, int term, double wall, double t_io, OscRunSummary* out) {
    double nd = 0.0;
    const int rc = osc_max_norm_dev(g, &nd);
    if (rc != OSC_OK) throw Error(rc, g_last_error);
    const Ctl& h = hctl(g);
    out->final_r = h.r;
    out->iterations = h.iter - ctl->iter;
    out->accepted = h.accepted;
    out->rejected = h.rejected;
    out->wall_s = wall;
    out->phase_hamiltonian_s = 0.0;  // (fused into the stage kernels)
    out->phase_evolve_s = wall - t_io;
    out->phase_io_s = t_io;
    out->max_worker_wait_s = 0.0;
    out->final_max_norm_dev = nd;
    out->termination = term == 2 ? 2 : (term == 3 ? 3 : 1);
}

}  // namespace

extern "C" {

int osc_extract_mode2(OscCtx* g, double* out, size_t n) {
    return guarded([&] {
        if (n != mode2_total(g)) throw Error(OSC_ERR_IO, "extract_mode2: payload size mismatch");
        size_t off = 0;
        for (OscCtx* c : ranks_of(g)) {
            use(c);
            enqueue_mode2(c);
            CUDA_OK(cudaMemcpyAsync(out + off, c->mode2buf.p, mode2_local(c) * sizeof(double), cudaMemcpyDeviceToHost,
                                    c->stream));
            off += mode2_local(c);
        }
        g_sync(g);
    });
}

int osc_run_dumps(OscCtx* g, const OscStepControl* ctl, const OscDumpGates* gates, int mode_mask,
                  osc_dump_fn fn, void* user, OscRunSummary* out) {
    return guarded([&] {
        using Clock = std::chrono::steady_clock;
        if (!ctl || !out || (mode_mask && (!gates || !fn)))
            throw Error(OSC_ERR_CONFIG, "osc_run_dumps: null argument");
        mode_mask &= 3;
        const std::vector<OscCtx*> R = ranks_of(g);
        const auto t0 = Clock::now();
        auto secs = [&] { return std::chrono::duration<double>(Clock::now() - t0).count(); };
        g_begin(g, *ctl, 1);
        // arm the device gates on every rank (DumpDriver::reset_marks: marks
        // at the start)
        for (OscCtx* c : R) {
            use(c);
            c->download_ctl();
            Ctl& h = *c->h_ctl;
            h.dump_mask = mode_mask;
            h.pause = 0;
            for (int m = 0; m < 2; ++m) {
                h.dump_r_step[m] = (mode_mask >> m & 1) ? gates[m].r_step : 0.0;
                h.dump_itr_step[m] = (mode_mask >> m & 1) ? gates[m].itr_step : 0;
                h.mark_r[m] = ctl->r;
                h.mark_iter[m] = ctl->iter;
            }
            c->upload_ctl();
        }
        double mark_t[2] = {0.0, 0.0};
        const size_t n1 = total_doubles(g), n2 = mode2_total(g);
        for (OscCtx* c : R) {
            use(c);
            const size_t l1 = local_doubles(c), l2 = mode2_local(c);
            if (mode_mask & 1) {
                if (c->staging.n < l1) c->staging.alloc(l1);
                if (c->staging2.n < l1) c->staging2.alloc(l1);
            }
            if (mode_mask & 2 && c->mode2buf.n < l2) c->mode2buf.alloc(l2);
            if (mode_mask && !c->copy_stream) CUDA_OK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        }
        const size_t pin_n = std::max((mode_mask & 1) ? n1 : 0, (mode_mask & 2) ? n2 : 0);
        if (pin_n > g->pinned_n) {
            for (double*& p : g->pinned) {
                if (p) cudaFreeHost(p);
                p = nullptr;
                CUDA_OK(cudaMallocHost(&p, pin_n * sizeof(double)));
            }
            g->pinned_n = pin_n;
        }

        // Two dump slots in flight: packed on each rank's compute stream into
        // a device staging buffer, copied (rank slices at their payload
        // offsets) to pinned memory on the rank's copy stream while the next
        // steps run; delivered in order.
        struct Pending {
            int mode = 0;
            size_t n = 0;
            OscRecordMeta meta{};
            std::vector<cudaEvent_t> done;  // per rank
            bool busy = false;
        } slot[2];
        for (Pending& p : slot) {
            p.done.resize(R.size(), nullptr);
            for (size_t q = 0; q < R.size(); ++q) {
                use(R[q]);
                CUDA_OK(cudaEventCreateWithFlags(&p.done[q], cudaEventDisableTiming));
            }
        }
        std::vector<int> fifo;
        double t_io = 0.0;
        auto deliver = [&](bool wait_all, int need_free) {
            while (!fifo.empty()) {
                Pending& p = slot[fifo.front()];
                if (!wait_all && need_free < 0) {
                    bool ready = true;
                    for (cudaEvent_t e : p.done) ready = ready && cudaEventQuery(e) != cudaErrorNotReady;
                    if (!ready) break;
                }
                for (cudaEvent_t e : p.done) CUDA_OK(cudaEventSynchronize(e));
                const auto ti = Clock::now();
                fn(user, p.mode, &p.meta, g->pinned[fifo.front()], p.n);
                t_io += std::chrono::duration<double>(Clock::now() - ti).count();
                p.busy = false;
                const int freed = fifo.front();
                fifo.erase(fifo.begin());
                if (!wait_all && need_free >= 0 && freed == need_free) break;
            }
        };
        auto take_dump = [&](int mode, const OscRecordMeta& meta) {
            int k = !slot[0].busy ? 0 : (!slot[1].busy ? 1 : -1);
            if (k < 0) {  // both in flight: deliver the oldest
                deliver(false, fifo.front());
                k = !slot[0].busy ? 0 : 1;
            }
            Pending& p = slot[k];
            size_t off = 0;
            for (size_t q = 0; q < R.size(); ++q) {
                OscCtx* c = R[q];
                use(c);
                const double* src;
                size_t len;
                if (mode == 1) {
                    double* st = k == 0 ? c->staging.p : c->staging2.p;
                    len = local_doubles(c);
                    k_pack<<<c->nsm * 8, 256, 0, c->stream>>>(c->args, st, 0, len);
                    c->count();
                    CUDA_OK(cudaGetLastError());
                    src = st;
                } else {
                    enqueue_mode2(c);
                    src = c->mode2buf.p;
                    len = mode2_local(c);
                }
                CUDA_OK(cudaEventRecord(p.done[q], c->stream));
                CUDA_OK(cudaStreamWaitEvent(c->copy_stream, p.done[q], 0));
                CUDA_OK(cudaMemcpyAsync(g->pinned[k] + off, src, len * sizeof(double), cudaMemcpyDeviceToHost,
                                        c->copy_stream));
                CUDA_OK(cudaEventRecord(p.done[q], c->copy_stream));
                if (mode == 2) CUDA_OK(cudaStreamWaitEvent(c->stream, p.done[q], 0));  // mode2buf reuse
                off += len;
            }
            p.n = off;
            p.mode = mode;
            p.meta = meta;
            p.busy = true;
            fifo.push_back(k);
        };

        int term = hctl(g).terminate;
        uint64_t last_acc = 0;
        Batcher bt{ctl};
        auto next_batch = [&]() {
            bt.last = bt.next(hctl(g).iter, secs());
            g_enqueue_steps(g, bt.last);
        };
        double tb = secs();
        if (!term) next_batch();
        while (!term) {
            Ctl& h = g_download(g);
            bt.measured(bt.last, secs() - tb);
            term = h.terminate;
            int due = h.pause & mode_mask;
            const double t = secs();
            if (h.accepted != last_acc) {  // wall-time gates at batch boundaries
                for (int m = 0; m < 2; ++m)
                    if ((mode_mask >> m & 1) && gates[m].t_step > 0.0 && t - mark_t[m] >= gates[m].t_step)
                        due |= 1 << m;
                last_acc = h.accepted;
            }
            if (due) {
                const OscRecordMeta meta{h.iter, h.r, h.dr, t};
                for (int m = 0; m < 2; ++m) {
                    if (!(due >> m & 1)) continue;
                    mark_t[m] = t;
                    take_dump(m + 1, meta);
                }
                for (OscCtx* c : R) {  // (every rank paused identically)
                    use(c);
                    Ctl& hc = *c->h_ctl;
                    for (int m = 0; m < 2; ++m)
                        if (due >> m & 1) {
                            hc.mark_r[m] = hc.r;  // (already moved by the device for its own gates)
                            hc.mark_iter[m] = hc.iter;
                        }
                    hc.pause = 0;
                    CUDA_OK(cudaMemcpyAsync(c->ctl_cur(), c->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, c->stream));
                }
            }
            if (!term && ctl->Tn > 0.0 && secs() >= ctl->Tn) term = 3;
            // keep the device busy while the host delivers finished dumps
            tb = secs();
            if (!term) next_batch();
            deliver(false, -1);
        }
        deliver(true, -1);
        for (Pending& p : slot)
            for (cudaEvent_t e : p.done)
                if (e) cudaEventDestroy(e);
        fill_summary(g, ctl, term, secs(), t_io, out);
    });
}

int osc_run(OscCtx* g, const OscStepControl* ctl, osc_hook_fn hook, void* user, OscRunSummary* out) {
    return guarded([&] {
        using Clock = std::chrono::steady_clock;
        if (!ctl || !out) throw Error(OSC_ERR_CONFIG, "osc_run: null argument");
        const auto t0 = Clock::now();
        auto secs = [&] { return std::chrono::duration<double>(Clock::now() - t0).count(); };
        g_begin(g, *ctl, 1);
        double t_io = 0.0;
        int term = hctl(g).terminate;
        std::vector<double> host_state;
        uint64_t last_acc = 0;
        Batcher bt{ctl};
        // batch size: one step at a time when a hook must see every accepted
        // state, else graph batches with a host check between batches
        while (!term) {
            const double tb = secs();
            bt.last = hook ? 1 : bt.next(hctl(g).iter, tb);
            g_enqueue_steps(g, bt.last);
            const Ctl& h = g_download(g);
            bt.measured(bt.last, secs() - tb);
            term = h.terminate;
            if (hook && h.accepted != last_acc) {
                last_acc = h.accepted;
                const auto ti = Clock::now();
                host_state.resize(total_doubles(g));
                get_state_impl(g, host_state.data(), host_state.size(), cudaMemcpyDeviceToHost);
                OscHookInfo info{h.iter, h.r, h.dr, secs()};
                hook(user, &info, host_state.data(), host_state.size());
                t_io += std::chrono::duration<double>(Clock::now() - ti).count();
            }
            if (!term && ctl->Tn > 0.0 && secs() >= ctl->Tn) term = 3;
        }
        fill_summary(g, ctl, term, secs(), t_io, out);
    });
}

}  // extern "C"
