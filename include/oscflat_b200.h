/*
 * oscflat_b200 — C-ABI drop-in for the reference's per-step beam evolution.
 *
 * The seam is the pimpl of the reference's solver::Engine
 * (/root/reference/proj/core/include/oscflat/solver.hpp:128-153): a
 * replacement Engine::Impl fills an OscDesc from its solver::Environment,
 * creates one context per GPU and forwards init_states / trial_step_error /
 * run / state() to the entry points below.  INTEGRATION.md shows that shim.
 *
 * Conventions
 *  - Plain C types only: pointers + sizes, no torch / CUDA types in the
 *    signatures (streams are passed as void*).
 *  - Exceptions never cross the ABI.  Every entry point returns an OscStatus;
 *    the message of the last failure on the calling thread is available from
 *    osc_last_error().  The status values map 1:1 onto the reference's
 *    exception types (types.hpp:43-51, parallel.hpp:15-17).
 *  - State payloads on the host are the reference's mode-1 order
 *    [traj][species][comp][ebin] (solver.cpp:127-140), traj = theta*pbins+phi,
 *    species NuE, NuEBar, NuX, NuXBar, comps ar, ai, br, bi, logical ebins
 *    (no padding).  With several ranks each context holds the contiguous theta
 *    block [t_lo, t_hi) given by make_partitions (parallel.cpp:11-24) and the
 *    payload covers only those trajectories.
 */
#ifndef OSCFLAT_B200_H
#define OSCFLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    OSC_OK = 0,
    OSC_ERR_CONFIG = 1,   /* oscflat::ConfigError   (types.hpp:43-45) */
    OSC_ERR_NUMERIC = 2,  /* oscflat::NumericError  (types.hpp:46-48) */
    OSC_ERR_IO = 3,       /* oscflat::IoError       (types.hpp:49-51) */
    OSC_ERR_PARALLEL = 4, /* par::ParallelError     (parallel.hpp:15-17) */
    OSC_ERR_CUDA = 5      /* device / driver failure (no reference analogue) */
} OscStatus;

/* geom::Model (geometry.hpp:11), extended with the plane (BASELINE configs[3],
 * paper Eq. 3.19) and cylinder (configs[4], Eq. 3.20) geometries, which the
 * reference does not implement. */
enum {
    OSC_MODEL_SINGLE_ANGLE = 0,
    OSC_MODEL_BULB = 1,
    OSC_MODEL_EXT_BULB = 2,
    OSC_MODEL_PLANE = 3,
    OSC_MODEL_CYLINDER = 4
};
/* matter::Profile (matter.hpp:9) */
enum { OSC_MATTER_POWERLAW = 0, OSC_MATTER_EXP = 1, OSC_MATTER_SUM = 2, OSC_MATTER_OFF = 3 };

/* Everything solver::Environment carries into the step (solver.hpp:71-85).
 * Tables are copied at osc_create; the caller keeps ownership. */
typedef struct OscDesc {
    int model;          /* OSC_MODEL_*                                        */
    int abins, pbins;   /* AngleGrid::abins / pbins (geometry.hpp:24-36)      */
    int ebins;          /* logical energy bins                                */
    double Rnu;         /* km                                                 */
    /* angle tables; models 0-2: AngleGrid::cos2_theta0 / sin_theta0 /
     * cos_phi / sin_phi.  Plane: cos(theta), sin(theta) of the zenith bins
     * and cos/sin(phi).  Cylinder: cos(a0), sin(a0) of the in-plane emission
     * angle and cos(b), sin(b) of the axial tilt. */
    const double* cos2_theta0; /* [abins] */
    const double* sin_theta0;  /* [abins] */
    const double* cos_phi;     /* [pbins] */
    const double* sin_phi;     /* [pbins] */
    const double* vac_h11;     /* [ebins]  VacuumTable::h11 (geometry.hpp:118)*/
    const double* vac_h12;     /* [ebins]  VacuumTable::h12                   */
    const double* fw;          /* [4][ebins] SpectrumTable::weights() f*dE    */
    double couplings[4];       /* Environment::couplings, 1/km                */
    double perturb;            /* Environment::perturb                        */
    int matter_profile;        /* OSC_MATTER_*  (MatterParams, matter.hpp:11) */
    double Ye, nb0, hNS, Mns, gs, S;
    /* 3-flavour extension (BASELINE configs[1]; not in the reference).
     * nflav 0 or 2: the fields above; nflav 3: species nu_e, nubar_e, nu_mu,
     * nubar_mu, nu_tau, nubar_tau, state comps re/im of (e, mu, tau), and the
     * tables below replace vac_h11/vac_h12/fw/couplings.  Models 0-1 only. */
    int nflav;
    const double* vac3;        /* [ebins][9] H_vac: d_e d_mu d_tau, re/im h_emu h_etau h_mutau */
    const double* fw6;         /* [6][ebins] f*dE per species */
    double couplings6[6];
} OscDesc;

/* One process per GPU.  nranks == 1 -> no collectives.  For nranks > 1 all
 * ranks pass the same 128-byte NCCL unique id (from osc_comm_unique_id on
 * rank 0, distributed by the caller). */
typedef struct OscComm {
    int rank, nranks, device;
    const void* nccl_unique_id; /* 128 bytes, ignored when nranks == 1 */
    int flags;                  /* OSC_COMM_FORCE_COLLECTIVES: run the multi-GPU
                                   exchange path (NCCL all-gather + control
                                   kernel) even when nranks == 1 (tests it on
                                   one GPU) */
} OscComm;
#define OSC_COMM_FORCE_COLLECTIVES 1
#define OSC_COMM_GROUP 2 /* (set by osc_create_group on its ranks: the group
                            drives the exchange, no NCCL communicator) */

/* solver::StepControl (solver.hpp:20-34) */
typedef struct OscStepControl {
    double dr, dr_max, dr_min, eps0, kappa, r, R0, Rn;
    uint64_t iter, Ts;
    double Tn;
} OscStepControl;

/* solver::RunSummary (solver.hpp:85-99); termination 1 radius, 2 iterations,
 * 3 walltime. */
typedef struct OscRunSummary {
    double final_r;
    uint64_t iterations, accepted, rejected;
    double wall_s, phase_hamiltonian_s, phase_evolve_s, phase_io_s, max_worker_wait_s;
    double final_max_norm_dev;
    int termination;
} OscRunSummary;

/* solver::HookInfo (solver.hpp:101-106) */
typedef struct OscHookInfo {
    uint64_t iter;
    double r, dr, t_wall;
} OscHookInfo;

/* solver::IoHook (solver.hpp:108-110): called on the host after each accepted
 * step with the committed local state (mode-1 payload, n doubles); must not
 * retain the pointer. */
typedef void (*osc_hook_fn)(void* user, const OscHookInfo* info, const double* state, size_t n);

/* io::DumpGates (snapshot.hpp:134-138): a dump is due after an accepted step
 * once r, wall time or iterations moved by the step since the last dump of
 * that mode (io::should_dump, snapshot.cpp:237-243); 0 disables a gate. */
typedef struct OscDumpGates {
    double r_step, t_step;
    uint64_t itr_step;
} OscDumpGates;

/* io::RecordMeta (snapshot.hpp:40-45) of a dump. */
typedef struct OscRecordMeta {
    uint64_t iter;
    double r, dr, t_wall;
} OscRecordMeta;

/* Snapshot callback: mode 1 = whole local state (mode-1 payload layout,
 * solver::extract_mode1 solver.cpp:127-140), mode 2 = energy-averaged
 * |psi_e|^2 per (trajectory, species) (solver::extract_mode2
 * solver.cpp:160-174).  Delivered in dump order on the calling thread; the
 * payload lives in pinned host memory owned by the engine and is valid only
 * during the call. */
typedef void (*osc_dump_fn)(void* user, int mode, const OscRecordMeta* meta, const double* payload, size_t n);

typedef struct OscCtx OscCtx;

const char* osc_last_error(void);
int osc_version(void);

/* NCCL unique id for a multi-GPU context (rank 0 calls, caller broadcasts). */
int osc_comm_unique_id(void* out128);

/* Device-initiated exchange (multi-rank contexts): replaces the per-stage NCCL
 * all-gather by peer stores over NVLink.  Every rank exports 128 bytes (the
 * CUDA IPC handle of its receive buffer), the caller all-gathers them (rank
 * order) and hands the nranks x 128 bytes to osc_comm_connect.  The last
 * block of each stage then stores its rank's moment slot into every rank's
 * buffer as sequence-flagged 64-bit words (no fences); the consumers poll the
 * words.  Without connect the NCCL path is used. */
int osc_comm_export(OscCtx* ctx, void* out128);
int osc_comm_connect(OscCtx* ctx, const void* handles);

/* Engine(env, lanes) — solver.cpp:459-466 (lanes -> GPUs, one per process). */
int osc_create(const OscDesc* desc, const OscComm* comm, OscCtx** out);
int osc_destroy(OscCtx* ctx);

/* Engine(env, lanes) in ONE process over several GPUs — the in-process
 * counterpart of par::run_lanes (parallel.cpp:224-253): nranks contexts, rank
 * q on devices[q] (NULL: q mod the device count) holding theta block q of
 * make_partitions (parallel.cpp:11-24), driven by the calling thread through
 * the returned group handle, which every entry point below accepts like a
 * single context (state payloads then cover all trajectories, in order).
 * Moment exchange between the stages:
 *   - stream-ordered (default): the rank slots are copied between the ranks'
 *     exchange buffers (peer copies) behind cross-stream events after every
 *     stage, a control kernel per rank after S4.  No kernel ever waits on
 *     another rank's kernel, so any placement works, several ranks per GPU
 *     included (how the tests run 2 and 3 ranks on one GPU);
 *   - device-initiated (OSC_GROUP_PEER, when every rank has its own GPU and
 *     all pairs have peer access; else the ordered exchange): the last block
 *     of each stage stores its rank's slot into every rank's buffer over
 *     NVLink through peer pointers (the osc_comm_connect path without IPC),
 *     consumers poll sequence-flagged words.  Opt-in until it has run on
 *     several GPUs (the same kernels run with a one-rank communicator).
 * nranks == 1 returns a plain context (osc_create with OscComm{0, 1, dev}). */
#define OSC_GROUP_ORDERED 1 /* (the default; kept for callers that pass it) */
#define OSC_GROUP_PEER 2
int osc_create_group(const OscDesc* desc, int nranks, const int* devices, int flags, OscCtx** out);
/* Ranks of a context (1 unless a group) and its exchange (1: stream-ordered). */
int osc_group_info(const OscCtx* ctx, int* nranks, int* ordered);
/* Visible CUDA devices (0 when none). */
int osc_device_count(int* n);

/* Local theta block [t_lo, t_hi) and local state size in doubles (a group:
 * [0, abins) and the whole state). */
int osc_local_range(const OscCtx* ctx, int* t_lo, int* t_hi, size_t* state_doubles);

/* Engine::init_states — solver.cpp:475-478 / 255-271 (splitmix64 noise with
 * seed = global beam index, beam.cpp:41-57). */
int osc_init_states(OscCtx* ctx);

/* Engine::state() as host mode-1 payloads (copy in / copy out). */
int osc_set_state(OscCtx* ctx, const double* mode1, size_t n);
int osc_get_state(OscCtx* ctx, double* mode1, size_t n);
/* Same, from/to device memory on the context's device (mode-1 order). */
int osc_set_state_device(OscCtx* ctx, const double* dev_mode1, size_t n);
int osc_get_state_device(OscCtx* ctx, double* dev_mode1, size_t n);

/* Engine::trial_step_error — solver.cpp:480-484: S1-S4 from (r, dr); returns
 * the global embedded error; never commits. */
int osc_trial_step_error(OscCtx* ctx, double r, double dr, double* err);

/* Engine::run — solver.cpp:486-525: the full adaptive loop (fixed-step when
 * eps0 is huge).  hook may be NULL. */
int osc_run(OscCtx* ctx, const OscStepControl* ctl, osc_hook_fn hook, void* user,
            OscRunSummary* out);

/* Engine::run with the CLI's dump gating (DumpDriver, tools/oscflat.cpp:
 * 46-118) moved next to the device: gates[0] for mode 1, gates[1] for mode 2,
 * mode_mask bit 0/1 enables them.  Radius and iteration gates are evaluated
 * by the device control update after every accepted step, which pauses the
 * step sequence only when a dump is due; the state is packed on the device
 * and copied to pinned host memory on a separate stream while the next steps
 * run (async device-to-host snapshot I/O), and the callback fires when the
 * copy has landed.  Wall-time gates are evaluated at batch boundaries. */
int osc_run_dumps(OscCtx* ctx, const OscStepControl* ctl, const OscDumpGates* gates, int mode_mask,
                  osc_dump_fn fn, void* user, OscRunSummary* out);

/* solver::extract_mode2 (solver.cpp:160-174) on the device: n = local
 * trajectories x species doubles (species: 4 for 2 flavours, 6 for 3). */
int osc_extract_mode2(OscCtx* ctx, double* out, size_t n);

/* max over local beams of |norm - 1| (beam.cpp:147-155). */
int osc_max_norm_dev(OscCtx* ctx, double* out);

/* ---- measurement helpers (bench.py) ------------------------------------ */
/* Arm a fixed-step walk (as osc_run would) without running it. */
int osc_begin(OscCtx* ctx, const OscStepControl* ctl);
/* Enqueue nsteps evolution steps on the context stream; no host sync. */
int osc_enqueue_steps(OscCtx* ctx, int nsteps);
/* Copy the device control block to the host (syncs the stream): r, dr, iter,
 * accepted, rejected, err, status, terminate. */
int osc_query(OscCtx* ctx, double* r, double* dr, uint64_t* iter, uint64_t* accepted,
              uint64_t* rejected, double* err, int* status, int* terminate);
int osc_synchronize(OscCtx* ctx);
void* osc_stream(OscCtx* ctx);
/* Kernel launches per evolution step and the kernel-name of the dominant one. */
int osc_launches_per_step(const OscCtx* ctx);
/* Last reduced moment sums: out[5][12] = sums0..sums3, next. */
int osc_debug_sums(OscCtx* ctx, double* out60);
/* Configure the stage schedule: 0 = recompute intermediates from psi0,
 * 1 = stash half2 in HBM between S3 and S4. */
int osc_set_schedule(OscCtx* ctx, int schedule);
/* How step batches launch (single-GPU 2-flavour contexts; multi-GPU and
 * 3-flavour contexts always use 0):
 *   0  stage kernels with programmatic dependent launch, CUDA graphs of 8 steps;
 *   2  one persistent cooperative kernel with the whole local state resident
 *      in shared memory (default when it fits: small problems, configs[0]).
 * (1, a persistent kernel streaming the state from HBM with grid barriers
 * between stages, measured slower than 0 on every config and was removed.)
 * Env OSC_LAUNCH=0/2 overrides the default.  OSC_ERR_CONFIG when the mode is
 * unavailable for this context. */
int osc_set_launch_mode(OscCtx* ctx, int mode);
int osc_get_launch_mode(OscCtx* ctx);
/* Number of kernels this context has launched so far (graph launches count
 * every kernel node) — the bench's gpu_launches evidence. */
unsigned long long osc_launch_count(const OscCtx* ctx);

/* Measured FP64 FMA throughput (thread-level DFMA instructions per second)
 * from a DFMA-chain microkernel on `device` — the FP64 roofline denominator. */
int osc_fp64_peak(int device, double* dfma_per_s, double* ms);
/* Average device time of each stage kernel (S2, S3, S4) over nsteps steps,
 * bracketed by CUDA events on the context stream (single-GPU contexts). */
int osc_profile_stages(OscCtx* ctx, int nsteps, float* ms_out3);
/* flavor::evolve_bin (beam.hpp:105-121) through the device propagator code,
 * for known-answer tests of its edge paths (lambda = 0, lambda dl < 1e-12,
 * |lambda dl| > 1e9, subnormal lambda^2): h [n][3] (h11, h12_re, h12_im),
 * dl [n], psi [n][4] (ar, ai, br, bi) -> out [n][4].  path 0: the stage
 * kernels' branch-free chain with its fallback branch; 1: the safe path. */
int osc_debug_evolve_bin(int device, size_t n, const double* h, const double* dl, const double* psi,
                         double* out, int path);
/* exp(-i H tau) of 3x3 Hermitian matrices through the device code of the
 * 3-flavour stages (csrc/su3_exp.cuh; generalises flavor::evolve_bin,
 * beam.hpp:105-121, to configs[1]) for known-answer tests: H [n][9] packed
 * (d0, d1, d2, re/im of h01, h02, h12), tau [n] -> U [n][18] row-major re/im.
 * path 0: one-call exponential; 1: shared decomposition + phases (S2). */
int osc_debug_exp3(int device, size_t n, const double* H, const double* tau, double* U, int path);
/* Development: per-block %globaltimer stamps of the stage launches of four
 * iterations (layout in csrc/step_kernels.cuh, trace_mark); OSC_ERR_CONFIG
 * unless the library was built with -DOSC_TRACE. */
int osc_debug_trace(unsigned long long* out, size_t n);

/* ---- host-side Environment builder (setup, not the hot path) ----------- */
/* Mirrors solver::Environment::from_config (solver.cpp:62-95): angle grid,
 * vacuum table, Fermi-Dirac spectra and couplings from physics parameters. */
typedef struct OscParams {
    int model, abins, pbins, ebins;
    double Rnu, E0, E1, dm2, theta, hvv_scale, perturb;
    double L[4], T[4], Emean[4], eta[4];
    int matter_profile;
    double Ye, nb0, hNS, Mns, gs, S;
    /* nflav = 3: dm2 / theta above are dm2_21 / theta12; the tau species take
     * L_tau / T_tau / Emean_tau / eta_tau (index 0 nu_tau, 1 nubar_tau); the
     * mu species take the x entries (index 2, 3) of the arrays above. */
    int nflav;
    double dm2_31, theta13, theta23, delta_cp;
    double L_tau[2], T_tau[2], Emean_tau[2], eta_tau[2];
} OscParams;
typedef struct OscEnv OscEnv;
int osc_env_build(const OscParams* p, OscEnv** out);
/* Pointers inside desc stay valid until osc_env_destroy. emean may be NULL. */
int osc_env_desc(const OscEnv* env, OscDesc* desc, double* emean4);
int osc_env_destroy(OscEnv* env);
double osc_fermi_integral(int k, double eta);

#ifdef __cplusplus
}
#endif
#endif
