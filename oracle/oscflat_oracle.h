/* TEST INFRASTRUCTURE ONLY — the CPU oracle (checker), never the product.
 *
 * Plain-C restatement of the reference's per-step beam evolution
 * (reference: /root/reference/proj/core, "oscflat").  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Parity status: PINNED against the compiled reference (oracle/_ref, built
 * by oracle/Makefile from the reference's own sources) and against the
 * golden fixtures in tests/golden/ generated from it
 * (tests/golden/make_golden.py).
 *
 * State layout is the reference's mode-1 order [traj][species][comp][ebin]
 * (solver.cpp:127-140) with traj = theta*pbins + phi.
 */
#ifndef OSCFLAT_ORACLE_H
#define OSCFLAT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Models 0-2 restate the reference (geom::Model).  3 (plane, paper Eq. 3.19)
 * and 4 (cylinder, Eq. 3.20) are BASELINE configs[3]/[4], which the reference
 * does not implement: PARITY UNPINNED for those two (self-consistency tests
 * only; see DESIGN.md §9 for the geometry chosen). */
enum { ORC_SINGLE_ANGLE = 0, ORC_BULB = 1, ORC_EXT_BULB = 2, ORC_PLANE = 3, ORC_CYLINDER = 4 };
enum { ORC_MATTER_POWERLAW = 0, ORC_MATTER_EXP = 1, ORC_MATTER_SUM = 2, ORC_MATTER_OFF = 3 };

typedef struct {
    int model, abins, pbins, ebins;
    double Rnu, E0, E1, dm2, theta, hvv_scale, perturb;
    double L[4], T[4], Emean[4], eta[4]; /* species order NuE, NuEBar, NuX, NuXBar */
    int matter_profile;
    double Ye, nb0, hNS, Mns, gs, S;
} OrcParams;

typedef struct OrcEnv OrcEnv;
typedef struct OrcEngine OrcEngine;

const char* orc_last_error(void);

/* Environment (solver::Environment::from_config, solver.cpp:62-95). */
int orc_env_create(const OrcParams* p, OrcEnv** out);
void orc_env_destroy(OrcEnv* env);
/* Copies the tables out (logical lengths): cos2[T] sin0[T] cphi[P] sphi[P]
 * vac11[E] vac12[E] fw[4*E] couplings[4] emean[4]. */
void orc_env_tables(const OrcEnv* env, double* cos2, double* sin0, double* cphi,
                    double* sphi, double* vac11, double* vac12, double* fw,
                    double* couplings, double* emean);
double orc_fermi_integral(int k, double eta);
double orc_matter_potential(const OrcEnv* env, double r_km);

/* Kernels (beam.hpp / beam.cpp). */
void orc_evolve_bin(const double* h, double dl, const double* psi, double* out);
void orc_density(const double* psi, double* out);
void orc_init_state(int species, int ebins, double eps, uint64_t seed, double* out);

/* Engine over the theta partition [t_lo, t_hi) (one rank / lane). */
int orc_engine_create(const OrcEnv* env, int t_lo, int t_hi, OrcEngine** out);
void orc_engine_destroy(OrcEngine* eng);
void orc_init_states(OrcEngine* eng);
/* local mode-1 payload for trajectories [t_lo*P, t_hi*P) */
void orc_set_state(OrcEngine* eng, const double* mode1);
void orc_get_state(const OrcEngine* eng, double* mode1);

/* Staged step with an external exchange (the multi-rank contract):
 *   stage 0: S1  partial moments of psi0 at r          -> 12 doubles
 *   stage 1: S2  evolve mid/full1; partial H1||H2      -> 24 doubles
 *   stage 2: S3  full2/avgA, half2; partial H3         -> 12 doubles
 *   stage 3: S4  full3/result; local err               ->  1 double
 * After each stage the caller combines the partials of all ranks (in rank
 * order) and hands the totals back with orc_stage_set.  orc_prepare must be
 * called first with (r, dr). */
int orc_prepare(OrcEngine* eng, double r, double dr);
int orc_stage(OrcEngine* eng, int stage, double* partial_out);
int orc_stage_set(OrcEngine* eng, int stage, const double* total);
void orc_commit(OrcEngine* eng); /* swap(psi0, result) */

/* Single-rank conveniences. */
int orc_trial_step(OrcEngine* eng, double r, double dr, double* err);

typedef struct {
    double dr, dr_max, dr_min, eps0, kappa, r, R0, Rn;
    uint64_t iter, Ts;
} OrcCtl;
typedef struct {
    double final_r;
    uint64_t iterations, accepted, rejected;
    double final_max_norm_dev;
    int termination; /* 1 radius, 2 iterations */
} OrcSummary;
/* Engine::run loop (solver.cpp:414-456, 486-525) on a single rank. */
int orc_run(OrcEngine* eng, const OrcCtl* ctl, OrcSummary* out);
double orc_step_size_update(const OrcCtl* ctl, double err, int accepted, int* collapse);
double orc_max_norm_dev(const OrcEngine* eng);

/* fold_rows + combine_stage + assemble_hvv on given rows at radius r (tests). */
int orc_hvv_from_rows(OrcEngine* eng, double r, const double* rows, double* sums12, double* hvv);

/* make_partitions (parallel.cpp:11-24): out = [workers][2] (lo, hi). */
int orc_make_partitions(int len, int workers, int* out);

/* ---- 3-flavour restatement (oscflat3_oracle.c; BASELINE configs[1];
 * PARITY UNPINNED w.r.t. the reference, which supports Flvs = 2 only). */
typedef struct {
    int model, abins, pbins, ebins;
    double Rnu, E0, E1, dm21, dm31, th12, th13, th23, dcp, hvv_scale, perturb;
    double L[6], T[6], Emean[6], eta[6];
    int matter_profile;
    double Ye, nb0, hNS, Mns, gs, S;
} Orc3Params;

typedef struct Orc3Env Orc3Env;
typedef struct Orc3Engine Orc3Engine;
const char* orc3_last_error(void);
int orc3_env_create(const Orc3Params* p, Orc3Env** out);
void orc3_env_destroy(Orc3Env* env);
void orc3_env_tables(const Orc3Env* env, double* vac9E, double* fw6E, double* couplings6);
void orc3_expm(const double* h9, double tau, double* out18);
void orc3_init_state(int species, int ebins, double eps, uint64_t seed, double* out6E);
int orc3_engine_create(const Orc3Env* env, int t_lo, int t_hi, Orc3Engine** out);
void orc3_engine_destroy(Orc3Engine* eng);
void orc3_init_states(Orc3Engine* eng);
void orc3_set_state(Orc3Engine* eng, const double* mode1);
void orc3_get_state(const Orc3Engine* eng, double* mode1);
int orc3_prepare(Orc3Engine* eng, double r, double dr);
int orc3_stage(Orc3Engine* eng, int stage, double* partial);
int orc3_stage_set(Orc3Engine* eng, int stage, const double* total);
void orc3_commit(Orc3Engine* eng);
int orc3_trial_step(Orc3Engine* eng, double r, double dr, double* err);
int orc3_run(Orc3Engine* eng, const OrcCtl* ctl, OrcSummary* out);

#ifdef __cplusplus
}
#endif
#endif
