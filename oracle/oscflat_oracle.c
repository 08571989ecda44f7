/* TEST INFRASTRUCTURE ONLY — CPU oracle (checker), never the product path.
 *
 * Plain-C restatement of the reference "oscflat" per-step beam evolution.
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/proj/core).  Parity: pinned against the compiled reference
 * (oracle/_ref) and tests/golden/ (see oscflat_oracle.h).
 */
#include "oscflat_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];
static void set_err(const char* msg) { snprintf(g_err, sizeof g_err, "%s", msg); }
const char* orc_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- units
 * include/oscflat/units.hpp:13-61 */
#define K_PI 3.14159265358979323846
static const double kGF = 1.166e-5 * 1e-6;        /* MeV^-2 */
static const double kHcCm = 197.327e-13;          /* MeV cm */
static const double kHcKm = 197.327e-18;          /* MeV km */
static const double kHbarS = 6.582119569e-22;     /* MeV s */
static const double kErgPerMeV = 1.602176634e-6;

static double per_km(double e_mev) { return e_mev / kHcKm; }

static double matter_A(double ne_cm3) { /* units.hpp:38-42 */
    const double hc3 = kHcCm * kHcCm * kHcCm;
    return per_km(sqrt(2.0) * kGF * ne_cm3 * hc3);
}
static double vacuum_delta(double dm2, double E) { /* units.hpp:46-49 */
    return per_km(dm2 * 1e-12 / (2.0 * E));
}
static double hvv_coupling(double L, double Em, double Rnu) { /* units.hpp:55-61 */
    const double flux = (L / kErgPerMeV) / Em;
    const double Rcm = Rnu * 1e5;
    const double a = sqrt(2.0) * kGF * flux * kHbarS * kHcCm * kHcCm / (2.0 * K_PI * Rcm * Rcm);
    return per_km(a);
}

/* -------------------------------------------------------------- spectra
 * src/spectra.cpp:17-125 (adaptive Simpson + closed-form tail) */
typedef struct { int k; double eta; int evals; int failed; } Quad;

static double fd_f(int k, double eta, double x) {
    const double t = x - eta;
    if (t > 500.0) return pow(x, k) * exp(-t);
    return pow(x, k) / (exp(t) + 1.0);
}
static double simpson(double a, double b, double fa, double fm, double fb) {
    return (b - a) / 6.0 * (fa + 4.0 * fm + fb);
}
static double adapt(Quad* q, double a, double b, double fa, double fm, double fb,
                    double whole, double tol, int depth) {
    if (q->evals > 200000 || depth > 60) { q->failed = 1; return 0.0; }
    const double m = 0.5 * (a + b);
    const double fl = fd_f(q->k, q->eta, 0.5 * (a + m));
    const double fr = fd_f(q->k, q->eta, 0.5 * (m + b));
    q->evals += 2;
    const double left = simpson(a, m, fa, fl, fm);
    const double right = simpson(m, b, fm, fr, fb);
    if (fabs(left + right - whole) <= 15.0 * tol)
        return left + right + (left + right - whole) / 15.0;
    return adapt(q, a, m, fa, fl, fm, left, 0.5 * tol, depth + 1) +
           adapt(q, m, b, fm, fr, fb, right, 0.5 * tol, depth + 1);
}
double orc_fermi_integral(int k, double eta) { /* spectra.cpp:77-83 */
    const double X = (eta > 0.0 ? eta : 0.0) + 40.0;
    Quad q = {k, eta, 0, 0};
    const double fa = fd_f(k, eta, 0.0), fb = fd_f(k, eta, X), fm = fd_f(k, eta, 0.5 * X);
    q.evals = 3;
    const double body = adapt(&q, 0.0, X, fa, fm, fb, simpson(0.0, X, fa, fm, fb), 1e-10, 0);
    if (q.failed) { set_err("fermi_integral: quadrature did not converge"); return NAN; }
    /* tail: e^{eta-X} sum_j k!/j! X^j  (spectra.cpp:63-73) */
    double poly = 0.0, fact = 1.0;
    for (int j = k; j >= 0; --j) { poly += fact * pow(X, j); fact *= j; }
    return body + exp(eta - X) * poly;
}

/* ------------------------------------------------------------------ env */
struct OrcEnv {
    int model, T, P, E;
    double Rnu;
    double *cos2, *sin0, *cphi, *sphi, *vac11, *vac12, *fw;
    double coupling[4], emean[4];
    int matter_profile;
    double Ye, nb0, hNS, Mns, gs, S;
    double perturb;
};

int orc_env_create(const OrcParams* p, OrcEnv** out) {
    OrcEnv* v = calloc(1, sizeof *v);
    v->model = p->model;
    v->T = p->abins;
    v->P = p->pbins;
    if (p->model == ORC_SINGLE_ANGLE) { v->T = 1; v->P = 1; } /* geometry.cpp:36-42 */
    if (p->model == ORC_BULB) v->P = 1;
    v->E = p->ebins;
    v->Rnu = p->Rnu;
    if (v->T < 1 || v->P < 1 || v->E < 1) { free(v); set_err("bins must be >= 1"); return 1; }
    v->cos2 = malloc(sizeof(double) * v->T);
    v->sin0 = malloc(sizeof(double) * v->T);
    v->cphi = malloc(sizeof(double) * v->P);
    v->sphi = malloc(sizeof(double) * v->P);
    if (v->model == ORC_CYLINDER) {
        /* in-plane emission angle a0 uniform on (-pi/2, pi/2); axial tilt b
         * uniform in sin(b) on (-1, 1): tables carry cos/sin of each */
        for (int t = 0; t < v->T; ++t) {
            const double a0 = -0.5 * K_PI + (t + 0.5) * K_PI / v->T;
            v->cos2[t] = cos(a0);
            v->sin0[t] = sin(a0);
        }
        for (int q = 0; q < v->P; ++q) {
            const double sb = -1.0 + (q + 0.5) * 2.0 / v->P;
            v->sphi[q] = sb;
            v->cphi[q] = sqrt(1.0 - sb * sb);
        }
    } else {
        for (int t = 0; t < v->T; ++t) { /* geometry.cpp:52-55; plane: cos(theta) midpoints */
            const double u = (t + 0.5) / v->T;
            v->cos2[t] = u;
            v->sin0[t] = (v->model == ORC_PLANE) ? sqrt(1.0 - u * u) : sqrt(1.0 - u);
        }
        const double dphi = 2.0 * K_PI / v->P;
        for (int q = 0; q < v->P; ++q) {
            const double phi = (q + 0.5) * dphi;
            v->cphi[q] = cos(phi);
            v->sphi[q] = sin(phi);
        }
    }
    /* VacuumTable::make, geometry.cpp:218-240 */
    v->vac11 = malloc(sizeof(double) * v->E);
    v->vac12 = malloc(sizeof(double) * v->E);
    const double dE = (p->E1 - p->E0) / v->E;
    const double c2 = cos(2.0 * p->theta), s2 = sin(2.0 * p->theta);
    for (int e = 0; e < v->E; ++e) {
        const double E = p->E0 + (e + 0.5) * dE;
        const double d = vacuum_delta(p->dm2, E);
        v->vac11[e] = -0.5 * d * c2;
        v->vac12[e] = 0.5 * d * s2;
    }
    /* SpectrumTable + couplings, spectra.cpp:87-125, solver.cpp:71-85 */
    v->fw = malloc(sizeof(double) * 4 * v->E);
    for (int s = 0; s < 4; ++s) {
        double T, Em;
        const double eta = p->eta[s];
        if (p->T[s] > 0.0) {
            T = p->T[s];
            Em = T * orc_fermi_integral(3, eta) / orc_fermi_integral(2, eta);
        } else if (p->Emean[s] > 0.0) {
            Em = p->Emean[s];
            T = Em * orc_fermi_integral(2, eta) / orc_fermi_integral(3, eta);
        } else {
            orc_env_destroy(v);
            set_err("one of T or Emean must be positive");
            return 1;
        }
        /* the coupling uses the configured Emean when given (solver.cpp:79-81) */
        const double Em_c = (p->Emean[s] > 0.0) ? p->Emean[s]
                                                : p->T[s] * orc_fermi_integral(3, eta) /
                                                      orc_fermi_integral(2, eta);
        v->coupling[s] = p->hvv_scale * hvv_coupling(p->L[s], Em_c, p->Rnu);
        v->emean[s] = Em;
        const double norm = 1.0 / (orc_fermi_integral(2, eta) * T * T * T);
        for (int e = 0; e < v->E; ++e) {
            const double E = p->E0 + (e + 0.5) * dE;
            const double t = E / T - eta;
            const double den = (t > 500.0) ? exp(t) : exp(t) + 1.0;
            const double f = norm * E * E / den;
            v->fw[s * v->E + e] = f * dE;
        }
    }
    v->matter_profile = p->matter_profile;
    v->Ye = p->Ye;
    v->nb0 = p->nb0;
    v->hNS = p->hNS;
    v->Mns = p->Mns;
    v->gs = p->gs;
    v->S = p->S;
    v->perturb = p->perturb;
    *out = v;
    return 0;
}

void orc_env_destroy(OrcEnv* v) {
    if (!v) return;
    free(v->cos2); free(v->sin0); free(v->cphi); free(v->sphi);
    free(v->vac11); free(v->vac12); free(v->fw);
    free(v);
}

void orc_env_tables(const OrcEnv* v, double* cos2, double* sin0, double* cphi, double* sphi,
                    double* vac11, double* vac12, double* fw, double* couplings, double* emean) {
    memcpy(cos2, v->cos2, sizeof(double) * v->T);
    memcpy(sin0, v->sin0, sizeof(double) * v->T);
    memcpy(cphi, v->cphi, sizeof(double) * v->P);
    memcpy(sphi, v->sphi, sizeof(double) * v->P);
    memcpy(vac11, v->vac11, sizeof(double) * v->E);
    memcpy(vac12, v->vac12, sizeof(double) * v->E);
    memcpy(fw, v->fw, sizeof(double) * 4 * v->E);
    memcpy(couplings, v->coupling, sizeof(double) * 4);
    memcpy(emean, v->emean, sizeof(double) * 4);
}

/* matter.cpp:12-42; returns NaN below the neutrino sphere (reference throws) */
double orc_matter_potential(const OrcEnv* v, double r) {
    if (v->matter_profile == ORC_MATTER_OFF) return 0.0;
    if (r < v->Rnu) return NAN;
    const double m = v->Mns / 1.4, s = 100.0 / v->S, x = 10.0 / r;
    const double pl = 4.2e30 * v->gs * m * m * m * s * s * s * s * x * x * x;
    const double ex = v->nb0 * exp(-(r - v->Rnu) / v->hNS);
    double nb = 0.0;
    switch (v->matter_profile) {
        case ORC_MATTER_POWERLAW: nb = pl; break;
        case ORC_MATTER_EXP: nb = ex; break;
        case ORC_MATTER_SUM: nb = pl + ex; break;
    }
    return matter_A(v->Ye * nb);
}

/* -------------------------------------------------------------- kernels */
/* flavor::evolve_bin, beam.hpp:105-121 */
static void evolve_bin(double h11, double hre, double him, double dl, double ar, double ai,
                       double br, double bi, double* o) {
    const double lam = sqrt(h11 * h11 + hre * hre + him * him);
    const double ldl = lam * dl;
    const double c = cos(ldl);
    const double s = (ldl < 1e-12) ? dl : sin(ldl) / lam;
    const double a = h11 * s, b = hre * s, d = him * s;
    o[0] = c * ar + a * ai + d * br + b * bi;
    o[1] = c * ai - a * ar + d * bi - b * br;
    o[2] = c * br - a * bi - d * ar + b * ai;
    o[3] = c * bi + a * br - d * ai - b * ar;
}
void orc_evolve_bin(const double* h, double dl, const double* psi, double* out) {
    evolve_bin(h[0], h[1], h[2], dl, psi[0], psi[1], psi[2], psi[3], out);
}
/* flavor::density, beam.hpp:96-100 */
static void density(double ar, double ai, double br, double bi, double* r) {
    r[0] = ar * ar + ai * ai - br * br - bi * bi;
    r[1] = 2.0 * (ar * br + ai * bi);
    r[2] = 2.0 * (ai * br - ar * bi);
}
void orc_density(const double* psi, double* out) { density(psi[0], psi[1], psi[2], psi[3], out); }

/* splitmix64 noise, beam.cpp:10-21 */
static uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
static double unit_noise(uint64_t seed, uint64_t bin, uint64_t comp) {
    const uint64_t h = mix64(seed ^ mix64(bin * 4 + comp));
    return ((double)(h >> 11) * 0x1.0p-53) - 0.5;
}
/* BeamState::init_flavor_state(eps, seed), beam.cpp:30-57; out=[4][E] */
void orc_init_state(int species, int E, double eps, uint64_t seed, double* out) {
    const int e_flav = species < 2;
    for (int e = 0; e < E; ++e) {
        out[0 * E + e] = e_flav ? 1.0 : 0.0;
        out[1 * E + e] = 0.0;
        out[2 * E + e] = e_flav ? 0.0 : 1.0;
        out[3 * E + e] = 0.0;
    }
    if (eps == 0.0) return;
    for (int e = 0; e < E; ++e) {
        const double u = eps * unit_noise(seed, (uint64_t)e, 0);
        const double v = eps * unit_noise(seed, (uint64_t)e, 1);
        const double q = 1.0 - u * u - v * v;
        const double w = sqrt(q > 0.0 ? q : 0.0);
        if (e_flav) { out[0 * E + e] = w; out[2 * E + e] = u; }
        else { out[0 * E + e] = u; out[2 * E + e] = w; }
        out[3 * E + e] = v;
    }
}

/* --------------------------------------------------------------- engine */
enum { S_PSI0, S_MID, S_FULL1, S_FULL2, S_AVGA, S_HALF2, S_FULL3, S_RESULT, S_NSETS };

typedef struct { double cos_t, sin_t, w, dl; } CacheRow;

struct OrcEngine {
    const OrcEnv* env;
    int t_lo, t_hi, ntraj; /* local trajectories = (t_hi-t_lo)*P */
    size_t nbeam;          /* doubles per set: ntraj*4*4*E */
    double* set[S_NSETS];
    CacheRow* cache[3];    /* [abins] each, local range filled */
    double* dlj[3];        /* [local traj] dl slots (per trajectory) */
    double r, dr, A[3];
    double sums[4][12];    /* sums0..sums3 totals */
    double (*hvvA)[3], (*hvvB)[3], (*hvvC)[3];
    double (*rows_a)[3], (*rows_b)[3];
};

static double* beam_ptr(OrcEngine* g, int set, int j_local, int s) {
    return g->set[set] + ((size_t)j_local * 4 + s) * 4 * g->env->E;
}

int orc_make_partitions(int len, int workers, int* out) { /* parallel.cpp:11-24 */
    if (workers < 1 || len < 0) { set_err("make_partitions: bad arguments"); return 1; }
    const int base = len / workers, extra = len % workers;
    int at = 0;
    for (int w = 0; w < workers; ++w) {
        const int n = base + (w < extra ? 1 : 0);
        out[2 * w] = at;
        out[2 * w + 1] = at + n;
        at += n;
    }
    return 0;
}

int orc_engine_create(const OrcEnv* env, int t_lo, int t_hi, OrcEngine** out) {
    if (t_lo < 0 || t_hi > env->T || t_lo > t_hi) { set_err("bad theta range"); return 1; }
    OrcEngine* g = calloc(1, sizeof *g);
    g->env = env;
    g->t_lo = t_lo;
    g->t_hi = t_hi;
    g->ntraj = (t_hi - t_lo) * env->P;
    g->nbeam = (size_t)g->ntraj * 16 * env->E;
    for (int k = 0; k < S_NSETS; ++k) g->set[k] = calloc(g->nbeam ? g->nbeam : 1, sizeof(double));
    for (int k = 0; k < 3; ++k) g->cache[k] = calloc(env->T, sizeof(CacheRow));
    for (int k = 0; k < 3; ++k) g->dlj[k] = calloc(g->ntraj ? g->ntraj : 1, sizeof(double));
    const size_t nt = g->ntraj ? g->ntraj : 1;
    g->hvvA = calloc(nt, sizeof *g->hvvA);
    g->hvvB = calloc(nt, sizeof *g->hvvB);
    g->hvvC = calloc(nt, sizeof *g->hvvC);
    g->rows_a = calloc(nt * 4, sizeof *g->rows_a);
    g->rows_b = calloc(nt * 4, sizeof *g->rows_b);
    *out = g;
    return 0;
}

void orc_engine_destroy(OrcEngine* g) {
    if (!g) return;
    for (int k = 0; k < S_NSETS; ++k) free(g->set[k]);
    for (int k = 0; k < 3; ++k) free(g->cache[k]);
    for (int k = 0; k < 3; ++k) free(g->dlj[k]);
    free(g->hvvA); free(g->hvvB); free(g->hvvC); free(g->rows_a); free(g->rows_b);
    free(g);
}

/* init_lane_states, solver.cpp:255-271: psi0 seeded with the global beam
 * index idx = j*4 + s (partition independent); other sets pure flavour. */
void orc_init_states(OrcEngine* g) {
    const int E = g->env->E;
    for (int jl = 0; jl < g->ntraj; ++jl) {
        const int j = g->t_lo * g->env->P + jl;
        for (int s = 0; s < 4; ++s) {
            orc_init_state(s, E, g->env->perturb, (uint64_t)(j * 4 + s), beam_ptr(g, S_PSI0, jl, s));
            for (int k = 1; k < S_NSETS; ++k) orc_init_state(s, E, 0.0, 0, beam_ptr(g, k, jl, s));
        }
    }
}

void orc_set_state(OrcEngine* g, const double* mode1) {
    memcpy(g->set[S_PSI0], mode1, sizeof(double) * g->nbeam);
}
void orc_get_state(const OrcEngine* g, double* mode1) {
    memcpy(mode1, g->set[S_PSI0], sizeof(double) * g->nbeam);
}

/* Plane / cylinder geometry of trajectory (t, q) at radius r (restatement,
 * parity unpinned): weight w, direction factors n (1 - v.v' = 1 - n.n'
 * after the constant term) and path cosine cdl. */
static void geo34(const OrcEnv* v, int t, int q, double r, double* w, double* n, double* cdl) {
    if (v->model == ORC_PLANE) {
        const double ct = v->cos2[t], st = v->sin0[t];
        *w = 1.0 / ((double)v->T * v->P);
        n[0] = ct;
        n[1] = st * v->cphi[q];
        n[2] = st * v->sphi[q];
        *cdl = ct;
    } else {
        const double ra = v->Rnu / r;
        const double sa = ra * v->sin0[t];
        const double ca = sqrt(1.0 - sa * sa);
        *w = ra * (v->cos2[t] / ca) / ((double)v->T * v->P);
        n[0] = v->cphi[q] * ca;
        n[1] = v->cphi[q] * sa;
        n[2] = v->sphi[q];
        *cdl = n[0];
    }
}

/* fill_cache, geometry.cpp:66-87 */
static void fill_cache(const OrcEngine* g, CacheRow* c, double r) {
    const OrcEnv* v = g->env;
    if (v->model == ORC_SINGLE_ANGLE) {
        c[0].cos_t = 1.0;
        c[0].sin_t = 0.0;
        c[0].w = 1.0;
        return;
    }
    const double ra = v->Rnu / r;
    const double dcos2 = 1.0 / v->T;
    const double pm = (v->model == ORC_EXT_BULB) ? 1.0 / v->P : 1.0;
    for (int t = g->t_lo; t < g->t_hi; ++t) {
        const double ct = sqrt(1.0 - ra * ra * (1.0 - v->cos2[t]));
        c[t].cos_t = ct;
        c[t].sin_t = ra * v->sin0[t];
        c[t].w = 0.5 * ra * ra * dcos2 / ct * pm;
    }
}
/* calc_delta_ls, geometry.cpp:89-97 */
static void delta_ls(const OrcEngine* g, CacheRow* dst, const CacheRow* s, const CacheRow* e,
                     double dr) {
    for (int t = g->t_lo; t < g->t_hi; ++t) dst[t].dl = dr / (0.5 * (s[t].cos_t + e[t].cos_t));
}

/* e_sum (beam.cpp:84-103): sequential low -> high over bins */
static void e_sum(const double* b, const double* fw, int E, double* row) {
    double r0 = 0.0, r1 = 0.0, r2 = 0.0;
    for (int e = 0; e < E; ++e) {
        double rho[3];
        density(b[e], b[E + e], b[2 * E + e], b[3 * E + e], rho);
        r0 += rho[0] * fw[e];
        r1 += rho[1] * fw[e];
        r2 += rho[2] * fw[e];
    }
    row[0] = r0; row[1] = r1; row[2] = r2;
}

/* combine_species + fold_rows + (partial) combine_stage,
 * geometry.cpp:119-182: local theta ascending, 12 doubles (a,b,c,d). */
static void fold(const OrcEngine* g, const CacheRow* c, double (*rows)[3], double* out12) {
    const OrcEnv* v = g->env;
    for (int k = 0; k < 12; ++k) out12[k] = 0.0;
    if (v->model >= ORC_PLANE) { /* per-trajectory weights, ascending trajectory order */
        for (int jl = 0; jl < g->ntraj; ++jl) {
            const int t = g->t_lo + jl / v->P, q = jl % v->P;
            double R[3] = {0, 0, 0};
            for (int s = 0; s < 4; ++s) {
                const double* rw = rows[jl * 4 + s];
                const double cs = v->coupling[s];
                if (s & 1) { R[0] -= cs * rw[0]; R[1] -= cs * rw[1]; R[2] -= cs * (-rw[2]); }
                else { R[0] += cs * rw[0]; R[1] += cs * rw[1]; R[2] += cs * rw[2]; }
            }
            double w, n[3], cdl;
            geo34(v, t, q, c[0].w /* radius carried in w slot, see orc_prepare */, &w, n, &cdl);
            for (int k = 0; k < 3; ++k) {
                out12[k] += R[k] * w;
                out12[3 + k] += R[k] * (w * n[0]);
                out12[6 + k] += R[k] * (w * n[1]);
                out12[9 + k] += R[k] * (w * n[2]);
            }
        }
        return;
    }
    for (int t = g->t_lo; t < g->t_hi; ++t) {
        double acc[3] = {0, 0, 0}, acc_c[3] = {0, 0, 0}, acc_s[3] = {0, 0, 0};
        for (int q = 0; q < v->P; ++q) {
            const int jl = (t - g->t_lo) * v->P + q;
            double R[3] = {0, 0, 0};
            for (int s = 0; s < 4; ++s) {
                const double* rw = rows[jl * 4 + s];
                const double cs = v->coupling[s];
                if (s & 1) { /* antiparticle: minus the conjugate row */
                    R[0] -= cs * rw[0];
                    R[1] -= cs * rw[1];
                    R[2] -= cs * (-rw[2]);
                } else {
                    R[0] += cs * rw[0];
                    R[1] += cs * rw[1];
                    R[2] += cs * rw[2];
                }
            }
            for (int k = 0; k < 3; ++k) acc[k] += R[k];
            if (v->model == ORC_EXT_BULB)
                for (int k = 0; k < 3; ++k) {
                    acc_c[k] += R[k] * v->cphi[q];
                    acc_s[k] += R[k] * v->sphi[q];
                }
        }
        double rs[12] = {0};
        switch (v->model) {
            case ORC_SINGLE_ANGLE:
                for (int k = 0; k < 3; ++k) rs[k] = acc[k];
                break;
            case ORC_BULB:
                for (int k = 0; k < 3; ++k) {
                    rs[k] = acc[k] * c[t].w;
                    rs[3 + k] = acc[k] * (c[t].w * c[t].cos_t);
                }
                break;
            default:
                for (int k = 0; k < 3; ++k) {
                    rs[k] = acc[k] * c[t].w;
                    rs[3 + k] = acc[k] * (c[t].w * c[t].cos_t);
                    rs[6 + k] = acc_c[k] * (c[t].w * c[t].sin_t);
                    rs[9 + k] = acc_s[k] * (c[t].w * c[t].sin_t);
                }
        }
        for (int k = 0; k < 12; ++k) out12[k] += rs[k];
    }
}

/* assemble_hvv, geometry.cpp:192-216 (with D, geometry.cpp:28-34) */
static void assemble(const OrcEngine* g, const CacheRow* c, const double* s12, double r,
                     double (*dst)[3]) {
    const OrcEnv* v = g->env;
    if (v->model >= ORC_PLANE) {
        for (int jl = 0; jl < g->ntraj; ++jl) {
            const int t = g->t_lo + jl / v->P, q = jl % v->P;
            double w, n[3], cdl;
            geo34(v, t, q, r, &w, n, &cdl);
            for (int k = 0; k < 3; ++k)
                dst[jl][k] = 0.5 * (s12[k] + s12[3 + k] * (-n[0]) + s12[6 + k] * (-n[1]) + s12[9 + k] * (-n[2]));
        }
        return;
    }
    for (int t = g->t_lo; t < g->t_hi; ++t)
        for (int q = 0; q < v->P; ++q) {
            const int jl = (t - g->t_lo) * v->P + q;
            double row[3];
            if (v->model == ORC_SINGLE_ANGLE) {
                const double ra = v->Rnu / r;
                const double tt = 1.0 - sqrt(1.0 - ra * ra);
                const double D = 0.5 * tt * tt;
                for (int k = 0; k < 3; ++k) row[k] = s12[k] * D;
            } else if (v->model == ORC_BULB) {
                const double ct = c[t].cos_t;
                for (int k = 0; k < 3; ++k) row[k] = s12[k] + s12[3 + k] * (-ct);
            } else {
                const double ct = c[t].cos_t, st = c[t].sin_t;
                for (int k = 0; k < 3; ++k)
                    row[k] = s12[k] + s12[3 + k] * (-ct) + s12[6 + k] * (-st * v->cphi[q]) +
                             s12[9 + k] * (-st * v->sphi[q]);
            }
            for (int k = 0; k < 3; ++k) dst[jl][k] = 0.5 * row[k];
        }
}

/* evolve_pass (solver.cpp:276-311) with beam_ham (beam.hpp:134-138).
 * mode: 0 plain evolve (+rows if rows != NULL), 1 evolve_avg, 2 evolve_avg_err */
static double pass(OrcEngine* g, double (*hvv)[3], int dl_slot, double A, int in, int out,
                   double (*rows)[3], int avg, int err_ref) {
    const OrcEnv* v = g->env;
    const int E = v->E;
    double err = 0.0;
    for (int jl = 0; jl < g->ntraj; ++jl) {
        const int t = g->t_lo + jl / v->P;
        const double dl = g->dlj[dl_slot][jl];
        (void)t;
        for (int s = 0; s < 4; ++s) {
            double hb[3];
            if (s & 1) { hb[0] = -(hvv[jl][0] + 0.5 * A); hb[1] = -hvv[jl][1]; hb[2] = hvv[jl][2]; }
            else { hb[0] = hvv[jl][0] + 0.5 * A; hb[1] = hvv[jl][1]; hb[2] = hvv[jl][2]; }
            const double* pi = beam_ptr(g, in, jl, s);
            double* po = beam_ptr(g, out, jl, s);
            for (int e = 0; e < E; ++e) {
                double o[4];
                evolve_bin(v->vac11[e] + hb[0], v->vac12[e] + hb[1], hb[2], dl, pi[e], pi[E + e],
                           pi[2 * E + e], pi[3 * E + e], o);
                for (int k = 0; k < 4; ++k) po[k * E + e] = o[k];
            }
            if (rows) e_sum(po, v->fw + s * E, E, rows[jl * 4 + s]);
            if (avg >= 0) {
                double* pa = beam_ptr(g, avg, jl, s);
                for (int k = 0; k < 4 * E; ++k) pa[k] = (pa[k] + po[k]) * 0.5;
                if (err_ref >= 0) { /* calc_err over logical bins, beam.cpp:125-136 */
                    const double* pr = beam_ptr(g, err_ref, jl, s);
                    for (int e = 0; e < E; ++e)
                        for (int k = 0; k < 4; ++k) {
                            const double d = fabs(pr[k * E + e] - pa[k * E + e]);
                            if (d > err || d != d) err = (d != d) ? d : (err > d ? err : d);
                        }
                }
            }
        }
    }
    return err;
}

static void copy_set(OrcEngine* g, int dst, int src) {
    memcpy(g->set[dst], g->set[src], sizeof(double) * g->nbeam);
}

/* do_step prologue: caches, dl slots, matter (solver.cpp:349-359) */
int orc_prepare(OrcEngine* g, double r, double dr) {
    g->r = r;
    g->dr = dr;
    if (g->env->model >= ORC_PLANE) {
        const OrcEnv* v = g->env;
        const double rk[3] = {r, r + 0.5 * dr, r + dr};
        if (v->model == ORC_CYLINDER && r < v->Rnu) {
            set_err("cylinder: r below the emitting surface");
            return 2;
        }
        for (int k = 0; k < 3; ++k) g->cache[k][0].w = rk[k]; /* radius for fold() */
        for (int jl = 0; jl < g->ntraj; ++jl) {
            const int t = g->t_lo + jl / v->P, q = jl % v->P;
            double w, n[3], c[3];
            for (int k = 0; k < 3; ++k) geo34(v, t, q, rk[k], &w, n, &c[k]);
            g->dlj[0][jl] = 0.5 * dr / (0.5 * (c[0] + c[1]));
            g->dlj[1][jl] = 0.5 * dr / (0.5 * (c[1] + c[2]));
            g->dlj[2][jl] = dr / (0.5 * (c[0] + c[2]));
        }
        g->A[0] = orc_matter_potential(v, r);
        g->A[1] = orc_matter_potential(v, r + 0.5 * dr);
        g->A[2] = orc_matter_potential(v, r + dr);
        return 0;
    }
    if (g->env->model != ORC_SINGLE_ANGLE && r < g->env->Rnu) {
        set_err("fill_cache: r below the neutrino sphere");
        return 2;
    }
    fill_cache(g, g->cache[0], r);
    fill_cache(g, g->cache[1], r + 0.5 * dr);
    fill_cache(g, g->cache[2], r + dr);
    if (g->env->model == ORC_SINGLE_ANGLE) {
        g->cache[0][0].dl = 0.5 * dr / (0.5 * (g->cache[0][0].cos_t + g->cache[1][0].cos_t));
        g->cache[1][0].dl = 0.5 * dr / (0.5 * (g->cache[1][0].cos_t + g->cache[2][0].cos_t));
        g->cache[2][0].dl = dr / (0.5 * (g->cache[0][0].cos_t + g->cache[2][0].cos_t));
    } else {
        delta_ls(g, g->cache[0], g->cache[0], g->cache[1], 0.5 * dr);
        delta_ls(g, g->cache[1], g->cache[1], g->cache[2], 0.5 * dr);
        delta_ls(g, g->cache[2], g->cache[0], g->cache[2], dr);
    }
    for (int jl = 0; jl < g->ntraj; ++jl)
        for (int k = 0; k < 3; ++k) g->dlj[k][jl] = g->cache[k][g->t_lo + jl / g->env->P].dl;
    g->A[0] = orc_matter_potential(g->env, r);
    g->A[1] = orc_matter_potential(g->env, r + 0.5 * dr);
    g->A[2] = orc_matter_potential(g->env, r + dr);
    return 0;
}

/* S1-S4 of do_step (solver.cpp:361-411), split at the reduction points. */
int orc_stage(OrcEngine* g, int stage, double* partial) {
    switch (stage) {
        case 0: /* S1 */
            for (int jl = 0; jl < g->ntraj; ++jl)
                for (int s = 0; s < 4; ++s)
                    e_sum(beam_ptr(g, S_PSI0, jl, s), g->env->fw + s * g->env->E, g->env->E,
                          g->rows_a[jl * 4 + s]);
            fold(g, g->cache[0], g->rows_a, partial);
            return 0;
        case 1: /* S2 */
            pass(g, g->hvvA, 0, g->A[0], S_PSI0, S_MID, g->rows_b, -1, -1);
            pass(g, g->hvvA, 2, g->A[0], S_PSI0, S_FULL1, g->rows_a, -1, -1);
            fold(g, g->cache[2], g->rows_a, partial);
            fold(g, g->cache[1], g->rows_b, partial + 12);
            return 0;
        case 2: /* S3 */
            copy_set(g, S_AVGA, S_FULL1);
            pass(g, g->hvvB, 2, g->A[2], S_PSI0, S_FULL2, NULL, S_AVGA, -1);
            pass(g, g->hvvC, 1, g->A[1], S_MID, S_HALF2, g->rows_a, -1, -1);
            fold(g, g->cache[2], g->rows_a, partial);
            return 0;
        case 3: /* S4 */
            copy_set(g, S_RESULT, S_HALF2);
            partial[0] = pass(g, g->hvvA, 2, g->A[2], S_PSI0, S_FULL3, NULL, S_RESULT, S_AVGA);
            return 0;
    }
    set_err("bad stage");
    return 1;
}

static int finite12(const double* s) {
    for (int k = 0; k < 12; ++k)
        if (!isfinite(s[k])) return 0;
    return 1;
}

int orc_stage_set(OrcEngine* g, int stage, const double* total) {
    switch (stage) {
        case 0:
            memcpy(g->sums[0], total, sizeof(double) * 12);
            assemble(g, g->cache[0], g->sums[0], g->r, g->hvvA);
            return 0;
        case 1:
            memcpy(g->sums[1], total, sizeof(double) * 12);
            memcpy(g->sums[2], total + 12, sizeof(double) * 12);
            assemble(g, g->cache[2], g->sums[1], g->r + g->dr, g->hvvB);
            assemble(g, g->cache[1], g->sums[2], g->r + 0.5 * g->dr, g->hvvC);
            return 0;
        case 2:
            memcpy(g->sums[3], total, sizeof(double) * 12);
            for (int k = 0; k < 4; ++k) /* check_sums_finite, solver.cpp:243-253 */
                if (!finite12(g->sums[k])) {
                    set_err("non-finite Hamiltonian sum");
                    return 2;
                }
            assemble(g, g->cache[2], g->sums[3], g->r + g->dr, g->hvvA);
            return 0;
    }
    return 0;
}

void orc_commit(OrcEngine* g) {
    double* t = g->set[S_PSI0];
    g->set[S_PSI0] = g->set[S_RESULT];
    g->set[S_RESULT] = t;
}

int orc_trial_step(OrcEngine* g, double r, double dr, double* err) {
    double buf[24];
    int rc = orc_prepare(g, r, dr);
    for (int st = 0; st < 4 && rc == 0; ++st) {
        rc = orc_stage(g, st, buf);
        if (rc == 0 && st < 3) rc = orc_stage_set(g, st, buf);
    }
    *err = buf[0];
    return rc;
}

/* step_size_update, solver.cpp:44-52 */
double orc_step_size_update(const OrcCtl* c, double err, int accepted, int* collapse) {
    *collapse = 0;
    const double raw = c->kappa * c->dr * sqrt(c->eps0 / (err > 1e-300 ? err : 1e-300));
    if (!accepted && raw < c->dr_min) { *collapse = 1; return raw; }
    return raw < c->dr_min ? c->dr_min : (c->dr_max < raw ? c->dr_max : raw);
}

double orc_max_norm_dev(const OrcEngine* g) { /* norm_deviation, beam.cpp:147-155 */
    const int E = g->env->E;
    double m = 0.0;
    for (int b = 0; b < g->ntraj * 4; ++b) {
        const double* p = g->set[S_PSI0] + (size_t)b * 4 * E;
        for (int e = 0; e < E; ++e) {
            const double n2 = p[e] * p[e] + p[E + e] * p[E + e] + p[2 * E + e] * p[2 * E + e] +
                              p[3 * E + e] * p[3 * E + e];
            const double d = fabs(n2 - 1.0);
            if (d > m) m = d;
        }
    }
    return m;
}

/* Engine::run + lane_body on one rank, solver.cpp:414-456, 486-525 */
int orc_run(OrcEngine* g, const OrcCtl* in, OrcSummary* out) {
    OrcCtl c = *in;
    double pr = c.r, pdr = c.dr < (c.Rn - c.r > 0 ? c.Rn - c.r : 0) ? c.dr : (c.Rn - c.r > 0 ? c.Rn - c.r : 0);
    uint64_t piter = c.iter;
    const double r_eps = 1e-12 * (fabs(c.Rn) > 1.0 ? fabs(c.Rn) : 1.0);
    int term = (c.r >= c.Rn - r_eps) ? 1 : 0;
    if (c.Ts > 0 && c.iter >= c.Ts) term = 2;
    uint64_t acc = 0, rej = 0;
    while (!term) {
        double err;
        int rc = orc_trial_step(g, pr, pdr, &err);
        if (rc) return rc;
        if (!isfinite(err)) { set_err("non-finite amplitudes"); return 2; }
        const int accept = err <= c.eps0;
        c.iter = piter + 1;
        c.dr = pdr;
        if (accept) { orc_commit(g); c.r = pr + pdr; ++acc; }
        else ++rej;
        int collapse;
        double next = orc_step_size_update(&c, err, accept, &collapse);
        if (collapse) { set_err("step collapse"); return 2; }
        if (c.r + next > c.Rn) next = c.Rn - c.r;
        pr = c.r;
        pdr = next;
        piter = c.iter;
        if (c.r >= c.Rn - r_eps) term = 1;
        else if (c.Ts > 0 && c.iter >= c.Ts) term = 2;
    }
    out->final_r = c.r;
    out->iterations = c.iter - in->iter;
    out->accepted = acc;
    out->rejected = rej;
    out->final_max_norm_dev = orc_max_norm_dev(g);
    out->termination = term;
    return 0;
}

/* fold_rows + combine_stage + assemble_hvv on caller-supplied rows
 * ([local traj*4+s][3]) at radius r (test hook; mirrors ref_partial_hvv). */
int orc_hvv_from_rows(OrcEngine* g, double r, const double* rows, double* sums12, double* hvv) {
    int rc = orc_prepare(g, r, 0.0);
    if (rc) return rc;
    memcpy(g->rows_a, rows, sizeof(double) * 3 * 4 * (size_t)g->ntraj);
    fold(g, g->cache[0], g->rows_a, sums12);
    assemble(g, g->cache[0], sums12, r, (double(*)[3])hvv);
    return 0;
}
