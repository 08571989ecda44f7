/* TEST INFRASTRUCTURE ONLY — CPU oracle for the 3-flavour path (BASELINE
 * configs[1]).  PARITY UNPINNED w.r.t. the reference, which rejects Flvs != 2
 * (config.cpp:298).  This is a restatement of the reference's
 * 2-flavour step (solver.cpp:343-412) generalised from SU(2) to SU(3):
 *   psi in C^3 per (trajectory, species, energy bin), species
 *     0 nu_e, 1 nubar_e, 2 nu_mu, 3 nubar_mu, 4 nu_tau, 5 nubar_tau;
 *   rho = psi psi^dagger (paper Eq. 3.9 without the traceless shift, which
 *     only adds a multiple of the identity to H);
 *   H_nu = U diag(0, dm21, dm31)/2E U^dagger + diag(A,0,0)
 *          + sum_s +-c_s int f (1 - v.v') rho_s  (antiparticles conjugated,
 *          Eq. 3.8); H_nubar = conj(H_vac) - diag(A,0,0) - conj(H_nunu);
 *   exp(-i H dl) by scaling-and-squaring Taylor in long double (independent
 *   of the closed form used on the device).
 * Self-consistency pins (tests/test_flavor3.py): with theta13 = theta23 = 0
 * and a dark tau sector the e-mu densities reproduce the 2-flavour reference;
 * unitarity; series exponential.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oscflat_oracle.h"

typedef long double complex lcx;

struct Orc3Env {
    Orc3Params p;
    int T, P, E;
    double *cos2, *sin0, *cphi, *sphi;
    double* vac;  /* [E][9]: d0 d1 d2, re/im h01, h02, h12 */
    double* fw;   /* [6][E] */
    double coupling[6];
    OrcEnv* env2; /* matter / Fermi helpers of the 2-flavour oracle */
};

static char g3_err[256];
const char* orc3_last_error(void) { return g3_err; }



static double per_km(double mev) { return mev / 197.327e-18; }

int orc3_env_create(const Orc3Params* p, Orc3Env** out) {
    Orc3Env* v = calloc(1, sizeof *v);
    v->p = *p;
    v->T = p->abins;
    v->P = p->pbins;
    if (p->model == ORC_SINGLE_ANGLE) v->T = v->P = 1;
    if (p->model == ORC_BULB) v->P = 1;
    v->E = p->ebins;
    /* 2-flavour env for grid, spectra of species 0..3 and matter */
    OrcParams q;
    memset(&q, 0, sizeof q);
    q.model = p->model;
    q.abins = p->abins;
    q.pbins = p->pbins;
    q.ebins = p->ebins;
    q.Rnu = p->Rnu;
    q.E0 = p->E0;
    q.E1 = p->E1;
    q.dm2 = p->dm21;
    q.theta = p->th12;
    q.hvv_scale = p->hvv_scale;
    q.perturb = p->perturb;
    for (int s = 0; s < 4; ++s) {
        q.L[s] = p->L[s];
        q.T[s] = p->T[s];
        q.Emean[s] = p->Emean[s];
        q.eta[s] = p->eta[s];
    }
    q.matter_profile = p->matter_profile;
    q.Ye = p->Ye;
    q.nb0 = p->nb0;
    q.hNS = p->hNS;
    q.Mns = p->Mns;
    q.gs = p->gs;
    q.S = p->S;
    if (orc_env_create(&q, &v->env2)) { free(v); snprintf(g3_err, sizeof g3_err, "%s", orc_last_error()); return 1; }
    /* tau sector spectra: a second 2-flavour env whose species 2,3 are tau */
    OrcParams qt = q;
    qt.L[2] = p->L[4]; qt.L[3] = p->L[5];
    qt.T[2] = p->T[4]; qt.T[3] = p->T[5];
    qt.Emean[2] = p->Emean[4]; qt.Emean[3] = p->Emean[5];
    qt.eta[2] = p->eta[4]; qt.eta[3] = p->eta[5];
    OrcEnv* et;
    if (orc_env_create(&qt, &et)) { free(v); snprintf(g3_err, sizeof g3_err, "%s", orc_last_error()); return 1; }
    const int T = v->T, P = v->P, E = v->E;
    v->cos2 = malloc(sizeof(double) * T);
    v->sin0 = malloc(sizeof(double) * T);
    v->cphi = malloc(sizeof(double) * P);
    v->sphi = malloc(sizeof(double) * P);
    double* fw4 = malloc(sizeof(double) * 4 * E);
    double* fwt = malloc(sizeof(double) * 4 * E);
    double* tmpE = malloc(sizeof(double) * E);
    double c4[4], ct4[4], em[4];
    orc_env_tables(v->env2, v->cos2, v->sin0, v->cphi, v->sphi, tmpE, tmpE, fw4, c4, em);
    double* dummyT = malloc(sizeof(double) * (T > P ? T : P));
    orc_env_tables(et, dummyT, dummyT, dummyT, dummyT, tmpE, tmpE, fwt, ct4, em);
    v->fw = malloc(sizeof(double) * 6 * E);
    for (int s = 0; s < 4; ++s) {
        memcpy(v->fw + s * E, fw4 + s * E, sizeof(double) * E);
        v->coupling[s] = c4[s];
    }
    memcpy(v->fw + 4 * E, fwt + 2 * E, sizeof(double) * 2 * E);
    v->coupling[4] = ct4[2];
    v->coupling[5] = ct4[3];
    free(fw4); free(fwt); free(tmpE); free(dummyT);
    orc_env_destroy(et);
    /* vacuum: U diag(0, d21, d31) U^dagger, standard PMNS parametrisation */
    const double c12 = cos(p->th12), s12 = sin(p->th12), c13 = cos(p->th13), s13 = sin(p->th13);
    const double c23 = cos(p->th23), s23 = sin(p->th23);
    const double complex ed = cexp(I * p->dcp);
    double complex U[3][3] = {
        {c12 * c13, s12 * c13, s13 * conj(ed)},
        {-s12 * c23 - c12 * s23 * s13 * ed, c12 * c23 - s12 * s23 * s13 * ed, s23 * c13},
        {s12 * s23 - c12 * c23 * s13 * ed, -c12 * s23 - s12 * c23 * s13 * ed, c23 * c13}};
    v->vac = malloc(sizeof(double) * 9 * E);
    const double dE = (p->E1 - p->E0) / E;
    for (int e = 0; e < E; ++e) {
        const double Ec = p->E0 + (e + 0.5) * dE;
        const double lam[3] = {0.0, per_km(p->dm21 * 1e-12 / (2.0 * Ec)), per_km(p->dm31 * 1e-12 / (2.0 * Ec))};
        double complex H[3][3];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                double complex acc = 0;
                for (int k = 0; k < 3; ++k) acc += U[i][k] * lam[k] * conj(U[j][k]);
                H[i][j] = acc;
            }
        double* o = v->vac + 9 * e;
        o[0] = creal(H[0][0]); o[1] = creal(H[1][1]); o[2] = creal(H[2][2]);
        o[3] = creal(H[0][1]); o[4] = cimag(H[0][1]);
        o[5] = creal(H[0][2]); o[6] = cimag(H[0][2]);
        o[7] = creal(H[1][2]); o[8] = cimag(H[1][2]);
    }
    *out = v;
    return 0;
}

void orc3_env_destroy(Orc3Env* v) {
    if (!v) return;
    orc_env_destroy(v->env2);
    free(v->cos2); free(v->sin0); free(v->cphi); free(v->sphi); free(v->vac); free(v->fw);
    free(v);
}

/* tables: vac[E*9], fw[6*E], couplings[6] */
void orc3_env_tables(const Orc3Env* v, double* vac, double* fw, double* couplings) {
    memcpy(vac, v->vac, sizeof(double) * 9 * v->E);
    memcpy(fw, v->fw, sizeof(double) * 6 * v->E);
    memcpy(couplings, v->coupling, sizeof(double) * 6);
}

/* ---- exp(-i H tau) by scaling and squaring (long double) */
static void mat_mul(lcx a[3][3], lcx b[3][3], lcx c[3][3]) {
    lcx t[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            t[i][j] = 0;
            for (int k = 0; k < 3; ++k) t[i][j] += a[i][k] * b[k][j];
        }
    memcpy(c, t, sizeof t);
}
void orc3_expm(const double* h9, double tau, double* out18) {
    lcx M[3][3];
    const long double d[3] = {h9[0], h9[1], h9[2]};
    const lcx o01 = h9[3] + I * (long double)h9[4], o02 = h9[5] + I * (long double)h9[6],
              o12 = h9[7] + I * (long double)h9[8];
    lcx H[3][3] = {{d[0], o01, o02}, {conjl(o01), d[1], o12}, {conjl(o02), conjl(o12), d[2]}};
    long double nrm = 0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            M[i][j] = -I * (long double)tau * H[i][j];
            nrm += cabsl(M[i][j]);
        }
    int sq = 0;
    while (nrm > 0.125L) { nrm *= 0.5L; ++sq; }
    const long double sc = ldexpl(1.0L, -sq);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) M[i][j] *= sc;
    lcx S[3][3], T[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) S[i][j] = T[i][j] = (i == j);
    for (int k = 1; k <= 22; ++k) {
        mat_mul(T, M, T);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                T[i][j] /= k;
                S[i][j] += T[i][j];
            }
    }
    for (int s = 0; s < sq; ++s) mat_mul(S, S, S);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            out18[2 * (3 * i + j)] = (double)creall(S[i][j]);
            out18[2 * (3 * i + j) + 1] = (double)cimagl(S[i][j]);
        }
}

/* ---- engine */
enum { Q_PSI0, Q_MID, Q_FULL1, Q_FULL2, Q_AVGA, Q_HALF2, Q_FULL3, Q_RESULT, Q_NSETS };
struct Orc3Engine {
    const Orc3Env* env;
    int t_lo, t_hi, ntraj;
    size_t n;
    double* set[Q_NSETS];
    double r, dr, A[3];
    double sums[4][36];
    double* hvv[4];   /* [traj][9] for H0..H3 (beam part, particle convention) */
    double* rows_a;   /* [traj][6][9] */
    double* rows_b;
    double* dlj[3];
};

static double* beam3(Orc3Engine* g, int set, int jl, int s) {
    return g->set[set] + ((size_t)jl * 6 + s) * 6 * g->env->E;
}

static uint64_t mix64b(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
static double noise3(uint64_t seed, uint64_t bin, uint64_t comp) {
    const uint64_t h = mix64b(seed ^ mix64b(bin * 4 + comp));
    return ((double)(h >> 11) * 0x1.0p-53) - 0.5;
}

/* pure initial flavour f = s/2 plus eps noise on the two other flavours
 * (generalises init_flavor_state, beam.cpp:41-57); comps re/im of e, mu, tau */
void orc3_init_state(int species, int E, double eps, uint64_t seed, double* out) {
    const int f = species / 2;
    for (int k = 0; k < 6 * E; ++k) out[k] = 0.0;
    for (int e = 0; e < E; ++e) out[(2 * f) * E + e] = 1.0;
    if (eps == 0.0) return;
    for (int e = 0; e < E; ++e) {
        const int o1 = (f + 1) % 3, o2 = (f + 2) % 3;
        const double u1 = eps * noise3(seed, e, 0), v1 = eps * noise3(seed, e, 1);
        const double u2 = eps * noise3(seed, e, 2), v2 = eps * noise3(seed, e, 3);
        const double q = 1.0 - u1 * u1 - v1 * v1 - u2 * u2 - v2 * v2;
        out[(2 * f) * E + e] = sqrt(q > 0 ? q : 0);
        out[(2 * o1) * E + e] = u1;
        out[(2 * o1 + 1) * E + e] = v1;
        out[(2 * o2) * E + e] = u2;
        out[(2 * o2 + 1) * E + e] = v2;
    }
}

int orc3_engine_create(const Orc3Env* env, int t_lo, int t_hi, Orc3Engine** out) {
    Orc3Engine* g = calloc(1, sizeof *g);
    g->env = env;
    g->t_lo = t_lo;
    g->t_hi = t_hi;
    g->ntraj = (t_hi - t_lo) * env->P;
    g->n = (size_t)g->ntraj * 36 * env->E;
    for (int k = 0; k < Q_NSETS; ++k) g->set[k] = calloc(g->n ? g->n : 1, sizeof(double));
    for (int k = 0; k < 4; ++k) g->hvv[k] = calloc((size_t)g->ntraj * 9 + 1, sizeof(double));
    g->rows_a = calloc((size_t)g->ntraj * 54 + 1, sizeof(double));
    g->rows_b = calloc((size_t)g->ntraj * 54 + 1, sizeof(double));
    for (int k = 0; k < 3; ++k) g->dlj[k] = calloc(g->ntraj + 1, sizeof(double));
    *out = g;
    return 0;
}
void orc3_engine_destroy(Orc3Engine* g) {
    if (!g) return;
    for (int k = 0; k < Q_NSETS; ++k) free(g->set[k]);
    for (int k = 0; k < 4; ++k) free(g->hvv[k]);
    free(g->rows_a); free(g->rows_b);
    for (int k = 0; k < 3; ++k) free(g->dlj[k]);
    free(g);
}
void orc3_init_states(Orc3Engine* g) {
    const int E = g->env->E;
    for (int jl = 0; jl < g->ntraj; ++jl) {
        const int j = g->t_lo * g->env->P + jl;
        for (int s = 0; s < 6; ++s)
            orc3_init_state(s, E, g->env->p.perturb, (uint64_t)(j * 6 + s), beam3(g, Q_PSI0, jl, s));
    }
}
void orc3_set_state(Orc3Engine* g, const double* m) { memcpy(g->set[Q_PSI0], m, sizeof(double) * g->n); }
void orc3_get_state(const Orc3Engine* g, double* m) { memcpy(m, g->set[Q_PSI0], sizeof(double) * g->n); }

/* geometry: w, direction n (bulb / ext-bulb / single angle), path cosine */
static void geo3(const Orc3Engine* g, int t, int q, double r, double* w, double* n, double* cdl) {
    const Orc3Env* v = g->env;
    if (v->p.model == ORC_SINGLE_ANGLE) { *w = 1; n[0] = 1; n[1] = n[2] = 0; *cdl = 1; return; }
    const double ra = v->p.Rnu / r;
    const double ct = sqrt(1.0 - ra * ra * (1.0 - v->cos2[t]));
    const double st = ra * v->sin0[t];
    const double pm = v->p.model == ORC_EXT_BULB ? 1.0 / v->P : 1.0;
    *w = 0.5 * ra * ra * (1.0 / v->T) / ct * pm;
    n[0] = ct;
    n[1] = v->p.model == ORC_EXT_BULB ? st * v->cphi[q] : 0.0;
    n[2] = v->p.model == ORC_EXT_BULB ? st * v->sphi[q] : 0.0;
    *cdl = ct;
}

/* rho = psi psi^dagger packed as 9 reals (d0 d1 d2, re/im 01, 02, 12) */
static void rho3(const double* x, double* r9) {
    const double complex a = x[0] + I * x[1], b = x[2] + I * x[3], c = x[4] + I * x[5];
    r9[0] = creal(a * conj(a)); r9[1] = creal(b * conj(b)); r9[2] = creal(c * conj(c));
    const double complex ab = a * conj(b), ac = a * conj(c), bc = b * conj(c);
    r9[3] = creal(ab); r9[4] = cimag(ab); r9[5] = creal(ac); r9[6] = cimag(ac);
    r9[7] = creal(bc); r9[8] = cimag(bc);
}

static void esum3(const double* b, const double* fw, int E, double* row9) {
    for (int k = 0; k < 9; ++k) row9[k] = 0;
    for (int e = 0; e < E; ++e) {
        double x[6], r9[9];
        for (int c = 0; c < 6; ++c) x[c] = b[c * E + e];
        rho3(x, r9);
        for (int k = 0; k < 9; ++k) row9[k] += r9[k] * fw[e];
    }
}

/* fold: 36 doubles = 4 geometric moments x 9 (a, b, c, d) */
static void fold3(const Orc3Engine* g, double r, const double* rows, double* out) {
    const Orc3Env* v = g->env;
    for (int k = 0; k < 36; ++k) out[k] = 0;
    for (int jl = 0; jl < g->ntraj; ++jl) {
        const int t = g->t_lo + jl / v->P, q = jl % v->P;
        double R[9] = {0};
        for (int s = 0; s < 6; ++s) {
            const double* rw = rows + ((size_t)jl * 6 + s) * 9;
            const double c = v->coupling[s];
            for (int k = 0; k < 9; ++k) {
                const double x = (s & 1) ? -((k == 4 || k == 6 || k == 8) ? -rw[k] : rw[k]) : rw[k];
                R[k] += c * x;
            }
        }
        double w, n[3], cdl;
        geo3(g, t, q, r, &w, n, &cdl);
        for (int k = 0; k < 9; ++k) {
            out[k] += w * R[k];
            out[9 + k] += w * n[0] * R[k];
            out[18 + k] += w * n[1] * R[k];
            out[27 + k] += w * n[2] * R[k];
        }
    }
}

static void assemble3(const Orc3Engine* g, double r, const double* s36, double A, double* dst) {
    const Orc3Env* v = g->env;
    for (int jl = 0; jl < g->ntraj; ++jl) {
        const int t = g->t_lo + jl / v->P, q = jl % v->P;
        double w, n[3], cdl;
        geo3(g, t, q, r, &w, n, &cdl);
        double* h = dst + (size_t)jl * 9;
        if (v->p.model == ORC_SINGLE_ANGLE) {
            const double ra = v->p.Rnu / r, tt = 1.0 - sqrt(1.0 - ra * ra), D = 0.5 * tt * tt;
            for (int k = 0; k < 9; ++k) h[k] = s36[k] * D;
        } else {
            for (int k = 0; k < 9; ++k) h[k] = s36[k] - n[0] * s36[9 + k] - n[1] * s36[18 + k] - n[2] * s36[27 + k];
        }
        h[0] += A; /* matter diag(A, 0, 0) */
    }
}

/* evolve one beam set; returns err when avg/err_ref given */
static double pass3(Orc3Engine* g, int hslot, int dl_slot, int in, int out, double* rows, int avg, int err_ref) {
    const Orc3Env* v = g->env;
    const int E = v->E;
    double err = 0.0;
    for (int jl = 0; jl < g->ntraj; ++jl) {
        const double* hb = g->hvv[hslot] + (size_t)jl * 9;
        const double dl = g->dlj[dl_slot][jl];
        for (int e = 0; e < E; ++e) {
            const double* hv = v->vac + 9 * e;
            double U[2][18];
            for (int pc = 0; pc < 2; ++pc) {
                double h9[9];
                for (int k = 0; k < 9; ++k) {
                    const double bpart = pc ? -((k == 4 || k == 6 || k == 8) ? -hb[k] : hb[k]) : hb[k];
                    const double vpart = (pc && (k == 4 || k == 6 || k == 8)) ? -hv[k] : hv[k];
                    h9[k] = vpart + bpart;
                }
                orc3_expm(h9, dl, U[pc]);
            }
            for (int s = 0; s < 6; ++s) {
                const double* pi = beam3(g, in, jl, s);
                double* po = beam3(g, out, jl, s);
                const double* u = U[s & 1];
                for (int i = 0; i < 3; ++i) {
                    double re = 0, im = 0;
                    for (int j = 0; j < 3; ++j) {
                        const double ur = u[2 * (3 * i + j)], ui = u[2 * (3 * i + j) + 1];
                        const double xr = pi[(2 * j) * E + e], xi = pi[(2 * j + 1) * E + e];
                        re += ur * xr - ui * xi;
                        im += ur * xi + ui * xr;
                    }
                    po[(2 * i) * E + e] = re;
                    po[(2 * i + 1) * E + e] = im;
                }
            }
        }
        for (int s = 0; s < 6; ++s) {
            double* po = beam3(g, out, jl, s);
            if (rows) esum3(po, v->fw + s * E, E, rows + ((size_t)jl * 6 + s) * 9);
            if (avg >= 0) {
                double* pa = beam3(g, avg, jl, s);
                for (int k = 0; k < 6 * E; ++k) pa[k] = (pa[k] + po[k]) * 0.5;
                if (err_ref >= 0) {
                    const double* pr = beam3(g, err_ref, jl, s);
                    for (int k = 0; k < 6 * E; ++k) {
                        const double d = fabs(pr[k] - pa[k]);
                        if (d > err) err = d;
                    }
                }
            }
        }
    }
    return err;
}

int orc3_prepare(Orc3Engine* g, double r, double dr) {
    const Orc3Env* v = g->env;
    g->r = r;
    g->dr = dr;
    if (v->p.model != ORC_SINGLE_ANGLE && r < v->p.Rnu) { snprintf(g3_err, sizeof g3_err, "r below Rnu"); return 2; }
    const double rk[3] = {r, r + 0.5 * dr, r + dr};
    for (int jl = 0; jl < g->ntraj; ++jl) {
        const int t = g->t_lo + jl / v->P, q = jl % v->P;
        double w, n[3], c[3];
        for (int k = 0; k < 3; ++k) geo3(g, t, q, rk[k], &w, n, &c[k]);
        g->dlj[0][jl] = 0.5 * dr / (0.5 * (c[0] + c[1]));
        g->dlj[1][jl] = 0.5 * dr / (0.5 * (c[1] + c[2]));
        g->dlj[2][jl] = dr / (0.5 * (c[0] + c[2]));
    }
    for (int k = 0; k < 3; ++k) g->A[k] = orc_matter_potential(v->env2, rk[k]);
    return 0;
}

/* stages as the 2-flavour oracle: 0 -> 36, 1 -> 72, 2 -> 36, 3 -> 1 */
int orc3_stage(Orc3Engine* g, int stage, double* partial) {
    const int E = g->env->E;
    switch (stage) {
        case 0:
            for (int jl = 0; jl < g->ntraj; ++jl)
                for (int s = 0; s < 6; ++s)
                    esum3(beam3(g, Q_PSI0, jl, s), g->env->fw + s * E, E, g->rows_a + ((size_t)jl * 6 + s) * 9);
            fold3(g, g->r, g->rows_a, partial);
            return 0;
        case 1:
            pass3(g, 0, 0, Q_PSI0, Q_MID, g->rows_b, -1, -1);
            pass3(g, 0, 2, Q_PSI0, Q_FULL1, g->rows_a, -1, -1);
            fold3(g, g->r + g->dr, g->rows_a, partial);
            fold3(g, g->r + 0.5 * g->dr, g->rows_b, partial + 36);
            return 0;
        case 2:
            memcpy(g->set[Q_AVGA], g->set[Q_FULL1], sizeof(double) * g->n);
            pass3(g, 1, 2, Q_PSI0, Q_FULL2, NULL, Q_AVGA, -1);
            pass3(g, 2, 1, Q_MID, Q_HALF2, g->rows_a, -1, -1);
            fold3(g, g->r + g->dr, g->rows_a, partial);
            return 0;
        case 3:
            memcpy(g->set[Q_RESULT], g->set[Q_HALF2], sizeof(double) * g->n);
            partial[0] = pass3(g, 3, 2, Q_PSI0, Q_FULL3, NULL, Q_RESULT, Q_AVGA);
            return 0;
    }
    return 1;
}

int orc3_stage_set(Orc3Engine* g, int stage, const double* total) {
    switch (stage) {
        case 0:
            memcpy(g->sums[0], total, sizeof(double) * 36);
            assemble3(g, g->r, g->sums[0], g->A[0], g->hvv[0]);
            return 0;
        case 1:
            memcpy(g->sums[1], total, sizeof(double) * 36);
            memcpy(g->sums[2], total + 36, sizeof(double) * 36);
            assemble3(g, g->r + g->dr, g->sums[1], g->A[2], g->hvv[1]);
            assemble3(g, g->r + 0.5 * g->dr, g->sums[2], g->A[1], g->hvv[2]);
            return 0;
        case 2:
            memcpy(g->sums[3], total, sizeof(double) * 36);
            for (int k = 0; k < 4; ++k)
                for (int i = 0; i < 36; ++i)
                    if (!isfinite(g->sums[k][i])) { snprintf(g3_err, sizeof g3_err, "non-finite sum"); return 2; }
            assemble3(g, g->r + g->dr, g->sums[3], g->A[2], g->hvv[3]);
            return 0;
    }
    return 0;
}

void orc3_commit(Orc3Engine* g) {
    double* t = g->set[Q_PSI0];
    g->set[Q_PSI0] = g->set[Q_RESULT];
    g->set[Q_RESULT] = t;
}

int orc3_trial_step(Orc3Engine* g, double r, double dr, double* err) {
    double buf[72];
    int rc = orc3_prepare(g, r, dr);
    for (int st = 0; st < 4 && rc == 0; ++st) {
        rc = orc3_stage(g, st, buf);
        if (rc == 0 && st < 3) rc = orc3_stage_set(g, st, buf);
    }
    *err = buf[0];
    return rc;
}

/* fixed/adaptive run (solver.cpp:414-456) on one rank */
int orc3_run(Orc3Engine* g, const OrcCtl* in, OrcSummary* out) {
    OrcCtl c = *in;
    const double rem = c.Rn - c.r > 0 ? c.Rn - c.r : 0;
    double pr = c.r, pdr = c.dr < rem ? c.dr : rem;
    uint64_t piter = c.iter;
    const double r_eps = 1e-12 * (fabs(c.Rn) > 1.0 ? fabs(c.Rn) : 1.0);
    int term = (c.r >= c.Rn - r_eps) ? 1 : 0;
    if (c.Ts > 0 && c.iter >= c.Ts) term = 2;
    uint64_t acc = 0, rej = 0;
    while (!term) {
        double err;
        int rc = orc3_trial_step(g, pr, pdr, &err);
        if (rc) return rc;
        if (!isfinite(err)) return 2;
        const int accept = err <= c.eps0;
        c.iter = piter + 1;
        c.dr = pdr;
        if (accept) { orc3_commit(g); c.r = pr + pdr; ++acc; }
        else ++rej;
        int collapse;
        double next = orc_step_size_update(&c, err, accept, &collapse);
        if (collapse) return 2;
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
    double m = 0;
    for (size_t b = 0; b < (size_t)g->ntraj * 6; ++b) {
        const double* p = g->set[Q_PSI0] + b * 6 * g->env->E;
        for (int e = 0; e < g->env->E; ++e) {
            double n2 = 0;
            for (int k = 0; k < 6; ++k) n2 += p[k * g->env->E + e] * p[k * g->env->E + e];
            if (fabs(n2 - 1) > m) m = fabs(n2 - 1);
        }
    }
    out->final_max_norm_dev = m;
    out->termination = term;
    return 0;
}
