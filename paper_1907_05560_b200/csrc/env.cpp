// Host-side Environment builder (setup, runs once; not the hot path).
//
// Produces the tables the device step consumes, following
// solver::Environment::from_config (reference solver.cpp:62-95):
//   angle grid     AngleGrid::make          geometry.cpp:36-64
//   vacuum table   VacuumTable::make        geometry.cpp:218-240
//   spectra        SpectrumTable ctor       spectra.cpp:87-125
//   Fermi integral fermi_integral           spectra.cpp:17-83
//   couplings      hvv_coupling_per_km      units.hpp:55-61
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "oscflat_b200.h"
#include "status.hpp"

namespace oscb200 {
namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kGF = 1.166e-5 * 1e-6;       // MeV^-2
constexpr double kHcCm = 197.327e-13;         // MeV cm
constexpr double kHcKm = 197.327e-18;         // MeV km
constexpr double kHbarS = 6.582119569e-22;    // MeV s
constexpr double kErgPerMeV = 1.602176634e-6;

// Adaptive Simpson on the Fermi-Dirac integrand with the reference's
// tolerance schedule (tol halves per level, Richardson correction /15).
class FermiQuad {
public:
    FermiQuad(int k, double eta) : k_(k), eta_(eta) {}

    double integrand(double x) const {
        const double t = x - eta_;
        return t > 500.0 ? std::pow(x, k_) * std::exp(-t) : std::pow(x, k_) / (std::exp(t) + 1.0);
    }

    double integrate(double a, double b, double tol) {
        const double fa = integrand(a), fb = integrand(b), fm = integrand(0.5 * (a + b));
        evals_ = 3;
        return refine(a, b, fa, fm, fb, panel(a, b, fa, fm, fb), tol, 0);
    }

private:
    static double panel(double a, double b, double fa, double fm, double fb) {
        return (b - a) / 6.0 * (fa + 4.0 * fm + fb);
    }
    double refine(double a, double b, double fa, double fm, double fb, double whole, double tol,
                  int depth) {
        if (evals_ > 200000 || depth > 60)
            throw Error(OSC_ERR_NUMERIC, "fermi_integral: quadrature did not converge");
        const double m = 0.5 * (a + b);
        const double fl = integrand(0.5 * (a + m)), fr = integrand(0.5 * (m + b));
        evals_ += 2;
        const double l = panel(a, m, fa, fl, fm), r = panel(m, b, fm, fr, fb);
        const double delta = l + r - whole;
        if (std::fabs(delta) <= 15.0 * tol) return l + r + delta / 15.0;
        return refine(a, m, fa, fl, fm, l, 0.5 * tol, depth + 1) +
               refine(m, b, fm, fr, fb, r, 0.5 * tol, depth + 1);
    }
    int k_;
    double eta_;
    int evals_ = 0;
};

double fermi_integral(int k, double eta) {
    if (k < 0) throw Error(OSC_ERR_CONFIG, "fermi_integral: k must be >= 0");
    const double X = std::max(eta, 0.0) + 40.0;
    FermiQuad q(k, eta);
    const double body = q.integrate(0.0, X, 1e-10);
    // closed-form tail of x^k e^{eta-x} beyond X: e^{eta-X} sum_j k!/j! X^j
    double poly = 0.0, coef = 1.0;
    for (int j = k; j >= 0; --j) {
        poly += coef * std::pow(X, j);
        coef *= j;
    }
    return body + std::exp(eta - X) * poly;
}

double mean_energy(double T, double eta) { return T * fermi_integral(3, eta) / fermi_integral(2, eta); }

double coupling_per_km(double L, double Em, double Rnu) {
    const double flux = (L / kErgPerMeV) / Em;
    const double Rcm = Rnu * 1e5;
    const double mev = std::sqrt(2.0) * kGF * flux * kHbarS * kHcCm * kHcCm / (2.0 * kPi * Rcm * Rcm);
    return mev / kHcKm;
}

}  // namespace
}  // namespace oscb200

struct OscEnv {
    OscDesc desc{};
    std::vector<double> cos2, sin0, cphi, sphi, vac11, vac12, fw;
    std::vector<double> vac3, fw6;  // 3-flavour tables
    double cpl6[6]{};
    double emean[4]{};
};

using oscb200::Error;
using oscb200::guarded;

extern "C" {

double osc_fermi_integral(int k, double eta) {
    double v = NAN;
    guarded([&] { v = oscb200::fermi_integral(k, eta); });
    return v;
}

int osc_env_build(const OscParams* p, OscEnv** out) {
    return guarded([&] {
        if (!p || !out) throw Error(OSC_ERR_CONFIG, "osc_env_build: null argument");
        auto env = std::make_unique<OscEnv>();
        int T = p->abins, P = p->pbins;
        if (p->model == OSC_MODEL_SINGLE_ANGLE) T = P = 1;
        if (p->model == OSC_MODEL_BULB) P = 1;
        const int E = p->ebins;
        if (T < 1 || P < 1 || E < 1) throw Error(OSC_ERR_CONFIG, "AngleGrid: bins must be >= 1");
        if (!(p->E1 > p->E0) || p->E0 < 0.0)
            throw Error(OSC_ERR_CONFIG, "build_spectrum: need E1 > E0 >= 0");
        env->cos2.resize(T);
        env->sin0.resize(T);
        env->cphi.resize(P);
        env->sphi.resize(P);
        if (p->model == OSC_MODEL_CYLINDER) {
            // in-plane emission angle a0: midpoints uniform on (-pi/2, pi/2);
            // axial tilt b: midpoints uniform in sin(b) on (-1, 1)
            for (int t = 0; t < T; ++t) {
                const double a0 = -0.5 * oscb200::kPi + (t + 0.5) * oscb200::kPi / T;
                env->cos2[t] = std::cos(a0);
                env->sin0[t] = std::sin(a0);
            }
            for (int q = 0; q < P; ++q) {
                const double sb = -1.0 + (q + 0.5) * 2.0 / P;
                env->sphi[q] = sb;
                env->cphi[q] = std::sqrt(1.0 - sb * sb);
            }
        } else {
            for (int t = 0; t < T; ++t) {
                // bulb: midpoints in cos^2(theta0) (geometry.cpp:52-55);
                // plane: midpoints in cos(theta) on (0, 1]
                const double u = (t + 0.5) / T;
                env->cos2[t] = u;
                env->sin0[t] = p->model == OSC_MODEL_PLANE ? std::sqrt(1.0 - u * u) : std::sqrt(1.0 - u);
            }
            const double dphi = 2.0 * oscb200::kPi / P;
            for (int q = 0; q < P; ++q) {
                env->cphi[q] = std::cos((q + 0.5) * dphi);
                env->sphi[q] = std::sin((q + 0.5) * dphi);
            }
        }
        const double dE = (p->E1 - p->E0) / E;
        const double c2 = std::cos(2.0 * p->theta), s2 = std::sin(2.0 * p->theta);
        env->vac11.resize(E);
        env->vac12.resize(E);
        for (int e = 0; e < E; ++e) {
            const double Ec = p->E0 + (e + 0.5) * dE;
            const double delta = (p->dm2 * 1e-12 / (2.0 * Ec)) / oscb200::kHcKm;
            env->vac11[e] = -0.5 * delta * c2;
            env->vac12[e] = 0.5 * delta * s2;
        }
        // SpectrumTable (spectra.cpp:87-125) + coupling (solver.cpp:71-85)
        auto spectrum = [&](double L, double Tin, double Emean, double eta, double* row, double* em) {
            double T_s, Em;
            if (Tin > 0.0) {
                T_s = Tin;
                Em = oscb200::mean_energy(T_s, eta);
            } else if (Emean > 0.0) {
                Em = Emean;
                T_s = Em * oscb200::fermi_integral(2, eta) / oscb200::fermi_integral(3, eta);
            } else {
                throw Error(OSC_ERR_CONFIG, "build_spectrum: one of T or Emean must be positive");
            }
            // the coupling takes the configured mean energy when given
            const double Em_c = Emean > 0.0 ? Emean : oscb200::mean_energy(Tin, eta);
            *em = Em;
            const double norm = 1.0 / (oscb200::fermi_integral(2, eta) * T_s * T_s * T_s);
            for (int e = 0; e < E; ++e) {
                const double Ec = p->E0 + (e + 0.5) * dE;
                const double x = Ec / T_s - eta;
                const double den = x > 500.0 ? std::exp(x) : std::exp(x) + 1.0;
                row[e] = norm * Ec * Ec / den * dE;
            }
            return p->hvv_scale * oscb200::coupling_per_km(L, Em_c, p->Rnu);
        };
        env->fw.resize(4 * static_cast<size_t>(E));
        double cpl[4];
        for (int s = 0; s < 4; ++s)
            cpl[s] = spectrum(p->L[s], p->T[s], p->Emean[s], p->eta[s], env->fw.data() + (size_t)s * E,
                              &env->emean[s]);
        const bool three = p->nflav == 3;
        if (three) {
            if (p->model > OSC_MODEL_BULB)
                throw Error(OSC_ERR_CONFIG, "3 flavours: single-angle and bulb models only");
            // species nu_e, nubar_e, nu_mu, nubar_mu (= the x spectra), nu_tau, nubar_tau
            env->fw6.resize(6 * static_cast<size_t>(E));
            std::copy(env->fw.begin(), env->fw.end(), env->fw6.begin());
            for (int s = 0; s < 4; ++s) env->cpl6[s] = cpl[s];
            double em;
            for (int k = 0; k < 2; ++k)
                env->cpl6[4 + k] = spectrum(p->L_tau[k], p->T_tau[k], p->Emean_tau[k], p->eta_tau[k],
                                            env->fw6.data() + (size_t)(4 + k) * E, &em);
            // H_vac = U diag(0, dm21, dm31) U^dagger / 2E, standard PMNS
            // parametrisation (theta12 = theta, dm21 = dm2)
            using cd = std::complex<double>;
            const double c12 = std::cos(p->theta), s12 = std::sin(p->theta);
            const double c13 = std::cos(p->theta13), s13 = std::sin(p->theta13);
            const double c23 = std::cos(p->theta23), s23 = std::sin(p->theta23);
            const cd ed = std::exp(cd(0.0, p->delta_cp));
            const cd U[3][3] = {{c12 * c13, s12 * c13, s13 * std::conj(ed)},
                                {-s12 * c23 - c12 * s23 * s13 * ed, c12 * c23 - s12 * s23 * s13 * ed, s23 * c13},
                                {s12 * s23 - c12 * c23 * s13 * ed, -c12 * s23 - s12 * c23 * s13 * ed, c23 * c13}};
            env->vac3.resize(9 * static_cast<size_t>(E));
            for (int e = 0; e < E; ++e) {
                const double Ec = p->E0 + (e + 0.5) * dE;
                const double lam[3] = {0.0, (p->dm2 * 1e-12 / (2.0 * Ec)) / oscb200::kHcKm,
                                       (p->dm2_31 * 1e-12 / (2.0 * Ec)) / oscb200::kHcKm};
                cd H[3][3];
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) {
                        cd acc = 0.0;
                        for (int k = 0; k < 3; ++k) acc += U[i][k] * lam[k] * std::conj(U[j][k]);
                        H[i][j] = acc;
                    }
                double* o = env->vac3.data() + 9 * (size_t)e;
                o[0] = H[0][0].real(); o[1] = H[1][1].real(); o[2] = H[2][2].real();
                o[3] = H[0][1].real(); o[4] = H[0][1].imag();
                o[5] = H[0][2].real(); o[6] = H[0][2].imag();
                o[7] = H[1][2].real(); o[8] = H[1][2].imag();
            }
        }
        OscDesc& d = env->desc;
        d.model = p->model;
        d.abins = T;
        d.pbins = P;
        d.ebins = E;
        d.Rnu = p->Rnu;
        d.cos2_theta0 = env->cos2.data();
        d.sin_theta0 = env->sin0.data();
        d.cos_phi = env->cphi.data();
        d.sin_phi = env->sphi.data();
        d.vac_h11 = env->vac11.data();
        d.vac_h12 = env->vac12.data();
        d.fw = env->fw.data();
        std::memcpy(d.couplings, cpl, sizeof cpl);
        d.perturb = p->perturb;
        d.matter_profile = p->matter_profile;
        d.Ye = p->Ye;
        d.nb0 = p->nb0;
        d.hNS = p->hNS;
        d.Mns = p->Mns;
        d.gs = p->gs;
        d.S = p->S;
        d.nflav = three ? 3 : 2;
        if (three) {
            d.vac3 = env->vac3.data();
            d.fw6 = env->fw6.data();
            std::memcpy(d.couplings6, env->cpl6, sizeof env->cpl6);
        }
        *out = env.release();
    });
}

int osc_env_desc(const OscEnv* env, OscDesc* desc, double* emean4) {
    return guarded([&] {
        if (!env || !desc) throw Error(OSC_ERR_CONFIG, "osc_env_desc: null argument");
        *desc = env->desc;
        if (emean4) std::memcpy(emean4, env->emean, sizeof env->emean);
    });
}

int osc_env_destroy(OscEnv* env) {
    delete env;
    return OSC_OK;
}

}  // extern "C"
