// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI harness around the *unmodified* reference core library
// (/root/reference/proj/core, compiled from its own sources by
// oracle/Makefile into oracle/_ref/).  Tests, smoke() and bench.py's
// cpu_baseline / --impl reference legs call these entry points through
// ctypes to (a) pin the C restatement in oracle/oscflat_oracle.c,
// (b) generate golden fixtures, and (c) time the reference CPU path.
//
// Every function maps onto a reference API:
//   ref_env_*          -> solver::Environment::from_config   (solver.cpp:62-95)
//   ref_run            -> solver::Engine::{init_states,run}  (solver.cpp:475-525)
//   ref_trial_step     -> solver::Engine::trial_step_error   (solver.cpp:480-484)
//   ref_evolve_bin     -> flavor::evolve_bin                  (beam.hpp:105-121)
//   ref_density        -> flavor::density                     (beam.hpp:96-100)
//   ref_e_sum          -> flavor::e_sum                       (beam.cpp:84-103)
//   ref_partial_hvv    -> geom::fold_rows+combine_stage       (geometry.cpp:138-190)
//   ref_assemble_hvv   -> geom::assemble_hvv                  (geometry.cpp:192-216)
//   ref_fermi_integral -> spectra::fermi_integral             (spectra.cpp:77-83)
//   ref_matter         -> matter::matter_potential            (matter.cpp:39-42)
//   ref_init_state     -> BeamState::init_flavor_state        (beam.cpp:41-57)
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "oscflat/beam.hpp"
#include "oscflat/config.hpp"
#include "oscflat/geometry.hpp"
#include "oscflat/matter.hpp"
#include "oscflat/snapshot.hpp"
#include "oscflat/solver.hpp"
#include "oscflat/spectra.hpp"

using namespace oscflat;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const NumericError& e) {
        g_err = e.what();
        return 2;
    } catch (const IoError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

io::RunConfig cfg_of(const char* text) {
    io::RunConfig c = io::parse_config(text);
    io::require_runnable(c);
    return c;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

/// dims[0..4] = model, abins, pbins, ebins, padded
int ref_env_dims(const char* cfg_text, int* dims) {
    return guard([&] {
        const auto cfg = cfg_of(cfg_text);
        const auto env = solver::Environment::from_config(cfg);
        dims[0] = static_cast<int>(env.grid.model);
        dims[1] = env.grid.abins;
        dims[2] = env.grid.pbins;
        dims[3] = env.ebins;
        dims[4] = padded_len(env.ebins);
    });
}

/// Environment tables, logical (unpadded) lengths.
/// cos2[abins] sin0[abins] cphi[pbins] sphi[pbins] vac11[E] vac12[E]
/// fw[4*E] (f*dE per species) couplings[4] emean[4]
int ref_env_tables(const char* cfg_text, double* cos2, double* sin0, double* cphi,
                   double* sphi, double* vac11, double* vac12, double* fw,
                   double* couplings, double* emean) {
    return guard([&] {
        const auto cfg = cfg_of(cfg_text);
        const auto env = solver::Environment::from_config(cfg);
        const int T = env.grid.abins, P = env.grid.pbins, E = env.ebins;
        for (int t = 0; t < T; ++t) {
            cos2[t] = env.grid.cos2_theta0[t];
            sin0[t] = env.grid.sin_theta0[t];
        }
        for (int p = 0; p < P; ++p) {
            cphi[p] = env.grid.cos_phi[p];
            sphi[p] = env.grid.sin_phi[p];
        }
        for (int e = 0; e < E; ++e) {
            vac11[e] = env.vacuum.h11[e];
            vac12[e] = env.vacuum.h12[e];
        }
        for (int s = 0; s < 4; ++s) {
            const auto w = env.tables[s].weights();
            for (int e = 0; e < E; ++e) fw[s * E + e] = w[e];
            couplings[s] = env.couplings[s];
            emean[s] = env.tables[s].Emean();
        }
    });
}

double ref_matter(const char* cfg_text, double r_km) {
    double out = NAN;
    guard([&] {
        const auto cfg = cfg_of(cfg_text);
        const auto env = solver::Environment::from_config(cfg);
        out = matter::matter_potential(r_km, env.matt);
    });
    return out;
}

double ref_fermi_integral(int k, double eta) {
    double out = NAN;
    guard([&] { out = spectra::fermi_integral(k, eta); });
    return out;
}

/// Mode-1 layout [traj][species][comp][ebin] for state_in / state_out.
/// state_in == NULL -> Engine::init_states().  r/dr/iter override the
/// config's StepControl when r >= 0.  ts > 0 overrides Ts.
/// summary[0..6] = final_r, iterations, accepted, rejected, wall_s,
///                 final_max_norm_dev, phase_evolve_s
int ref_run(const char* cfg_text, int lanes, const double* state_in, double r, double dr,
            uint64_t iter, uint64_t ts, double* state_out, double* summary) {
    return guard([&] {
        const auto cfg = cfg_of(cfg_text);
        const auto env = solver::Environment::from_config(cfg);
        solver::Engine engine(env, lanes);
        engine.init_states();
        const std::size_t n = static_cast<std::size_t>(env.grid.trajectories()) * 4 * 4 * env.ebins;
        if (state_in) solver::fill_mode1(engine.state(), env.grid, {state_in, n});
        auto ctl = solver::StepControl::from_config(cfg);
        if (r >= 0.0) {
            ctl.r = r;
            ctl.dr = dr;
            ctl.iter = iter;
        }
        if (ts > 0) ctl.Ts = ts;
        const auto s = engine.run(ctl);
        if (state_out) {
            std::vector<double> payload;
            solver::extract_mode1(engine.state(), env.grid, payload);
            std::memcpy(state_out, payload.data(), payload.size() * sizeof(double));
        }
        if (summary) {
            summary[0] = s.final_r;
            summary[1] = static_cast<double>(s.iterations);
            summary[2] = static_cast<double>(s.accepted);
            summary[3] = static_cast<double>(s.rejected);
            summary[4] = s.wall_s;
            summary[5] = s.final_max_norm_dev;
            summary[6] = s.phase_evolve_s;
        }
    });
}

/// Engine::run with the CLI's dump gating (tools/oscflat.cpp:46-118
/// DumpDriver::on_step + io::should_dump): gates[m*3 + {0,1,2}] = r_step,
/// t_step, itr_step of mode m+1; fn receives each due dump (mode 1:
/// extract_mode1, mode 2: extract_mode2) in order.
typedef void (*ref_dump_fn)(void* user, int mode, uint64_t iter, double r, double dr, const double* payload,
                            size_t n);
int ref_run_dumps(const char* cfg_text, int lanes, const double* state_in, const double* gates, int mode_mask,
                  ref_dump_fn fn, void* user, double* state_out) {
    return guard([&] {
        const auto cfg = cfg_of(cfg_text);
        const auto env = solver::Environment::from_config(cfg);
        solver::Engine engine(env, lanes);
        engine.init_states();
        const std::size_t n = static_cast<std::size_t>(env.grid.trajectories()) * 4 * 4 * env.ebins;
        if (state_in) solver::fill_mode1(engine.state(), env.grid, {state_in, n});
        const auto ctl = solver::StepControl::from_config(cfg);
        io::DumpGates g[2];
        io::DumpMarks marks[2];
        for (int m = 0; m < 2; ++m) {
            g[m] = {gates[m * 3], gates[m * 3 + 1], static_cast<std::uint64_t>(gates[m * 3 + 2])};
            marks[m] = {ctl.r, 0.0, ctl.iter};
        }
        std::vector<double> payload;
        engine.run(ctl, [&](const solver::HookInfo& info, const solver::BeamSet& set) {
            for (int m = 0; m < 2; ++m) {
                if (!(mode_mask >> m & 1)) continue;
                if (!io::should_dump(g[m], info.r, info.t_wall, info.iter, marks[m])) continue;
                if (m == 0)
                    solver::extract_mode1(set, env.grid, payload);
                else
                    solver::extract_mode2(set, env.grid, env, payload);
                fn(user, m + 1, info.iter, info.r, info.dr, payload.data(), payload.size());
                marks[m] = {info.r, info.t_wall, info.iter};
            }
        });
        if (state_out) {
            solver::extract_mode1(engine.state(), env.grid, payload);
            std::memcpy(state_out, payload.data(), payload.size() * sizeof(double));
        }
    });
}

/// solver::extract_mode2 of a mode-1 payload.
int ref_extract_mode2(const char* cfg_text, const double* state_in, double* out) {
    return guard([&] {
        const auto cfg = cfg_of(cfg_text);
        const auto env = solver::Environment::from_config(cfg);
        solver::Engine engine(env, 1);
        engine.init_states();
        const std::size_t n = static_cast<std::size_t>(env.grid.trajectories()) * 4 * 4 * env.ebins;
        solver::fill_mode1(engine.state(), env.grid, {state_in, n});
        std::vector<double> payload;
        solver::extract_mode2(engine.state(), env.grid, env, payload);
        std::memcpy(out, payload.data(), payload.size() * sizeof(double));
    });
}

/// Engine::trial_step_error on a single lane; state_in may be NULL.
int ref_trial_step(const char* cfg_text, const double* state_in, double r, double dr,
                   double* err, double* state_after) {
    return guard([&] {
        const auto cfg = cfg_of(cfg_text);
        const auto env = solver::Environment::from_config(cfg);
        solver::Engine engine(env, 1);
        engine.init_states();
        const std::size_t n = static_cast<std::size_t>(env.grid.trajectories()) * 4 * 4 * env.ebins;
        if (state_in) solver::fill_mode1(engine.state(), env.grid, {state_in, n});
        *err = engine.trial_step_error(r, dr);
        if (state_after) {
            std::vector<double> payload;
            solver::extract_mode1(engine.state(), env.grid, payload);
            std::memcpy(state_after, payload.data(), payload.size() * sizeof(double));
        }
    });
}

/// BeamState::init_flavor_state(eps, seed) for one beam; out = [4][ebins].
int ref_init_state(int species, int ebins, double eps, uint64_t seed, double* out) {
    return guard([&] {
        BeamState b(static_cast<Species>(species), ebins);
        b.init_flavor_state(eps, seed);
        for (int e = 0; e < ebins; ++e) {
            out[0 * ebins + e] = b.ar()[e];
            out[1 * ebins + e] = b.ai()[e];
            out[2 * ebins + e] = b.br()[e];
            out[3 * ebins + e] = b.bi()[e];
        }
    });
}

void ref_evolve_bin(const double* h, double dl, const double* psi, double* out) {
    flavor::evolve_bin(h[0], h[1], h[2], dl, psi[0], psi[1], psi[2], psi[3], out[0], out[1],
                       out[2], out[3]);
}

void ref_density(const double* psi, double* out) {
    const auto r = flavor::density(psi[0], psi[1], psi[2], psi[3]);
    out[0] = r.d;
    out[1] = r.o_re;
    out[2] = r.o_im;
}

/// e_sum over one beam given as [4][ebins] plus fw[ebins].
int ref_e_sum(int ebins, const double* beam, const double* fw, double* out) {
    return guard([&] {
        BeamState b(Species::NuE, ebins);
        b.init_flavor_state();
        for (int e = 0; e < ebins; ++e) {
            b.ar()[e] = beam[0 * ebins + e];
            b.ai()[e] = beam[1 * ebins + e];
            b.br()[e] = beam[2 * ebins + e];
            b.bi()[e] = beam[3 * ebins + e];
        }
        std::vector<double> w(padded_len(ebins), 0.0);
        for (int e = 0; e < ebins; ++e) w[e] = fw[e];
        const auto r = flavor::e_sum(b, {w.data(), w.size()});
        out[0] = r.d;
        out[1] = r.o_re;
        out[2] = r.o_im;
    });
}

/// partial_hvv for the config's grid at radius r; rows = [traj*4+s][3];
/// sums_out = 12 doubles; hvv_out = [traj][3] assembled Hamiltonians.
int ref_partial_hvv(const char* cfg_text, double r, const double* rows, double* sums_out,
                    double* hvv_out) {
    return guard([&] {
        const auto cfg = cfg_of(cfg_text);
        const auto env = solver::Environment::from_config(cfg);
        const auto& g = env.grid;
        geom::RadiusCache c;
        c.resize(g.abins);
        geom::fill_cache(g, c, r, 0, g.abins);
        std::vector<ReductionRow> rr(static_cast<std::size_t>(g.trajectories()) * 4);
        for (std::size_t i = 0; i < rr.size(); ++i)
            rr[i] = {rows[3 * i], rows[3 * i + 1], rows[3 * i + 2]};
        const auto sums = geom::partial_hvv(g, c, env.couplings, rr);
        sums.to_doubles(sums_out);
        for (int t = 0; t < g.abins; ++t)
            for (int p = 0; p < g.pbins; ++p) {
                const Ham2 h = geom::assemble_hvv(g, c, sums, t, p);
                const int j = g.traj_index(t, p);
                hvv_out[3 * j] = h.h11;
                hvv_out[3 * j + 1] = h.h12_re;
                hvv_out[3 * j + 2] = h.h12_im;
            }
    });
}

/// fill_cache at r for the config's grid: out = [4][abins] = cos, sin, w, (unused)
int ref_fill_cache(const char* cfg_text, double r, double* out) {
    return guard([&] {
        const auto cfg = cfg_of(cfg_text);
        const auto env = solver::Environment::from_config(cfg);
        const auto& g = env.grid;
        geom::RadiusCache c;
        c.resize(g.abins);
        geom::fill_cache(g, c, r, 0, g.abins);
        for (int t = 0; t < g.abins; ++t) {
            out[t] = c.cos_theta[t];
            out[g.abins + t] = c.sin_theta[t];
            out[2 * g.abins + t] = c.w[t];
        }
    });
}

}  // extern "C"
