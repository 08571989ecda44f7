// solver_b200.cpp — drop-in replacement of the reference's solver::Engine
// (proj/core/include/oscflat/solver.hpp:128-153, solver.cpp:198-527) over the
// B200 C-ABI (include/oscflat_b200.h).  A maintainer compiles this file
// instead of the Engine section of solver.cpp (the rest of solver.cpp —
// Environment::from_config, StepControl::from_config, extract/fill_mode1,
// extract_mode2, resume_from, RunSummary::to_kv — stays) and links
// paper_1907_05560_b200/_oscb200.so.  tests/test_host.py compiles it against
// the reference headers (-fsyntax-only) whenever /root/reference is present.
//
// Semantics kept: Engine(env, lanes) borrows env; init_states, trial_step_error
// (single lane), run(ctl, hook) with the IoHook called after every accepted
// step on the calling thread; ConfigError / NumericError / IoError /
// ParallelError from the C status codes.  One semantic change: state() is a
// host copy of the device state (refreshed on each call; writes through it —
// resume_from — are pushed before the next trial step or run).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "oscflat/parallel.hpp"
#include "oscflat/solver.hpp"
#include "oscflat/types.hpp"
#include "oscflat_b200.h"
#include "solver_b200.hpp"

namespace oscflat::solver {
namespace {

[[noreturn]] void rethrow(int rc) {
    const std::string m = osc_last_error();
    switch (rc) {
        case OSC_ERR_CONFIG: throw ConfigError(m);
        case OSC_ERR_NUMERIC: throw NumericError(m);
        case OSC_ERR_IO: throw IoError(m);
        default: throw par::ParallelError(m);
    }
}
void ok(int rc) {
    if (rc != OSC_OK) rethrow(rc);
}

}  // namespace

RunSummary summary_of(const OscRunSummary& s);

struct Engine::Impl {
    const Environment* env;
    OscCtx* ctx = nullptr;
    BeamSet host;                 // state() view
    std::vector<double> payload;  // mode-1 staging
    bool host_dirty = false;      // state() handed out mutably since the last push

    int lanes = 1;
    int gpus = 1;

    Impl(const Environment& e, int lanes_) : env(&e), host(e.grid, e.ebins), lanes(lanes_) {
        // the reference constructor's checks, same messages (solver.cpp:459-466)
        if (lanes < 1) throw ConfigError("Engine: lanes must be >= 1");
        if (e.grid.model == geom::Model::SingleAngle && lanes != 1)
            throw ConfigError("single-angle model does not support multiple workers");
        if (lanes > e.grid.abins) throw ConfigError("Engine: more lanes than theta bins");
        std::vector<double> fw(4 * static_cast<std::size_t>(e.ebins));
        for (int s = 0; s < 4; ++s) {
            const auto w = e.tables[static_cast<std::size_t>(s)].weights();
            std::memcpy(fw.data() + static_cast<std::size_t>(s) * e.ebins, w.data(),
                        sizeof(double) * static_cast<std::size_t>(e.ebins));
        }
        OscDesc d{};
        d.model = static_cast<int>(e.grid.model);  // Model and OSC_MODEL_* share 0-2
        d.abins = e.grid.abins;
        d.pbins = e.grid.pbins;
        d.ebins = e.ebins;
        d.Rnu = e.grid.Rnu;
        d.cos2_theta0 = e.grid.cos2_theta0.data();
        d.sin_theta0 = e.grid.sin_theta0.data();
        d.cos_phi = e.grid.cos_phi.data();
        d.sin_phi = e.grid.sin_phi.data();
        d.vac_h11 = e.vacuum.h11.data();
        d.vac_h12 = e.vacuum.h12.data();
        d.fw = fw.data();
        for (int s = 0; s < 4; ++s) d.couplings[s] = e.couplings[static_cast<std::size_t>(s)];
        d.perturb = e.perturb;
        d.matter_profile = static_cast<int>(e.matt.profile);  // Profile and OSC_MATTER_* share 0-3
        d.Ye = e.matt.Ye;
        d.nb0 = e.matt.nb0;
        d.hNS = e.matt.hNS;
        d.Mns = e.matt.Mns;
        d.gs = e.matt.gs;
        d.S = e.matt.S;
        d.nflav = 2;
        // GPUs: OSC_GPUS (default: every visible device), at most one per
        // theta bin, one for the single-angle model.  lanes stays what it is
        // in the reference — the worker count the interface validates — and
        // does not change the device decomposition, so results are
        // bit-identical for any lanes (test_solver.cpp:226-251).
        gpus = b200::device_count();
        if (const char* g = std::getenv("OSC_GPUS")) gpus = std::atoi(g);
        if (gpus < 1) gpus = 1;
        gpus = std::min(gpus, e.grid.abins);
        if (e.grid.model == geom::Model::SingleAngle) gpus = 1;
        // (OSC_GROUP_PEER=1: the device-initiated exchange between the GPUs)
        const char* peer = std::getenv("OSC_GROUP_PEER");
        ok(osc_create_group(&d, gpus, nullptr, peer && std::atoi(peer) ? OSC_GROUP_PEER : 0, &ctx));
    }
    ~Impl() {
        if (ctx) osc_destroy(ctx);
    }

    std::size_t doubles() const {
        std::size_t n = 0;
        ok(osc_local_range(ctx, nullptr, nullptr, &n));
        return n;
    }
    void pull() {
        payload.resize(doubles());
        ok(osc_get_state(ctx, payload.data(), payload.size()));
        fill_mode1(host, env->grid, payload);
    }
    void push_if_dirty() {
        if (!host_dirty) return;
        extract_mode1(host, env->grid, payload);
        ok(osc_set_state(ctx, payload.data(), payload.size()));
        host_dirty = false;
    }
};

Engine::Engine(const Environment& env, int lanes) : impl_(std::make_unique<Impl>(env, lanes)), env_(&env) {}
Engine::~Engine() = default;
Engine::Engine(Engine&&) noexcept = default;
Engine& Engine::operator=(Engine&&) noexcept = default;

BeamSet& Engine::state() {
    impl_->push_if_dirty();
    impl_->pull();
    impl_->host_dirty = true;  // the caller may write (resume_from)
    return impl_->host;
}

const BeamSet& Engine::state() const {
    impl_->push_if_dirty();
    impl_->pull();
    return impl_->host;
}

void Engine::init_states() {
    ok(osc_init_states(impl_->ctx));
    impl_->host_dirty = false;
}

double Engine::trial_step_error(double r, double dr) {
    if (impl_->lanes != 1) throw ConfigError("trial_step_error: single-lane engines only");  // solver.cpp:480-484
    impl_->push_if_dirty();
    double err = 0.0;
    ok(osc_trial_step_error(impl_->ctx, r, dr, &err));
    return err;
}

RunSummary Engine::run(StepControl c, const IoHook& hook) {
    impl_->push_if_dirty();
    const OscStepControl oc{c.dr, c.dr_max, c.dr_min, c.eps0, c.kappa, c.r, c.R0, c.Rn, c.iter, c.Ts, c.Tn};
    OscRunSummary s{};
    if (const b200::DeviceDumps* dd = b200::DeviceDumps::active()) {
        // device-gated dumps (solver_b200.hpp): no per-step hook
        if (hook) throw ConfigError("Engine::run: an IoHook and a DeviceDumps scope are exclusive");
        const b200::DumpSpec& sp = dd->spec();
        OscDumpGates g[2];
        for (int m = 0; m < 2; ++m) g[m] = {sp.gates[m].r_step, sp.gates[m].t_step, sp.gates[m].itr_step};
        auto cb = [](void* u, int mode, const OscRecordMeta* m, const double* p, std::size_t n) {
            const auto* d = static_cast<const b200::DeviceDumps*>(u);
            d->sink()(mode, io::RecordMeta{m->iter, m->r, m->dr, m->t_wall}, std::span<const double>(p, n));
        };
        ok(osc_run_dumps(impl_->ctx, &oc, g, sp.mode_mask, +cb, const_cast<b200::DeviceDumps*>(dd), &s));
        return summary_of(s);
    }
    struct Tramp {
        const IoHook* hook;
        const Environment* env;
        BeamSet* set;
    } t{&hook, env_, &impl_->host};
    auto cb = [](void* u, const OscHookInfo* i, const double* st, std::size_t n) {
        auto* tp = static_cast<Tramp*>(u);
        fill_mode1(*tp->set, tp->env->grid, std::span<const double>(st, n));
        (*tp->hook)(HookInfo{i->iter, i->r, i->dr, i->t_wall}, *tp->set);
    };
    ok(osc_run(impl_->ctx, &oc, hook ? +cb : nullptr, &t, &s));
    return summary_of(s);
}

namespace b200 {

namespace {
thread_local const DeviceDumps* t_active = nullptr;
}

DeviceDumps::DeviceDumps(const DumpSpec& spec, DumpSink sink) : spec_(spec), sink_(std::move(sink)), prev_(t_active) {
    t_active = this;
}
DeviceDumps::~DeviceDumps() { t_active = prev_; }
const DeviceDumps* DeviceDumps::active() { return t_active; }

int device_count() {
    int n = 0;
    return osc_device_count(&n) == OSC_OK ? n : 0;
}

}  // namespace b200

RunSummary summary_of(const OscRunSummary& s) {
    RunSummary out;
    out.final_r = s.final_r;
    out.iterations = s.iterations;
    out.accepted = s.accepted;
    out.rejected = s.rejected;
    out.wall_s = s.wall_s;
    out.phase_hamiltonian_s = s.phase_hamiltonian_s;
    out.phase_evolve_s = s.phase_evolve_s;
    out.phase_io_s = s.phase_io_s;
    out.max_worker_wait_s = s.max_worker_wait_s;
    out.final_max_norm_dev = s.final_max_norm_dev;
    out.termination = s.termination == 2 ? "iterations" : (s.termination == 3 ? "walltime" : "radius");
    return out;
}

}  // namespace oscflat::solver
