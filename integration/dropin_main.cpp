// dropin_main.cpp — the reference's run path (tools/oscflat.cpp cmd_run:
// parse_config_file -> require_runnable -> Environment::from_config ->
// StepControl::from_config -> Engine(env, lanes) -> init_states -> run) with
// the reference host code unchanged and solver::Engine replaced by
// solver_b200.cpp.  Writes the final mode-1 state (raw doubles) and prints
// RunSummary::to_kv().
//
// usage: oscflat_b200_dropin CONFIG OUT_STATE [dump_every]
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <fstream>
#include <iostream>
#include <vector>

#include "oscflat/config.hpp"
#include "oscflat/solver.hpp"

using namespace oscflat;

int main(int argc, char** argv) {
    if (argc < 3) {
        std::cerr << "usage: " << argv[0] << " CONFIG OUT_STATE [hook_every]\n";
        return 2;
    }
    try {
        io::RunConfig cfg = io::parse_config_file(argv[1]);
        io::require_runnable(cfg);
        const solver::Environment env = solver::Environment::from_config(cfg);
        const solver::StepControl ctl = solver::StepControl::from_config(cfg);
        solver::Engine engine(env, 1);
        engine.init_states();
        const std::uint64_t every = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 0;
        std::uint64_t hooks = 0;
        solver::IoHook hook;
        if (every)
            hook = [&](const solver::HookInfo& info, const solver::BeamSet&) {
                if (info.iter % every == 0) ++hooks;
            };
        const solver::RunSummary s = engine.run(ctl, hook);
        std::vector<double> payload;
        solver::extract_mode1(engine.state(), env.grid, payload);
        std::ofstream out(argv[2], std::ios::binary);
        out.write(reinterpret_cast<const char*>(payload.data()),
                  static_cast<std::streamsize>(payload.size() * sizeof(double)));
        std::cout << s.to_kv() << "hooks= " << hooks << "\n";
        return 0;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
