// oscflat_b200 — the reference CLI's `run` and `resume` commands
// (tools/oscflat.cpp:122-165 cmd_run, option wiring :245-319) over the B200
// drop-in Engine (solver_b200.cpp), with snapshot dumps gated on the device.
//
//   oscflat_b200 run     -c CONFIG [-o DIR] [--override k=v]... [--lanes N] [--gpus N] [-v]
//   oscflat_b200 resume  -c CONFIG -s SNAPSHOT [same options]
//   oscflat_b200 analyze -i SNAPSHOT [-o DIR] [--what survival|spectra|content|all]
//
// Same flow and outputs as the reference: parse + overrides, require_runnable,
// config hash, Environment / StepControl from the config, Engine(env, lanes),
// init_states, resume_from (resume: r, dr, iter from the last record), the
// dump writers (io::SnapshotFileWriter per enabled mode behind one
// io::WriterLane, file names <prefix>Snapshot<k>_0 / <prefix>Average<k>_0),
// the run, the unconditional final mode-1 dump, summary.kv, the one-line
// report, and the exit codes 2 config / 3 numeric / 4 io.
//
// Engine selection: --gpus N maps the run onto N GPUs of this process
// (OSC_GPUS; default every visible device).  The dump gates (r_step*,
// t_step*, itr_step*) are handed to the device control update through
// b200::DeviceDumps instead of a per-step IoHook (DumpDriver::on_step,
// tools/oscflat.cpp:97-115), so the state leaves the GPU only when a dump is
// due.  Built with -DOSC_REFERENCE_ENGINE (integration/Makefile target
// oscflat_ref_cli, test infrastructure) the same source drives the unmodified
// reference engine through the hook, which is the behaviour the tests compare
// against.
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <memory>
#include <string>
#include <vector>

#include "oscflat/analysis.hpp"
#include "oscflat/config.hpp"
#include "oscflat/parallel.hpp"
#include "oscflat/snapshot.hpp"
#include "oscflat/solver.hpp"
#ifndef OSC_REFERENCE_ENGINE
#include "solver_b200.hpp"
#endif

namespace {

using namespace oscflat;

constexpr int kExitConfig = 2;
constexpr int kExitNumeric = 3;
constexpr int kExitIo = 4;

struct Options {
    std::string command;
    std::string config_path, snapshot_path, output_dir = ".";
    std::string input_path, what = "all";  // analyze
    std::vector<std::string> overrides;
    int lanes = 0;  // 0: the config's
    int gpus = 0;   // 0: every visible device
    bool verbose = false;
};

[[noreturn]] void usage(const char* argv0) {
    std::cerr << "usage: " << argv0
              << " run|resume -c CONFIG [-s SNAPSHOT] [-o DIR] [--override key=value]... [--lanes N] [--gpus N] [-v]\n"
              << "       " << argv0 << " analyze -i SNAPSHOT [-o DIR] [--what survival|spectra|content|all]\n";
    std::exit(kExitConfig);
}

Options parse_args(int argc, char** argv) {
    Options o;
    if (argc < 2) usage(argv[0]);
    o.command = argv[1];
    if (o.command != "run" && o.command != "resume" && o.command != "analyze") usage(argv[0]);
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto value = [&]() -> std::string {
            if (i + 1 >= argc) throw ConfigError("option " + a + " needs a value");
            return argv[++i];
        };
        if (a == "-c" || a == "--config") o.config_path = value();
        else if (a == "-s" || a == "--snapshot") o.snapshot_path = value();
        else if (a == "-o" || a == "--output") o.output_dir = value();
        else if (a == "--override") o.overrides.push_back(value());
        else if (a == "--lanes") o.lanes = std::stoi(value());
        else if (a == "--gpus") o.gpus = std::stoi(value());
        else if (a == "-v" || a == "--verbose") o.verbose = true;
        else if (a == "-i" || a == "--input") o.input_path = value();
        else if (a == "--what") o.what = value();
        else throw ConfigError("unknown option " + a);
    }
    if (o.command == "analyze") {
        if (o.input_path.empty()) throw ConfigError("analyze needs --input");
        return o;
    }
    if (o.config_path.empty()) throw ConfigError("--config is required");
    if (o.command == "resume" && o.snapshot_path.empty()) throw ConfigError("resume needs --snapshot");
    return o;
}

/// The CLI's dump writers and gates.  Gating runs on the device (B200
/// engine) or in the per-step hook (reference engine, as DumpDriver does).
class Dumps {
public:
    Dumps(const io::RunConfig& cfg, const solver::Environment& env, const std::string& dir, std::uint64_t hash)
        : cfg_(cfg), env_(env) {
        const io::SnapshotDims dims{env.grid.abins, env.grid.pbins, kSpeciesCount, 4, env.ebins};
        std::unique_ptr<io::SnapshotFileWriter> w[2];
        for (int m = 0; m < 2; ++m)
            if (cfg.dumpMode & (1 << m))
                w[m] = std::make_unique<io::SnapshotFileWriter>(dir, cfg.filePrefix, m + 1, 0, cfg.newFile_step,
                                                                cfg.sync_step, dims, env.spectra_header(), hash);
        if (w[0] || w[1])
            lane_ = std::make_unique<io::WriterLane>(std::move(w[0]), std::move(w[1]), cfg.designatedWriter != 0);
        gates_[0] = {cfg.r_step1, cfg.t_step1, cfg.itr_step1};
        gates_[1] = {cfg.r_step2, cfg.t_step2, cfg.itr_step2};
    }

    int mode_mask() const { return lane_ ? (cfg_.dumpMode & 3) : 0; }

    void submit(int mode, const io::RecordMeta& meta, std::vector<double> payload) {
        io::WriterLane::Job job;
        job.mode = mode;
        job.meta = meta;
        job.payload = std::move(payload);
        lane_->submit(std::move(job));
    }

    solver::RunSummary run(solver::Engine& engine, const solver::StepControl& ctl) {
        if (!lane_) return engine.run(ctl);
#ifdef OSC_REFERENCE_ENGINE
        io::DumpMarks marks[2];
        for (auto& m : marks) m = {ctl.r, 0.0, ctl.iter};
        return engine.run(ctl, [&](const solver::HookInfo& info, const solver::BeamSet& set) {
            for (int mode = 1; mode <= 2; ++mode) {
                if (!(cfg_.dumpMode & mode)) continue;
                if (!io::should_dump(gates_[mode - 1], info.r, info.t_wall, info.iter, marks[mode - 1])) continue;
                std::vector<double> payload;
                if (mode == 1)
                    solver::extract_mode1(set, env_.grid, payload);
                else
                    solver::extract_mode2(set, env_.grid, env_, payload);
                submit(mode, {info.iter, info.r, info.dr, info.t_wall}, std::move(payload));
                marks[mode - 1] = {info.r, info.t_wall, info.iter};
            }
        });
#else
        solver::b200::DumpSpec spec;
        spec.mode_mask = mode_mask();
        spec.gates[0] = gates_[0];
        spec.gates[1] = gates_[1];
        solver::b200::DeviceDumps scope(spec, [&](int mode, const io::RecordMeta& meta, std::span<const double> p) {
            submit(mode, meta, std::vector<double>(p.begin(), p.end()));
        });
        return engine.run(ctl);
#endif
    }

    // final whole state, unconditionally (DumpDriver::dump_final)
    void final_state(const io::RecordMeta& meta, const solver::BeamSet& set) {
        if (!lane_ || !(cfg_.dumpMode & 1)) return;
        std::vector<double> payload;
        solver::extract_mode1(set, env_.grid, payload);
        submit(1, meta, std::move(payload));
    }

    void finish() {
        if (lane_) lane_->finish();
    }

private:
    const io::RunConfig& cfg_;
    const solver::Environment& env_;
    std::unique_ptr<io::WriterLane> lane_;
    io::DumpGates gates_[2];
};

int cmd_run(const Options& opt) {
    io::RunConfig cfg = io::parse_config_file(opt.config_path);
    for (const auto& ov : opt.overrides) io::apply_override(cfg, ov);
    for (const auto& w : cfg.warnings) std::cerr << "warning: " << w << "\n";
    io::require_runnable(cfg);
    const std::uint64_t hash = io::config_hash(cfg);
    if (opt.gpus > 0) setenv("OSC_GPUS", std::to_string(opt.gpus).c_str(), 1);

    const solver::Environment env = solver::Environment::from_config(cfg);
    solver::StepControl ctl = solver::StepControl::from_config(cfg);
    const int lanes = opt.lanes > 0 ? opt.lanes : std::max(1, cfg.lanes);
    solver::Engine engine(env, lanes);
    engine.init_states();

    if (opt.command == "resume") {
        std::vector<std::string> warnings;
        const io::RecordMeta meta = solver::resume_from(opt.snapshot_path, engine.state(), env.grid, hash, &warnings);
        ctl.r = meta.r;
        ctl.dr = meta.dr;
        ctl.iter = meta.iter;
        for (const auto& w : warnings) std::cerr << "warning: " << w << "\n";
        if (opt.verbose) std::cerr << "resumed at r = " << meta.r << " km, iteration " << meta.iter << "\n";
    }

    std::filesystem::create_directories(opt.output_dir);
    Dumps dumps(cfg, env, opt.output_dir, hash);
    const solver::RunSummary s = dumps.run(engine, ctl);
    dumps.final_state({s.iterations + ctl.iter, s.final_r, ctl.dr, s.wall_s}, engine.state());
    dumps.finish();

    const std::string kv = s.to_kv();
    {
        std::ofstream f(opt.output_dir + "/summary.kv");
        if (!f) throw IoError("cannot write " + opt.output_dir + "/summary.kv");
        f << kv;
    }
    std::cout << "run finished: r = " << s.final_r << " km after " << s.iterations << " iterations (" << s.accepted
              << " accepted, " << s.rejected << " rejected), " << s.wall_s << " s, termination: " << s.termination
              << "\n";
    if (opt.verbose) std::cout << kv;
    return 0;
}

// `analyze` (tools/oscflat.cpp:334-339): the reference's own post-processing
// (analysis::analyze_file, host code, unchanged) on snapshots the GPU wrote.
int cmd_analyze(const Options& opt) {
    for (const auto& f : analysis::analyze_file(opt.input_path, opt.output_dir, opt.what))
        std::cout << "wrote " << f << "\n";
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Options opt = parse_args(argc, argv);
        return opt.command == "analyze" ? cmd_analyze(opt) : cmd_run(opt);
    } catch (const ConfigError& e) {
        std::cerr << "config error: " << e.what() << "\n";
        return kExitConfig;
    } catch (const par::ParallelError& e) {
        std::cerr << "numeric error: " << e.what() << "\n";
        return kExitNumeric;
    } catch (const NumericError& e) {
        std::cerr << "numeric error: " << e.what() << "\n";
        return kExitNumeric;
    } catch (const IoError& e) {
        std::cerr << "io error: " << e.what() << "\n";
        return kExitIo;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
