// solver_b200.hpp — what the drop-in Engine (solver_b200.cpp) adds to the
// reference's solver::Engine interface (solver.hpp:128-153), for callers that
// know they run on the B200 engine (the CLI in oscflat_b200_cli.cpp).
//
// Device-gated dumps.  The reference CLI gates snapshots inside the per-step
// IoHook (DumpDriver::on_step, tools/oscflat.cpp:97-115), which through any
// device engine means a whole-state download after every accepted step.
// With a DeviceDumps scope alive on the calling thread, Engine::run instead
// hands the gates (io::DumpGates per mode, io::should_dump semantics,
// snapshot.cpp:237-243) to the device control update (osc_run_dumps): the
// step sequence pauses only when a dump is due, the payload is packed on the
// device (mode 1: extract_mode1 order, mode 2: extract_mode2) and copied to
// pinned memory while the next steps run, and `sink` receives it in dump
// order on the calling thread.
#pragma once

#include <functional>
#include <span>

#include "oscflat/snapshot.hpp"
#include "oscflat/solver.hpp"

namespace oscflat::solver::b200 {

struct DumpSpec {
    int mode_mask = 0;     // bit 0: mode 1 (whole state), bit 1: mode 2 (energy-averaged)
    io::DumpGates gates[2];  // [0] mode 1, [1] mode 2
};

using DumpSink = std::function<void(int mode, const io::RecordMeta& meta, std::span<const double> payload)>;

class DeviceDumps {
public:
    DeviceDumps(const DumpSpec& spec, DumpSink sink);
    ~DeviceDumps();
    DeviceDumps(const DeviceDumps&) = delete;
    DeviceDumps& operator=(const DeviceDumps&) = delete;

    const DumpSpec& spec() const { return spec_; }
    const DumpSink& sink() const { return sink_; }
    static const DeviceDumps* active();  // innermost scope on this thread

private:
    DumpSpec spec_;
    DumpSink sink_;
    const DeviceDumps* prev_;
};

/// GPUs the drop-in can map Engine lanes onto (0 without a usable device).
int device_count();

}  // namespace oscflat::solver::b200
