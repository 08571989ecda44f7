#!/usr/bin/env python
"""Benchmark: fp64 beam-steps/s of the fused evolution step on B200.

One "step" = one full S1-S4 evolution step (reference solver.cpp:343-412)
of every beam of the workload; one beam-step = one (angle, energy) cell with
all four species (BASELINE.md "Unit").  Default workload: BASELINE.json
configs[2] (bulb, 4096 angle x 256 energy bins, 2 flavours, fp64, fixed step
dr = 0.24 km from r = 10 km), the largest single-GPU configuration the
reference implements.

Arms
  (default)          our CUDA path; `value` = device-resident throughput
                     (CUDA events on the engine stream, max over ranks);
                     `e2e` = the reference-facing call sequence with HOST
                     buffers: set_state(host psi0) + run(K steps) +
                     state() -> host, timed on the device stream.
  --impl reference   the reference's own CPU implementation (oracle/_ref:
                     the unmodified reference core compiled from its sources)
                     on this box's host cores, same workload / metric.

Launch: python bench.py --gpus N --steps K --warmup W   (torchrun for N > 1)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 beam-steps/sec"
UNIT = "beam-steps/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="configs2")
    ap.add_argument("--schedule", type=int, default=-1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=0)
    ap.add_argument("--no-other-configs", action="store_true")
    ap.add_argument("--nccl-exchange", action="store_true", help="multi-GPU: NCCL instead of peer stores")
    return ap.parse_args()


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed regions.

    NVML is polled from a thread of this process (about every 2 ms, so even a
    20-step timed region of a few milliseconds is seen); `mark()` brackets the
    timed regions on the host clock and only samples inside them count.  When
    NVML cannot be loaded the sampler falls back to an `nvidia-smi -lms` child
    process (slow to start: it may miss a short region, and says so)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake"}

    def __init__(self, device: int):
        self.device = device
        self.samples = []   # (t, sm_mhz, reasons bitmask)
        self.windows = []   # (t0, t1) timed regions, host clock
        self.max_mhz = None
        self._stop = False
        self._thread = None
        self._nvml = None
        self._smi = None
        self._smi_path = None

    def _handle(self):
        import pynvml

        pynvml.nvmlInit()
        self._nvml = pynvml
        try:
            import torch

            uuid = str(torch.cuda.get_device_properties(self.device).uuid)
            if not uuid.startswith("GPU-"):
                uuid = "GPU-" + uuid
            return pynvml.nvmlDeviceGetHandleByUUID(uuid)
        except Exception:  # noqa: BLE001
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            ids = [v for v in vis.split(",") if v.strip().isdigit()]
            idx = int(ids[self.device]) if self.device < len(ids) else self.device
            return pynvml.nvmlDeviceGetHandleByIndex(idx)

    def _poll(self, h):
        nv = self._nvml
        while not self._stop:
            try:
                mhz = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                try:
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:  # noqa: BLE001
                    rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((time.perf_counter(), float(mhz), int(rs)))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def start(self):
        import threading

        try:
            h = self._handle()
            self.max_mhz = float(self._nvml.nvmlDeviceGetMaxClockInfo(h, self._nvml.NVML_CLOCK_SM))
            self._thread = threading.Thread(target=self._poll, args=(h,), daemon=True)
            self._thread.start()
            return
        except Exception:  # noqa: BLE001
            self._nvml = None
        fd, self._smi_path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._smi = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self._smi_path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self._smi = None

    def mark(self, t0: float, t1: float):
        self.windows.append((t0, t1))

    def stop(self) -> dict:
        if self._thread is not None:
            self._stop = True
            self._thread.join(timeout=2)
            inside = [s for s in self.samples if any(a <= s[0] <= b for a, b in self.windows)]
            bits = 0
            for s in inside:
                bits |= s[2]
            reasons = sorted(n for b, n in self.REASONS.items() if bits & b)
            sm = [s[1] for s in inside]
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                    "reasons": reasons, "samples": len(inside),
                    "source": "NVML polled in-process every ~2 ms; samples inside the timed regions "
                              "(device-resident steps and the end-to-end call)"}
        if self._smi is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.1)
        self._smi.terminate()
        try:
            self._smi.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self._smi.kill()
        rows = [[p.strip() for p in line.split(",")] for line in open(self._smi_path)]
        rows = [r for r in rows if len(r) >= 7]
        os.unlink(self._smi_path)
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:7]) if v.lower() == "active"})
        busy = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows),
                "source": "nvidia-smi -lms 20 over the whole run (NVML python binding unavailable)"}


# --------------------------------------------------------------- reference
def _ref_lib():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle  # checker / CPU baseline only

    return pyoracle


def cpu_reference(cfg, steps: int, warmup: int):
    """Time the reference CPU engine (oracle/_ref) on all host cores."""
    po = _ref_lib()
    ref = po.Ref()
    text = cfg.render()
    T = cfg.values["Abins"]
    lanes = max(1, min(os.cpu_count() or 1, T))
    cells = T * cfg.values["Pbins"] * cfg.values["Ebins"]
    if warmup > 0:
        ref.run(text, lanes=lanes, ts=warmup)
    t0 = time.perf_counter()
    _, summ = ref.run(text, lanes=lanes, ts=steps)
    wall = time.perf_counter() - t0
    run_wall = summ["wall_s"]
    return dict(value=cells * steps / run_wall, cores=lanes, wall=wall, steps=steps,
                variant=ref.variant, iterations=summ["iterations"])


def run_reference_arm(a, cfg):
    rank, world, _ = _dist()
    if rank != 0:
        return
    try:
        r = cpu_reference(cfg, a.steps, a.warmup)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"}))
        return
    cells = cfg.values["Abins"] * cfg.values["Pbins"] * cfg.values["Ebins"]
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT,
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": 1e3 * cells / r["value"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": a.config, "cells": cells, "parallelism": f"{r['cores']} host threads"},
        "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["cores"],
                         "kind": "reference",
                         "sample": f"{a.config}: solver::Engine::run of {a.steps} fixed steps "
                                   f"from R0 (after {a.warmup} warm-up steps), "
                                   f"{r['cores']} lanes, build x86-64-{r['variant']}"},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def main():
    a = _args()
    from paper_1907_05560_b200 import baseline_config

    cfg = baseline_config(a.config)
    if a.impl == "reference":
        run_reference_arm(a, cfg)
        return

    import torch

    from paper_1907_05560_b200 import Engine, Environment, StepControl, comm_unique_id
    from paper_1907_05560_b200.engine import fp64_peak

    rank, world, local = _dist()
    assert world == a.gpus or "RANK" not in os.environ, "--gpus must match WORLD_SIZE"
    torch.cuda.set_device(local)
    dist = None
    nccl_id = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    env = Environment.from_config(cfg)
    eng = Engine(env, rank=rank, nranks=world, device=local, nccl_id=nccl_id)
    exchange = "single GPU"
    if world > 1:
        # device-initiated stage exchange over NVLink (peer stores of flagged
        # words); NCCL all-gather if the peers cannot be mapped
        exchange = "NCCL all-gather per stage"
        if not a.nccl_exchange:
            tokens = [None] * world
            dist.all_gather_object(tokens, eng.comm_export())
            try:
                eng.comm_connect(tokens)
                exchange = "device-initiated peer stores over NVLink"
            except Exception as e:  # noqa: BLE001
                print(f"rank {rank}: peer exchange unavailable ({e}); using NCCL", file=sys.stderr)
    if a.schedule >= 0:
        eng.set_schedule(a.schedule)
    eng.init_states()
    stream = torch.cuda.ExternalStream(eng.stream())
    cells_total = env.cells
    ctl = StepControl.from_config(cfg)
    ctl.Ts = 0  # the timed walk is bounded by K, not by the config's Ts
    ctl.Rn = 1e9  # keep walking at max_dr for K steps

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    sampler = ClockSampler(local)
    sampler.start()
    # ---- warm-up (W steps), then exactly K timed steps
    eng.begin(ctl)
    eng.enqueue_steps(a.warmup)
    eng.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_launch0 = eng.launch_count()
    tw0 = time.perf_counter()
    e0.record(stream)
    eng.enqueue_steps(a.steps)
    e1.record(stream)
    n_launch = eng.launch_count() - n_launch0
    e1.synchronize()
    sampler.mark(tw0, time.perf_counter())
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    q = eng.query()
    if q["status"] != 0:
        raise SystemExit(f"device reported status {q['status']}")
    value = cells_total * a.steps / (ms * 1e-3)

    # ---- per-stage kernel durations (same stream, CUDA events)
    stage_ms = eng.profile_stages(20) if world == 1 else [None, None, None]

    # ---- e2e through the reference-facing API with host buffers
    import numpy as np

    n = eng.state_doubles
    host_in = torch.empty(n, dtype=torch.float64).pin_memory()
    host_out = torch.empty(n, dtype=torch.float64).pin_memory()
    eng.get_state_host_ptr(host_in.data_ptr(), n)
    e2e_steps = a.steps
    ctl_e2e = StepControl.from_config(cfg)
    ctl_e2e.Ts = e2e_steps
    ctl_e2e.Rn = 1e9
    # warm-up of the end-to-end path (untimed, as the W device steps): the
    # first transfers through freshly pinned buffers run at ~half the link
    # rate while their pages are mapped
    for _ in range(max(1, min(a.warmup, 2))):
        eng.set_state_host_ptr(host_in.data_ptr(), n)
        eng.run(ctl_e2e)
        eng.get_state_host_ptr(host_out.data_ptr(), n)
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    f0.record(stream)
    eng.set_state_host_ptr(host_in.data_ptr(), n)
    summ = eng.run(ctl_e2e)
    eng.get_state_host_ptr(host_out.data_ptr(), n)
    f1.record(stream)
    f1.synchronize()
    wall_e2e = time.perf_counter() - t0
    sampler.mark(t0, t0 + wall_e2e)
    clocks = sampler.stop()
    barrier()
    ms_e2e = max_over_ranks(max(f0.elapsed_time(f1), wall_e2e * 1e3))
    e2e_value = cells_total * summ.iterations / (ms_e2e * 1e-3)
    bytes_state = n * 8

    # ---- roofline (FP64 pipe) for the dominant kernel
    peak_dfma = fp64_peak(local)  # thread-DFMA/s; 2 flop each
    W = _work_per_cell()
    roof = None
    if stage_ms[0] is not None:
        names = ["S2", "S3", "S4"]
        k = max(range(3), key=lambda i: stage_ms[i])
        w_k = W["per_stage"][names[k]]
        achieved = w_k * cells_total / (stage_ms[k] * 1e-3) * 2 / 1e12  # TFLOP/s (DFMA-equiv)
        peak = peak_dfma * 2 / 1e12
        w_step = W.get("W_step", sum(W["per_stage"].values()))
        step_achieved = w_step * cells_total / (ms / a.steps * 1e-3) * 2 / 1e12
        hbm_peak = _hbm_peak()
        # HBM view: the step's compulsory state traffic (read
        # psi0 + write psi_new, 256 B per beam-step) all moves in S4; the
        # schedule adds its own intermediates (Bloch planes 48 B, P stash 64 B)
        alg_bytes = {"S2": 0, "S3": 0, "S4": 256}[names[k]]
        # (S2 -> S3 scalars: 32 B written by S2, read by S3; they and the P stash
        # stay in L2 and are dropped there after their one read)
        sched_bytes = {"S2": 48 + 32, "S3": 48 + 32 + 64, "S4": 128 + 64 + 128 + 48}[names[k]]
        hbm_ach = alg_bytes * cells_total / (stage_ms[k] * 1e-3) / 1e9
        hbm_frac = hbm_ach / hbm_peak[0]
        fp64_view = {"achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "work_unit": "algorithmic FP64 instructions of the reference schedule "
                                  "(DFMA-equivalent, 2 flop each) per beam-step",
                     "W_per_cell": w_k, "W_source": W["source"],
                     "peak_source": "measured live: DFMA-chain microkernel (osc_fp64_peak)"}
        traffic = W.get("traffic", {}).get(names[k])
        hbm_bound = alg_bytes > 0 and hbm_frac >= achieved / peak
        roof = {"bound": "hbm" if hbm_bound else "fp64", "kernel": f"k_stage<{names[k]}>",
                "achieved": hbm_ach if hbm_bound else achieved,
                "peak": hbm_peak[0] if hbm_bound else peak,
                "unit": "GB/s" if hbm_bound else "TFLOP/s",
                "frac": hbm_frac if hbm_bound else achieved / peak,
                "traffic": traffic,
                "traffic_warm": W.get("traffic_warm", {}).get(names[k]),
                "algorithmic_bytes_per_cell": alg_bytes,
                "peak_source": hbm_peak[1] if hbm_bound else fp64_view["peak_source"],
                "stage_ms": dict(zip(names, stage_ms)),
                "schedule_bytes_view": {"bytes_per_cell": sched_bytes,
                                        "achieved_gbs": sched_bytes * cells_total / (stage_ms[k] * 1e-3) / 1e9,
                                        "frac": sched_bytes * cells_total / (stage_ms[k] * 1e-3) / 1e9 / hbm_peak[0],
                                        "note": "all bytes this schedule moves in the kernel (state, "
                                                "propagator stash, Bloch planes)"},
                "fp64_view": fp64_view,
                "traffic_note": "ncu dram__bytes_read+write per launch (profiles/fp64_work.json): traffic from the "
                                "--set full capture (cold-cache replay; writes still in L2 at kernel end not "
                                "counted), traffic_warm with --cache-control none in the running pipeline",
                "step": {"W_per_cell": w_step, "achieved": step_achieved,
                         "frac_fp64": step_achieved / peak,
                         "hbm_compulsory_gbs": 256 * cells_total / (ms / a.steps * 1e-3) / 1e9,
                         "hbm_peak_gbs": hbm_peak[0], "hbm_peak_source": hbm_peak[1]}}

    others = None
    if world == 1 and not a.no_other_configs:
        others = {name: _other_config(name, local, a.no_cpu_baseline)
                  for name in ("configs0", "configs1", "configs3", "configs4") if name != a.config}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            steps_cpu = a.cpu_steps or max(4, int(40 * 1048576 / cells_total))
            r = cpu_reference(cfg, steps_cpu, 1)
            cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "reference",
                   "sample": f"{a.config}: reference solver::Engine::run, {steps_cpu} fixed steps "
                             f"from R0, {r['cores']} lanes, oracle/_ref x86-64-{r['variant']} build"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {type(e).__name__}: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": a.config, "cells": cells_total,
                       "angle_bins": env.abins, "energy_bins": env.ebins, "model": "bulb",
                       "steps_from_r_km": ctl.r, "dr_km": ctl.dr,
                       "parallelism": f"theta-sharded x{world}",
                       "exchange": exchange,
                       "l2": f"inputs larger than L2 (state {bytes_state / 2**20:.0f} MiB per buffer, "
                             f"2 buffers)",
                       "schedule": "recompute" if a.schedule == 0 else "stash-P",
                       "launch": LAUNCH_NAMES.get(eng.launch_mode, str(eng.launch_mode))},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": bytes_state / e2e_steps,
                    "d2h_bytes_per_step": bytes_state / e2e_steps,
                    "call": "osc_set_state(host) + osc_run(Ts=K) + osc_get_state(host)",
                    "steps": int(summ.iterations), "ms": ms_e2e},
            "gpu_launches": n_launch,
            "clocks": clocks,
            "roofline": roof,
            "cpu_baseline": cpu,
            "other_configs": others,
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if dist is not None:
        dist.destroy_process_group()


LAUNCH_NAMES = {0: "stage kernels (PDL, one-wave early release, partials reduced by the next stage, "
                   "control at the start of S2), CUDA graphs of 8 steps",
                2: "resident kernel (state in shared memory, grid all-reduce per stage)"}


def _other_config(name: str, device: int, no_cpu: bool) -> dict:
    """Device-resident throughput of another BASELINE config (same method as
    `value`), plus its CPU baseline: the reference engine for configs[0], the C
    restatement (1 thread, parity unpinned) for configs[1]/[3]/[4], which the
    reference does not implement."""
    import torch

    from paper_1907_05560_b200 import Engine, Environment, StepControl, baseline_config

    cfg = baseline_config(name)
    env = Environment.from_config(cfg)
    eng = Engine(env, device=device)
    eng.init_states()
    ctl = StepControl.from_config(cfg)
    ctl.Ts, ctl.Rn = 0, 1e9
    stream = torch.cuda.ExternalStream(eng.stream())
    steps = 200 if env.cells < 200000 else 60
    eng.begin(ctl)
    eng.enqueue_steps(5)
    eng.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    eng.enqueue_steps(steps)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    q = eng.query()
    launch = LAUNCH_NAMES.get(eng.launch_mode, str(eng.launch_mode))
    eng.close()
    out = {"value": env.cells * steps / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms / steps,
           "cells": env.cells, "flavours": env.nflav, "steps_timed": steps, "status": q["status"],
           "launch": launch}
    if no_cpu:
        return out
    try:
        if name == "configs0":
            r = cpu_reference(cfg, 20, 1)
            out["cpu"] = {"value": r["value"], "cores": r["cores"], "kind": "reference",
                          "sample": "20 fixed steps, reference engine"}
        else:
            po = _ref_lib()
            o = po.Oracle3(cfg) if env.nflav == 3 else po.Oracle(cfg)
            t0 = time.perf_counter()
            o.run(ts=1)
            wall = time.perf_counter() - t0
            out["cpu"] = {"value": env.cells / wall, "cores": 1, "kind": "port",
                          "sample": "1 step, C restatement (not in the reference; parity unpinned)"}
    except Exception as e:  # noqa: BLE001
        out["cpu"] = {"value": None, "sample": f"unavailable: {type(e).__name__}: {e}"}
    return out


def _hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        return json.load(open(path)).get("hbm_gbs"), "MEASURED_PEAKS.json (measured)"
    return 6650.0, "B200_PROFILING.md fallback"


def _work_per_cell() -> dict:
    """Algorithmic FP64 work per beam-step, frozen from ncu (profiles/)."""
    path = os.path.join(ROOT, "profiles", "fp64_work.json")
    if os.path.exists(path):
        return json.load(open(path))
    # SURVEY.md §8(d) estimate until the ncu measurement is frozen
    return {"source": "SURVEY.md §8(d) estimate (1.1e3 FP64 instr / beam-step)",
            "per_stage": {"S2": 1.1e3 * 0.35, "S3": 1.1e3 * 0.3, "S4": 1.1e3 * 0.35}}


if __name__ == "__main__":
    main()
