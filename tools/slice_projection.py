"""Per-rank step time of a 1/N theta slice on one B200 -> projected N-GPU
efficiency (the box has one GPU).

For each config, the slice a rank holds at N GPUs (make_partitions: T/N
theta bins, all phi and energy bins) runs as its own problem:
  * single-GPU kernels (what one rank's compute costs, no exchange);
  * the multi-rank kernels with a one-rank device-initiated exchange (the
    rank's last blocks publish their slot and every consumer polls it — the
    whole multi-rank code path except the NVLink hop).
The NVLink hop is added as a stated per-exchange latency (3 exchanges per
step).  Projected efficiency = T_full / (N * T_rank).
usage: python tools/slice_projection.py [N] [nvlink_us]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_05560_b200 import Engine, Environment, StepControl, baseline_config  # noqa: E402


def per_step(cfg, mode, n=64):
    env = Environment.from_config(cfg)
    eng = Engine(env, force_collectives=(mode == "multirank"))
    eng.init_states()
    if mode == "multirank":
        eng.comm_connect([eng.comm_export()])
    elif mode == "stages":
        eng.set_launch_mode(Engine.LAUNCH_STAGES)
    elif mode == "resident":
        try:
            eng.set_launch_mode(Engine.LAUNCH_RESIDENT)
        except Exception:
            eng.close()
            return None
    ctl = StepControl.from_config(cfg)
    ctl.Rn, ctl.Ts = 1e9, 0
    eng.begin(ctl)
    eng.enqueue_steps(16)
    eng.synchronize()
    best = 1e9
    for _ in range(5):
        t = time.perf_counter()
        eng.enqueue_steps(n)
        eng.synchronize()
        best = min(best, time.perf_counter() - t)
    eng.close()
    return best / n * 1e6


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    hop = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
    for name in ("configs2", "configs4", "configs3", "configs0"):
        full = baseline_config(name)
        T = full.Abins
        sl = baseline_config(name, Abins=T // N)
        t_full = per_step(full, "stages" if name != "configs0" else "resident", n=32)
        res = {m: per_step(sl, m) for m in ("stages", "resident", "multirank")}
        t_rank = res["multirank"] + 3 * hop
        best_single = min(v for v in (res["stages"], res["resident"]) if v is not None)
        print(f"{name}: full {t_full:.1f} us/step; 1/{N} slice ({sl.Abins}x{sl.Pbins}x{sl.Ebins}): "
              f"single-GPU kernels {res['stages']:.1f} (resident {res['resident']}), multi-rank kernels "
              f"{res['multirank']:.1f} us/step; + {3 * hop:.1f} us NVLink -> projected {N}-GPU efficiency "
              f"{t_full / (N * t_rank):.2f} (compute-only bound {t_full / (N * best_single):.2f})")


if __name__ == "__main__":
    main()
