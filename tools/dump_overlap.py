"""Cost of snapshot I/O on configs[2]: K steps with no dumps, with mode-1
dumps every N iterations through osc_run_dumps (device gating, async D2H),
and the same dumps through a per-step hook (reference IoHook semantics:
synchronous state download after every accepted step)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_05560_b200 import Engine, Environment, StepControl, baseline_config, should_dump  # noqa: E402

K, N = int(os.environ.get("K", 200)), int(os.environ.get("N", 50))
cfg = baseline_config(os.environ.get("CFG", "configs2"), Ts=K)
env = Environment.from_config(cfg)
eng = Engine(env)


def timed(fn):
    eng.init_states()
    t = time.perf_counter()
    out = fn()
    return time.perf_counter() - t, out


ctl = StepControl.from_config(cfg)
t0, s0 = timed(lambda: eng.run(ctl))
n1 = []
gates = [(0, 0, N), (0, 0, 0)]
eng.run_dumps(ctl, gates, 1, lambda m, meta, p: None, copy=False)  # allocate the pinned buffers
t1, s1 = timed(lambda: eng.run_dumps(ctl, gates, 1, lambda m, meta, p: n1.append(meta.iter), copy=False))
n3 = []
t3, s3 = timed(lambda: eng.run_dumps(ctl, gates, 1, lambda m, meta, p: n3.append(p.sum())))
n2 = []
mark = [ctl.r, 0.0, ctl.iter]


def hook(info, state):
    if should_dump((0, 0, N), info.r, 0.0, info.iter, mark):
        n2.append(info.iter)
        mark[:] = [info.r, 0.0, info.iter]


t2, s2 = timed(lambda: eng.run(ctl, hook))
mb = eng.state_doubles * 8 / 2**20
print(f"{cfg.values['Abins']}x{cfg.values['Ebins']}: {K} steps, state {mb:.0f} MiB")
print(f"  no dumps                         {t0 * 1e3:8.1f} ms")
print(f"  osc_run_dumps every {N:3d} (async)  {t1 * 1e3:8.1f} ms  dumps {len(n1)} (callback does nothing)")
print(f"  same, callback reads the payload  {t3 * 1e3:8.1f} ms  dumps {len(n3)}")
print(f"  per-step hook (sync download)    {t2 * 1e3:8.1f} ms  dumps {len(n2)}")
