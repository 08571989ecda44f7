"""Device time per step of one BASELINE config at full size (quick A/B).
usage: python tools/time_config.py configs1 [steps] [launch|-] [schedule]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1907_05560_b200 import Engine, Environment, StepControl, baseline_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "configs1"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = baseline_config(name)
env = Environment.from_config(cfg)
eng = Engine(env)
if len(sys.argv) > 3 and sys.argv[3] != "-":
    eng.set_launch_mode(int(sys.argv[3]))
if len(sys.argv) > 4:
    eng.set_schedule(int(sys.argv[4]))
eng.init_states()
ctl = StepControl.from_config(cfg)
ctl.Rn, ctl.Ts = 1e9, 0
eng.begin(ctl)
eng.enqueue_steps(16)
eng.synchronize()
s = torch.cuda.ExternalStream(eng.stream())
best = 1e9
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    eng.enqueue_steps(steps)
    e1.record(s)
    e1.synchronize()
    best = min(best, e0.elapsed_time(e1) / steps)
print(f"{name}: {best * 1e3:.1f} us/step, {env.cells / (best * 1e-3):.3e} beam-steps/s, status {eng.query()['status']}")
