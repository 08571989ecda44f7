"""One resident-kernel launch of N steps on a small config (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_05560_b200 import Engine, Environment, StepControl, baseline_config  # noqa: E402

cfg = baseline_config(os.environ.get("CFG", "configs0"))
env = Environment.from_config(cfg)
eng = Engine(env)
eng.init_states()
ctl = StepControl.from_config(cfg)
ctl.Ts = 0
eng.begin(ctl)
eng.enqueue_steps(int(os.environ.get("N", 50)))
eng.synchronize()
print(eng.query(), eng.launch_mode)
