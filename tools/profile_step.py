"""Small deterministic driver for ncu: configs[2] (or --config), S1 + N steps
launched directly (no graph) so each stage kernel appears as its own launch."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1907_05560_b200 import Engine, Environment, StepControl, baseline_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="configs2")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--schedule", type=int, default=0)
a = ap.parse_args()
cfg = baseline_config(a.config)
env = Environment.from_config(cfg)
eng = Engine(env)
eng.set_schedule(a.schedule)
eng.init_states()
ctl = StepControl.from_config(cfg)
eng.begin(ctl)
for _ in range(a.steps):
    eng.enqueue_steps(1)
eng.synchronize()
q = eng.query()
assert q["status"] == 0, q
print("ok", q)
