import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from paper_1907_05560_b200 import Engine, Environment, StepControl
from test_gpu import base_config
cfg = base_config()
for kv in ("Lve=1e51", "Lvae=1e51", "Lvt=1e51", "Lvat=1e51", "Abins=6", "R0=50", "Rn=53"):
    cfg.override(kv)
def run(on, n, sched):
    env = Environment.from_config(cfg); eng = Engine(env); eng.init_states(); eng.set_schedule(sched); eng.set_persistent(on)
    ctl = StepControl.from_config(cfg); eng.begin(ctl); eng.enqueue_steps(n); eng.synchronize()
    return eng.state()
for sched in (1, 0):
    for n in (2016, 51713):
        print(os.environ.get("OSC_LIB", "in-tree"), "sched", sched, n, np.abs(run(True, n, sched) - run(False, n, sched)).max())
