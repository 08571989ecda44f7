import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from paper_1907_05560_b200 import Engine, Environment, StepControl
from test_gpu import base_config
cfg = base_config()
for kv in ("Lve=1e51", "Lvae=1e51", "Lvt=1e51", "Lvat=1e51", "Abins=6", "R0=50", "Rn=53"):
    cfg.override(kv)
def run(on, n, single=False):
    env = Environment.from_config(cfg); eng = Engine(env); eng.init_states(); eng.set_persistent(on)
    ctl = StepControl.from_config(cfg); eng.begin(ctl)
    if single:
        for i in range(n): eng.enqueue_steps(1)
    else:
        eng.enqueue_steps(n)
    eng.synchronize()
    return eng.state()
n = 2016
a = run(False, n); b = run(False, n); c = run(False, n, True); d = run(True, n); e = run(True, n, True)
print("s-s", np.abs(a - b).max(), "graph-vs-single", np.abs(a - c).max(), "p-vs-single", np.abs(d - c).max(), "p1-vs-single", np.abs(e - c).max())
