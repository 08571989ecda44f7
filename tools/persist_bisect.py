import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from paper_1907_05560_b200 import Engine, Environment, StepControl
from test_gpu import base_config

cfg = base_config()
for kv in ("Lve=1e51", "Lvae=1e51", "Lvt=1e51", "Lvat=1e51", "Abins=6", "R0=50", "Rn=53"):
    cfg.override(kv)

def run(on, n):
    env = Environment.from_config(cfg); eng = Engine(env); eng.init_states(); eng.set_launch_mode(1 if on else 0)
    ctl = StepControl.from_config(cfg)
    eng.begin(ctl)
    eng.enqueue_steps(n); eng.synchronize()
    return eng.state(), eng.query(), eng.debug_sums()

lo, hi = 0, 51713
a, qa, sa = run(True, hi); b, qb, sb = run(False, hi)
print("full", np.abs(a - b).max(), qa == qb)
while hi - lo > 1:
    mid = (lo + hi) // 2
    a, qa, sa = run(True, mid); b, qb, sb = run(False, mid)
    same = np.array_equal(a, b) and qa == qb and np.array_equal(sa, sb)
    if same: lo = mid
    else: hi = mid
print("first differing step count", hi)
a, qa, sa = run(True, hi); b, qb, sb = run(False, hi)
print(qa); print(qb)
print("state diff", np.abs(a - b).max(), "where", np.argwhere(a != b)[:10].ravel())
print("sums diff rows/cols", np.argwhere(sa != sb)[:20].tolist())
a2, qa2, _ = run(True, hi - 1); b2, qb2, _ = run(False, hi - 1)
print(qa2)
