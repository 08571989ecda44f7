import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from paper_1907_05560_b200 import Engine, Environment, StepControl
from test_gpu import base_config

cfg = base_config()
for kv in ("Lve=1e51", "Lvae=1e51", "Lvt=1e51", "Lvat=1e51", "Abins=6", "R0=50", "Rn=53"):
    cfg.override(kv)
res = {}
for on in (True, False):
    env = Environment.from_config(cfg); eng = Engine(env); eng.init_states(); eng.set_persistent(on)
    s = eng.run(StepControl.from_config(cfg))
    res[on] = eng.state()
    print(on, s.iterations, s.accepted, s.rejected, s.final_r, eng.query())
print("diff", np.abs(res[True] - res[False]).max())
for on in (True, False):
    env = Environment.from_config(cfg); eng = Engine(env); eng.init_states(); eng.set_persistent(on)
    ctl = StepControl.from_config(cfg); ctl.Ts = 0
    eng.begin(ctl)
    for k in range(200):
        eng.enqueue_steps(2); q = eng.query()
        if q["terminate"]: break
    print(on, q)
st = []
for on in (True, True, False):
    env = Environment.from_config(cfg); eng = Engine(env); eng.init_states(); eng.set_persistent(on)
    s = eng.run(StepControl.from_config(cfg))
    st.append(eng.state())
print("p-p", np.abs(st[0] - st[1]).max(), "p-s", np.abs(st[0] - st[2]).max())
