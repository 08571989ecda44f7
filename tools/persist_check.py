"""Compare the persistent kernel with the per-stage kernels step by step."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1907_05560_b200 import Engine, Environment, StepControl, baseline_config

cfg = baseline_config("configs0", Abins=6, Ebins=20, R0=50, Rn=53, dr=0.01, max_dr=0.5, eps0=1e-9)
for nsteps in (2, 3, 4, 8, 16):
    st, sums, q = [], [], []
    for on in (True, False):
        env = Environment.from_config(cfg); eng = Engine(env); eng.init_states()
        eng.set_persistent(on)
        ctl = StepControl.from_config(cfg)
        eng.begin(ctl); eng.enqueue_steps(nsteps); eng.synchronize()
        st.append(eng.state()); sums.append(eng.debug_sums()); q.append(eng.query())
    d = np.abs(st[0] - st[1]).max()
    ds = np.abs(sums[0] - sums[1]).max()
    print(nsteps, "state diff", d, "sums diff", ds, q[0], q[1] if q[0] != q[1] else "same ctl")
    if ds:
        print(np.argwhere(sums[0] != sums[1]))
