"""Quick GPU sanity/timing probe (development aid)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import pyoracle as po
from paper_1907_05560_b200 import *

def cmp(name, cfg, steps):
    env = Environment.from_config(cfg)
    eng = Engine(env); eng.init_states()
    orc = po.Oracle(cfg)
    e1 = eng.trial_step_error(cfg.values["R0"], cfg.values["dr"])
    e2 = orc.trial_step(cfg.values["R0"], cfg.values["dr"])
    s = eng.run(StepControl.from_config(cfg))
    orc2 = po.Oracle(cfg); so = orc2.run()
    d = np.max(np.abs(eng.state() - orc2.get_state()))
    print(f"{name}: err gpu {e1:.6e} orc {e2:.6e}; steps {s.iterations}/{so['iterations']} r {s.final_r}/{so['final_r']} max|dpsi| {d:.3e} normdev {s.final_max_norm_dev:.3e}/{so['final_max_norm_dev']:.3e}", flush=True)

cmp("bulb", baseline_config("configs0", Abins=24, Ebins=40, R0=50, Rn=51, dr=1e-4, max_dr=1e-4, Ts=20), 20)
cmp("bulb-unres", baseline_config("configs0", Abins=24, Ebins=40, Ts=5), 5)
c = baseline_config("configs0", Abins=12, Ebins=20, R0=50, Rn=51, dr=1e-4, max_dr=1e-4, Ts=20); c.override("model=ebulb"); c.override("Pbins=6")
cmp("ebulb", c, 20)
c = baseline_config("configs0", Abins=1, Ebins=20, R0=50, Rn=51, dr=1e-4, max_dr=1e-4, Ts=20); c.override("model=sa")
cmp("sa", c, 20)
c = baseline_config("configs0", Abins=16, Ebins=24, R0=50, Rn=60, dr=1e-3, max_dr=1e-2, Ts=30); c.override("eps0=1e-9"); c.override("hasMatter=1"); c.override("matterProfile=sum"); c.override("Ye=0.5"); c.override("nb0=1e30"); c.override("hNS=5"); c.override("Mns=1.4"); c.override("gs=1"); c.override("S=100")
cmp("adaptive+matter", c, 30)

for name in ("configs0", "configs2"):
    cfg = baseline_config(name)
    env = Environment.from_config(cfg); eng = Engine(env); eng.init_states()
    for sched in (0, 1):
        eng.set_schedule(sched)
        ctl = StepControl.from_config(cfg)
        eng.begin(ctl); eng.enqueue_steps(16); eng.synchronize()
        n = 64 if name == "configs2" else 512
        eng.begin(ctl); eng.synchronize()
        t = time.perf_counter(); eng.enqueue_steps(n); eng.synchronize(); dt = time.perf_counter() - t
        q = eng.query()
        print(f"{name} sched{sched}: {dt/n*1e6:.1f} us/step, {env.cells*n/dt:.3e} cell-steps/s, q={q}", flush=True)
