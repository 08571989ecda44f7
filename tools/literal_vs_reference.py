"""Literal BASELINE configs (unresolved fixed steps) on the GPU vs the reference engine and vs the
reference built without FMA contraction (its own build-to-build spread).  usage: tools/literal_vs_reference.py configs0 [configs2]"""
import sys, os, time
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import numpy as np
import pyoracle
from paper_1907_05560_b200 import Engine, Environment, StepControl, baseline_config
def dens(m, E):
    s = m.reshape(-1, 4, 4, E); ar, ai, br, bi = s[:, :, 0], s[:, :, 1], s[:, :, 2], s[:, :, 3]
    return np.stack([ar*ar+ai*ai-br*br-bi*bi, 2*(ar*br+ai*bi), 2*(ai*br-ar*bi)])
for name in sys.argv[1:] or ("configs0",):
    cfg = baseline_config(name)
    env = Environment.from_config(cfg)
    res = {}
    for mode in (0, 2):
        e = Engine(env)
        try:
            e.set_launch_mode(mode)
        except Exception:
            continue
        e.init_states(); s = e.run(StepControl.from_config(cfg)); res[mode] = e.state(); print("gpu", mode, s.iterations, s.final_r)
    t = time.time(); ra, sa = pyoracle.Ref("v4").run(cfg.render(), lanes=min(os.cpu_count() or 1, 32)); print("ref", sa["iterations"], time.time() - t)
    t = time.time(); rb, sb = pyoracle.Ref("v4_nofma").run(cfg.render(), lanes=min(os.cpu_count() or 1, 32)); print("ref nofma", sb["iterations"], time.time() - t)
    E = env.ebins
    print("ref vs nofma", np.max(np.abs(dens(ra, E) - dens(rb, E))))
    for m in res:
        print("gpu", m, "vs ref", np.max(np.abs(dens(res[m], E) - dens(ra, E))), "vs nofma", np.max(np.abs(dens(res[m], E) - dens(rb, E))))
    if len(res) == 2:
        print("gpu stage vs resident", np.max(np.abs(dens(res[0], E) - dens(res[2], E))))
