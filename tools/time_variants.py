"""Time configs[2] (and configs[0]) steps for each library variant in
tools/_variants/*.so (development sweep; one subprocess per variant)."""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, time
sys.path.insert(0, %r)
from paper_1907_05560_b200 import *
out = []
for name, n in [(c, n) for c, n in (("configs2", 64), ("configs0", 256), ("configs1", 128), ("configs3", 64), ("configs4", 64)) if c in os.environ.get("TV_CONFIGS", "configs2,configs0,configs1,configs3,configs4")]:
    cfg = baseline_config(name)
    env = Environment.from_config(cfg); eng = Engine(env); eng.init_states()
    for sched, pers in [sp for sp in ((1, 0), (1, 2), (0, 0)) if f"s{sp[0]}p{sp[1]}" in os.environ.get("TV_MODES", "s1p0,s1p2,s0p0")]:
        eng.set_schedule(sched)
        try:
            eng.set_launch_mode(pers)
        except Exception:
            continue
        ctl = StepControl.from_config(cfg); ctl.Rn = 1e9; ctl.Ts = 0
        eng.begin(ctl); eng.enqueue_steps(16); eng.synchronize()
        best = 1e9
        for rep in range(3):
            t = time.perf_counter(); eng.enqueue_steps(n); eng.synchronize(); best = min(best, time.perf_counter() - t)
        st = eng.profile_stages(10)
        out.append(f"{name} s{sched}p{pers}: {best/n*1e6:7.1f} us/step  {env.cells*n/best:.3e}/s  stages " + " ".join(f"{x*1e3:6.1f}" for x in st))
print("\n".join(out))
''' % ROOT

for so in sorted(glob.glob(os.path.join(ROOT, "tools", "_variants", "*.so"))) + [None]:
    env = dict(os.environ)
    if so:
        env["OSC_LIB"] = so
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print("==", os.path.basename(so) if so else "in-tree", flush=True)
    print(r.stdout.strip() or r.stderr[-2000:], flush=True)
