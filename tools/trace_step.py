"""Stage timeline of a few steps from a -DOSC_TRACE build (development aid).

usage: python tools/trace_step.py [config]   (builds tools/_variants/trace.so)
Prints, per stage launch, block-averaged and extreme times (us) relative to
the previous launch's last block: entry, ready (control + dependency),
main-loop start, main-loop end, exit, last block done."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SO = os.path.join(ROOT, "tools", "_variants", "trace.so")
if not os.environ.get("OSC_LIB"):
    os.environ["OSC_LIB"] = SO
from paper_1907_05560_b200 import Engine, Environment, StepControl, baseline_config  # noqa: E402
from paper_1907_05560_b200.native import lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "configs2"
cfg = baseline_config(name)
env = Environment.from_config(cfg)
eng = Engine(env)
eng.set_launch_mode(Engine.LAUNCH_STAGES)
eng.init_states()
ctl = StepControl.from_config(cfg)
ctl.Rn, ctl.Ts = 1e9, 0
eng.begin(ctl)
eng.enqueue_steps(32)
eng.synchronize()
L, B, P = 12, 1024, 10
buf = (C.c_ulonglong * (L * B * P))()
assert lib().osc_debug_trace(buf, L * B * P) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(L, B, P).astype(np.float64)
nb = int((t[0, :, 0] > 0).sum())
t = t[:, :nb]
base = t[:, :, 0].min()
t = (t - base) * 1e-3  # us
names = ["S2", "S3", "S4"]
prev_done = 0.0
print(f"{name}: {nb} blocks; times in us relative to the previous launch's last block")
print("launch   entry(min/avg/max)        ready(avg/max)   loop0(avg/max)   loop1(min/avg/max)      exit(avg/max)  last: ticket reduced published done")
for l in range(L):
    x = t[l]
    done = x[:, 5].max()
    rel = x - prev_done
    ent = rel[:, 0]
    ex = np.where(x[:, 4] > 0, rel[:, 4], rel[:, 5])
    lb = int(np.argmax(x[:, 5]))  # the last block
    print(f"{l // 3}:{names[l % 3]}  {ent.min():6.2f} {ent.mean():6.2f} {ent.max():6.2f}   "
          f"{rel[:, 1].mean():6.2f} {rel[:, 1].max():6.2f}   {rel[:, 2].mean():6.2f} {rel[:, 2].max():6.2f}   "
          f"{rel[:, 3].min():6.2f} {rel[:, 3].mean():6.2f} {rel[:, 3].max():6.2f}   {ex.mean():6.2f} {ex.max():6.2f}  "
          f"{rel[lb, 6]:6.2f} {rel[lb, 7]:6.2f} {rel[lb, 8]:6.2f} {done - prev_done:6.2f}")
    prev_done = done
