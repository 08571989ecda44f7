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
cfg = baseline_config(name, **({"Abins": int(os.environ["TRACE_ABINS"])} if os.environ.get("TRACE_ABINS") else {}))
env = Environment.from_config(cfg)
eng = Engine(env)
eng.set_launch_mode(Engine.LAUNCH_STAGES)
eng.init_states()
ctl = StepControl.from_config(cfg)
ctl.Rn, ctl.Ts = 1e9, 0
eng.begin(ctl)
eng.enqueue_steps(32)
eng.synchronize()
L, B, P = 12, 1024, 14
buf = (C.c_ulonglong * (L * B * P))()
assert lib().osc_debug_trace(buf, L * B * P) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(L, B, P).astype(np.float64)
smid = t[:, :, 9].copy()
t[:, :, 9] = 0
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
          f"{rel[lb, 6]:6.2f} {rel[lb, 7]:6.2f} {rel[lb, 8]:6.2f} {done - prev_done:6.2f}"
          + ("" if not (x[:, 6] > 0).all() else
             f"   [cr: waited {rel[:, 6].mean():6.2f} totals {rel[:, 7].mean():6.2f} ktab {rel[:, 8].mean():6.2f}]")
          + ("" if not (x[:, 10] > 0).all() else
             f"   [S2: wait done {rel[:, 10].mean():6.2f} reduced {rel[:, 11].mean():6.2f} decided {rel[:, 12].mean():6.2f}"
             f" tma issued {rel[:, 13].mean():6.2f}]"))
    prev_done = done

# per-block main-loop durations of the last traced S4 and S2: by SM and by block
for l in (L - 1, L - 3):
    x = t[l]
    dur = x[:, 3] - x[:, 2]
    sm = smid[l].astype(int)
    order = np.argsort(dur)
    print(f"{names[l % 3]} loop durations: min {dur.min():.2f} median {np.median(dur):.2f} max {dur.max():.2f} us")
    print("  slowest blocks (block, sm, dur, start):", [(int(b), int(sm[b]), round(dur[b], 2), round(x[b, 2] - x[:, 2].min(), 2)) for b in order[-12:]])
    print("  fastest blocks:", [(int(b), int(sm[b]), round(dur[b], 2)) for b in order[:6]])
    # blocks sharing an SM: duration of the pair
    per_sm = {}
    for b in range(nb):
        per_sm.setdefault(sm[b], []).append(dur[b])
    sm_max = np.array([max(v) for v in per_sm.values()])
    print(f"  per-SM max duration: min {sm_max.min():.2f} median {np.median(sm_max):.2f} max {sm_max.max():.2f}; SMs used {len(per_sm)}")
    # correlation with block index (memory position)
    q = np.array_split(np.arange(nb), 8)
    print("  mean duration by block-index octile:", [round(float(dur[i].mean()), 2) for i in q])
    st0 = x[:, 2] - x[:, 2].min()
    print("  mean loop start by octile:", [round(float(st0[i].mean()), 2) for i in q])
    print("  mean loop end by octile:  ", [round(float((x[:, 3] - x[:, 2].min())[i].mean()), 2) for i in q])
    sm = sm[:nb]
    print("  mean duration by SM-id group of 18:",
          [round(float(dur[sm // 18 == g].mean()), 2) for g in range(int(sm.max()) // 18 + 1) if (sm // 18 == g).any()])
