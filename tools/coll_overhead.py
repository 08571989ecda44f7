"""Per-step cost of the multi-GPU exchange path (NCCL all-gather of the stage
partials + control kernel) measured with a one-rank communicator."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_05560_b200 import Engine, Environment, StepControl, baseline_config  # noqa: E402

for name, n in (("configs2", 64), ("configs0", 256)):
    cfg = baseline_config(name)
    env = Environment.from_config(cfg)
    res = []
    for coll, p2p in ((False, False), (True, False), (True, True)):
        eng = Engine(env, force_collectives=coll)
        eng.init_states()
        if p2p:
            eng.comm_connect([eng.comm_export()])
        if not coll:
            eng.set_launch_mode(Engine.LAUNCH_STAGES)
        ctl = StepControl.from_config(cfg)
        ctl.Rn, ctl.Ts = 1e9, 0
        eng.begin(ctl)
        eng.enqueue_steps(16)
        eng.synchronize()
        best = 1e9
        for _ in range(3):
            t = time.perf_counter()
            eng.enqueue_steps(n)
            eng.synchronize()
            best = min(best, time.perf_counter() - t)
        res.append(best / n * 1e6)
        eng.close()
    print(f"{name}: stage kernels {res[0]:.1f} us/step; exchange path with one rank: NCCL {res[1]:.1f}, "
          f"device-initiated peer stores {res[2]:.1f} us/step")
