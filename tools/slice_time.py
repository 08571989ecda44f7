import sys, os
sys.path.insert(0, ".")
import torch
from paper_1907_05560_b200 import Engine, Environment, StepControl, baseline_config
for name, A in (("configs2", 512), ("configs4", 64), ("configs2", 4096)):
    cfg = baseline_config(name, Abins=A)
    env = Environment.from_config(cfg)
    eng = Engine(env); eng.set_launch_mode(Engine.LAUNCH_STAGES); eng.init_states()
    ctl = StepControl.from_config(cfg); ctl.Rn, ctl.Ts = 1e9, 0
    eng.begin(ctl); eng.enqueue_steps(16); eng.synchronize()
    s = torch.cuda.ExternalStream(eng.stream())
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); eng.enqueue_steps(200); e1.record(s); e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 200)
    print(name, A, os.environ.get("OSC_BLOCKS_PER_SM", "2"), f"{best*1e3:.1f} us/step")
