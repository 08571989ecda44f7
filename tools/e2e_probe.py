import sys, time
sys.path.insert(0, ".")
import torch
from paper_1907_05560_b200 import Engine, Environment, StepControl, baseline_config
cfg = baseline_config("configs2")
env = Environment.from_config(cfg)
eng = Engine(env)
eng.init_states()
n = eng.state_doubles
hin = torch.empty(n, dtype=torch.float64).pin_memory()
hout = torch.empty(n, dtype=torch.float64).pin_memory()
eng.get_state_host_ptr(hin.data_ptr(), n)
dev = torch.empty(n, dtype=torch.float64, device="cuda")
s = torch.cuda.ExternalStream(eng.stream())
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); dev.copy_(hin, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    hout.copy_(dev, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"raw H2D {128*1.048576/(t1-t0)/1e3:.1f} GB/s ({(t1-t0)*1e3:.2f} ms), D2H {128*1.048576/(t2-t1)/1e3:.1f} GB/s ({(t2-t1)*1e3:.2f} ms)")
ctl = StepControl.from_config(cfg); ctl.Ts = 20; ctl.Rn = 1e9
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); eng.set_state_host_ptr(hin.data_ptr(), n); t1 = time.perf_counter()
    summ = eng.run(ctl); t2 = time.perf_counter()
    eng.get_state_host_ptr(hout.data_ptr(), n); t3 = time.perf_counter()
    print(f"set_state {1e3*(t1-t0):.2f} ms, run(20) {1e3*(t2-t1):.2f} ms (wall_s {summ.wall_s*1e3:.2f}), get_state {1e3*(t3-t2):.2f} ms, total {1e3*(t3-t0):.2f}")
