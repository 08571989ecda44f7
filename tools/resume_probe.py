"""Where does a resumed stage-kernel run leave the uninterrupted one?

Runs K steps, restores the state into a fresh engine (S1 rebuilds the Bloch
planes and sums0), and compares the sums0 the two engines start the next
step from, then the states after M more steps.  Usage:
    python tools/resume_probe.py [configs2|small] K M [batch]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1907_05560_b200 import Engine, Environment, StepControl, baseline_config  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "configs2"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    M = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    batch = int(sys.argv[4]) if len(sys.argv) > 4 else K
    if which == "configs2":
        cfg = baseline_config("configs2", R0=50, Rn=1e9, dr=5e-5, max_dr=5e-5, Ts=0)
    else:
        cfg = baseline_config("configs0", Abins=64, Ebins=40, R0=50, Rn=1e9, dr=5e-5, max_dr=5e-5, Ts=0)
    env = Environment.from_config(cfg)
    a = Engine(env)
    a.set_launch_mode(Engine.LAUNCH_STAGES)
    a.init_states()
    ctl = StepControl.from_config(cfg)
    a.begin(ctl)
    done = 0
    while done < K:
        n = min(batch, K - done)
        a.enqueue_steps(n)
        done += n
    a.synchronize()
    q = a.query()
    x = a.state()
    sa = a.debug_sums()
    b = Engine(env)
    b.set_launch_mode(Engine.LAUNCH_STAGES)
    b.init_states()
    b.set_state(x)
    c2 = StepControl.from_config(cfg)
    c2.r, c2.dr, c2.iter = q["r"], q["dr"], q["iter"]
    b.begin(c2)
    b.synchronize()
    sb = b.debug_sums()
    print("query", q)
    print("sums0 A", sa[:12])
    print("sums0 B", sb[:12])
    print("next  A", sa[48:60])
    print("sums0 bit-equal:", np.array_equal(sa[:12], sb[:12]), "max diff", np.max(np.abs(sa[:12] - sb[:12])))
    a.enqueue_steps(M)
    b.enqueue_steps(M)
    xa, xb = a.state(), b.state()
    qa, qb = a.query(), b.query()
    print("after", M, "steps: iters", qa["iter"], qb["iter"], "r", qa["r"], qb["r"],
          "states bit-equal:", np.array_equal(xa, xb), "max diff", np.max(np.abs(xa - xb)))


if __name__ == "__main__":
    main()
