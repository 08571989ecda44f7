"""In-process multi-rank engine (osc_create_group: the reference's lanes ->
GPUs, par::run_lanes parallel.cpp:224-253 / make_partitions :11-24) on real
hardware.  The round-end box has one GPU, so the ranks share it and exchange
their stage moments stream-ordered (no kernel ever waits on another rank's
kernel); the multi-rank stage kernels, the per-rank rank-slot publication,
the rank-order totals and the per-rank control kernel all run with >= 2
ranks.  Results must match the single-GPU engine: same accept/reject
sequence, states within 1e-12 (the rank partials are combined in rank
order, so the sums associate differently)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1907_05560_b200 import Engine, Environment, StepControl, baseline_config

pytestmark = pytest.mark.gpu


def _single(cfg, **kw):
    env = Environment.from_config(cfg)
    eng = Engine(env)
    return env, eng


def _group(cfg, n):
    env = Environment.from_config(cfg)
    return env, Engine.group(env, n, devices=[0] * n)


CASES = {
    # resolved windows (R0 = 50 km), adaptive with rejections, uneven theta split
    "bulb": lambda: baseline_config("configs0", Abins=25, Ebins=20, R0=50, Rn=50.2, dr=1e-3, max_dr=0.05, eps0=1e-8,
                                    Ts=60),
    "ebulb": lambda: baseline_config("configs0", Abins=12, Ebins=16, R0=50, Rn=50.2, dr=1e-3, max_dr=0.05, eps0=1e-8,
                                     Ts=40).override("model=ebulb").override("Pbins=6").override("perturb=1e-6"),
    "plane": lambda: baseline_config("configs3", Abins=12, Pbins=6, Ebins=16, Ts=20, dr=1e-4, max_dr=1e-4),
    "flavour3": lambda: baseline_config("configs1", Abins=14, Ebins=8, R0=50, Rn=60, Ts=12, dr=1e-4, max_dr=1e-4),
}


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("name", list(CASES))
def test_group_matches_single_gpu(name, nranks):
    cfg = CASES[name]()
    _, a = _single(cfg)
    a.init_states()
    sa = a.run(StepControl.from_config(cfg))
    env, g = _group(cfg, nranks)
    assert g.nranks == nranks and g.ordered and g.state_doubles == a.state_doubles
    g.init_states()
    assert np.array_equal(g.state(), _init_state(cfg))  # init_states seeds by global beam index
    sg = g.run(StepControl.from_config(cfg))
    assert (sg.iterations, sg.accepted, sg.rejected) == (sa.iterations, sa.accepted, sa.rejected)
    assert sg.iterations > 0 and (sa.rejected > 0 or name in ("plane", "flavour3"))
    assert sg.final_r == pytest.approx(sa.final_r, rel=1e-14)
    assert np.max(np.abs(g.state() - a.state())) <= 1e-12
    assert sg.final_max_norm_dev == pytest.approx(sa.final_max_norm_dev, rel=1e-6, abs=1e-15)
    assert g.launch_count() > 0


def _init_state(cfg):
    env = Environment.from_config(cfg)
    e = Engine(env)
    e.init_states()
    return e.state()


def test_group_trial_step_error_and_state_roundtrip():
    """trial_step_error through the group equals the single engine's (the
    global max over ranks) and never commits; set_state/get_state scatter
    and gather the rank slices in trajectory order; mode 2 likewise."""
    cfg = baseline_config("configs0", Abins=21, Ebins=24, R0=50, Rn=60, dr=1e-3, max_dr=1e-3)
    env, a = _single(cfg)
    _, g = _group(cfg, 3)
    a.init_states()
    g.init_states()
    rng = np.random.default_rng(7)
    x = a.state() * (1.0 + 1e-3 * rng.standard_normal(a.state_doubles))
    a.set_state(x)
    g.set_state(x)
    assert np.array_equal(g.state(), a.state())
    assert np.array_equal(g.mode2(), a.mode2())
    ea, eg = a.trial_step_error(50.0, 0.5), g.trial_step_error(50.0, 0.5)
    assert eg == pytest.approx(ea, rel=1e-9) and ea > 0
    assert np.array_equal(g.state(), a.state())


def test_group_dumps_and_hook_match_single_gpu():
    """Device-gated dumps (iteration and radius gates) and the per-step hook
    through a 2-rank group: the same dump sequence as the single engine,
    payloads gathered over the ranks (mode 1 within 1e-12, mode 2 within
    1e-12 rel)."""
    cfg = baseline_config("configs0", Abins=16, Ebins=20, R0=50, Rn=50.2, dr=1e-3, max_dr=0.05, eps0=1e-8, Ts=60)
    gates = [(0.0, 0.0, 4), (0.001, 0.0, 0)]
    out = []
    for mk in (_single, lambda c: _group(c, 2)):
        env, e = mk(cfg)
        e.init_states()
        got = []
        e.run_dumps(StepControl.from_config(cfg), gates, 3, lambda m, meta, p: got.append((m, meta.iter, meta.r, p)))
        hooks = []
        e.init_states()
        e.run(StepControl.from_config(cfg), hook=lambda info, st: hooks.append((info.iter, st)))
        out.append((got, hooks))
    (ga, ha), (gb, hb) = out
    assert [(m, i) for m, i, *_ in ga] == [(m, i) for m, i, *_ in gb] and len(ga) > 8
    assert any(m == 2 for m, *_ in ga)
    for (m, _, ra, pa), (_, _, rb, pb) in zip(ga, gb):
        assert ra == pytest.approx(rb, rel=1e-14)
        assert np.max(np.abs(pa - pb)) <= 1e-12 * max(1.0, np.max(np.abs(pa)))
    assert [i for i, _ in ha] == [i for i, _ in hb] and len(ha) > 5
    assert max(np.max(np.abs(x - y)) for (_, x), (_, y) in zip(ha, hb)) <= 1e-12
