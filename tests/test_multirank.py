"""World-size-2 gloo test of the multi-GPU contract on CPU.

Each rank owns the theta block given by make_partitions (parallel.cpp:11-24),
computes its partial moment sums per stage, all-gathers them, and combines
them in ascending rank order — the same protocol the CUDA path runs with
NCCL (engine.cu exchange() + slot_total()).  The oracle supplies the stage
arithmetic; the result must equal the single-rank run.
"""
import os
import socket

import numpy as np
import pytest

from paper_1907_05560_b200.config import baseline_config


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, cfg_text, steps, out):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    import torch
    import torch.distributed as dist

    import pyoracle
    from paper_1907_05560_b200.config import parse_config

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = parse_config(cfg_text)
    parts = pyoracle.make_partitions(cfg.values["Abins"], world)
    lo, hi = parts[rank]
    o = pyoracle.Oracle(cfg, lo, hi)

    def allreduce_ordered(partial):
        bufs = [torch.zeros(len(partial), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(bufs, torch.tensor(partial, dtype=torch.float64))
        total = bufs[0].clone()
        for q in range(1, world):  # fixed ascending rank order
            total += bufs[q]
        return total.numpy(), [b.numpy() for b in bufs]

    r, dr = cfg.values["R0"], cfg.values["dr"]
    for _ in range(steps):
        o.prepare(r, dr)
        for st in range(3):
            tot, _ = allreduce_ordered(o.stage(st))
            o.stage_set(st, tot)
        _, errs = allreduce_ordered(o.stage(3))
        err = max(float(e[0]) for e in errs)  # reduce_max
        assert np.isfinite(err)
        o.commit()  # eps0 = 1e30: every step accepted (fixed-step walk)
        r = r + dr
    states = [None] * world
    dist.all_gather_object(states, o.get_state())
    if rank == 0:
        out.put(np.concatenate(states))
    dist.destroy_process_group()


@pytest.mark.parametrize("model", ["bulb", "ebulb"])
def test_two_rank_gloo_matches_single_rank(pyoracle, model):
    import torch.multiprocessing as mp

    cfg = baseline_config("configs0", Abins=9, Ebins=12, R0=50, Rn=51, dr=1e-4, max_dr=1e-4,
                          Ts=8)
    if model == "ebulb":
        cfg.override("model=ebulb").override("Pbins=3").override("perturb=1e-8")
    steps = 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, cfg.render(), steps, q))
             for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = pyoracle.Oracle(cfg)
    single.run()
    want = single.get_state()
    assert got.shape == want.shape
    assert np.max(np.abs(got - want)) <= 1e-13


def test_partitions_cover_and_order(pyoracle):
    for n in (1, 7, 9, 256, 4096):
        for w in (1, 2, 3, 4, 8):
            if w > n:
                continue
            parts = pyoracle.make_partitions(n, w)
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
