"""The drop-in at the reference's own seams, on the GPU:

* the reference's solver unit suite (proj/tests/unit/test_solver.cpp, all 14
  cases, compiled unchanged against the drop-in Engine with a doctest
  stand-in: integration/_build/test_solver_b200), on one GPU and with the
  Engine spread over two ranks;
* the run/resume/analyze CLI (integration/oscflat_b200_cli.cpp;
  tools/oscflat.cpp cmd_run, analyze) with device-gated dumps through the reference's WriterLane /
  SnapshotFileWriter, compared file by file with the same CLI source driving
  the unmodified reference engine (integration/_build/oscflat_ref_cli), and
  run -> dump -> resume bit-exactness at the configs[2] size.
"""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(__file__))
import snapfile  # noqa: E402

from paper_1907_05560_b200 import baseline_config  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "integration", "_build")
SUITE = os.path.join(BUILD, "test_solver_b200")
CLI = os.path.join(BUILD, "oscflat_b200")
REF_CLI = os.path.join(BUILD, "oscflat_ref_cli")
RHO_TOL = 1e-8  # north star: every rho component within 1e-8

pytestmark = pytest.mark.gpu


def _need(path):
    if not os.path.exists(path):
        pytest.fail(f"{path} is not built (integration/Makefile, run __graft_entry__.build() with the reference present)")


@pytest.mark.parametrize("gpus", ["1", "2"])
def test_reference_solver_suite_through_dropin(gpus):
    """All TEST_CASEs of the reference's test_solver.cpp pass with
    solver::Engine replaced by the B200 drop-in: step control, O(dr^3)
    error order, trial steps, Ts/Rn termination, step collapse, single-angle
    closed form, series exponential with matter, collective unitarity,
    1-vs-2-lane bit invariance, run -> dump (OSCFSNAP) -> resume exactness,
    dims/hash checks, single-angle lane rejection, summary rendering.
    OSC_GPUS=2 spreads every multi-angle Engine over two ranks (one GPU:
    stream-ordered exchange)."""
    _need(SUITE)
    env = dict(os.environ, OSC_GPUS=gpus)
    r = subprocess.run([SUITE], capture_output=True, text=True, timeout=600, env=env)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0, r.stdout + r.stderr
    assert "14 passed | 0 failed" in r.stdout


def _density(payload, ebins):
    """rho components (|a|^2-|b|^2, 2 Re ab*, 2 Im ab*) of a mode-1 payload."""
    p = payload.reshape(-1, 4, ebins)
    ar, ai, br, bi = p[:, 0], p[:, 1], p[:, 2], p[:, 3]
    return np.stack([ar * ar + ai * ai - br * br - bi * bi, 2 * (ar * br + ai * bi), 2 * (ai * br - ar * bi)])


def _run(exe, cfg_path, out_dir, *extra, env=None):
    r = subprocess.run([exe, *extra[:1], "-c", str(cfg_path), "-o", str(out_dir), *extra[1:]], capture_output=True,
                       text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    kv = dict(line.split("= ", 1) for line in open(os.path.join(out_dir, "summary.kv")).read().splitlines()
              if "= " in line)
    return kv


def _files(d):
    return sorted(f for f in os.listdir(d) if "Snapshot" in f or "Average" in f)


def _cfg(**kw):
    cfg = baseline_config("configs0", **kw)
    for k in ("dumpMode=3", "itr_step1=70", "r_step2=0.004", "newFile_step=2", "filePrefix=cli_"):
        cfg.override(k)
    return cfg


def _compare_dirs(da, db, ebins, rho_tol=RHO_TOL):
    fa, fb = _files(da), _files(db)
    assert fa == fb and len(fa) >= 4, (fa, fb)
    for name in fa:
        ha, ra = snapfile.read(os.path.join(da, name))
        hb, rb = snapfile.read(os.path.join(db, name))
        assert ha["dims"] == hb["dims"] and ha["config_hash"] == hb["config_hash"]
        assert ha["spectra"]["E0"] == hb["spectra"]["E0"]
        assert [x[0] for x in ra] == [x[0] for x in rb], name
        for (ia, r_a, dr_a, _, pa), (_, r_b, dr_b, _, pb) in zip(ra, rb):
            # (adaptive steps: dr follows err, which differs at ~1e-9 relative)
            assert r_a == pytest.approx(r_b, rel=1e-11) and dr_a == pytest.approx(dr_b, rel=1e-8)
            if ha["mode"] == 1:
                assert np.max(np.abs(_density(pa, ebins) - _density(pb, ebins))) <= rho_tol, (name, ia)
            else:
                # (energy averages of |psi_e|^2: as close as the states, 1e-8)
                assert np.max(np.abs(pa - pb)) <= rho_tol * np.max(np.abs(pb)), (name, ia)


def test_cli_run_and_resume_match_reference_cli(tmp_path):
    """`run` then `resume` from the second mode-1 file: the same snapshot
    files (names, rotation every newFile_step records, record iterations,
    r, dr, payloads: rho within 1e-8, mode 2 within 1e-8 rel) and the same
    summary counts as the unmodified reference engine behind the same CLI —
    an adaptive resolved run, dumps gated by iteration
    (mode 1) and by radius (mode 2)."""
    _need(CLI)
    _need(REF_CLI)
    cfg = _cfg(Abins=48, Ebins=40, R0=50, Rn=50.05, dr=1e-3, max_dr=0.05, eps0=1e-8, Ts=0)
    path = tmp_path / "run.cfg"
    path.write_text(cfg.render())
    runs = {}
    for tag, exe in (("gpu", CLI), ("ref", REF_CLI)):
        d = tmp_path / tag
        runs[tag] = _run(exe, path, d, "run", "--lanes", "4")
    assert runs["gpu"]["iterations"] == runs["ref"]["iterations"]
    assert runs["gpu"]["accepted"] == runs["ref"]["accepted"] and int(runs["ref"]["accepted"]) > 20
    assert float(runs["gpu"]["final_r"]) == pytest.approx(float(runs["ref"]["final_r"]), rel=1e-11)
    _compare_dirs(tmp_path / "gpu", tmp_path / "ref", 40)
    snap = sorted(f for f in _files(tmp_path / "ref") if "Snapshot" in f)[1]
    for tag, exe in (("gpu", CLI), ("ref", REF_CLI)):
        d = tmp_path / (tag + "_resume")
        runs[tag + "_resume"] = _run(exe, path, d, "resume", "-s", str(tmp_path / "ref" / snap))
    assert runs["gpu_resume"]["iterations"] == runs["ref_resume"]["iterations"]
    _compare_dirs(tmp_path / "gpu_resume", tmp_path / "ref_resume", 40)
    # `analyze` (the reference's analysis::analyze_file, host code) on the
    # last mode-1 and mode-2 files each engine wrote: survival grids, final
    # spectra and the content series agree
    for kind in ("Snapshot", "Average"):
        last = sorted((f for f in _files(tmp_path / "ref") if kind in f),
                      key=lambda f: int(f.split(kind)[1].split("_")[0]))[-1]
        outs = []
        for tag, exe in (("gpu", CLI), ("ref", REF_CLI)):
            od = tmp_path / f"an_{tag}_{kind}"
            r = subprocess.run([exe, "analyze", "-i", str(tmp_path / tag / last), "-o", str(od)], capture_output=True,
                               text=True, timeout=300)
            assert r.returncode == 0, r.stdout + r.stderr
            outs.append(od)
        names = sorted(os.listdir(outs[0]))
        assert names == sorted(os.listdir(outs[1])) and len(names) == (8 if kind == "Snapshot" else 1)
        for n in names:
            a = np.loadtxt(outs[0] / n, delimiter=",", skiprows=1, ndmin=2)
            b = np.loadtxt(outs[1] / n, delimiter=",", skiprows=1, ndmin=2)
            assert a.shape == b.shape and a.size > 0, n
            assert np.allclose(a, b, rtol=1e-8, atol=1e-10), (n, np.max(np.abs(a - b)))


def test_cli_resume_is_bit_exact_at_configs2_size(tmp_path):
    """configs[2] shape (4096 theta x 256 E, 1,048,576 cells, 128 MiB per
    mode-1 record): run 24 fixed steps dumping every 8 iterations into one
    file per record, resume from the second file, and the resumed run's
    final record is bit-identical to the uninterrupted run's (the reference's
    own exactness test, test_solver.cpp:253-320, at the headline size)."""
    _need(CLI)
    cfg = baseline_config("configs2", R0=50, Rn=1e9, dr=5e-5, max_dr=5e-5, Ts=24)
    for k in ("dumpMode=1", "itr_step1=8", "newFile_step=1", "filePrefix=big_"):
        cfg.override(k)
    path = tmp_path / "run.cfg"
    path.write_text(cfg.render())
    _run(CLI, path, tmp_path / "a", "run")
    files = sorted(_files(tmp_path / "a"), key=lambda f: int(f.split("Snapshot")[1].split("_")[0]))
    assert len(files) == 4  # iterations 8, 16, 24 + the final state
    _, last = snapfile.read(str(tmp_path / "a" / files[-1]))
    _run(CLI, path, tmp_path / "b", "resume", "-s", str(tmp_path / "a" / files[1]))
    fb = sorted(_files(tmp_path / "b"), key=lambda f: int(f.split("Snapshot")[1].split("_")[0]))
    _, last_b = snapfile.read(str(tmp_path / "b" / fb[-1]))
    assert last_b[-1][0] == last[-1][0] == 24
    assert np.array_equal(last_b[-1][4], last[-1][4])
