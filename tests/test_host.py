"""CPU tests of the product's host side: library loading / exported symbols,
the Environment builder against the reference's golden tables, and the
config vocabulary (reference config.cpp)."""
import ctypes as C
import json
import os
import re

import numpy as np
import pytest

from paper_1907_05560_b200 import (BASELINE_CONFIGS, ConfigError, Environment, baseline_config,
                                   fermi_integral, parse_config)
from paper_1907_05560_b200 import native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def header_symbols():
    syms = set()
    for f in os.listdir(os.path.join(ROOT, "include")):
        if f.endswith(".h"):
            txt = open(os.path.join(ROOT, "include", f)).read()
            syms |= set(re.findall(r"^\s*(?:int|double|unsigned long long|void\s*\*|const char\s*\*|void)\s+(osc_\w+)\s*\(",
                                   txt, flags=re.M))
    return syms


def test_library_exports_every_header_symbol():
    L = native.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert set(native.SYMBOLS) == syms


def test_library_is_sm100a():
    so = native.LIB
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {so} 2>&1").read()
    assert "sm_100a" in out, out


def test_env_tables_match_reference_golden():
    g = np.load(os.path.join(GOLD, "golden.npz"))
    meta = json.load(open(os.path.join(GOLD, "golden_meta.json")))
    for name, text in meta["cases"].items():
        t = Environment.from_config(parse_config(text)).tables()
        for k, v in t.items():
            np.testing.assert_allclose(v, g[f"{name}/tab_{k}"], rtol=1e-14, atol=0,
                                       err_msg=f"{name}:{k}")


def test_fermi_integral_golden():
    g = np.load(os.path.join(GOLD, "golden.npz"))
    for k, eta, want in g["kat_fermi"]:
        assert fermi_integral(int(k), eta) == pytest.approx(want, rel=1e-14)


def test_config_parse_and_validation():
    cfg = parse_config("Abins= 8 # comment\nunknownKey= 3\n\nmodel= ebulb\n")
    assert cfg.values["Abins"] == 8 and cfg.model_id == 2
    assert any("unknownKey" in w for w in cfg.warnings)
    with pytest.raises(ConfigError):
        parse_config("Abins 8\n")
    with pytest.raises(ConfigError):
        cfg.require_runnable()  # physics keys missing
    c = baseline_config("configs0")
    c.require_runnable()
    c.override("Flvs=4")
    with pytest.raises(ConfigError):
        c.require_runnable()
    c.override("Flvs=3")
    c.require_runnable()  # 3 flavours: sa / bulb (configs[1])


def test_baseline_configs_shapes():
    c0 = baseline_config("configs0")
    assert (c0.Abins, c0.Ebins, c0.Ts, c0.max_dr) == (256, 100, 2000, 0.12)
    assert c0.R0 + c0.Ts * c0.max_dr == pytest.approx(250.0)
    c2 = baseline_config("configs2")
    assert (c2.Abins, c2.Ebins, c2.Ts) == (4096, 256, 1000)
    assert c2.R0 + c2.Ts * c2.max_dr == pytest.approx(250.0)
    assert set(BASELINE_CONFIGS) >= {"configs0", "configs2"}


def test_bad_descriptor_is_config_error():
    env = Environment.from_config(baseline_config("configs0", Abins=4, Ebins=8))
    d = env.desc
    d2 = native.OscDesc.from_buffer_copy(d)
    d2.model = 7
    ctx = C.c_void_p()
    rc = native.lib().osc_create(C.byref(d2), None, C.byref(ctx))
    assert rc == 1  # OSC_ERR_CONFIG, raised before any device call


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/core/include"), reason="reference headers absent")
def test_engine_shim_compiles_against_reference_headers():
    """integration/solver_b200.cpp implements the reference's solver::Engine
    declaration (solver.hpp:128-153) over include/oscflat_b200.h."""
    import subprocess

    r = subprocess.run(["g++", "-std=gnu++20", "-fsyntax-only", "-include", "cstdint",
                        "-I", "/root/reference/proj/core/include", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "integration", "solver_b200.cpp")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
