"""Generate tests/golden/golden.npz from the reference itself.

Runs the UNMODIFIED reference core (compiled by oracle/Makefile from
/root/reference/proj/core into oracle/_ref, driven by oracle/ref_harness.cpp)
on small seeded cases and stores inputs + outputs.  Only needs to run where
/root/reference exists; the fixtures are committed and travel with the repo.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle  # noqa: E402

from paper_1907_05560_b200.config import baseline_config  # noqa: E402


def cases():
    """name -> RunConfig (small shapes the CPU reference finishes instantly)."""
    out = {}
    c = baseline_config("configs0", Abins=8, Ebins=16, R0=50, Rn=51, dr=1e-4, max_dr=1e-4, Ts=20)
    out["bulb_resolved"] = c
    c = baseline_config("configs0", Abins=8, Ebins=16, Ts=6)
    out["bulb_unresolved"] = c  # literal configs[0] step near R_nu
    c = baseline_config("configs0", Abins=6, Ebins=12, R0=50, Rn=51, dr=1e-4, max_dr=1e-4, Ts=20)
    c.override("model=ebulb").override("Pbins=4").override("perturb=1e-8")
    out["ebulb_resolved"] = c
    c = baseline_config("configs0", Abins=1, Ebins=16, R0=50, Rn=51, dr=1e-3, max_dr=1e-3, Ts=20)
    c.override("model=sa")
    out["sa_resolved"] = c
    c = baseline_config("configs0", Abins=9, Ebins=10, R0=50, Rn=60, dr=1e-3, max_dr=1e-2, Ts=40)
    for kv in ("eps0=1e-9", "hasMatter=1", "matterProfile=sum", "Ye=0.5", "nb0=1e30", "hNS=5",
               "eta_ve=3", "eta_vae=3", "Eve=11", "Evae=16", "Mns=1.4", "gs=1", "S=100"):
        c.override(kv)
    out["bulb_adaptive_matter"] = c
    return out


def main():
    ref = pyoracle.Ref()
    rng = np.random.default_rng(20191907)
    g = {}
    meta = {"reference": "/root/reference/proj/core (oscflat)", "variant": ref.variant,
            "cases": {}}
    # --- kernels: evolve_bin / density KATs (beam.hpp:96-121)
    H = rng.uniform(-2, 2, size=(256, 3))
    H[:8] = 0.0  # lambda = 0 -> identity branch
    DL = rng.uniform(0.01, 2.0, size=256)
    PSI = rng.uniform(-1, 1, size=(256, 4))
    PSI /= np.linalg.norm(PSI, axis=1, keepdims=True)
    g["kat_h"], g["kat_dl"], g["kat_psi"] = H, DL, PSI
    g["kat_evolve"] = np.array([ref.evolve_bin(H[i], DL[i], PSI[i]) for i in range(256)])
    g["kat_density"] = np.array([ref.density(PSI[i]) for i in range(256)])
    # --- init_flavor_state (beam.cpp:41-57)
    inits = []
    for s in range(4):
        for eps, seed in ((1e-10, 7), (1e-8, 12345), (0.3, 2**40 + 3)):
            inits.append(ref.init_state(s, 37, eps, seed))
    g["kat_init"] = np.array(inits)
    # --- Fermi integrals (spectra.cpp:77-83)
    g["kat_fermi"] = np.array([[k, eta, ref.fermi_integral(k, eta)]
                               for k in (2, 3) for eta in (-2.0, 0.0, 3.0)])
    # --- per-case tables, partial sums, trial step, short run
    for name, cfg in cases().items():
        text = cfg.render()
        meta["cases"][name] = text
        t = ref.tables(text)
        for k, v in t.items():
            g[f"{name}/tab_{k}"] = v
        d = ref.dims(text)
        ntraj = d["abins"] * d["pbins"]
        rows = rng.uniform(-1, 1, size=(ntraj * 4, 3))
        r_probe = cfg.values["R0"] + 0.37
        sums, hvv = ref.partial_hvv(text, r_probe, rows)
        g[f"{name}/rows"], g[f"{name}/r_probe"] = rows, np.array([r_probe])
        g[f"{name}/sums"], g[f"{name}/hvv"] = sums, hvv
        g[f"{name}/cache"] = ref.fill_cache(text, r_probe)
        g[f"{name}/matter"] = np.array([[r, ref.matter(text, r)] for r in (10.0, 30.0, 50.5, 200.0)])
        err, _ = ref.trial_step(text, cfg.values["R0"], cfg.values["dr"])
        g[f"{name}/trial_err"] = np.array([err])
        init, _ = ref.run(text, lanes=1, ts=0, r=cfg.values["Rn"], dr=0.0)  # no steps: init state
        g[f"{name}/init_state"] = init
        state, summ = ref.run(text, lanes=1)
        g[f"{name}/final_state"] = state
        g[f"{name}/summary"] = np.array([summ["final_r"], summ["iterations"], summ["accepted"],
                                         summ["rejected"], summ["final_max_norm_dev"]])
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **g)
    json.dump(meta, open(os.path.join(HERE, "golden_meta.json"), "w"), indent=1)
    print("wrote", len(g), "arrays")


if __name__ == "__main__":
    main()
