"""Plane (BASELINE configs[3]) and cylinder (configs[4]) geometries.

The reference does not implement these models (config.cpp:298),
so parity is UNPINNED: the C oracle's factorised moment reduction is checked
against a brute-force pairwise (1 - v.v') double sum, the same way the
reference pins its bulb / extended-bulb reduction
(proj/tests/unit/test_geometry.cpp:26-48, 183-227).
"""
import numpy as np
import pytest

from paper_1907_05560_b200 import baseline_config


def directions(model, tab, T, P, r, Rnu):
    """Unit propagation vectors and weights per trajectory."""
    v = np.zeros((T * P, 3))
    w = np.zeros(T * P)
    for t in range(T):
        for q in range(P):
            j = t * P + q
            if model == 3:
                ct, st = tab["cos2"][t], tab["sin0"][t]
                v[j] = (ct, st * tab["cphi"][q], st * tab["sphi"][q])
                w[j] = 1.0 / (T * P)
            else:
                ra = Rnu / r
                sa = ra * tab["sin0"][t]
                ca = np.sqrt(1 - sa * sa)
                cb, sb = tab["cphi"][q], tab["sphi"][q]
                v[j] = (cb * ca, cb * sa, sb)
                w[j] = ra * tab["cos2"][t] / ca / (T * P)
    return v, w


@pytest.mark.parametrize("name,r", [("configs3", 3.7), ("configs4", 17.0), ("configs4", 10.5)])
def test_factorised_moments_equal_pairwise_sum(pyoracle, name, r):
    cfg = baseline_config(name, Abins=7, Pbins=5, Ebins=3)
    o = pyoracle.Oracle(cfg)
    tab = o.tables()
    T, P = 7, 5
    rng = np.random.default_rng(11)
    rows = rng.uniform(-1, 1, size=(T * P * 4, 3))
    sums, hvv = o.hvv_from_rows(r, rows)
    c = tab["couplings"]
    R = np.zeros((T * P, 3))
    for j in range(T * P):
        for s in range(4):
            row = rows[j * 4 + s].copy()
            if s & 1:
                row[2] = -row[2]
                R[j] -= c[s] * row
            else:
                R[j] += c[s] * row
    v, w = directions(cfg.model_id, tab, T, P, r, cfg.values["Rv"])
    brute = 0.5 * np.einsum("ij,j,jk->ik", 1.0 - v @ v.T, w, R)
    scale = np.abs(brute).max()
    assert np.abs(hvv - brute).max() <= 1e-12 * scale


def test_plane_azimuthal_symmetry_cancels_transverse_moments(pyoracle):
    cfg = baseline_config("configs3", Abins=6, Pbins=8, Ebins=3)
    o = pyoracle.Oracle(cfg)
    rng = np.random.default_rng(3)
    theta_rows = rng.uniform(-1, 1, size=(6, 4, 3))
    rows = np.repeat(theta_rows[:, None], 8, axis=1).reshape(-1, 3)  # phi-symmetric data
    sums, hvv = o.hvv_from_rows(1.0, rows)
    assert np.abs(sums[6:]).max() <= 1e-13 * np.abs(sums[:6]).max()
    h = hvv.reshape(6, 8, 3)
    assert np.abs(h - h[:, :1]).max() <= 1e-13 * np.abs(h).max()  # H independent of phi


def test_cylinder_weights_normalised_at_surface(pyoracle):
    cfg = baseline_config("configs4", Abins=64, Pbins=16, Ebins=3)
    o = pyoracle.Oracle(cfg)
    tab = o.tables()
    _, w = directions(4, tab, 64, 16, cfg.values["Rv"], cfg.values["Rv"])
    assert w.sum() == pytest.approx(1.0, rel=1e-12)  # isotropic half-plane emission


def test_plane_and_cylinder_runs_conserve_norm_when_resolved(pyoracle):
    for name, r0 in (("configs3", 0.0), ("configs4", 30.0)):
        cfg = baseline_config(name, Abins=6, Pbins=4, Ebins=8, R0=r0, Rn=r0 + 1,
                              dr=1e-7, max_dr=1e-7, Ts=30)
        o = pyoracle.Oracle(cfg)
        s = o.run()
        assert s["iterations"] == 30
        assert s["final_max_norm_dev"] <= 1e-12
