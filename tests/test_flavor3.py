"""Three-flavour path (BASELINE configs[1]).

The reference rejects Flvs != 2 (config.cpp:298), so parity is UNPINNED; the
3-flavour C restatement (oracle/oscflat3_oracle.c) is pinned by:
  * its series exponential against scipy's expm (the SU(3) analogue of
    testutil.hpp:56-95);
  * the decoupled-flavour reduction: with theta13 = theta23 = 0 and a dark tau
    sector, the e-mu densities reproduce the unmodified 2-flavour reference.
"""
import numpy as np
import pytest
import scipy.linalg as sl

from paper_1907_05560_b200 import baseline_config


def herm9(H):
    return np.array([H[0, 0].real, H[1, 1].real, H[2, 2].real, H[0, 1].real, H[0, 1].imag,
                     H[0, 2].real, H[0, 2].imag, H[1, 2].real, H[1, 2].imag])


def test_oracle_series_exponential(pyoracle):
    o = pyoracle.Oracle3(baseline_config("configs1", Abins=2, Ebins=2))
    rng = np.random.default_rng(5)
    for k in range(300):
        A = rng.normal(size=(3, 3)) + 1j * rng.normal(size=(3, 3))
        H = (A + A.conj().T) * 10 ** rng.uniform(-3, 2)
        tau = 10 ** rng.uniform(-3, 0)
        U = o.expm(herm9(H), tau)
        np.testing.assert_allclose(U, sl.expm(-1j * H * tau), atol=1e-12 * max(1, np.abs(H).max() * tau))
        assert np.abs(U @ U.conj().T - np.eye(3)).max() <= 1e-13


def decoupled_pair(r0=50.0, steps=12):
    """(3-flavour config, matching 2-flavour config): theta12 = theta, dm21 = dm2,
    theta13 = theta23 = 0, tau luminosity 0."""
    kw = dict(Abins=6, Ebins=10, R0=r0, Rn=r0 + 1, dr=2e-4, max_dr=2e-4, Ts=steps)
    c2 = baseline_config("configs0", **kw)
    c3 = baseline_config("configs1", **kw)
    for kv in ("dm2_21=-2.35e-3", "theta12=0.1", "theta13=0", "theta23=0", "dm2_31=-2.4e-3",
               "Lvtau=0", "Lvatau=0", "hasMatter=0"):
        c3.override(kv)
    return c3, c2


def embed(s2, ntraj, E):
    """2-flavour mode-1 payload -> 3-flavour payload (tau species pure tau)."""
    a = s2.reshape(ntraj, 4, 4, E)
    s3 = np.zeros((ntraj, 6, 6, E))
    s3[:, :4, :4] = a
    s3[:, 4, 4] = 1.0
    s3[:, 5, 4] = 1.0
    return s3.ravel()


def rho_emu(s3, ntraj, E):
    x = s3.reshape(ntraj, 6, 6, E)[:, :4]
    ae, be = x[:, :, 0] + 1j * x[:, :, 1], x[:, :, 2] + 1j * x[:, :, 3]
    return np.stack([abs(ae) ** 2 - abs(be) ** 2, 2 * (ae * be.conj()).real,
                     2 * (ae * be.conj()).imag])


def rho2(s2, ntraj, E):
    x = s2.reshape(ntraj, 4, 4, E)
    a, b = x[:, :, 0] + 1j * x[:, :, 1], x[:, :, 2] + 1j * x[:, :, 3]
    return np.stack([abs(a) ** 2 - abs(b) ** 2, 2 * (a * b.conj()).real, 2 * (a * b.conj()).imag])


def test_decoupled_tau_reproduces_two_flavour_reference(pyoracle, ref):
    c3, c2 = decoupled_pair()
    init2, _ = ref.run(c2.render(), lanes=1, ts=0, r=c2.values["Rn"], dr=0.0)  # reference init
    want, summ = ref.run(c2.render(), lanes=1)
    o3 = pyoracle.Oracle3(c3)
    o3.set_state(embed(init2, 6, 10))
    s = o3.run()
    assert s["iterations"] == summ["iterations"] == 12
    got = rho_emu(o3.get_state(), 6, 10)
    assert np.abs(got - rho2(want, 6, 10)).max() <= 1e-12


def test_three_flavour_resolved_run_is_unitary(pyoracle):
    cfg = baseline_config("configs1", Abins=8, Ebins=6, R0=50, Rn=51, dr=1e-6, max_dr=1e-6, Ts=10)
    o = pyoracle.Oracle3(cfg)
    s = o.run()
    assert s["iterations"] == 10 and s["final_max_norm_dev"] <= 1e-12


def test_three_flavour_config_validation():
    from paper_1907_05560_b200 import ConfigError

    c = baseline_config("configs1")
    c.require_runnable()
    c.override("model=ebulb")
    with pytest.raises(ConfigError):
        c.require_runnable()
