"""The closed-form 3x3 exponential of the 3-flavour stages (csrc/su3_exp.cuh;
the SU(3) analogue of flavor::evolve_bin, beam.hpp:105-121 — outside the
reference, so pinned against scipy's expm and the restatement's series
exponential instead).

CPU: the header's host build (plain C++, same algorithm as the device code)
on random, degenerate and badly scaled spectra.  GPU: the device code through
osc_debug_exp3, same cases, plus host-vs-device agreement."""
import ctypes as C
import os
import subprocess
import tempfile

import numpy as np
import pytest
import scipy.linalg as sl

from conftest import ROOT, gpu_available

HARNESS = r"""
#include "su3_exp.cuh"
using namespace oscb200;
extern "C" void su3_exp_host(int n, const double* H, const double* tau, double* U, int path) {
    for (int i = 0; i < n; ++i) {
        Herm3 h;
        for (int k = 0; k < 3; ++k) h.d[k] = H[9 * i + k];
        h.o01 = Cx{H[9 * i + 3], H[9 * i + 4]};
        h.o02 = Cx{H[9 * i + 5], H[9 * i + 6]};
        h.o12 = Cx{H[9 * i + 7], H[9 * i + 8]};
        const Mat3 u = path == 0 ? exp_herm3(h, tau[i]) : exp_from_eig(eig_herm3(h), tau[i]);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                U[18 * i + (r * 3 + c) * 2] = u.m[r][c].re;
                U[18 * i + (r * 3 + c) * 2 + 1] = u.m[r][c].im;
            }
    }
}
"""


@pytest.fixture(scope="module")
def host_exp():
    d = tempfile.mkdtemp(prefix="su3host_")
    src, lib = os.path.join(d, "h.cpp"), os.path.join(d, "h.so")
    open(src, "w").write(HARNESS)
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-shared", "-fPIC", "-x", "c++", src,
                    "-I", os.path.join(ROOT, "paper_1907_05560_b200", "csrc"), "-o", lib], check=True)
    L = C.CDLL(lib)
    dp = C.POINTER(C.c_double)
    L.su3_exp_host.argtypes = [C.c_int, dp, dp, dp, C.c_int]

    def run(H9, tau, path=0):
        H9 = np.ascontiguousarray(H9, dtype=np.float64).reshape(-1, 9)
        n = H9.shape[0]
        tau = np.ascontiguousarray(tau, dtype=np.float64).reshape(n)
        out = np.zeros((n, 18))
        L.su3_exp_host(n, H9.ctypes.data_as(dp), tau.ctypes.data_as(dp), out.ctypes.data_as(dp), path)
        return (out[:, 0::2] + 1j * out[:, 1::2]).reshape(n, 3, 3)

    return run


def pack(H):
    return np.array([H[0, 0].real, H[1, 1].real, H[2, 2].real, H[0, 1].real, H[0, 1].imag,
                     H[0, 2].real, H[0, 2].imag, H[1, 2].real, H[1, 2].imag])


def from_spectrum(rng, lam):
    """A Hermitian matrix with the given eigenvalues and a random eigenbasis."""
    Z = rng.normal(size=(3, 3)) + 1j * rng.normal(size=(3, 3))
    Qm, _ = np.linalg.qr(Z)
    H = (Qm * np.asarray(lam)) @ Qm.conj().T
    return 0.5 * (H + H.conj().T)


def cases():
    rng = np.random.default_rng(20240607)
    Hs, taus = [], []
    for _ in range(200):  # generic
        A = rng.normal(size=(3, 3)) + 1j * rng.normal(size=(3, 3))
        Hs.append(0.5 * (A + A.conj().T) * 10.0 ** rng.uniform(-3, 2))
        taus.append(10.0 ** rng.uniform(-3, 1))
    for gap in (0.0, 1e-15, 1e-12, 1e-9, 1e-6, 1e-3):  # (near-)degenerate pairs, both sides
        for sgn in (1.0, -1.0):
            for _ in range(5):
                Hs.append(from_spectrum(rng, [sgn * 2.0, sgn * (-1.0 + gap), sgn * (-1.0 - gap)]) + 0.3 * np.eye(3))
                taus.append(rng.uniform(0.1, 3.0))
    for eps in (0.0, 1e-14, 1e-10, 1e-6):  # all three (nearly) equal
        for _ in range(4):
            Hs.append(from_spectrum(rng, [1.0 + eps, 1.0, 1.0 - 2 * eps]))
            taus.append(rng.uniform(0.1, 3.0))
    for _ in range(20):  # symmetric spectrum (q = 0: either root is "most isolated")
        x = rng.uniform(0.1, 5.0)
        Hs.append(from_spectrum(rng, [x, 0.0, -x]))
        taus.append(rng.uniform(0.1, 3.0))
    for _ in range(20):  # diagonal and block-diagonal (a decoupled flavour)
        H = np.diag(rng.normal(size=3)).astype(complex)
        if rng.random() < 0.5:
            H[0, 1] = rng.normal() + 1j * rng.normal()
            H[1, 0] = np.conj(H[0, 1])
        Hs.append(H)
        taus.append(rng.uniform(0.1, 3.0))
    for s in (1e-60, 1e-30, 1e30):  # badly scaled
        A = rng.normal(size=(3, 3)) + 1j * rng.normal(size=(3, 3))
        Hs.append(0.5 * (A + A.conj().T) * s)
        taus.append(1.0 / s)
    Hs.append(np.zeros((3, 3), complex))
    taus.append(1.0)
    Hs.append(0.7 * np.eye(3, dtype=complex))
    taus.append(2.0)
    # phases large enough for the argument reduction to matter (|H| tau ~ 1e4,
    # the literal configs[1] steps near R_nu)
    for _ in range(20):
        A = rng.normal(size=(3, 3)) + 1j * rng.normal(size=(3, 3))
        Hs.append(0.5 * (A + A.conj().T) * 1e3)
        taus.append(rng.uniform(1.0, 30.0))
    return np.array(Hs), np.array(taus)


def check(run, path):
    Hs, taus = cases()
    U = run(np.array([pack(H) for H in Hs]), taus, path)
    worst = 0.0
    for H, tau, u in zip(Hs, taus, U):
        # scale-free reference: expm of the dimensionless matrix
        want = sl.expm(-1j * (H * tau))
        scale = max(1.0, np.abs(H).max() * tau)
        err = np.abs(u - want).max() / scale
        worst = max(worst, err)
        assert err <= 4e-15, (H, tau, err)
        assert np.abs(u @ u.conj().T - np.eye(3)).max() <= 2e-14 * max(1.0, np.abs(H).max() * tau * 1e-2)
    return worst


@pytest.mark.parametrize("path", [0, 1])
def test_host_exponential_matches_expm(host_exp, path):
    check(host_exp, path)


def test_host_exponential_matches_the_restatement(host_exp, pyoracle):
    """The oracle's series exponential (oscflat3_oracle.c), the checker of the
    3-flavour GPU runs, agrees with the closed form."""
    from paper_1907_05560_b200 import baseline_config

    o = pyoracle.Oracle3(baseline_config("configs1", Abins=2, Ebins=2))
    rng = np.random.default_rng(5)
    for _ in range(50):
        A = rng.normal(size=(3, 3)) + 1j * rng.normal(size=(3, 3))
        H = 0.5 * (A + A.conj().T)
        tau = rng.uniform(0.1, 2.0)
        assert np.abs(host_exp(pack(H), [tau])[0] - o.expm(pack(H), tau)).max() <= 1e-13


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a GPU")
@pytest.mark.parametrize("path", [0, 1])
def test_device_exponential_matches_expm(path):
    from paper_1907_05560_b200.engine import debug_exp3

    check(lambda H9, tau, p: debug_exp3(H9, tau, path=p), path)


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a GPU")
def test_device_and_host_exponentials_agree(host_exp):
    from paper_1907_05560_b200.engine import debug_exp3

    Hs, taus = cases()
    H9 = np.array([pack(H) for H in Hs])
    a, b = debug_exp3(H9, taus), host_exp(H9, taus)
    scale = np.maximum(1.0, np.abs(Hs).max(axis=(1, 2)) * taus)
    assert (np.abs(a - b).max(axis=(1, 2)) / scale).max() <= 2e-15
