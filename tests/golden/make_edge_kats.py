"""Edge-path known answers of flavor::evolve_bin (beam.hpp:105-121), produced
by the unmodified reference (oracle/_ref, built from /root/reference by
oracle/Makefile).  Run in the build container:

    python tests/golden/make_edge_kats.py      -> tests/golden/kat_edge.npz

Cases: lambda = 0 (identity), lambda*dl < 1e-12 (s = dl branch) and just
above it, |lambda*dl| > 1e9 (outside the device fast sincos range),
lambda^2 subnormal, lambda^2 above 1e300 (outside the fast rsqrt range),
and ordinary values for contrast."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle  # noqa: E402


def cases():
    rng = np.random.default_rng(1907055602)
    H, DL, TAG = [], [], []

    def add(h, dl, tag):
        H.append(h)
        DL.append(dl)
        TAG.append(tag)

    unit = lambda: (v := rng.normal(size=3)) / np.linalg.norm(v)  # noqa: E731
    for _ in range(8):
        add(np.zeros(3), rng.uniform(1e-3, 10.0), "lambda0")
    for _ in range(8):  # lambda*dl in [1e-16, 1e-13): the s = dl branch
        lam = 10 ** rng.uniform(-16, -13)
        add(lam * unit(), 1.0, "tiny_ldl")
    for _ in range(8):  # lambda*dl in (1e-12, 1e-11]: just above it
        lam = 10 ** rng.uniform(-12 + 1e-3, -11)
        add(lam * unit(), 1.0, "small_ldl")
    for _ in range(8):  # |lambda dl| in [2e9, 1e13]
        lam = 10 ** rng.uniform(4, 7)
        add(lam * unit(), 10 ** rng.uniform(5.5, 6), "huge_ldl")
    for _ in range(8):  # lambda^2 subnormal (< 2.2e-308)
        lam = 10 ** rng.uniform(-162, -155)
        add(lam * unit(), 10 ** rng.uniform(0, 3), "subnormal_l2")
    for _ in range(8):  # lambda^2 in (1e300, 1e307)
        lam = 10 ** rng.uniform(150.1, 153.4)
        add(lam * unit(), 10 ** rng.uniform(-153, -151), "large_l2")
    for _ in range(16):
        add(rng.uniform(-2, 2, size=3), rng.uniform(0.01, 2.0), "ordinary")
    psi = rng.uniform(-1, 1, size=(len(H), 4))
    psi /= np.linalg.norm(psi, axis=1, keepdims=True)
    return np.array(H), np.array(DL), psi, np.array(TAG)


def main():
    ref = pyoracle.Ref()
    H, DL, PSI, TAG = cases()
    OUT = np.array([ref.evolve_bin(H[i], DL[i], PSI[i]) for i in range(len(H))])
    np.savez(os.path.join(HERE, "kat_edge.npz"), h=H, dl=DL, psi=PSI, tag=TAG, evolve=OUT,
             variant=np.array(ref.variant))
    print(f"{len(H)} edge KATs, reference build {ref.variant}")


if __name__ == "__main__":
    main()
