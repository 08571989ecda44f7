"""Builds the in-tree sm_100a shared library ``_oscb200.so`` with nvcc.

The library is the product: the C-ABI of ``include/oscflat_b200.h`` over the
hand-written FP64 kernels in ``csrc/``.  It is built in-tree so the ``.so``
travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "_oscb200.so")
SOURCES = ["engine.cu", "env.cpp"]
HEADERS = ["step_kernels.cuh", "status.hpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-shared", "-Xcompiler", "-fPIC,-O3",
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "oscflat_b200.h"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    cmd = [NVCC, *ARCH, *FLAGS, "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           *[os.path.join(CSRC, s) for s in SOURCES], "-o", LIB + ".tmp", "-ldl"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(PKG, "_build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + out.stdout + out.stderr)
    if out.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + out.stderr[-6000:])
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        print(out.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
