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
HEADERS = ["step_kernels.cuh", "step3_kernels.cuh", "resident_kernels.cuh", "su3_exp.cuh", "fastmath.cuh", "status.hpp"]
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


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile to ``out`` (default: the in-tree ``_oscb200.so``).  ``defines``
    are extra -D tuning knobs (e.g. OSC_MIN_BLOCKS=3) for variant sweeps."""
    target = out or LIB
    if target == LIB and not defines and not force and not _stale():
        return LIB
    cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"),
           "-I", CSRC, *[os.path.join(CSRC, s) for s in SOURCES], "-o", target + ".tmp", "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(PKG, "_build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stderr[-6000:])
    os.replace(target + ".tmp", target)
    if verbose:
        print(res.stderr)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
