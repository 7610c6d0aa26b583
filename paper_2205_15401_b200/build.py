"""In-tree build of the CUDA library (sm_100a) and, for tests, the oracle.

``python -m paper_2205_15401_b200.build`` or ``__graft_entry__.build()``.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgvr_cuda.so")
SOURCES = ["gvr_cuda.cu"]
DEPS = ["gvr_cuda.cu", "gvr_common.cuh", "project.cuh", "forward.cuh", "backward.cuh", "sampler.cuh", "fit.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-warn-spills",
]


def _nvcc() -> str:
    for cand in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.isabs(cand) and os.path.exists(cand):
            return cand
    return "nvcc"


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_cuda(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(CSRC, d) for d in DEPS] + [os.path.join(ROOT, "include", "gvr_cuda.h")]
    if force or _stale(LIB, deps):
        cmd = [_nvcc(), *NVCC_FLAGS, *[os.path.join(CSRC, s) for s in SOURCES], "-o", LIB]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return LIB


def build_oracle(verbose: bool = False) -> None:
    """Checker only: the C port always; the reference build when /root/reference exists."""
    odir = os.path.join(ROOT, "oracle")
    subprocess.run(["make", "-s", "-C", odir, "port"], check=True)
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-j8", "-C", odir, "ref"], check=True)


if __name__ == "__main__":
    build_cuda(force="--force" in sys.argv, verbose=True)
    build_oracle(verbose=True)
