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
DEPS = ["gvr_cuda.cu", "gvr_common.cuh", "project.cuh", "forward.cuh", "backward.cuh", "sampler.cuh", "fit.cuh",
        "blocks.cuh"]

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


def source_hash() -> str:
    """SHA-256 (first 16 hex digits) of every CUDA source and the C ABI header:
    embedded in libgvr_cuda.so (gvr_build_hash) and checked at load time, so a
    stale library cannot silently stand in for the sources next to it."""
    import hashlib

    h = hashlib.sha256()
    for f in [os.path.join(CSRC, d) for d in DEPS] + [os.path.join(ROOT, "include", "gvr_cuda.h")]:
        with open(f, "rb") as fh:
            h.update(os.path.basename(f).encode() + b"\0" + fh.read())
    return h.hexdigest()[:16]


def build_cuda(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(CSRC, d) for d in DEPS] + [os.path.join(ROOT, "include", "gvr_cuda.h")]
    stale = force or _stale(LIB, deps)
    if not stale:  # same mtimes, other sources (e.g. a checkout): the embedded hash decides
        with open(LIB, "rb") as fh:
            stale = source_hash().encode() not in fh.read()
    if stale:
        cmd = [_nvcc(), *NVCC_FLAGS, f"-DGVR_SOURCE_HASH=\"{source_hash()}\"",
               *[os.path.join(CSRC, s) for s in SOURCES], "-o", LIB]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return LIB


NLOHMANN = None
for _cand in [os.path.join(p, "include", "cudnn_frontend", "thirdparty", "nlohmann") for p in sys.path if p] + [
        "/usr/include/nlohmann"]:
    if os.path.exists(os.path.join(_cand, "json.hpp")):
        NLOHMANN = _cand
        break
CLI = os.path.join(HERE, "gvr")


def build_cli(verbose: bool = False) -> str:
    """The `gvr` command-line tool (paper_2205_15401_b200/cli/gvr_main.cpp) over the
    C++ drop-in; JSON through nlohmann::json (header shipped with the Python env)."""
    src = os.path.join(HERE, "cli", "gvr_main.cpp")
    deps = [src, LIB] + [os.path.join(ROOT, "include", "gvr", f)
                         for f in ("gvr.hpp", "scene_io.hpp", "image_io.hpp", "fit.hpp")]
    if NLOHMANN is None:
        raise RuntimeError("nlohmann/json.hpp not found: the CLI needs it")
    if _stale(CLI, deps):
        cmd = ["g++", "-std=c++20", "-O2", "-Wall", f"-I{ROOT}/include", f"-I{NLOHMANN}", src, f"-L{HERE}",
               "-lgvr_cuda", "-Wl,-rpath,$ORIGIN", "-o", CLI]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return CLI


REF_TESTS = ("test_scene", "test_tracer", "test_blender", "test_grad", "test_fit")
CLI_DATA = os.path.join(ROOT, "tests", "cpp", "_build", "cli_data")


def write_cli_data() -> str:
    """JSON inputs of the reference's CLI tests (tests/data/{test,gradcheck,texture}_
    {scene,camera}.json), re-serialised from the committed golden vectors (the
    same doubles; tests/golden/make_golden.py read them from the reference)."""
    import numpy as np

    sys.path.insert(0, ROOT)
    from paper_2205_15401_b200 import scene_io
    from paper_2205_15401_b200.types import Camera, GaussianScene

    os.makedirs(CLI_DATA, exist_ok=True)
    for name in ("test", "gradcheck", "texture"):
        g = np.load(os.path.join(ROOT, "tests", "golden", f"{name}_scene.npz"))
        scene_io.save_scene_json(GaussianScene(g["centers"], g["inv_cov"], g["attr"], float(g["tau"])),
                                 os.path.join(CLI_DATA, f"{name}_scene.json"))
        c = g["camera"]
        scene_io.save_camera_json(Camera(c[:9].reshape(3, 3), c[9:12], c[12], c[13], c[14], int(c[15]), int(c[16])),
                                  os.path.join(CLI_DATA, f"{name}_camera.json"))
    # the fitting fixtures are read from the reference's data at build time (like
    # tests/golden/make_golden.py) and re-serialised into the ignored build tree
    ref_data = "/root/reference/proj/tests/data"
    for name in ("part_red", "part_blue"):
        scene_io.save_scene_json(scene_io.load_scene_json(os.path.join(ref_data, f"{name}.json")),
                                 os.path.join(CLI_DATA, f"{name}.json"))
    scene_io.save_camera_json(scene_io.load_camera_json(os.path.join(ref_data, "fit_camera.json")),
                              os.path.join(CLI_DATA, "fit_camera.json"))
    return CLI_DATA
REF_TEST_DIR = os.path.join(ROOT, "tests", "cpp", "_build")


def build_reference_suites(verbose: bool = False) -> list:
    """The reference's own hot-path test suites (/root/reference/proj/tests/
    test_{scene,tracer,blender,grad,fit}.cpp), compiled UNMODIFIED against the C++
    drop-in (include/gvr/*.hpp -> libgvr_cuda.so), with Eigen and doctest from
    the repo's test shims (oracle/shim). Only where /root/reference exists (this
    container); the binaries travel to the GPU box with the tree and are run by
    tests/test_gpu_reference_suites.py. Returns the binaries built."""
    src = "/root/reference/proj/tests"
    if not os.path.isdir(src):
        return []
    os.makedirs(REF_TEST_DIR, exist_ok=True)
    out = []
    for t in REF_TESTS:
        exe = os.path.join(REF_TEST_DIR, "ref_" + t)
        cpp = os.path.join(src, t + ".cpp")
        deps = [cpp, os.path.join(ROOT, "include", "gvr_cuda.h")] + [
            os.path.join(ROOT, "include", "gvr", f) for f in ("gvr.hpp", "fit.hpp", "shapes.hpp", "convert.hpp")]
        if _stale(exe, deps):
            cmd = ["g++", "-std=c++20", "-O2", "-DGVR_WITH_EIGEN", f"-I{ROOT}/include", f"-I{ROOT}/oracle/shim",
                   f"-I{src}", cpp, f"-L{HERE}", "-lgvr_cuda", "-Wl,-rpath,$ORIGIN/../../../paper_2205_15401_b200",
                   "-o", exe]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.run(cmd, check=True)
        out.append(exe)
    # the CLI suite (test_cli.cpp) against the `gvr` tool
    if NLOHMANN is not None and os.path.exists(CLI):
        write_cli_data()
        exe = os.path.join(REF_TEST_DIR, "ref_test_cli")
        cpp = os.path.join(src, "test_cli.cpp")
        deps = [cpp] + [os.path.join(ROOT, "include", "gvr", f) for f in ("gvr.hpp", "scene_io.hpp", "image_io.hpp")]
        if _stale(exe, deps):
            cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", f"-I{ROOT}/oracle/shim", f"-I{NLOHMANN}",
                   f'-DGVR_CLI_PATH="{CLI}"', f'-DGVR_TEST_DATA="{CLI_DATA}"', cpp, f"-L{HERE}", "-lgvr_cuda",
                   "-Wl,-rpath,$ORIGIN/../../../paper_2205_15401_b200", "-o", exe]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.run(cmd, check=True)
        out.append(exe)
    return out


def build_oracle(verbose: bool = False) -> None:
    """Checker only: the C port always; the reference build when /root/reference exists."""
    odir = os.path.join(ROOT, "oracle")
    subprocess.run(["make", "-s", "-C", odir, "port"], check=True)
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-j8", "-C", odir, "ref"], check=True)


if __name__ == "__main__":
    build_cuda(force="--force" in sys.argv, verbose=True)
    build_cli(verbose=True)
    build_reference_suites(verbose=True)
    build_oracle(verbose=True)
