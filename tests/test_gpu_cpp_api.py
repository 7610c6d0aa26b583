"""GPU: the C++ drop-in (include/gvr/gvr.hpp) — reference test cases ported to
C++ (tests/cpp/test_cpp_api.cpp), compiled with g++ against libgvr_cuda.so and
run as a reference-style test executable."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_api_suite():
    out_dir = os.path.join(ROOT, "tests", "cpp", "_build")
    os.makedirs(out_dir, exist_ok=True)
    exe = os.path.join(out_dir, "test_cpp_api")
    pkg = os.path.join(ROOT, "paper_2205_15401_b200")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", f"-I{ROOT}/include", f"-I{ROOT}/oracle/shim",
                    os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp"), f"-L{pkg}", "-lgvr_cuda",
                    f"-Wl,-rpath,{pkg}", "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
