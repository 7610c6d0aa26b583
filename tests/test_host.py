"""CPU: host-side logic and the C-ABI surface (no GPU compute).

* synthetic benchmark inputs == the reference's generators (golden / oracle/_ref);
* libgvr_cuda.so loads and exports every entry point declared in include/gvr_cuda.h;
* without a usable sm_100 device the library fails loudly (no CPU fallback);
* the product package never imports the oracle;
* JSON fixtures load like the reference's scene_io.
"""
import ast
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from conftest import Golden
from paper_2205_15401_b200 import _lib, synthetic
from paper_2205_15401_b200.types import ValidationError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gvr_cuda.h")
PKG = os.path.join(ROOT, "paper_2205_15401_b200")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gvr_[a-z0-9_]+)\s*\(", text)))


def test_bench_scene_matches_reference_golden():
    g = Golden("bench_c1")
    s = synthetic.make_bench_scene(1000)
    assert s.size == 1016
    assert np.array_equal(s.centers, g["centers"])
    assert np.array_equal(s.inv_cov, g["inv_cov"])
    assert np.array_equal(s.attr, g["attr"])
    assert np.array_equal(synthetic.make_bench_camera(128).as_array(), g["camera"])


def test_orbit_camera_matches_reference_golden():
    g = Golden("orbit_rect")
    cam = synthetic.make_orbit_camera(0.7, 0.3, 4.0, (0, 0, 4), 40, 56, 60.0)
    assert np.array_equal(cam.as_array(), g["camera"])


@pytest.mark.skipif(not oracle.ref_available(), reason="reference build not present")
@pytest.mark.parametrize("n", [50000, 100000])
def test_large_bench_scenes_match_reference(n):
    c, s, a, tau = oracle.ref_make_bench_scene(n)
    scene = synthetic.make_bench_scene(n)
    assert np.array_equal(scene.centers, c) and np.array_equal(scene.inv_cov, s) and np.array_equal(scene.attr, a)
    for v in range(4):
        ref = oracle.ref_make_orbit_camera(2 * np.pi * v / 64, 0.3, 4.0, (0, 0, 4), 512, 512, 819.2)
        cam = synthetic.make_orbit_camera(2 * np.pi * v / 64, 0.3, 4.0, (0, 0, 4), 512, 512, 819.2)
        assert np.array_equal(cam.as_array(), ref)


def test_library_exports_every_declared_entry_point():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = declared_functions()
    assert len(declared) >= 20
    missing = [f for f in declared if not hasattr(lib, f)]
    assert not missing, missing
    assert sorted(_lib.EXPORTED_SYMBOLS) == declared


def test_library_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = _lib.load()
    h = ctypes.c_void_p()
    assert lib.gvr_context_create(0, ctypes.byref(h)) == _lib.GVR_ERR_RUNTIME
    import paper_2205_15401_b200 as gvr

    with pytest.raises(gvr.GvrRuntimeError):
        gvr.Context(0)


def test_product_never_imports_the_oracle():
    for fname in os.listdir(PKG):
        if not fname.endswith(".py"):
            continue
        tree = ast.parse(open(os.path.join(PKG, fname)).read())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                assert all(not a.name.startswith("oracle") for a in node.names), fname
            if isinstance(node, ast.ImportFrom):
                assert not (node.module or "").startswith("oracle"), fname


def test_scene_json_loading():
    from paper_2205_15401_b200.scene_io import load_camera_json, load_scene_json

    data = "/root/reference/proj/tests/data"
    if not os.path.isdir(data):
        pytest.skip("reference fixtures not present")
    g = Golden("test_scene")
    s = load_scene_json(f"{data}/test_scene.json")
    assert np.array_equal(s.centers, g["centers"]) and np.array_equal(s.inv_cov, g["inv_cov"])
    c = load_camera_json(f"{data}/test_camera.json")
    assert np.array_equal(c.as_array(), g["camera"])


def test_mixed_attribute_dims_rejected():
    from paper_2205_15401_b200.types import GaussianScene

    with pytest.raises(ValidationError, match="attribute dimension is not uniform"):
        GaussianScene.from_kernels([((0, 0, 4), np.eye(3), [1, 2, 3]), ((0, 0, 5), np.eye(3), [1, 2])])


def test_cpp_dropin_header_compiles_and_links():
    """include/gvr/gvr.hpp + the ported reference cases compile and link against
    libgvr_cuda.so on the CPU (they run in the GPU suite)."""
    import shutil
    import subprocess
    import tempfile

    if shutil.which("g++") is None or not os.path.exists(_lib.LIB_PATH):
        pytest.skip("g++ or the built library missing")
    root = os.path.dirname(PKG)
    with tempfile.TemporaryDirectory() as tmp:
        exe = os.path.join(tmp, "t")
        r = subprocess.run(["g++", "-std=c++17", "-O0", "-Wall", "-Werror", f"-I{root}/include", f"-I{root}/oracle/shim",
                            os.path.join(root, "tests", "cpp", "test_cpp_api.cpp"), f"-L{PKG}", "-lgvr_cuda",
                            f"-Wl,-rpath,{PKG}", "-o", exe], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]


def test_so3_chart_round_trip():
    import importlib

    gvr_so3 = importlib.import_module("paper_2205_15401_b200.gradcheck")

    """so3_log(so3_exp(w)) == w and so3_exp_gradient matches central differences."""
    rng = np.random.default_rng(3)
    for _ in range(5):
        w = rng.normal(size=3) * 0.7
        assert np.allclose(gvr_so3.so3_log(gvr_so3.so3_exp(w)), w, atol=1e-12)
        dr = rng.normal(size=(3, 3))
        g = gvr_so3.so3_exp_gradient(w, dr)
        num = np.zeros(3)
        for i in range(3):
            e = np.zeros(3)
            e[i] = 1e-6
            num[i] = ((gvr_so3.so3_exp(w + e) - gvr_so3.so3_exp(w - e)) * dr).sum() / 2e-6
        assert np.allclose(g, num, rtol=1e-6, atol=1e-8)
