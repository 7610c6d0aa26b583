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


# ---------------------------------------------------------------- data formats (test_io.cpp)

def _random_scene(seed, k):
    from paper_2205_15401_b200.types import GaussianScene
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((k, 3, 3)))
    s = q @ (rng.uniform(0.5, 9.0, (k, 3))[:, :, None] * np.transpose(q, (0, 2, 1)))
    return GaussianScene(rng.normal(0, 1, (k, 3)) + [0, 0, 5], s, rng.uniform(0, 1, (k, 3)), float(rng.uniform(0.5, 2)))


def test_scene_json_round_trip_is_exact(tmp_path):
    """test_io.cpp:30-47 and :233-244 (identical bytes for the same scene)."""
    import paper_2205_15401_b200 as gvr
    scene = _random_scene(101, 7)
    path = tmp_path / "scene.json"
    gvr.save_scene_json(scene, path)
    loaded = gvr.load_scene_json(path)
    assert loaded.tau == scene.tau
    assert np.array_equal(loaded.centers, scene.centers)
    assert np.array_equal(loaded.inv_cov, scene.inv_cov)
    assert np.array_equal(loaded.attr, scene.attr)
    assert not (tmp_path / "scene.json.tmp").exists()
    gvr.save_scene_json(scene, tmp_path / "b.json")
    assert path.read_bytes() == (tmp_path / "b.json").read_bytes()


@pytest.mark.skipif(not os.path.exists(_lib.LIB_PATH), reason="library not built")
def test_camera_json_round_trip_is_exact_and_validated(tmp_path):
    """test_io.cpp:49-70; the loader validates like Camera::validate (types.cpp:44-63)."""
    import paper_2205_15401_b200 as gvr
    from paper_2205_15401_b200.gradcheck import so3_exp
    cam = gvr.Camera(so3_exp([0.3, -0.2, 0.9]), np.array([0.5, -1.0, 2.0]), 123.5, 31.25, 63.5, 128, 64)
    path = tmp_path / "camera.json"
    gvr.save_camera_json(cam, path)
    loaded = gvr.load_camera_json(path)
    assert np.array_equal(loaded.rotation, cam.rotation) and np.array_equal(loaded.translation, cam.translation)
    assert (loaded.focal, loaded.ox, loaded.oy, loaded.height, loaded.width) == (123.5, 31.25, 63.5, 128, 64)
    bad = gvr.Camera(np.diag([2.0, 1.0, 1.0]), np.zeros(3), 10.0, 1.0, 1.0, 4, 4)
    gvr.save_camera_json(bad, path)
    with pytest.raises(ValidationError, match="camera rotation is not orthonormal"):
        gvr.load_camera_json(path)
    gvr.save_camera_json(gvr.Camera(np.eye(3), np.zeros(3), -1.0, 1.0, 1.0, 4, 4), path)
    with pytest.raises(ValidationError, match="camera focal length must be > 0"):
        gvr.load_camera_json(path)


def test_loading_rejects_missing_and_malformed_files(tmp_path):
    """test_io.cpp:72-83."""
    import paper_2205_15401_b200 as gvr
    with pytest.raises(ValidationError, match="cannot open file"):
        gvr.load_scene_json(tmp_path / "nope.json")
    (tmp_path / "bad.json").write_text("{ not json")
    with pytest.raises(ValidationError, match="invalid JSON"):
        gvr.load_scene_json(tmp_path / "bad.json")
    (tmp_path / "v2.json").write_text('{"version":2,"tau":1.0,"kernels":[]}')
    with pytest.raises(ValidationError, match="unsupported format version"):
        gvr.load_scene_json(tmp_path / "v2.json")


def test_attrs_json_round_trip(tmp_path):
    """test_io.cpp:85-100."""
    import paper_2205_15401_b200 as gvr
    from paper_2205_15401_b200.types import SampledAttributes
    attrs = SampledAttributes(np.array([[0.1, 0.2, 0.3], [0.0, 0.0, 0.0]]), np.array([1.5, 0.0]),
                              np.array([False, True]))
    gvr.save_attrs_json(attrs, tmp_path / "attrs.json")
    loaded = gvr.load_attrs_json(tmp_path / "attrs.json")
    assert np.array_equal(loaded.attrs, attrs.attrs) and np.array_equal(loaded.support, attrs.support)
    assert np.array_equal(loaded.masked, attrs.masked) and loaded.masked_count() == 1
    (tmp_path / "bad.json").write_text('{"version":1,"attrs":[[1,2]],"support":[1,2],"masked":[false]}')
    with pytest.raises(ValidationError, match="inconsistent attrs file"):
        gvr.load_attrs_json(tmp_path / "bad.json")


def test_pfm_round_trips_at_float_precision(tmp_path):
    """test_io.cpp:213-231, plus the byte layout (image_io.cpp:124-157): header,
    little-endian float32, rows bottom-up."""
    import paper_2205_15401_b200 as gvr
    rng = np.random.default_rng(103)
    for ch in (1, 3):
        img = rng.uniform(-5, 5, (9, 11, ch))
        path = tmp_path / f"img{ch}.pfm"
        gvr.write_pfm(img, path)
        raw = path.read_bytes()
        header = f"{'PF' if ch == 3 else 'Pf'}\n11 9\n-1.0\n".encode()
        assert raw.startswith(header) and len(raw) == len(header) + 4 * img.size
        first_row_on_disk = np.frombuffer(raw, "<f4", count=11 * ch, offset=len(header))
        assert np.array_equal(first_row_on_disk, img[-1].reshape(-1).astype(np.float32))
        loaded = gvr.read_pfm(path)
        assert loaded.shape == img.shape
        np.testing.assert_allclose(loaded, img, rtol=1e-7, atol=0)
    with pytest.raises(ValidationError, match="write_pfm supports 1 or 3 channels"):
        gvr.write_pfm(np.zeros((2, 2, 2)), tmp_path / "x.pfm")
    (tmp_path / "be.pfm").write_bytes(b"PF\n1 1\n1.0\n" + b"\0" * 12)
    with pytest.raises(ValidationError, match="big-endian PFM is not supported"):
        gvr.read_pfm(tmp_path / "be.pfm")
    (tmp_path / "short.pfm").write_bytes(b"PF\n2 2\n-1.0\n" + b"\0" * 12)
    with pytest.raises(ValidationError, match="truncated PFM data"):
        gvr.read_pfm(tmp_path / "short.pfm")
    (tmp_path / "magic.pfm").write_bytes(b"P6\n2 2\n255\n")
    with pytest.raises(ValidationError, match="not a PFM file"):
        gvr.read_pfm(tmp_path / "magic.pfm")
