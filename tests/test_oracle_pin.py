"""CPU: pin the oracles.

* The reference, compiled unmodified from /root/reference against the Eigen /
  doctest shims (oracle/_ref), passes the reference's own hot-path suites.
* The plain-C restatement (oracle/gvr_oracle.c) reproduces the reference's
  golden vectors (tests/golden, made by the reference build) bit for bit.
* Where the reference build is present, port == reference on random inputs,
  including the validation error messages.
"""
import os
import subprocess

import numpy as np
import pytest

import oracle
from conftest import Golden, golden_names
from paper_2205_15401_b200.types import Camera, GaussianScene, SelectionConfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = ["test_scene", "test_tracer", "test_blender", "test_grad", "test_convert", "test_sampler"]


@pytest.mark.parametrize("suite", REF_TESTS)
def test_reference_suites_pass_against_shim(suite):
    exe = os.path.join(ROOT, "oracle", "_ref", suite)
    if not os.path.exists(exe):
        pytest.skip("reference build not present (make -C oracle ref needs /root/reference)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "0 failed" in out.stdout


@pytest.mark.parametrize("name", golden_names())
def test_port_forward_bit_identical_to_golden(name):
    g = Golden(name)
    out = oracle.port_render(g.scene, g.camera, g.cfg, threads=8)
    for key in ("topk_idx", "topk_w", "image", "alpha", "depth"):
        assert np.array_equal(out[key], g[key]), key
    if "topk_l" in g:
        for key in ("topk_l", "topk_q", "topk_sigma"):
            assert np.array_equal(out[key], g[key]), key


@pytest.mark.parametrize("name", golden_names())
def test_port_backward_bit_identical_to_golden(name):
    g = Golden(name)
    gr = oracle.port_backward(g.scene, g.camera, g.cfg, g["d_image"], g["d_alpha"], bool(g["through_transmittance"]),
                              bool(g["through_density"]), threads=8)
    for key in ("d_center", "d_inv_cov", "d_attr", "d_rotation", "d_translation"):
        assert np.array_equal(gr[key], g[key]), key


def _random_scene(seed, k=60, d=3):
    rng = np.random.default_rng(seed)
    c = np.stack([rng.uniform(-1, 1, k), rng.uniform(-1, 1, k), rng.uniform(2.5, 6, k)], 1)
    inv = []
    for _ in range(k):
        q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        m = q @ np.diag(rng.uniform(2, 80, 3)) @ q.T
        inv.append(0.5 * (m + m.T))
    return GaussianScene(c, np.array(inv), rng.uniform(0, 1, (k, d)), float(rng.uniform(0.5, 3)))


@pytest.mark.skipif(not oracle.ref_available(), reason="reference build not present")
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_port_equals_reference_random(seed):
    scene = _random_scene(seed)
    rng = np.random.default_rng(100 + seed)
    ang = rng.normal(size=3) * 0.2
    from scipy.spatial.transform import Rotation

    cam = Camera(Rotation.from_rotvec(ang).as_matrix(), rng.normal(size=3) * 0.1, 30.0, 19.5, 17.0, 36, 40)
    for cfg in (SelectionConfig(), SelectionConfig(eta=0.2, k_prime=5, coarse_downsample=3),
                SelectionConfig(coarse_enabled=False, k_prime=9)):
        a = oracle.port_render(scene, cam, cfg, threads=3)
        b = oracle.ref_render(scene, cam, cfg, threads=3)
        for key in a:
            assert np.array_equal(a[key], b[key]), key
        di = rng.uniform(-1, 1, (cam.height, cam.width, 3))
        da = rng.uniform(-1, 1, (cam.height, cam.width, 1))
        ga = oracle.port_backward(scene, cam, cfg, di, da, threads=3)
        gb = oracle.ref_backward(scene, cam, cfg, di, da, threads=3)
        for key in ga:
            assert np.array_equal(ga[key], gb[key]), key


@pytest.mark.skipif(not oracle.ref_available(), reason="reference build not present")
def test_port_coarse_boxes_equal_reference():
    scene = _random_scene(7, k=200)
    cam = Camera(np.eye(3), np.zeros(3), 40.0, 31.5, 31.5, 64, 64)
    for cfg in (SelectionConfig(), SelectionConfig(coarse_downsample=5, eta=0.05)):
        a, da = oracle.port_coarse_boxes(scene, cam, cfg)
        b, db = oracle.ref_coarse_boxes(scene, cam, cfg)
        assert da == db
        assert np.array_equal(a, b)


@pytest.mark.skipif(not oracle.ref_available(), reason="reference build not present")
def test_validation_messages_match_reference():
    base = _random_scene(3, k=4)
    cam = Camera(np.eye(3), np.zeros(3), 20.0, 7.5, 7.5, 16, 16)
    cases = []
    s = base.copy()
    s.inv_cov[2, 0, 1] += 0.5
    cases.append((s, cam, SelectionConfig()))
    s = base.copy()
    s.inv_cov[1] = -np.eye(3)
    cases.append((s, cam, SelectionConfig()))
    s = base.copy()
    s.centers[3, 1] = np.nan
    cases.append((s, cam, SelectionConfig()))
    s = base.copy()
    s.tau = -1.0
    cases.append((s, cam, SelectionConfig()))
    bad_cam = Camera(np.diag([2.0, 1.0, 1.0]), np.zeros(3), 20.0, 7.5, 7.5, 16, 16)
    cases.append((base, bad_cam, SelectionConfig()))
    cases.append((base, Camera(np.eye(3), np.zeros(3), 0.0, 7.5, 7.5, 16, 16), SelectionConfig()))
    cases.append((base, cam, SelectionConfig(eta=1.5)))
    cases.append((base, cam, SelectionConfig(k_prime=0)))
    for scene, c, cfg in cases:
        with pytest.raises(oracle.OracleError) as ea:
            oracle.port_render(scene, c, cfg, threads=1)
        with pytest.raises(oracle.OracleError) as eb:
            oracle.ref_render(scene, c, cfg, threads=1)
        assert str(ea.value) == str(eb.value)
        assert ea.value.code == eb.value.code == 1


def test_port_sampler_and_helpers_bit_identical_to_golden():
    """sample_attributes / resynthesize inputs, transmittance_at, normalized_weights,
    shade_lambert (sampler.cpp:11-66, blender.cpp:19-25, 55-62, 146-172)."""
    g = Golden("sampler_random")
    for norm, pre in ((False, "s_"), (True, "n_")):
        a, s, m = oracle.port_sample_attributes(g.scene, g.camera, g.cfg, g["observed"], norm, threads=8)
        assert np.array_equal(a, g[pre + "attrs"])
        assert np.array_equal(s, g[pre + "support"])
        assert np.array_equal(m, g[pre + "masked"])
    trans, nw = oracle.port_pixel_helpers(g.scene, g.camera, g.cfg, g["t_query"], 1e-8, threads=8)
    assert np.array_equal(trans, g["trans_at"])
    assert np.array_equal(nw, g["norm_w"])
    sh = oracle.port_shade_lambert(g.camera, g["image"], g["alpha"], g["depth"], g["light_pos"], g["light_color"])
    assert np.array_equal(sh, g["shade"])
    assert g["s_masked"][-1] and not g["s_masked"].all()


@pytest.mark.skipif(not oracle.ref_available(), reason="reference build not present")
def test_port_sampler_equals_reference_random():
    scene = _random_scene(21, k=80)
    cam = Camera(np.eye(3), np.zeros(3), 30.0, 15.5, 13.0, 32, 28)
    cfg = SelectionConfig(k_prime=7, coarse_downsample=4)
    rng = np.random.default_rng(5)
    obs = rng.uniform(0, 1, (32, 28, 2))
    for norm in (False, True):
        a = oracle.port_sample_attributes(scene, cam, cfg, obs, norm, threads=3)
        b = oracle.ref_sample_attributes(scene, cam, cfg, obs, norm, threads=3)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    with pytest.raises(oracle.OracleError) as ea:
        oracle.port_sample_attributes(scene, cam, cfg, obs[:16], False)
    with pytest.raises(oracle.OracleError) as eb:
        oracle.ref_sample_attributes(scene, cam, cfg, obs[:16], False)
    assert str(ea.value) == str(eb.value) == "observed image size does not match the camera"
    n = rng.normal(size=(32, 28, 3))
    al = rng.uniform(-0.2, 1, (32, 28, 1))
    de = rng.uniform(2, 6, (32, 28, 1))
    assert np.array_equal(oracle.port_shade_lambert(cam, n, al, de, [1.0, 2.0, -3.0], [0.9, 0.5, 0.1]),
                          oracle.ref_shade_lambert(cam, n, al, de, [1.0, 2.0, -3.0], [0.9, 0.5, 0.1]))


@pytest.mark.skipif(not oracle.ref_available(), reason="reference build not present")
def test_reference_regularizers_reproduce_golden():
    """tests/golden/aux/fit_regularizers.npz was made by the reference build (fit.cpp:44-113)."""
    g = np.load(os.path.join(ROOT, "tests", "golden", "aux", "fit_regularizers.npz"))
    ev, eg, lv, lg = oracle.ref_shape_reg(g["edges"], g["rest"], g["centers"])
    assert ev == g["edge_value"] and lv == g["laplacian_value"]
    assert np.array_equal(eg, g["edge_grad"]) and np.array_equal(lg, g["laplacian_grad"])


def test_mesh_edges_of_the_box_mesh():
    """mesh_edges (convert.cpp:39-51): unique sorted pairs; a closed box grid has E = 3V - 6."""
    from paper_2205_15401_b200 import synthetic

    verts, faces = synthetic.make_box_mesh((1.0, 1.0, 1.0), 6, (0.0, 0.0, 4.0))
    e = synthetic.mesh_edges(faces)
    assert np.all(e[:, 0] < e[:, 1])
    assert len(np.unique(e[:, 0].astype(np.int64) * len(verts) + e[:, 1])) == len(e)
    assert len(e) == 3 * len(verts) - 6
