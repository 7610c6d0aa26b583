"""GPU: more of the reference's hot-path test cases (test_scene.cpp, test_tracer.cpp,
test_blender.cpp), expressed through renders. A traced triple (l, q, sigma) on
the optical axis is realised by an isotropic kernel of width sigma centred at
(v, 0, l) with v = sigma sqrt(-2 q): the axis ray (pixel (0, 0) of a camera
with its principal point there) traces it to exactly (l, q, sigma)."""
import math

import numpy as np
import pytest

import paper_2205_15401_b200 as gvr
from paper_2205_15401_b200.types import Camera, GaussianScene, SelectionConfig
from test_gpu_properties import default_camera, random_scene

pytestmark = pytest.mark.gpu


def axis_camera():
    return Camera(np.eye(3), np.zeros(3), 10.0, 0.0, 0.0, 1, 1)


def axis_scene(triples, tau=1.0, attr=None):
    """Kernels whose axis trace is (l, q, sigma)."""
    c, s = [], []
    for l, q, sg in triples:
        c.append([sg * math.sqrt(max(-2.0 * q, 0.0)), 0.0, l])
        s.append(np.eye(3) / sg**2)
    n = len(triples)
    a = np.ones((n, 3)) if attr is None else np.asarray(attr, dtype=np.float64)
    return GaussianScene(np.array(c), np.array(s), a, tau)


def random_rotation(rng):
    q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


# ----------------------------------------------------------------- test_scene.cpp

def test_view_transform_with_identity_extrinsics_is_a_no_op(ctx):
    """test_scene.cpp:9-19."""
    scene = random_scene(11, 4)
    fr = gvr.render_with_tape(scene, default_camera(), ctx=ctx)
    c, s = fr.tape.cam_scene()
    assert np.abs(c - scene.centers).max() == pytest.approx(0.0, abs=1e-12)
    assert np.abs(s - scene.inv_cov).max() == pytest.approx(0.0, abs=1e-12)


def test_pure_translation_moves_centers_and_keeps_inv_cov(ctx):
    """test_scene.cpp:21-35."""
    scene = GaussianScene(np.array([[1.0, 2, 3]]), (2.0 * np.eye(3))[None], np.ones((1, 3)), 1.0)
    cam = default_camera()
    cam = Camera(cam.rotation, np.array([0, 0, 5.0]), cam.focal, cam.ox, cam.oy, cam.height, cam.width)
    c, s = gvr.render_with_tape(scene, cam, ctx=ctx).tape.cam_scene()
    assert np.allclose(c[0], [1, 2, 8]) and np.allclose(s[0], 2.0 * np.eye(3))


def test_rotation_preserves_inv_cov_eigenvalues(ctx):
    """test_scene.cpp:37-56."""
    rng = np.random.default_rng(7)
    for _ in range(20):
        q = random_rotation(rng)
        spd = q @ np.diag(rng.uniform(0.5, 8.0, 3)) @ q.T
        spd = 0.5 * (spd + spd.T)
        scene = GaussianScene(np.array([[0.1, -0.2, 4.0]]), spd[None], np.zeros((1, 1)), 1.0)
        cam = default_camera()
        cam = Camera(random_rotation(rng), np.zeros(3), cam.focal, cam.ox, cam.oy, cam.height, cam.width)
        _, s = gvr.render_with_tape(scene, cam, ctx=ctx).tape.cam_scene()
        assert np.abs(np.linalg.eigvalsh(spd) - np.linalg.eigvalsh(s[0])).max() < 1e-9
        assert np.linalg.eigvalsh(s[0]).min() > 0.0


def test_view_transform_composition_equals_composed_extrinsics(ctx):
    """test_scene.cpp:58-78: (scene -> first -> second) == scene -> (second o first)."""
    rng = np.random.default_rng(13)
    for _ in range(10):
        scene = random_scene(int(rng.integers(1 << 30)), 3)
        r1, t1 = random_rotation(rng), np.array([0.3, -0.4, 1.0])
        r2, t2 = random_rotation(rng), np.array([-0.1, 0.2, 0.5])
        cam1 = Camera(r1, t1, 16.0, 15.5, 15.5, 32, 32)
        c1, s1 = gvr.render_with_tape(scene, cam1, ctx=ctx).tape.cam_scene()
        mid = GaussianScene(c1, s1, scene.attr, scene.tau)
        cam2 = Camera(r2, t2, 16.0, 15.5, 15.5, 32, 32)
        c12, s12 = gvr.render_with_tape(mid, cam2, ctx=ctx).tape.cam_scene()
        comp = Camera(r2 @ r1, r2 @ t1 + t2, 16.0, 15.5, 15.5, 32, 32)
        cc, sc = gvr.render_with_tape(scene, comp, ctx=ctx).tape.cam_scene()
        assert np.abs(c12 - cc).max() < 1e-9 and np.abs(s12 - sc).max() < 1e-9


# ----------------------------------------------------------------- test_tracer.cpp

def test_q_equals_the_log_density_at_the_peak(ctx):
    """test_tracer.cpp:67-84 on every selected entry of a random render."""
    scene = random_scene(42, 30, 3, 0.5, 8.0)
    cam = default_camera(24, 12.0)
    fr = gvr.render_with_tape(scene, cam, ctx=ctx)
    idx, l, q, sg = fr.tape.traced()
    checked = 0
    for i in range(cam.height):
        for j in range(cam.width):
            d = np.array([(i - cam.oy) / cam.focal, (j - cam.ox) / cam.focal, 1.0])
            d /= np.linalg.norm(d)
            for s in range(idx.shape[2]):
                k = idx[i, j, s]
                if k < 0:
                    break
                v = l[i, j, s] * d - scene.centers[k]
                assert abs(q[i, j, s] - (-0.5 * v @ scene.inv_cov[k] @ v)) < 1e-9
                checked += 1
    assert checked > 100


def test_fine_select_keeps_everything_under_the_cap_sorted_by_depth(ctx):
    """test_tracer.cpp:118-128: depths 6, 4, 5 -> order 1, 2, 0."""
    scene = axis_scene([(6.0, -0.5, 1.0), (4.0, -0.1, 1.0), (5.0, -0.2, 1.0)])
    fr = gvr.render_with_tape(scene, axis_camera(), SelectionConfig(k_prime=20), ctx=ctx)
    assert list(fr.buffers.topk_idx[0, 0, :3]) == [1, 2, 0]
    assert fr.buffers.topk_idx[0, 0, 3] == -1


def test_fine_select_drops_vanished_kernels(ctx):
    """test_tracer.cpp:112-116: q far below ln(eta) -> nothing selected, empty outputs."""
    scene = axis_scene([(5.0, -800.0, 1.0), (6.0, -900.0, 1.0)])
    fr = gvr.render_with_tape(scene, axis_camera(), ctx=ctx)
    assert fr.buffers.topk_idx[0, 0, 0] == -1 and fr.buffers.alpha[0, 0, 0] == 0.0


def test_raising_eta_shrinks_the_selection(ctx):
    """test_tracer.cpp:170-183 (boxes shrink with eta): per-pixel selections only lose kernels."""
    scene = random_scene(45, 60)
    cam = default_camera(32, 16.0)
    lo = gvr.render(scene, cam, SelectionConfig(eta=0.01, k_prime=64), ctx=ctx).topk_idx
    hi = gvr.render(scene, cam, SelectionConfig(eta=0.3, k_prime=64), ctx=ctx).topk_idx
    for p in range(cam.height * cam.width):
        a = set(lo.reshape(-1, 64)[p][lo.reshape(-1, 64)[p] >= 0])
        b = set(hi.reshape(-1, 64)[p][hi.reshape(-1, 64)[p] >= 0])
        assert b <= a
    assert (hi >= 0).sum() < (lo >= 0).sum()


# ----------------------------------------------------------------- test_blender.cpp

def test_front_kernels_win_the_depth_ordering(ctx):
    """test_blender.cpp:166-176."""
    for triples, front in (([(4.0, 0.0, 0.5), (6.0, 0.0, 0.5)], 0), ([(6.0, 0.0, 0.5), (4.0, 0.0, 0.5)], 1)):
        buf = gvr.render(axis_scene(triples), axis_camera(), ctx=ctx)
        w = dict(zip(buf.topk_idx[0, 0, :2], buf.topk_w[0, 0, :2]))
        assert w[front] > w[1 - front]


def test_coincident_stacks_follow_the_closed_form(ctx):
    """test_blender.cpp:120-138: for n coincident kernels with peaks g_i (sum G),
    the closed form gives W_i = g_i exp(-G / 2) (Phi(0) = 1/2 for every pair)."""
    rng = np.random.default_rng(58)
    for n in range(1, 6):
        g = rng.uniform(0.05, 1.0, n)
        scene = axis_scene([(5.0, math.log(gi), 0.5) for gi in g])
        buf = gvr.render(scene, axis_camera(), ctx=ctx)
        for s in range(n):
            k = buf.topk_idx[0, 0, s]
            assert buf.topk_w[0, 0, s] == pytest.approx(g[k] * math.exp(-g.sum() / 2.0), rel=1e-6)


def test_blend_weights_are_permutation_invariant(ctx):
    """test_blender.cpp:67-91: shuffling the scene's kernel order permutes ids only."""
    rng = np.random.default_rng(52)
    scene = random_scene(52, 40)
    cam = default_camera(24, 12.0)
    perm = rng.permutation(scene.size)
    shuffled = GaussianScene(scene.centers[perm], scene.inv_cov[perm], scene.attr[perm], scene.tau)
    a = gvr.render(scene, cam, ctx=ctx)
    b = gvr.render(shuffled, cam, ctx=ctx)
    ids_b = np.where(b.topk_idx >= 0, perm[np.maximum(b.topk_idx, 0)], -1)
    assert np.array_equal(a.topk_idx, ids_b)
    np.testing.assert_allclose(b.topk_w, a.topk_w, rtol=1e-12, atol=0)
    np.testing.assert_allclose(b.alpha, a.alpha, rtol=1e-12, atol=0)
    assert np.all(a.topk_w >= 0.0) and np.all(a.topk_w <= 1.0) and np.all(a.alpha <= 1.0)


def test_transmittance_is_non_increasing_and_in_unit_interval(ctx):
    """test_blender.cpp:35-50."""
    scene = axis_scene([(4.0, -0.3, 0.5), (5.0, 0.0, 0.8), (6.5, -1.0, 0.3)])
    fr = gvr.render_with_tape(scene, axis_camera(), ctx=ctx)
    prev = 1.0
    for t in np.linspace(-5.0, 15.0, 200):
        cur = gvr.transmittance_at(fr, np.array([[t]]))[0, 0]
        assert 0.0 < cur <= 1.0 and cur <= prev + 1e-15
        prev = cur


@pytest.mark.parametrize("k_prime", [8, 20, 32])
def test_batch_merge_with_near_ties_matches_the_oracle(ctx, k_prime):
    """Many candidates of one 32-candidate batch on the same ray with depths equal
    or within FP32 resolution of each other: the warp batch merge must defer to the
    exact (l, idx) order (fine_select, tracer.cpp:119-122) exactly like the oracle."""
    import oracle
    rng = np.random.default_rng(60 + k_prime)
    triples = []
    for _ in range(40):
        base = float(rng.choice([5.0, 5.0 + 1e-7, 5.0 * (1 + 3e-7), 6.0, 7.25]))
        triples.append((base * (1.0 + float(rng.integers(-2, 3)) * 1e-16), float(rng.uniform(-2.0, 0.0)), 0.5))
    triples += [(float(l), float(rng.uniform(-2.0, 0.0)), 0.5) for l in rng.uniform(3.0, 9.0, 30)]
    scene = axis_scene(triples)
    cfg = SelectionConfig(k_prime=k_prime)
    buf = gvr.render(scene, axis_camera(), cfg, ctx=ctx)
    ref = oracle.port_render(scene, axis_camera(), cfg)
    assert np.array_equal(buf.topk_idx, ref["topk_idx"])
    assert (buf.topk_idx >= 0).sum() == k_prime
