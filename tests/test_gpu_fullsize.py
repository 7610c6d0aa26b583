"""GPU: full-size parity of the BASELINE.json configs the other suites only cover
at reduced size, against the C oracle (bit-pinned to the reference build):

* C4 — one 1024x1024 view of make_bench_scene(1e6) (1,003,688 kernels,
  bench.cpp:9-24), forward + backward, and the same view tile-sharded over 2
  "ranks" (gvr_render_shard) whose outputs union / gradients sum to the full
  render;
* C5 — one full Fitter iteration: make_bench_scene(5e4) (50,786 kernels),
  32 orbit views at 256x256 (fit.cpp:117-158 loss_and_grad semantics).

Every render also reports its tile-list layout: no tile may overflow the list
pool (an overflowing tile would stream every kernel) at these sizes.
"""
import numpy as np
import pytest

import oracle
import paper_2205_15401_b200 as gvr
from conftest import assert_close_rel, assert_grad_close
from paper_2205_15401_b200.types import SelectionConfig

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c4():
    scene = gvr.make_bench_scene(1_000_000)
    assert scene.size == 1_003_688
    cam = gvr.make_bench_camera(1024)
    cfg = SelectionConfig()
    o = oracle.port_render(scene, cam, cfg, threads=0)
    rng = np.random.default_rng(4)
    di = o["image"] - rng.uniform(0, 1, o["image"].shape)
    da = o["alpha"] - rng.uniform(0, 1, o["alpha"].shape)
    go = oracle.port_backward(scene, cam, cfg, di, da, threads=0)
    return scene, cam, cfg, o, di, da, go


def test_c4_full_size_parity(ctx, c4):
    scene, cam, cfg, o, di, da, go = c4
    fr = gvr.render_with_tape(scene, cam, cfg, ctx=ctx)
    st = fr.tape.list_stats()
    print(f"\nC4 tile lists: {st}")
    assert st["overflow_tiles"] == 0
    assert np.array_equal(fr.buffers.topk_idx, o["topk_idx"])
    for key in ("image", "alpha", "depth", "topk_w"):
        assert_close_rel(getattr(fr.buffers, key), o[key], what=f"c4 {key}")
    g = gvr.backward(fr, di, da)
    for key in ("d_center", "d_inv_cov", "d_attr", "d_rotation", "d_translation"):
        assert_grad_close(getattr(g, key), go[key], what=f"c4 {key}")
    assert np.array_equal(g.d_inv_cov, np.transpose(g.d_inv_cov, (0, 2, 1)))


def test_c4_two_shards_union_to_the_full_render(ctx, c4):
    """C4 tile sharding: the shards' outputs union to the oracle's
    render and their gradients sum to the oracle's gradient."""
    scene, cam, cfg, o, di, da, go = c4
    parts, grads = [], []
    for shard in range(2):
        fr = gvr.render_with_tape(scene, cam, cfg, ctx=ctx, shard=(shard, 2))
        st = fr.tape.list_stats()
        assert st["overflow_tiles"] == 0
        parts.append(fr.buffers)
        grads.append(gvr.backward(fr, di, da))
    th = (np.arange(1024) // 8)[:, None] * 128 + (np.arange(1024) // 8)[None, :]
    own = [(th % 2) == s for s in range(2)]
    img = np.where(own[0][..., None], parts[0].image, parts[1].image)
    idx = np.where(own[0][..., None], parts[0].topk_idx, parts[1].topk_idx)
    assert np.array_equal(idx, o["topk_idx"])
    assert_close_rel(img, o["image"], what="c4 shard image")
    for s in range(2):  # other shards' pixels hold the empty render
        assert np.all(parts[s].image[~own[s]] == 0.0) and np.all(parts[s].topk_idx[~own[s]] == -1)
    for key in ("d_center", "d_inv_cov", "d_attr", "d_rotation", "d_translation"):
        assert_grad_close(getattr(grads[0], key) + getattr(grads[1], key), go[key], what=f"c4 shard {key}")


def test_c5_full_size_fit_iteration(ctx):
    """One C5 iteration (50,786 kernels, 32 orbit views 256x256): the Fitter's
    loss and view-summed gradients equal the oracle's loss_and_grad."""
    from paper_2205_15401_b200.fit import Fitter

    target = gvr.make_bench_scene(50_000)
    assert target.size == 50_786
    target.attr[:] = (0.2, 0.5, 0.8)
    cfg = SelectionConfig()
    views = []
    for v in range(32):
        cam = gvr.make_orbit_camera(2 * np.pi * v / 32, 0.3, 4.0, (0, 0, 4), 256, 256, 1.6 * 256)
        t = oracle.port_render(target, cam, cfg, threads=0)
        views.append((cam, t["image"], t["alpha"]))
    scene = target.copy()
    scene.attr[:] = (0.8, 0.3, 0.2)
    scene.centers = scene.centers + np.random.default_rng(5).normal(0.0, 0.002, scene.centers.shape)
    fitter = Fitter(ctx, scene, views, rgb_weight=1.0, silhouette_weight=1.0)
    fitter.loss_and_grad()
    loss = fitter.loss()
    g_center = fitter.g_center.cpu().numpy().reshape(-1, 3)
    g_attr = fitter.g_attr.cpu().numpy().reshape(-1, 3)
    want_loss, want_c, want_a = 0.0, np.zeros_like(g_center), np.zeros_like(g_attr)
    for cam, ti, ta in views:
        o = oracle.port_render(scene, cam, cfg, threads=0)
        di = 2.0 * (o["image"] - ti) / (ti.size * len(views))
        da = 2.0 * (o["alpha"] - ta) / (ta.size * len(views))
        want_loss += (((o["image"] - ti) ** 2).sum() / ti.size + ((o["alpha"] - ta) ** 2).sum() / ta.size) / len(views)
        g = oracle.port_backward(scene, cam, cfg, di, da, threads=0)
        want_c += g["d_center"]
        want_a += g["d_attr"]
    assert loss == pytest.approx(want_loss, rel=1e-6)
    assert_grad_close(g_center, want_c, what="c5 d_center")
    assert_grad_close(g_attr, want_a, what="c5 d_attr")
