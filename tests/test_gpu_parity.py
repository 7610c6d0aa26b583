"""GPU parity against the reference's golden vectors (tests/golden, made by the
reference build) and against the C oracle port, through the C ABI.

Bars (SURVEY.md §8a "Parity criteria", north star):
  * top-K index sets and their order: bit-exact (the deciding arithmetic is
    exact FP64 in the reference's evaluation order);
  * Tape::traced (l, q, sigma): bit-exact, same reason;
  * W, image, alpha, depth: |x - x_ref| <= 1e-4 |x_ref| + 1e-7;
  * gradients: |g - g_ref| <= 1e-4 max(|g_ref|, 1e-3 max_k |g_ref|) per class,
    d_inv_cov exactly symmetric.
"""
import numpy as np
import pytest

import paper_2205_15401_b200 as gvr
from conftest import assert_close_rel, assert_grad_close  # noqa: E402

pytestmark = pytest.mark.gpu


def test_forward_matches_reference(golden, ctx):
    fr = gvr.render_with_tape(golden.scene, golden.camera, golden.cfg, ctx=ctx)
    b = fr.buffers
    assert np.array_equal(b.topk_idx, golden["topk_idx"]), "top-K index sets / order differ"
    assert_close_rel(b.topk_w, golden["topk_w"], what="W")
    assert_close_rel(b.image, golden["image"], what="image")
    assert_close_rel(b.alpha, golden["alpha"], what="alpha")
    assert_close_rel(b.depth, golden["depth"], what="depth")


def test_tape_traced_bit_exact(golden, ctx):
    if "topk_l" not in golden:
        pytest.skip("golden file stores no traced values")
    fr = gvr.render_with_tape(golden.scene, golden.camera, golden.cfg, ctx=ctx)
    idx, l, q, s = fr.tape.traced()
    assert np.array_equal(idx, golden["topk_idx"])
    assert np.array_equal(l, golden["topk_l"]), f"l max diff {np.abs(l - golden['topk_l']).max()}"
    assert np.array_equal(q, golden["topk_q"]), f"q max diff {np.abs(q - golden['topk_q']).max()}"
    assert np.array_equal(s, golden["topk_sigma"]), f"sigma max diff {np.abs(s - golden['topk_sigma']).max()}"


def test_backward_matches_reference(golden, ctx):
    fr = gvr.render_with_tape(golden.scene, golden.camera, golden.cfg, ctx=ctx)
    gb = gvr.backward(fr, golden["d_image"], golden["d_alpha"], golden.flags)
    assert_grad_close(gb.d_attr, golden["d_attr"], what="d_attr")
    assert_grad_close(gb.d_center, golden["d_center"], what="d_center")
    assert_grad_close(gb.d_inv_cov, golden["d_inv_cov"], what="d_inv_cov")
    assert_grad_close(gb.d_rotation, golden["d_rotation"], what="d_rotation")
    assert_grad_close(gb.d_translation, golden["d_translation"], what="d_translation")
    assert np.array_equal(gb.d_inv_cov, np.transpose(gb.d_inv_cov, (0, 2, 1))), "d_inv_cov not exactly symmetric"


def test_prefilter_is_conservative(golden, ctx):
    """The FP32 pre-filter never rejects what the exact FP64 path accepts:
    sending every candidate through FP64 gives bit-identical outputs."""
    a = gvr.render(golden.scene, golden.camera, golden.cfg, ctx=ctx)
    ctx.set_prefilter_guard(1e30)
    try:
        b = gvr.render(golden.scene, golden.camera, golden.cfg, ctx=ctx)
    finally:
        ctx.set_prefilter_guard(0.02)
    assert np.array_equal(a.topk_idx, b.topk_idx)
    assert np.array_equal(a.image, b.image)


def test_forward_deterministic(ctx):
    from conftest import Golden

    g = Golden("texture_scene")
    a = gvr.render(g.scene, g.camera, g.cfg, ctx=ctx)
    b = gvr.render(g.scene, g.camera, g.cfg, ctx=ctx)
    for k in ("image", "alpha", "depth", "topk_idx", "topk_w"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_tile_list_overflow_path(golden, ctx):
    """Tiles whose candidate list does not fit the list pool stream every kernel
    with the same exact tests: outputs are bit-identical."""
    a = gvr.render_with_tape(golden.scene, golden.camera, golden.cfg, ctx=ctx)
    assert a.tape.list_stats()["overflow_tiles"] == 0
    ctx.set_tile_capacity(8)
    try:
        b = gvr.render_with_tape(golden.scene, golden.camera, golden.cfg, ctx=ctx)
        st = b.tape.list_stats()
    finally:
        ctx.set_tile_capacity(0)
    if st["entries"] > 8:
        assert st["overflow_tiles"] > 0
    assert np.array_equal(a.buffers.topk_idx, b.buffers.topk_idx)
    assert np.array_equal(a.buffers.image, b.buffers.image)
    # the same cap leaves kernels without a mask rectangle: the backward's atomic fallback
    ctx.set_tile_capacity(8)
    try:
        c = gvr.render_with_tape(golden.scene, golden.camera, golden.cfg, ctx=ctx)
        gb = gvr.backward(c, golden["d_image"], golden["d_alpha"], golden.flags)
    finally:
        ctx.set_tile_capacity(0)
    for key in ("d_attr", "d_center", "d_inv_cov", "d_rotation", "d_translation"):
        assert_grad_close(getattr(gb, key), golden[key], what=f"fallback {key}")


def test_backward_is_bit_deterministic(ctx):
    """test_grad.cpp:279-296: repeated backwards give bit-identical bundles (the
    per-kernel gather sums every gradient in one fixed order)."""
    scene = gvr.make_bench_scene(100000)
    cam = gvr.make_orbit_camera(0.7, 0.3, 4.0, (0, 0, 4), 256, 256, 1.6 * 256)
    rng = np.random.default_rng(9)
    bundles = []
    for _ in range(3):
        fr = gvr.render_with_tape(scene, cam, ctx=ctx)
        st = fr.tape.list_stats()
        assert st["mask_tiles"] <= st["mask_capacity"]
        di = rng.uniform(-1, 1, fr.buffers.image.shape) if not bundles else di
        da = rng.uniform(-1, 1, fr.buffers.alpha.shape) if not bundles else da
        bundles.append(gvr.backward(fr, di, da))
        bundles.append(gvr.backward(fr, di, da))
    for b in bundles[1:]:
        for key in ("d_center", "d_inv_cov", "d_attr", "d_rotation", "d_translation"):
            assert np.array_equal(getattr(b, key), getattr(bundles[0], key)), key


def test_lists_sorted_in_global_memory(golden, ctx):
    """Lists longer than the shared-memory stage are depth-sorted in the global
    sorted pool (same bucket order, same early exit): bit-identical outputs."""
    a = gvr.render_with_tape(golden.scene, golden.camera, golden.cfg, ctx=ctx)
    ctx.set_list_smem(1)
    try:
        b = gvr.render_with_tape(golden.scene, golden.camera, golden.cfg, ctx=ctx)
        st = b.tape.list_stats()
    finally:
        ctx.set_list_smem(2048)
    assert st["overflow_tiles"] == 0
    if st["max_list"] > 1:
        assert st["global_sorted_tiles"] > 0
    assert np.array_equal(a.buffers.topk_idx, b.buffers.topk_idx)
    assert np.array_equal(a.buffers.image, b.buffers.image)
    assert np.array_equal(a.buffers.topk_w, b.buffers.topk_w)


def test_graph_replay_matches_eager(ctx):
    """A captured render -> loss -> backward graph replays to the eager results."""
    import torch

    from conftest import Golden

    g = Golden("texture_scene")
    dev = torch.device("cuda:0")
    stream = torch.cuda.ExternalStream(int(ctx.lib.gvr_context_stream(ctx.handle)), device=dev)
    torch.cuda.set_stream(stream)
    s = g.scene
    ds = gvr.DeviceScene(ctx).set_raw(s.size, s.attr_dim(), s.tau, torch.from_numpy(s.centers).to(dev),
                                      torch.from_numpy(s.inv_cov).to(dev), torch.from_numpy(s.attr).to(dev))
    tape = gvr.Tape(ctx)
    h, w = g.camera.height, g.camera.width
    img = torch.empty((h, w, s.attr_dim()), dtype=torch.float64, device=dev)
    ti = torch.rand((h, w, s.attr_dim()), dtype=torch.float64, device=dev)
    ta = torch.rand((h, w, 1), dtype=torch.float64, device=dev)
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    gc = torch.empty((s.size, 3), dtype=torch.float64, device=dev)

    def step():
        gvr.render_into(ctx, ds, g.camera, g.cfg, tape, img)
        gvr.scalar_loss_into(tape, ti, ta, 1.0, 1.0, loss)
        gvr.backward_into(tape, None, None, gvr.GradFlags(), gc)

    step()
    ctx.synchronize()
    eager_img, eager_loss, eager_gc = img.clone(), loss.clone(), gc.clone()
    with ctx.capture() as graph:
        step()
    img.zero_()
    gc.zero_()
    graph.launch()
    ctx.synchronize()
    assert torch.equal(img, eager_img)
    assert torch.allclose(loss, eager_loss, rtol=1e-14, atol=0)
    assert torch.allclose(gc, eager_gc, rtol=1e-12, atol=1e-15)
    torch.cuda.set_stream(torch.cuda.default_stream(dev))


@pytest.mark.parametrize("kp", [80, 128])
def test_large_k_prime_matches_the_oracle(ctx, kp):
    """K' beyond the warp selection (CTA selection + sorting blend), up to the
    backend's 128: bit-exact selection, tolerance parity of outputs and gradients."""
    import oracle
    from paper_2205_15401_b200.types import Camera, GaussianScene, SelectionConfig

    rng = np.random.default_rng(kp)
    k = 220
    centers = np.stack([rng.uniform(-0.4, 0.4, k), rng.uniform(-0.4, 0.4, k), rng.uniform(3.0, 6.0, k)], 1)
    inv_cov = np.stack([np.eye(3) / rng.uniform(0.2, 0.5) ** 2 for _ in range(k)])
    scene = GaussianScene(centers, inv_cov, rng.uniform(0, 1, (k, 3)), 0.3)
    cam = Camera(np.eye(3), np.zeros(3), 20.0, 11.5, 11.5, 24, 24)
    cfg = SelectionConfig(k_prime=kp)
    fr = gvr.render_with_tape(scene, cam, cfg, ctx=ctx)
    o = oracle.port_render(scene, cam, cfg, threads=0)
    assert (fr.buffers.topk_idx >= 0).sum(axis=2).max() > 64  # the case is really beyond 64
    assert np.array_equal(fr.buffers.topk_idx, o["topk_idx"])
    for key in ("image", "alpha", "depth", "topk_w"):
        assert_close_rel(getattr(fr.buffers, key), o[key], what=f"kp{kp} {key}")
    di = rng.uniform(-1, 1, fr.buffers.image.shape)
    da = rng.uniform(-1, 1, fr.buffers.alpha.shape)
    g = gvr.backward(fr, di, da)
    go = oracle.port_backward(scene, cam, cfg, di, da, threads=0)
    for key in ("d_center", "d_inv_cov", "d_attr", "d_rotation", "d_translation"):
        assert_grad_close(getattr(g, key), go[key], what=f"kp{kp} {key}")
