"""GPU: multi-view batches (gvr_render_views / gvr_scalar_loss_views /
gvr_backward_views) — the C3 view-sharded workload and the C5 per-iteration
view loop. A batch must equal the same views rendered one by one: forward bit
for bit (the forward is deterministic), gradients to FP64 atomic-order noise,
and the view sum to the sum of the per-view bundles; one view against the
oracle (the reference restated) closes the loop."""
import numpy as np
import pytest
import torch

import oracle
import paper_2205_15401_b200 as gvr
from conftest import assert_close_rel, assert_grad_close
from paper_2205_15401_b200.types import GradFlags, SelectionConfig, ValidationError

pytestmark = pytest.mark.gpu

KEYS = ("d_center", "d_inv_cov", "d_attr", "d_rotation", "d_translation")


def _views(n, size=48):
    return [gvr.make_orbit_camera(2 * np.pi * v / n, 0.3, 4.0, (0, 0, 4), size, size, 1.6 * size) for v in range(n)]


def _grad_bufs(k, d, dev):
    shapes = dict(d_center=(k, 3), d_inv_cov=(k, 3, 3), d_attr=(k, d), d_rotation=(3, 3), d_translation=(3,))
    return {n: torch.zeros(s, dtype=torch.float64, device=dev) for n, s in shapes.items()}


@pytest.mark.parametrize("k_prime", [20, 40])
def test_views_equal_single_renders(ctx, k_prime):
    """K' = 20 (warp selection, presorted) and K' = 40 (CTA selection, blend sorts)."""
    scene = gvr.make_bench_scene(2000)
    cams = _views(11)
    cfg = SelectionConfig(k_prime=k_prime)
    dev = torch.device("cuda:0")
    ds = gvr.DeviceScene(ctx).set(scene)
    tapes = [gvr.Tape(ctx) for _ in cams]
    imgs = [torch.empty((48, 48, 3), dtype=torch.float64, device=dev) for _ in cams]
    alphas = [torch.empty((48, 48, 1), dtype=torch.float64, device=dev) for _ in cams]
    tk = [np.empty((48, 48, k_prime), dtype=np.int32) for _ in cams]  # host outputs in a batch
    gvr.render_views_into(ctx, ds, cams, cfg, tapes, images=imgs, alphas=alphas, topk_idx=tk)
    rng = np.random.default_rng(0)
    ti = [torch.tensor(rng.uniform(0, 1, (48, 48, 3)), device=dev) for _ in cams]
    ta = [torch.tensor(rng.uniform(0, 1, (48, 48, 1)), device=dev) for _ in cams]
    losses = torch.zeros(len(cams), dtype=torch.float64, device=dev)
    gvr.scalar_loss_views_into(ctx, tapes, ti, ta, 1.0, 1.0, losses)
    outs = [_grad_bufs(scene.size, 3, dev) for _ in cams]
    total = _grad_bufs(scene.size, 3, dev)
    gvr.backward_views_into(ctx, tapes, GradFlags(), outs, total)
    ctx.synchronize()
    acc = {k: np.zeros(v.shape) for k, v in total.items()}
    for v, cam in enumerate(cams):
        fr = gvr.render_with_tape(ds, cam, cfg, ctx=ctx)
        assert np.array_equal(imgs[v].cpu().numpy(), fr.buffers.image)
        assert np.array_equal(alphas[v].cpu().numpy(), fr.buffers.alpha)
        assert np.array_equal(tk[v], fr.buffers.topk_idx)
        loss, di, da = gvr.scalar_loss(fr.tape, gvr.ScalarLoss(ti[v].cpu().numpy(), ta[v].cpu().numpy()))
        assert losses[v].item() == pytest.approx(loss, rel=1e-12)
        gb = gvr.backward(fr, None, None)
        for key in KEYS:
            got = outs[v][key].cpu().numpy()
            ref = getattr(gb, key)
            np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-12 * max(np.abs(ref).max(), 1e-300))
            acc[key] += got
    for key in KEYS:
        np.testing.assert_allclose(total[key].cpu().numpy(), acc[key], rtol=1e-12, atol=1e-15)


def test_one_view_of_a_batch_matches_the_oracle(ctx):
    scene = gvr.make_bench_scene(2000)
    cams = _views(4, 40)
    cfg = SelectionConfig()
    ds = gvr.DeviceScene(ctx).set(scene)
    tapes = [gvr.Tape(ctx) for _ in cams]
    imgs = [np.empty((40, 40, 3)) for _ in cams]
    tk = [np.empty((40, 40, 20), dtype=np.int32) for _ in cams]
    gvr.render_views_into(ctx, ds, cams, cfg, tapes, images=imgs, topk_idx=tk)
    ref = oracle.port_render(scene, cams[2], cfg)
    assert np.array_equal(tk[2], ref["topk_idx"])
    assert_close_rel(imgs[2], ref["image"], what="views image")
    rng = np.random.default_rng(1)
    ti = [rng.uniform(0, 1, (40, 40, 3)) for _ in cams]
    ta = [rng.uniform(0, 1, (40, 40, 1)) for _ in cams]
    gvr.scalar_loss_views_into(ctx, tapes, ti, ta)
    dev = torch.device("cuda:0")
    outs = [_grad_bufs(scene.size, 3, dev) for _ in cams]
    gvr.backward_views_into(ctx, tapes, GradFlags(), outs)
    ctx.synchronize()
    g = oracle.port_backward(scene, cams[2], cfg, ref["image"] - ti[2], ref["alpha"] - ta[2])
    for key in KEYS:
        assert_grad_close(outs[2][key].cpu().numpy(), g[key], what=f"views {key}")


def test_views_are_capturable_in_one_graph(ctx):
    scene = gvr.make_bench_scene(2000)
    cams = _views(9)
    cfg = SelectionConfig()
    dev = torch.device("cuda:0")
    ds = gvr.DeviceScene(ctx).set(scene)
    tapes = [gvr.Tape(ctx) for _ in cams]
    imgs = [torch.empty((48, 48, 3), dtype=torch.float64, device=dev) for _ in cams]
    ti = [torch.full((48, 48, 3), 0.5, dtype=torch.float64, device=dev) for _ in cams]
    ta = [torch.full((48, 48, 1), 0.5, dtype=torch.float64, device=dev) for _ in cams]
    total = _grad_bufs(scene.size, 3, dev)

    def step():
        for t in total.values():
            t.zero_()
        gvr.render_views_into(ctx, ds, cams, cfg, tapes, images=imgs)
        gvr.scalar_loss_views_into(ctx, tapes, ti, ta)
        gvr.backward_views_into(ctx, tapes, GradFlags(), None, total)

    stream = torch.cuda.ExternalStream(int(ctx.lib.gvr_context_stream(ctx.handle)), device=dev)
    with torch.cuda.stream(stream):
        step()
        ctx.synchronize()
        eager = {k: v.clone() for k, v in total.items()}
        eager_img = imgs[5].clone()
        with ctx.capture() as g:
            step()
        for im in imgs:
            im.zero_()
        g.launch()
        ctx.synchronize()
    assert torch.equal(imgs[5], eager_img)
    for k in KEYS:
        torch.testing.assert_close(total[k], eager[k], rtol=1e-10, atol=1e-14)


def test_views_validation(ctx):
    scene = gvr.make_bench_scene(200)
    ds = gvr.DeviceScene(ctx).set(scene)
    cams = _views(3, 16)
    t = gvr.Tape(ctx)
    with pytest.raises(gvr.GvrRuntimeError, match="share a tape"):
        gvr.render_views_into(ctx, ds, cams[:2], SelectionConfig(), [t, t])
    bad = gvr.Camera(np.diag([2.0, 1.0, 1.0]), np.zeros(3), 20.0, 7.5, 7.5, 16, 16)
    with pytest.raises(ValidationError, match="camera rotation is not orthonormal"):
        gvr.render_views_into(ctx, ds, [cams[0], bad], SelectionConfig(), [gvr.Tape(ctx), gvr.Tape(ctx)])
    # the context is still usable after a rejected batch
    fr = gvr.render_with_tape(ds, cams[0], SelectionConfig(), ctx=ctx)
    assert fr.buffers.alpha.max() > 0
