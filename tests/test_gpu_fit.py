"""GPU: the fitting loop (C5) and tile sharding (C4) against the oracle.

* one Fitter iteration's loss and summed per-view gradients == the oracle's
  loss_and_grad semantics (fit.cpp:117-158) on the same inputs;
* gvr_adam_step == AdamState::update (fit.cpp:20-42);
* fitting reduces the loss (test_fit.cpp spirit);
* the union of tile-sharded renders equals the full render bit for bit and the
  shard gradients sum to the full gradient (C4 invariants).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2205_15401_b200 as gvr
from conftest import assert_grad_close
from paper_2205_15401_b200 import synthetic
from paper_2205_15401_b200.fit import AdamConfig, Fitter, make_fit_views
from paper_2205_15401_b200.types import GaussianScene, SelectionConfig, ValidationError

pytestmark = pytest.mark.gpu


def _views(target, n, size):
    views = []
    for v in range(n):
        cam = gvr.make_orbit_camera(2 * np.pi * v / n, 0.3, 4.0, (0, 0, 4), size, size, 1.6 * size)
        o = oracle.port_render(target, cam, SelectionConfig(), threads=4)
        views.append((cam, o["image"], o["alpha"]))
    return views


def test_fitter_loss_and_grad_matches_oracle(ctx):
    scene = gvr.make_bench_scene(1000)
    target = scene.copy()
    target.attr = target.attr[:, ::-1].copy()  # recoloured target
    target.centers = target.centers * 1.02
    views = _views(target, 4, 48)
    fitter = Fitter(ctx, scene, views, rgb_weight=1.0, silhouette_weight=0.5)
    fitter.loss_and_grad()
    loss = fitter.loss()
    g_center = fitter.g_center.cpu().numpy().reshape(-1, 3)
    g_attr = fitter.g_attr.cpu().numpy().reshape(-1, 3)
    want_loss, want_c, want_a = 0.0, np.zeros_like(g_center), np.zeros_like(g_attr)
    for cam, ti, ta in views:
        o = oracle.port_render(scene, cam, SelectionConfig(), threads=4)
        di = 2.0 * (o["image"] - ti) / (ti.size * len(views))
        da = 2.0 * 0.5 * (o["alpha"] - ta) / (ta.size * len(views))
        want_loss += (((o["image"] - ti) ** 2).sum() / ti.size + 0.5 * ((o["alpha"] - ta) ** 2).sum() / ta.size) / len(views)
        g = oracle.port_backward(scene, cam, SelectionConfig(), di, da, threads=4)
        want_c += g["d_center"]
        want_a += g["d_attr"]
    assert loss == pytest.approx(want_loss, rel=1e-6)
    assert_grad_close(g_center, want_c, what="fit d_center")
    assert_grad_close(g_attr, want_a, what="fit d_attr")


def test_adam_step_matches_reference_formula(ctx):
    rng = np.random.default_rng(0)
    p = rng.normal(size=1000)
    g = rng.normal(size=1000)
    m = rng.normal(size=1000) * 0.1
    v = np.abs(rng.normal(size=1000)) * 0.1
    dev = torch.device("cuda:0")
    tp, tg, tm, tv = (torch.tensor(a, device=dev) for a in (p, g, m, v))
    gvr.adam_step(ctx, tp, tg, tm, tv, 3, 0.01)
    ctx.synchronize()
    b1, b2, lr, eps = 0.9, 0.999, 0.01, 1e-8
    m2 = b1 * m + (1 - b1) * g
    v2 = b2 * v + (1 - b2) * g * g
    p2 = p - lr * (m2 / (1 - b1**3)) / (np.sqrt(v2 / (1 - b2**3)) + eps)
    np.testing.assert_allclose(tp.cpu().numpy(), p2, rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(tm.cpu().numpy(), m2, rtol=1e-13, atol=1e-16)
    np.testing.assert_allclose(tv.cpu().numpy(), v2, rtol=1e-13, atol=1e-16)


def test_fitting_reduces_loss(ctx):
    scene = gvr.make_bench_scene(1000)
    target = scene.copy()
    target.attr = np.tile([0.2, 0.6, 0.9], (scene.size, 1))
    views = _views(target, 4, 48)
    fitter = Fitter(ctx, scene, views, adam=AdamConfig(lr=0.02))
    fitter.loss_and_grad()
    first = fitter.loss()
    for _ in range(15):
        fitter.step()
    fitter.loss_and_grad()
    assert fitter.loss() < 0.5 * first


@pytest.mark.parametrize("nshards", [2, 3, 8])
def test_tile_shards_union_equals_full_render(ctx, nshards):
    scene = gvr.make_bench_scene(20000)
    cam = gvr.make_orbit_camera(0.4, 0.3, 4.0, (0, 0, 4), 200, 232, 320.0)
    cfg = SelectionConfig()
    ds = gvr.DeviceScene(ctx).set(scene)
    full_tape = gvr.Tape(ctx)
    h, w = cam.height, cam.width
    img, alpha = np.empty((h, w, 3)), np.empty((h, w, 1))
    gvr.render_into(ctx, ds, cam, cfg, full_tape, img, alpha)
    rng = np.random.default_rng(1)
    di, da = rng.uniform(-1, 1, (h, w, 3)), rng.uniform(-1, 1, (h, w, 1))
    gfull = np.empty((scene.size, 3))
    gvr.backward_into(full_tape, di, da, gvr.GradFlags(), d_center=gfull)
    u_img, u_alpha, g_sum = np.zeros_like(img), np.zeros_like(alpha), np.zeros_like(gfull)
    for r in range(nshards):
        tape = gvr.Tape(ctx)
        si, sa = np.empty_like(img), np.empty_like(alpha)
        gvr.render_into(ctx, ds, cam, cfg, tape, si, sa, shard=(r, nshards))
        u_img += si
        u_alpha += sa
        gs = np.empty_like(gfull)
        gvr.backward_into(tape, di, da, gvr.GradFlags(), d_center=gs)
        g_sum += gs
    assert np.array_equal(u_img, img)
    assert np.array_equal(u_alpha, alpha)
    np.testing.assert_allclose(g_sum, gfull, rtol=1e-9, atol=1e-12 * np.abs(gfull).max())


def test_device_regularizers_match_the_reference(ctx):
    """edge_reg / laplacian_reg on the device against the reference's values and
    gradients (golden tests/golden/aux/fit_regularizers.npz, fit.cpp:66-113)."""
    import os

    from paper_2205_15401_b200.fit import ShapeRegularizer

    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "aux", "fit_regularizers.npz"))
    reg = ShapeRegularizer(ctx, g["edges"], g["rest"])
    ge, gl = np.zeros_like(g["centers"]), np.zeros_like(g["centers"])
    ev = reg.edge_reg(g["centers"], ge)
    lv = reg.laplacian_reg(g["centers"], gl)
    assert ev == pytest.approx(float(g["edge_value"]), rel=1e-12)
    assert lv == pytest.approx(float(g["laplacian_value"]), rel=1e-12)
    np.testing.assert_allclose(ge, g["edge_grad"], rtol=1e-10, atol=1e-15)
    np.testing.assert_allclose(gl, g["laplacian_grad"], rtol=1e-10, atol=1e-15)
    # weighted accumulation into an existing gradient
    acc = np.ones_like(ge)
    reg.edge_reg(g["centers"], acc, weight=0.5, accumulate=True)
    np.testing.assert_allclose(acc, 1.0 + 0.5 * g["edge_grad"], rtol=1e-10, atol=1e-15)


def test_regularizer_validation(ctx):
    from paper_2205_15401_b200.fit import LossSpec, ShapeRegularizer
    from paper_2205_15401_b200.types import ValidationError

    with pytest.raises(ValidationError, match="regularizer needs a non-empty neighbor graph"):
        ShapeRegularizer(ctx, np.zeros((0, 2), dtype=np.int32), np.zeros((3, 3)))
    with pytest.raises(ValidationError, match="loss weights must be non-negative"):
        LossSpec(edge_weight=-1.0).validate()
    with pytest.raises(ValidationError, match="at least one loss weight must be positive"):
        LossSpec(0.0, 0.0, 0.0, 0.0).validate()


def test_fitter_adds_the_regularizer_terms(ctx):
    """fit_shape adds w_e edge_reg + w_l laplacian_reg to the loss and their
    gradients to d_center (fit.cpp:227-238)."""
    from paper_2205_15401_b200.fit import ShapeRegularizer

    verts, faces = synthetic.make_box_mesh((1.0, 1.0, 1.0), 4, (0.0, 0.0, 4.0))
    scene = synthetic.mesh_to_gaussians_isotropic(verts, faces, 0.5, (0.8, 0.3, 0.2))
    views = make_fit_views(scene, 3, 32, ctx=ctx)
    start = scene.copy()
    start.centers = start.centers + np.random.default_rng(2).normal(0.0, 0.01, start.centers.shape)
    edges = synthetic.mesh_edges(faces)
    reg = ShapeRegularizer(ctx, edges, verts)
    plain = Fitter(ctx, start, views)
    plain.loss_and_grad()
    with_reg = Fitter(ctx, start, views, regularizer=reg, edge_weight=0.3, laplacian_weight=0.7)
    with_reg.loss_and_grad()
    ev, eg, lv, lg = (oracle.ref_shape_reg(edges, verts, start.centers) if oracle.ref_available() else
                      (None, None, None, None))
    if ev is None:
        pytest.skip("reference build not present")
    assert with_reg.loss() - plain.loss() == pytest.approx(0.3 * ev + 0.7 * lv, rel=1e-9)
    d = with_reg.g_center.cpu().numpy().reshape(-1, 3) - plain.g_center.cpu().numpy().reshape(-1, 3)
    np.testing.assert_allclose(d, 0.3 * eg + 0.7 * lg, rtol=1e-6, atol=1e-12)


def test_graph_fitter_matches_eager(ctx):
    """The captured iteration (deferred scene validation, all views in one CUDA
    graph) follows the same trajectory as the eager one (FP64 atomic-order noise)."""
    scene = gvr.make_bench_scene(1000)
    target = scene.copy()
    target.attr = np.tile([0.2, 0.6, 0.9], (scene.size, 1))
    target.centers = target.centers * 1.01
    views = _views(target, 5, 40)
    eager = Fitter(ctx, scene, views, adam=AdamConfig(lr=0.01), use_graph=False)
    graph = Fitter(ctx, scene, views, adam=AdamConfig(lr=0.01), use_graph=True)
    for it in range(6):
        eager.step()
        graph.step()
        assert graph._graph is not None or it == 0
        assert graph.loss() == pytest.approx(eager.loss(), rel=1e-9)
    np.testing.assert_allclose(graph.params.cpu().numpy(), eager.params.cpu().numpy(), rtol=1e-9, atol=1e-12)


def test_deferred_scene_validation_reports_at_check(ctx):
    import torch
    scene = gvr.make_bench_scene(200)
    dev = torch.device("cuda:0")
    c = torch.tensor(scene.centers, device=dev)
    s = torch.tensor(scene.inv_cov, device=dev)
    a = torch.tensor(scene.attr, device=dev)
    ds = gvr.DeviceScene(ctx)
    ds.set_raw(scene.size, 3, 1.0, c, s, a, deferred=True)
    ds.check()  # valid
    s[7, 0, 1] += 1.0  # not symmetric
    ds.set_raw(scene.size, 3, 1.0, c, s, a, deferred=True)
    with pytest.raises(ValidationError, match=r"inv_cov is not symmetric \(kernel 7\)"):
        ds.check()
    s[7, 0, 1] -= 1.0
    c[3, 2] = float("nan")
    ds.set_raw(scene.size, 3, 1.0, c, s, a, deferred=True)
    with pytest.raises(ValidationError, match=r"non-finite values \(kernel 3\)"):
        ds.check()


def test_deferred_validation_is_rechecked_after_graph_replays(ctx):
    """A captured deferred upload validates on every replay; check() reads the latest."""
    import torch
    scene = gvr.make_bench_scene(200)
    dev = torch.device("cuda:0")
    c = torch.tensor(scene.centers, device=dev)
    s = torch.tensor(scene.inv_cov, device=dev)
    a = torch.tensor(scene.attr, device=dev)
    ds = gvr.DeviceScene(ctx)
    ds.set_raw(scene.size, 3, 1.0, c, s, a, deferred=True)  # sizes the buffers
    ds.check()
    stream = torch.cuda.ExternalStream(int(ctx.lib.gvr_context_stream(ctx.handle)), device=dev)
    with torch.cuda.stream(stream):
        with ctx.capture() as g:
            ds.set_raw(scene.size, 3, 1.0, c, s, a, deferred=True)
        g.launch()
        ds.check()
        c[5, 0] = float("inf")
        g.launch()
        with pytest.raises(ValidationError, match=r"non-finite values \(kernel 5\)"):
            ds.check()
        c[5, 0] = 0.0
        g.launch()
        ds.check()


def test_device_render_reports_non_finite_outputs(ctx):
    """validate_finite (blender.cpp:132-134) for renders into device buffers:
    Tape.check_finite raises the reference's message (image channels included).
    A deferred upload renders the values as they are, so a NaN attribute reaches
    the image while the geometry (alpha, depth) stays finite."""
    import torch
    dev = torch.device("cuda:0")
    scene = gvr.make_bench_scene(200)
    cam = gvr.make_bench_camera(32)
    attr = torch.tensor(scene.attr, device=dev)
    attr[:, 1] = float("nan")
    ds = gvr.DeviceScene(ctx)
    ds.set_raw(scene.size, 3, scene.tau, torch.tensor(scene.centers, device=dev),
               torch.tensor(scene.inv_cov, device=dev), attr, deferred=True)
    tape = gvr.Tape(ctx)
    img = torch.empty((32, 32, 3), dtype=torch.float64, device=dev)
    alpha = torch.empty((32, 32, 1), dtype=torch.float64, device=dev)
    gvr.render_into(ctx, ds, cam, SelectionConfig(), tape, img, alpha)
    assert torch.isfinite(alpha).all() and not torch.isfinite(img).all()
    with pytest.raises(ValidationError, match="image contains non-finite values"):
        tape.check_finite()
    ok = gvr.Tape(ctx)
    gvr.render_into(ctx, gvr.DeviceScene(ctx).set(scene), cam, SelectionConfig(), ok, img)
    ok.check_finite()


def test_objects_of_another_context_are_rejected(ctx):
    other = gvr.Context(0)
    fr = gvr.render_with_tape(gvr.make_bench_scene(200), gvr.make_bench_camera(24), ctx=other)
    with pytest.raises(gvr.GvrRuntimeError, match="another context"):
        ctx.check(ctx.lib.gvr_backward(ctx.handle, fr.tape.handle, None, None, None, None))
    with pytest.raises(gvr.GvrRuntimeError, match="another context"):
        ctx.check(ctx.lib.gvr_tape_traced(ctx.handle, fr.tape.handle, None, None, None, None))


def test_fitter_stops_updating_after_a_non_finite_loss(ctx):
    """fit_shape (fit.cpp:246-250): a non-finite loss ends the fit before the
    update -- the device ADAM step is skipped and the divergence latches."""
    target = gvr.make_bench_scene(300)
    views = make_fit_views(target, 2, 32, ctx=ctx)
    start = target.copy()
    start.attr[:] = 1e200  # finite image, overflowing loss
    fitter = Fitter(ctx, start, views, adam=AdamConfig(lr=0.01))
    p0 = fitter.params.cpu().numpy().copy()
    fitter.step()
    fitter.step()
    assert fitter.diverged
    assert not np.isfinite(fitter.loss())
    assert np.array_equal(fitter.params.cpu().numpy(), p0)
    healthy = Fitter(ctx, target, views, adam=AdamConfig(lr=0.01))
    healthy.step()
    assert not healthy.diverged


def test_async_host_buffer_mode_matches_synchronous_calls():
    """gvr_context_set_async: host-buffer calls return before their copies finish;
    after synchronize the outputs equal the synchronous calls' bit for bit, and
    the deferred checks report an invalid upload."""
    import torch
    scene = gvr.make_bench_scene(2000)
    cam = gvr.make_bench_camera(64)
    rng = np.random.default_rng(2)
    ti = torch.tensor(rng.uniform(0, 1, (64, 64, 3))).pin_memory()
    ta = torch.tensor(rng.uniform(0, 1, (64, 64, 1))).pin_memory()
    results = []
    for mode in (False, True):
        c = gvr.Context(0)
        c.set_async(mode)
        ds = gvr.DeviceScene(c).set_raw(scene.size, 3, scene.tau, torch.tensor(scene.centers).pin_memory(),
                                        torch.tensor(scene.inv_cov).pin_memory(), torch.tensor(scene.attr).pin_memory())
        tp = gvr.Tape(c)
        img = torch.empty((64, 64, 3), dtype=torch.float64).pin_memory()
        loss = torch.zeros(1, dtype=torch.float64).pin_memory()
        gc = torch.empty((scene.size, 3), dtype=torch.float64).pin_memory()
        gvr.render_into(c, ds, cam, SelectionConfig(), tp, img)
        gvr.scalar_loss_into(tp, ti, ta, 1.0, 1.0, loss)
        gvr.backward_into(tp, None, None, gvr.GradFlags(), gc)
        c.synchronize()
        ds.check()
        tp.check_finite()
        results.append((img.clone(), loss.clone(), gc.clone()))
        if mode:
            bad = scene.inv_cov.copy()
            bad[3, 0, 1] += 1.0
            ds.set_raw(scene.size, 3, scene.tau, scene.centers, bad, scene.attr)  # returns: validated later
            with pytest.raises(ValidationError, match=r"not symmetric \(kernel 3\)"):
                ds.check()
    for a, b in zip(results[0], results[1]):
        assert torch.equal(a, b)


def test_packed_backward_equals_the_gradient_bundle(ctx):
    """gvr_backward_packed rows unpack to gvr_backward's bundle bit for bit."""
    import torch
    scene = gvr.make_bench_scene(3000)
    cam = gvr.make_orbit_camera(0.4, 0.3, 4.0, (0, 0, 4), 96, 96, 150.0)
    rng = np.random.default_rng(8)
    fr = gvr.render_with_tape(scene, cam, ctx=ctx)
    di = rng.uniform(-1, 1, fr.buffers.image.shape)
    da = rng.uniform(-1, 1, fr.buffers.alpha.shape)
    g = gvr.backward(fr, di, da)
    dev = torch.device("cuda:0")
    packed = torch.zeros((scene.size, 12), dtype=torch.float64, device=dev)
    d_rt = torch.zeros(12, dtype=torch.float64, device=dev)
    tdi, tda = torch.tensor(di, device=dev), torch.tensor(da, device=dev)
    torch.cuda.synchronize()  # torch's stream is not the context's: inputs ready before the backward
    gvr.backward_packed_into(fr.tape, tdi, tda, gvr.GradFlags(), packed, d_rt)
    ctx.synchronize()
    assert np.abs(g.d_center).max() > 0.0
    c, s, a, r, t = gvr.unpack_gradients(packed.cpu().numpy(), d_rt.cpu().numpy(), 3)
    for got, want in ((c, g.d_center), (s, g.d_inv_cov), (a, g.d_attr), (r, g.d_rotation), (t, g.d_translation)):
        assert np.array_equal(got, want)


def test_device_buffers_on_torchs_own_stream_are_ordered(ctx):
    """Tensors made on torch's current stream (not the context's) are safe to pass:
    the *_into calls order the two streams with events (no host sync needed)."""
    import torch
    assert torch.cuda.current_stream().cuda_stream != ctx.torch_stream().cuda_stream
    scene = gvr.make_bench_scene(2000)
    fr = gvr.render_with_tape(scene, gvr.make_bench_camera(96), ctx=ctx)
    rng = np.random.default_rng(3)
    di = rng.uniform(-1, 1, fr.buffers.image.shape)
    da = rng.uniform(-1, 1, fr.buffers.alpha.shape)
    want = gvr.backward(fr, di, da)
    dev = torch.device("cuda:0")
    for _ in range(3):
        big = torch.empty(64 << 20, dtype=torch.float64, device=dev).fill_(1.0)  # keeps torch's stream busy
        packed = torch.zeros((scene.size, 12), dtype=torch.float64, device=dev)
        d_rt = torch.zeros(12, dtype=torch.float64, device=dev)
        gvr.backward_packed_into(fr.tape, torch.tensor(di, device=dev), torch.tensor(da, device=dev),
                                 gvr.GradFlags(), packed, d_rt)
        c = packed[:, :3].cpu().numpy()  # torch's stream waits for the context's
        assert np.array_equal(c, want.d_center)
        del big


def test_pipelined_async_steps_with_side_stream_copies_match_synchronous():
    """Async host-buffer mode copies a call's host outputs on a side stream while
    the context stream runs the next call; the next call of the same kind waits
    for them. Steps pipelined over two contexts (as in bench.py's e2e loop), with
    changing targets, give the synchronous results bit for bit."""
    scene = gvr.make_bench_scene(3000)
    cam = gvr.make_bench_camera(64)
    rng = np.random.default_rng(5)
    targets = [(torch.tensor(rng.uniform(0, 1, (64, 64, 3))).pin_memory(),
                torch.tensor(rng.uniform(0, 1, (64, 64, 1))).pin_memory()) for _ in range(6)]
    pin = lambda a: torch.tensor(a).pin_memory()  # noqa: E731
    hc, hs, ha = pin(scene.centers), pin(scene.inv_cov), pin(scene.attr)

    def make_slot(async_mode):
        c = gvr.Context(0)
        c.set_async(async_mode)
        out = dict(img=torch.empty((64, 64, 3), dtype=torch.float64).pin_memory(),
                   loss=torch.zeros(1, dtype=torch.float64).pin_memory(),
                   gc=torch.empty((scene.size, 3), dtype=torch.float64).pin_memory(),
                   gs=torch.empty((scene.size, 3, 3), dtype=torch.float64).pin_memory())
        return c, gvr.DeviceScene(c), gvr.Tape(c), out

    def enqueue(slot, t):
        c, ds, tp, o = slot
        ds.set_raw(scene.size, 3, scene.tau, hc, hs, ha)
        gvr.render_into(c, ds, cam, SelectionConfig(), tp, o["img"])
        gvr.scalar_loss_into(tp, targets[t][0], targets[t][1], 1.0, 1.0, o["loss"])
        gvr.backward_into(tp, None, None, gvr.GradFlags(), o["gc"], o["gs"])

    def take(slot):
        c, ds, tp, o = slot
        c.synchronize()
        ds.check()
        tp.check_finite()
        return {k: v.clone() for k, v in o.items()}

    ref = []
    sync = make_slot(False)
    for t in range(len(targets)):
        enqueue(sync, t)
        ref.append(take(sync))
    slots = [make_slot(True), make_slot(True)]
    got = [None] * len(targets)
    for t in range(len(targets)):
        if t >= 2:
            got[t - 2] = take(slots[t % 2])
        enqueue(slots[t % 2], t)
    for t in range(len(targets) - 2, len(targets)):
        got[t] = take(slots[t % 2])
    for a, b in zip(ref, got):
        for k in a:
            assert torch.equal(a[k], b[k]), k
    assert len({float(r["loss"][0]) for r in ref}) == len(targets)  # the targets did change


def test_schedule_from_the_last_render_of_the_view_keeps_outputs():
    """The tile order of a render may come from the selection cycles of the last
    render of the same view on the tape (LPT costs); it only reorders work: a
    repeated view, a view after a different camera, and a fresh tape agree bit
    for bit (topk, image, gradients)."""
    scene = gvr.make_bench_scene(20000)
    cam_a = gvr.make_bench_camera(128)
    cam_b = gvr.make_orbit_camera(0.7, 0.2, 4.0, (0, 0, 4), 128, 128, 1.6 * 128)

    kp = SelectionConfig().k_prime

    def run(tape, cam):
        img = np.empty((128, 128, 3))
        tidx = np.empty((128, 128, kp), dtype=np.int32)
        gvr.render_into(c, ds, cam, SelectionConfig(), tape, img, None, None, tidx)
        dc = np.empty((scene.size, 3))
        ds_ = np.empty((scene.size, 3, 3))
        gvr.backward_into(tape, np.ones((128, 128, 3)), np.ones((128, 128, 1)), gvr.GradFlags(), dc, ds_)
        return tidx, img, dc, ds_

    c = gvr.Context(0)
    ds = gvr.DeviceScene(c).set(scene)
    fresh = run(gvr.Tape(c), cam_a)
    tape = gvr.Tape(c)
    seq = [run(tape, cam_a), run(tape, cam_a), run(tape, cam_b), run(tape, cam_a), run(tape, cam_a)]
    for r in (seq[0], seq[1], seq[3], seq[4]):
        for a, b in zip(fresh, r):
            assert np.array_equal(a, b)
    other = run(gvr.Tape(c), cam_b)
    for a, b in zip(other, seq[2]):
        assert np.array_equal(a, b)
