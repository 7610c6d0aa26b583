"""GPU, world size 2 (both ranks on cuda:0, gloo): the multi-GPU render paths
as bench.py / Fitter run them, on the one GPU of the test box.

* C4 tile sharding: the ranks' shard renders union to the 1-rank render bit
  for bit, and their all-reduced gradients equal the 1-rank gradients;
* C5 fitting: a 2-rank Fitter (views split, gradient all-reduce, replicated
  ADAM) keeps identical parameters on both ranks and follows the 1-rank
  trajectory (up to the summation order of the view gradients).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _c4_inputs():
    import paper_2205_15401_b200 as gvr

    scene = gvr.make_bench_scene(20000)
    cam = gvr.make_bench_camera(256)
    rng = np.random.default_rng(11)
    ti = rng.uniform(0, 1, (256, 256, 3))
    ta = rng.uniform(0, 1, (256, 256, 1))
    return scene, cam, ti, ta


def _c4_rank(rank, world):
    """One rank's C4 step: shard render, device loss, backward, gradient all-reduce."""
    import paper_2205_15401_b200 as gvr
    from paper_2205_15401_b200.distributed import allreduce_gradients

    scene, cam, ti, ta = _c4_inputs()
    ctx = gvr.Context(0)
    fr = gvr.render_with_tape(scene, cam, ctx=ctx, shard=(rank, world))
    gvr.scalar_loss(fr.tape, gvr.ScalarLoss(ti, ta), want_grads=False)
    # the bench's C4 path: packed rows (gvr_backward_packed), summed across ranks
    dev = torch.device("cuda:0")
    packed = torch.zeros((scene.size, 12), dtype=torch.float64, device=dev)
    d_rt = torch.zeros(12, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()  # torch's stream is not the context's
    gvr.backward_packed_into(fr.tape, None, None, gvr.GradFlags(), packed, d_rt)
    ctx.synchronize()
    assert float(packed.abs().max()) > 0.0
    allreduce_gradients([packed, d_rt])
    parts = gvr.unpack_gradients(packed.cpu().numpy(), d_rt.cpu().numpy(), 3)
    return fr.buffers, [np.ascontiguousarray(p) for p in parts]


def _fit_run(rank, world, steps=3):
    import paper_2205_15401_b200 as gvr
    from paper_2205_15401_b200.fit import AdamConfig, Fitter, make_fit_views

    ctx = gvr.Context(0)
    target = gvr.make_bench_scene(1000)
    target.attr[:] = (0.2, 0.5, 0.8)
    views = make_fit_views(target, 4, 48, ctx=ctx)
    start = target.copy()
    start.attr[:] = (0.8, 0.3, 0.2)
    start.centers = start.centers + np.random.default_rng(5).normal(0.0, 0.002, start.centers.shape)
    fitter = Fitter(ctx, start, views, adam=AdamConfig(lr=0.002), rank=rank, world=world,
                    device=torch.device("cuda:0"))
    for _ in range(steps):
        fitter.step()
    loss = fitter.loss()
    return fitter.params.cpu().numpy().copy(), loss


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        buf, grads = _c4_rank(rank, world)
        params, loss = _fit_run(rank, world)
        out[rank] = dict(image=buf.image, topk=buf.topk_idx, grads=grads, params=params, loss=loss)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _single(q):
    torch.cuda.set_device(0)
    buf, grads = _c4_rank(0, 1)
    params, loss = _fit_run(0, 1)
    q["single"] = dict(image=buf.image, topk=buf.topk_idx, grads=grads, params=params, loss=loss)


def test_two_ranks_match_one_rank():
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    out = manager.dict()
    p = ctx.Process(target=_single, args=(out,))
    p.start()
    p.join()
    assert p.exitcode == 0
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    one, r0, r1 = out["single"], out[0], out[1]
    # C4: union of the tile shards == the 1-rank render, bit for bit
    th = (np.arange(256) // 8)[:, None] * 32 + (np.arange(256) // 8)[None, :]
    own0 = (th % 2 == 0)[..., None]
    assert np.array_equal(np.where(own0, r0["topk"], r1["topk"]), one["topk"])
    assert np.array_equal(np.where(own0, r0["image"], r1["image"]), one["image"])
    for a, b, c in zip(r0["grads"], r1["grads"], one["grads"]):
        assert np.array_equal(a, b)  # every rank holds the same reduced gradient
        # the same sums in another grouping (per shard, then NCCL): FP64 rounding of the
        # per-kernel chain, which cancels up to (|m| / sigma)^2 (backward.cuh: entry_coeffs)
        np.testing.assert_allclose(a, c, rtol=1e-9, atol=1e-10 * np.abs(c).max())
    # C5: identical parameters on both ranks, the 1-rank trajectory
    assert np.array_equal(r0["params"], r1["params"])
    np.testing.assert_allclose(r0["params"], one["params"], rtol=1e-9, atol=1e-12)
    assert r0["loss"] == pytest.approx(one["loss"], rel=1e-9)
