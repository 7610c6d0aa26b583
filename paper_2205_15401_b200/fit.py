"""Device fitting loop.

Mirrors ``gvr::loss_and_grad`` + ``AdamState::update`` of ``fit_shape``
(/root/reference/proj/src/fit.cpp:117-158, :20-42, :176-265) with everything on
the GPU and the views sharded across ranks:

  per iteration, on each rank, for all of its views v at once (the views run
  concurrently on the context's worker streams):
      render_with_tape(scene, camera_v)                      (gvr_render_views)
      loss_v = rgb |img - t|^2 / #img + sil |alpha - t_a|^2 / #alpha, scaled 1/#views
      d_image = 2 rgb (img - t) / (#img #views), d_alpha likewise    (gvr_scalar_loss_views)
      gradients = sum_v backward(tape_v, d_image_v, d_alpha_v)   (gvr_backward_views, view sum)
  all-reduce(sum) of [d_center | d_attr | loss] across ranks (NCCL over NVLink;
  the only collective of the render path)
  ADAM on [centers | attrs] (gvr_adam_step), identical on every rank.

plus, when a ``ShapeRegularizer`` is given, the edge-length and uniform-Laplacian
terms on the centres (fit.cpp:66-113, device kernels, weights of LossSpec).

Difference from fit_shape: every view is used every iteration (the C5 config:
32 views, no random batch sampling).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .distributed import allreduce_gradients, shard_views
from .render import (Context, DeviceScene, Tape, adam_step, backward_views_into, render_views_into,
                     scalar_loss_views_into)
from .types import Camera, GaussianScene, GradFlags, SelectionConfig


@dataclass
class LossSpec:
    """``gvr::LossSpec`` (fit.hpp:9-16)."""

    rgb_weight: float = 1.0
    silhouette_weight: float = 1.0
    edge_weight: float = 0.0
    laplacian_weight: float = 0.0

    def validate(self) -> None:
        """fit.cpp:10-18, same messages."""
        from .types import ValidationError

        if min(self.rgb_weight, self.silhouette_weight, self.edge_weight, self.laplacian_weight) < 0.0:
            raise ValidationError("loss weights must be non-negative")
        if self.rgb_weight == 0.0 and self.silhouette_weight == 0.0 and self.edge_weight == 0.0 and \
                self.laplacian_weight == 0.0:
            raise ValidationError("at least one loss weight must be positive")


class ShapeRegularizer:
    """``gvr::ShapeRegularizer`` (fit.hpp:50-60) on the device: neighbour graph,
    rest edge lengths and rest Laplacian displacements (fit.cpp:44-64)."""

    def __init__(self, ctx: Context, edges, rest_centers):
        import ctypes

        self.ctx = ctx
        e = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 2)
        c = np.ascontiguousarray(rest_centers, dtype=np.float64).reshape(-1, 3)
        self.n_vertices, self.n_edges = c.shape[0], e.shape[0]
        h = ctypes.c_void_p()
        ctx.check(ctx.lib.gvr_regularizer_create(ctx.handle, self.n_vertices, self.n_edges,
                                                 e.ctypes.data if e.size else None, c.ctypes.data, ctypes.byref(h)))
        self.handle = h

    def _term(self, fn, centers, weight: float, grad, accumulate: bool):
        from .render import _ptr

        out = np.zeros(1)
        c = np.ascontiguousarray(centers, dtype=np.float64) if isinstance(centers, np.ndarray) else centers
        self.ctx.check(fn(self.ctx.handle, self.handle, _ptr(c), float(weight), _ptr(out), _ptr(grad),
                          int(bool(accumulate))))
        return float(out[0])

    def edge_reg(self, centers, grad=None, weight: float = 1.0, accumulate: bool = False) -> float:
        """``edge_reg`` (fit.cpp:66-85); grad [N, 3] receives weight * gradient."""
        return self._term(self.ctx.lib.gvr_edge_reg, centers, weight, grad, accumulate)

    def laplacian_reg(self, centers, grad=None, weight: float = 1.0, accumulate: bool = False) -> float:
        """``laplacian_reg`` (fit.cpp:87-113)."""
        return self._term(self.ctx.lib.gvr_laplacian_reg, centers, weight, grad, accumulate)

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.ctx.lib.gvr_regularizer_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class AdamConfig:
    """``gvr::AdamConfig`` (fit.hpp:18-23)."""

    lr: float = 0.01
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8


class Fitter:
    """Shape/texture fitting of centers and attributes against target views."""

    def __init__(self, ctx: Context, scene: GaussianScene, views: Sequence[Tuple[Camera, np.ndarray, np.ndarray]],
                 cfg: SelectionConfig = SelectionConfig(), rgb_weight: float = 1.0, silhouette_weight: float = 1.0,
                 adam: AdamConfig = AdamConfig(), rank: int = 0, world: int = 1, device=None,
                 regularizer: Optional["ShapeRegularizer"] = None, edge_weight: float = 0.0,
                 laplacian_weight: float = 0.0, use_graph: bool = True):
        import torch

        LossSpec(rgb_weight, silhouette_weight, edge_weight, laplacian_weight).validate()
        self.reg, self.edge_weight, self.laplacian_weight = regularizer, edge_weight, laplacian_weight

        self.torch = torch
        self.ctx = ctx
        self.cfg = cfg
        self.adam = adam
        self.rank, self.world = rank, world
        self.dev = device if device is not None else torch.device(f"cuda:{ctx.device}")
        self.K, self.D = scene.size, scene.attr_dim()
        self.tau = scene.tau
        k3 = 3 * self.K
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.params = torch.cat([torch.from_numpy(scene.centers.reshape(-1)), torch.from_numpy(scene.attr.reshape(-1))]).to(**f64)
        self.centers = self.params[:k3].view(self.K, 3)
        self.attr = self.params[k3:].view(self.K, self.D)
        self.inv_cov = torch.from_numpy(scene.inv_cov).to(**f64).contiguous()
        self.grads = torch.zeros_like(self.params)
        self.g_center = self.grads[:k3]
        self.g_attr = self.grads[k3:]
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.step_count = 0
        self.n_views = len(views)
        self.mine = shard_views(self.n_views, rank, world)
        # views grouped by loss weights (2 rgb / (#img #views) etc.): one batched call per group
        groups = {}
        for idx in self.mine:
            cam, ti, ta = views[idx]
            n_img = float(np.asarray(ti).size)
            n_alpha = float(np.asarray(ta).size)
            w = (2.0 * rgb_weight / (n_img * self.n_views), 2.0 * silhouette_weight / (n_alpha * self.n_views))
            g = groups.setdefault(w, ([], [], [], []))
            g[0].append(cam)
            g[1].append(torch.as_tensor(np.ascontiguousarray(ti)).to(**f64))
            g[2].append(torch.as_tensor(np.ascontiguousarray(ta)).to(**f64))
            g[3].append(Tape(ctx))
        self.groups: List[Tuple[Tuple[float, float], list, list, list, list, object]] = [
            (w, cams, tis, tas, tapes, torch.zeros(len(cams), **f64)) for w, (cams, tis, tas, tapes) in groups.items()]
        self.loss_acc = torch.zeros(1, **f64)
        self._diverged = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self._lsum = [torch.zeros(1, **f64) for _ in self.groups]
        self.dscene = DeviceScene(ctx)
        # the per-iteration device work (upload + validation, all views fwd + loss
        # + bwd) is captured once into a CUDA graph and replayed: no host launch
        # cost per view; the regularizers return host values, so they keep it eager
        self.use_graph = use_graph and regularizer is None
        self._graph = None
        self._warm = False
        self.total = dict(d_center=self.g_center.view(self.K, 3),
                          d_attr=self.g_attr.view(self.K, self.D) if self.D > 0 else None)
        # torch work (accumulations, NCCL) on the context's stream, ordered with our kernels
        self.stream = torch.cuda.ExternalStream(int(ctx.lib.gvr_context_stream(ctx.handle)), device=self.dev)

    def loss_and_grad(self) -> None:
        """Accumulate this rank's loss and gradients (device, asynchronous)."""
        with self.torch.cuda.stream(self.stream):
            self._run_loss_and_grad()

    def _run_loss_and_grad(self) -> None:
        if not self.use_graph:
            self._loss_and_grad()
            return
        if self._graph is None:
            if not self._warm:  # the first pass sizes every buffer (no allocation while capturing)
                self._loss_and_grad()
                self._warm = True
                return
            g = self.ctx.capture()
            with g:
                self._loss_and_grad()
            self._graph = g
        self._graph.launch()

    def _loss_and_grad(self) -> None:
        # deferred validation: no host synchronisation here; loss() reports it
        self.dscene.set_raw(self.K, self.D, self.tau, self.centers, self.inv_cov, self.attr, deferred=True)
        self.grads.zero_()
        self.loss_acc.zero_()
        for ((w_img, w_alpha), cams, tis, tas, tapes, losses), lsum in zip(self.groups, self._lsum):
            render_views_into(self.ctx, self.dscene, cams, self.cfg, tapes)
            scalar_loss_views_into(self.ctx, tapes, tis, tas, w_img, w_alpha, losses)
            backward_views_into(self.ctx, tapes, GradFlags(), None, self.total)
            self.torch.sum(losses, dim=0, keepdim=True, out=lsum)
            self.loss_acc.add_(lsum)
        if self.reg is not None and self.rank == 0:  # once per iteration (added before the rank sum)
            for w, fn in ((self.edge_weight, self.reg.edge_reg), (self.laplacian_weight, self.reg.laplacian_reg)):
                if w > 0.0:
                    self.loss_acc += w * fn(self.centers, self.g_center.view(self.K, 3), w, accumulate=True)

    def step(self, group=None) -> None:
        """One fit_shape iteration: loss_and_grad, NCCL all-reduce, ADAM."""
        with self.torch.cuda.stream(self.stream):
            self._run_loss_and_grad()
            allreduce_gradients([self.grads, self.loss_acc], group)
            self.step_count += 1
            adam_step(self.ctx, self.params, self.grads, self.m, self.v, self.step_count, self.adam.lr,
                      self.adam.beta1, self.adam.beta2, self.adam.eps, loss=self.loss_acc, diverged=self._diverged)

    def loss(self) -> float:
        """Loss of the last loss_and_grad / step (synchronises). Raises ValidationError
        like the reference's render would: invalid parameters (deferred scene
        validation) or non-finite render outputs (blender.cpp:132-134)."""
        self.stream.synchronize()
        self.dscene.check()  # the deferred validation of the last upload
        for group in self.groups:
            for tape in group[4]:
                tape.check_finite()
        return float(self.loss_acc.item())

    @property
    def diverged(self) -> bool:
        """FitReport::diverged (fit.cpp:248): a step saw a non-finite loss; the
        parameters stay as they were before it (every later update is skipped)."""
        self.stream.synchronize()
        return bool(self._diverged.item())

    def scene(self) -> GaussianScene:
        return GaussianScene(self.centers.cpu().numpy().copy(), self.inv_cov.cpu().numpy().copy(),
                             self.attr.cpu().numpy().copy(), self.tau)


def make_fit_views(target: GaussianScene, n_views: int, size: int, cfg: SelectionConfig = SelectionConfig(),
                   ctx: Optional[Context] = None):
    """Target images of `target` from n orbit cameras (shapes.cpp:118-141),
    rendered with this library (the reference renders its targets the same way,
    tools/gvr_main.cpp:92-109)."""
    from .render import default_context, render
    from .synthetic import make_orbit_camera

    ctx = ctx or default_context()
    center = target.centers.mean(axis=0)
    views = []
    for v in range(n_views):
        cam = make_orbit_camera(2 * np.pi * v / n_views, 0.3, 4.0, center, size, size, 1.6 * size)
        buf = render(target, cam, cfg, weights=False, ctx=ctx)
        views.append((cam, buf.image, buf.alpha))
    return views
