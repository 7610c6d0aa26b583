"""Host-side mirror of the reference render API over the C ABI.

Reference entry points (namespace ``gvr``, /root/reference/proj):

* ``render(scene, camera, cfg, threads)``            blender.hpp:40-41
* ``render_with_tape(scene, camera, cfg, threads)``  grad.hpp:41-42
* ``backward(tape, d_image, d_alpha, flags)``        grad.hpp:53-54
* ``ScalarLoss::value(buf, d_image*, d_alpha*)``     grad.hpp:68, grad.cpp:201-216
* ``sample_attributes`` / ``resynthesize``           sampler.hpp:23-30, sampler.cpp:11-66
* ``transmittance_at`` / ``normalized_weights``      blender.hpp:29-36 (per pixel of a tape)
* ``shade_lambert``                                  blender.hpp:46-47, blender.cpp:146-172

Same argument meaning and error behaviour: invalid inputs raise
:class:`ValidationError` with the reference's message text. ``threads`` is
accepted for signature parity and ignored (the GPU grid replaces
``parallel_for_partitions``). Every call goes through ``libgvr_cuda.so``.

Buffers may be numpy arrays (host; copied over PCIe inside the call) or CUDA
tensors / any object exposing ``data_ptr()`` (device-resident; no copy).
"""
from __future__ import annotations

import contextlib
import ctypes
import threading
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .types import (
    Camera,
    GaussianScene,
    GradFlags,
    GradientBundle,
    RenderBuffers,
    SampledAttributes,
    ScalarLoss,
    SelectionConfig,
    ValidationError,
)


class GvrRuntimeError(RuntimeError):
    """Runtime / CUDA failure inside libgvr_cuda.so (status 2)."""


def _ptr(x) -> Optional[int]:
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays must be C-contiguous")
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    raise TypeError(f"unsupported buffer type {type(x)!r}")


def _cuda_tensors(bufs):
    out = []
    for b in bufs:
        if isinstance(b, (list, tuple)):
            out += _cuda_tensors(b)
        elif isinstance(b, dict):
            out += _cuda_tensors(list(b.values()))
        elif b is not None and getattr(b, "is_cuda", False):
            out.append(b)
    return out


@contextlib.contextmanager
def _stream_order(ctx: "Context", *bufs):
    """Stream ordering for CUDA tensor arguments: the context's stream waits for
    torch's current stream before the call (inputs written by torch are ready)
    and torch's current stream waits for the context's stream after it (outputs
    are ready for torch). Asynchronous (events); nothing to do when torch already
    runs on the context's stream (bench.py, Fitter) or no tensor is on the GPU."""
    if not _cuda_tensors(bufs):
        yield
        return
    import torch

    cur = torch.cuda.current_stream()
    ext = ctx.torch_stream()
    if cur.cuda_stream == ext.cuda_stream:
        yield
        return
    ext.wait_stream(cur)
    try:
        yield
    finally:
        cur.wait_stream(ext)


class Context:
    """One CUDA device + stream + scratch arenas (``gvr_context``)."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = ctypes.c_void_p()
        rc = self.lib.gvr_context_create(device, ctypes.byref(h))
        if rc != _lib.GVR_OK:
            raise GvrRuntimeError(f"gvr_context_create(device={device}) failed: no usable sm_100 CUDA device")
        self.handle = h
        self.device = device

    def check(self, rc: int) -> None:
        if rc == _lib.GVR_OK:
            return
        msg = self.lib.gvr_last_error(self.handle).decode()
        if rc == _lib.GVR_ERR_VALIDATION:
            raise ValidationError(msg)
        raise GvrRuntimeError(msg)

    def set_stream(self, stream_handle: Optional[int]) -> None:
        self.check(self.lib.gvr_context_set_stream(self.handle, stream_handle))

    def synchronize(self) -> None:
        self.check(self.lib.gvr_context_synchronize(self.handle))

    @property
    def launch_count(self) -> int:
        return int(self.lib.gvr_context_launch_count(self.handle))

    @property
    def library_call_count(self) -> int:
        return int(self.lib.gvr_context_library_call_count(self.handle))

    STAGES = ("project", "emit", "ranges", "select", "blend", "loss", "backward", "object_space")

    def enable_timing(self, on: bool = True) -> None:
        self.check(self.lib.gvr_context_enable_timing(self.handle, int(on)))

    def stage_times(self) -> dict:
        """{stage: (total_ms, launches)} accumulated since enable_timing()."""
        n = len(self.STAGES)
        ms = np.zeros(n)
        cnt = np.zeros(n, dtype=np.int64)
        self.check(self.lib.gvr_context_stage_times(self.handle, ms.ctypes.data, cnt.ctypes.data, n))
        return {s: (float(ms[i]), int(cnt[i])) for i, s in enumerate(self.STAGES)}

    def pipe_peak(self, kind: str = "fp32") -> float:
        """Measured FMA-chain FLOP/s of the FP32 or FP64 pipe."""
        out = ctypes.c_double()
        self.check(self.lib.gvr_measure_pipe_peak(self.handle, 0 if kind == "fp32" else 1, ctypes.byref(out)))
        return out.value

    def capture(self) -> "Graph":
        return Graph(self)

    def set_tile_capacity(self, cap: int) -> None:
        """Test hook: tile-list pool capacity in entries, 0 = automatic (tiles whose list does not fit stream every kernel)."""
        self.check(self.lib.gvr_context_set_tile_capacity(self.handle, int(cap)))

    def torch_stream(self):
        """The context's stream as a torch stream (cached)."""
        st = getattr(self, "_torch_stream", None)
        ptr = int(self.lib.gvr_context_stream(self.handle) or 0)
        if st is None or st.cuda_stream != ptr:
            import torch

            st = torch.cuda.ExternalStream(ptr, device=torch.device(f"cuda:{self.device}"))
            self._torch_stream = st
        return st

    def set_async(self, on: bool = True) -> None:
        """Host-buffer calls enqueue their copies and return (gvr_context_set_async):
        synchronize() before reading results; scene validation and the non-finite
        check are then read with DeviceScene.check() / Tape.check_finite()."""
        self.check(self.lib.gvr_context_set_async(self.handle, int(bool(on))))

    def set_list_smem(self, n: int) -> None:
        """Test hook: tile lists longer than n (<= 2048) are sorted in global memory."""
        self.check(self.lib.gvr_context_set_list_smem(self.handle, int(n)))

    def set_precise(self, on: bool = True) -> None:
        """Verification mode: FP64 exact traces and erfc in the blend (gradcheck)."""
        self.check(self.lib.gvr_context_set_precise(self.handle, int(bool(on))))

    def set_tile_profile(self, on: bool = True) -> None:
        """Profiling hook: record per-tile selection cycles on each tape (Tape.tile_cycles)."""
        self.check(self.lib.gvr_context_set_tile_profile(self.handle, int(bool(on))))

    def set_prefilter_guard(self, guard: float) -> None:
        self.check(self.lib.gvr_context_set_prefilter_guard(self.handle, float(guard)))

    def close(self) -> None:
        if self.handle:
            self.lib.gvr_context_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Graph:
    """A captured sequence of device-resident calls (``gvr_graph``), replayed
    with one launch. Usage::

        with ctx.capture() as g:        # after one uncaptured warm-up call
            render_into(...); scalar_loss_into(...); backward_into(...)
        g.launch()
    """

    def __init__(self, ctx: "Context"):
        self.ctx = ctx
        self.handle = None

    def __enter__(self):
        self.ctx.check(self.ctx.lib.gvr_graph_begin(self.ctx.handle))
        return self

    def __exit__(self, exc_type, exc, tb):
        h = ctypes.c_void_p()
        rc = self.ctx.lib.gvr_graph_end(self.ctx.handle, ctypes.byref(h))
        if exc_type is None:
            self.ctx.check(rc)
            self.handle = h
        return False

    def launch(self) -> None:
        self.ctx.check(self.ctx.lib.gvr_graph_launch(self.ctx.handle, self.handle))

    def __del__(self):
        try:
            if self.handle:
                self.ctx.lib.gvr_graph_destroy(self.handle)
        except Exception:
            pass


_default = threading.local()


def default_context(device: int = 0) -> Context:
    ctx = getattr(_default, "ctx", None)
    if ctx is None or ctx.device != device:
        ctx = Context(device)
        _default.ctx = ctx
    return ctx


class DeviceScene:
    """A validated, device-resident scene (``gvr_scene``).

    ``set`` uploads + validates once (GaussianScene::validate, types.cpp:31-42);
    renders then reuse it without re-validation."""

    def __init__(self, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        h = ctypes.c_void_p()
        self.ctx.check(self.ctx.lib.gvr_scene_create(self.ctx.handle, ctypes.byref(h)))
        self.handle = h
        self.K = 0
        self.D = 0
        self.tau = 1.0

    def set(self, scene: GaussianScene) -> "DeviceScene":
        return self.set_raw(scene.size, scene.attr_dim(), scene.tau, scene.centers, scene.inv_cov, scene.attr)

    def set_raw(self, K: int, D: int, tau: float, centers, inv_cov, attr, deferred: bool = False) -> "DeviceScene":
        """Upload from host or device arrays. ``deferred``: validate on the device
        without synchronising (capturable); :meth:`check` reports the result."""
        fn = self.ctx.lib.gvr_scene_set_deferred if deferred else self.ctx.lib.gvr_scene_set
        with _stream_order(self.ctx, centers, inv_cov, attr):
            self.ctx.check(
                fn(self.ctx.handle, self.handle, int(K), int(D), float(tau), _ptr(centers), _ptr(inv_cov),
                   _ptr(attr) if D > 0 else None)
            )
        self.K, self.D, self.tau = int(K), int(D), float(tau)
        return self

    def check(self) -> None:
        """Raise the validation error of the last deferred upload, if any (synchronises)."""
        self.ctx.check(self.ctx.lib.gvr_scene_check(self.ctx.handle, self.handle))

    def close(self) -> None:
        if self.handle:
            self.ctx.lib.gvr_scene_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Tape:
    """``gvr::Tape`` (grad.hpp:26-33): the device record of a forward render."""

    def __init__(self, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        h = ctypes.c_void_p()
        self.ctx.check(self.ctx.lib.gvr_tape_create(self.ctx.handle, ctypes.byref(h)))
        self.handle = h
        self.scene: Optional[DeviceScene] = None
        self.camera: Optional[Camera] = None
        self.cfg: Optional[SelectionConfig] = None
        self.host_scene: Optional[GaussianScene] = None

    def shape(self):
        h, w, kp, d = (ctypes.c_int32() for _ in range(4))
        self.ctx.check(self.ctx.lib.gvr_tape_shape(self.handle, ctypes.byref(h), ctypes.byref(w), ctypes.byref(kp),
                                                   ctypes.byref(d)))
        return h.value, w.value, kp.value, d.value

    def traced(self):
        """Per-pixel selected kernels (Tape::traced): idx, l, q, sigma as [H, W, K'] arrays."""
        h, w, kp, _ = self.shape()
        idx = np.empty((h, w, kp), dtype=np.int32)
        l, q, s = (np.empty((h, w, kp)) for _ in range(3))
        self.ctx.check(self.ctx.lib.gvr_tape_traced(self.ctx.handle, self.handle, _ptr(idx), _ptr(l), _ptr(q),
                                                    _ptr(s)))
        return idx, l, q, s

    def cam_scene(self):
        """Tape::cam_scene (grad.hpp:29): camera-space centers [K, 3] and inv_cov [K, 3, 3]."""
        k = self.scene.K
        c, s = np.empty((k, 3)), np.empty((k, 3, 3))
        self.ctx.check(self.ctx.lib.gvr_tape_cam_scene(self.ctx.handle, self.handle, _ptr(c), _ptr(s)))
        return c, s

    def dropped_behind_camera(self) -> int:
        """PixelKernelMap::dropped_behind_camera (tracer.hpp:39)."""
        out = ctypes.c_int32()
        self.ctx.check(self.ctx.lib.gvr_tape_dropped_behind_camera(self.ctx.handle, self.handle, ctypes.byref(out)))
        return int(out.value)

    def check_finite(self) -> None:
        """validate_finite (blender.cpp:132-134) of a render with device outputs:
        raises ValidationError("image contains non-finite values")."""
        self.ctx.check(self.ctx.lib.gvr_tape_check_finite(self.ctx.handle, self.handle))

    def list_stats(self) -> dict:
        """Tile-list layout of the taped render (gvr_tape_list_stats): listed entries, longest
        list, tiles that overflowed the pool (streamed), lists sorted in global memory, pool capacity."""
        out = np.zeros(7, dtype=np.int64)
        self.ctx.check(self.ctx.lib.gvr_tape_list_stats(self.ctx.handle, self.handle,
                                                        out.ctypes.data_as(ctypes.c_void_p)))
        return {"entries": int(out[0]), "max_list": int(out[1]), "overflow_tiles": int(out[2]),
                "global_sorted_tiles": int(out[3]), "pool_capacity": int(out[4]),
                "mask_tiles": int(out[5]), "mask_capacity": int(out[6])}

    def tile_cycles(self) -> np.ndarray:
        """[tiles_y, tiles_x] SM cycles of each 8x8 tile's selection CTA (needs Context.set_tile_profile)."""
        h, w, _, _ = self.shape()
        ty, tx = (h + 7) // 8, (w + 7) // 8
        out = np.zeros((ty, tx), dtype=np.int64)
        self.ctx.check(self.ctx.lib.gvr_tape_tile_cycles(self.ctx.handle, self.handle,
                                                         out.ctypes.data_as(ctypes.c_void_p), out.size))
        return out

    def close(self) -> None:
        if self.handle:
            self.ctx.lib.gvr_tape_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class ForwardResult:
    """``gvr::ForwardResult`` (grad.hpp:35-38)."""

    buffers: RenderBuffers
    tape: Tape


def _camera_c(camera: Camera) -> _lib.GvrCamera:
    c = _lib.GvrCamera()
    c.rotation[:] = [float(v) for v in np.asarray(camera.rotation, dtype=np.float64).reshape(9)]
    c.translation[:] = [float(v) for v in np.asarray(camera.translation, dtype=np.float64).reshape(3)]
    c.focal, c.ox, c.oy = float(camera.focal), float(camera.ox), float(camera.oy)
    c.height, c.width = int(camera.height), int(camera.width)
    return c


def _selection_c(cfg: SelectionConfig) -> _lib.GvrSelection:
    return _lib.GvrSelection(float(cfg.eta), int(cfg.k_prime), int(bool(cfg.coarse_enabled)),
                             int(cfg.coarse_downsample))


def _as_device_scene(scene, ctx: Context) -> DeviceScene:
    if isinstance(scene, DeviceScene):
        return scene
    return DeviceScene(ctx).set(scene)


def render_into(ctx: Context, dscene: DeviceScene, camera: Camera, cfg: SelectionConfig, tape: Tape,
                image=None, alpha=None, depth=None, topk_idx=None, topk_w=None, shard=(0, 1)) -> None:
    """Low-level forward: outputs written into caller buffers (host or device, any may be None).
    ``shard=(r, n)`` renders only tiles with index % n == r (C4 tile sharding)."""
    out = _lib.GvrRenderOutputs(_ptr(image), _ptr(alpha), _ptr(depth), _ptr(topk_idx), _ptr(topk_w))
    cam_c, sel_c = _camera_c(camera), _selection_c(cfg)
    with _stream_order(ctx, image, alpha, depth, topk_idx, topk_w):
        ctx.check(ctx.lib.gvr_render_shard(ctx.handle, dscene.handle, ctypes.byref(cam_c), ctypes.byref(sel_c),
                                           tape.handle, ctypes.byref(out), int(shard[0]), int(shard[1])))
    tape.scene, tape.camera, tape.cfg = dscene, camera, cfg


def render_with_tape(scene, camera: Camera, cfg: SelectionConfig = SelectionConfig(), threads: int = 0, *,
                     weights: bool = True, ctx: Optional[Context] = None, shard=(0, 1)) -> ForwardResult:
    """``gvr::render_with_tape`` (grad.cpp:38-47): render and keep the tape for backward.
    ``shard=(r, n)``: only tiles with index % n == r (C4 tile sharding; the rest stay empty)."""
    del threads
    ctx = ctx or default_context()
    dscene = _as_device_scene(scene, ctx)
    h, w = int(camera.height), int(camera.width)
    dc = max(dscene.D, 1)
    kp = int(cfg.k_prime)
    image = np.empty((h, w, dc))
    alpha = np.empty((h, w, 1))
    depth = np.empty((h, w, 1))
    tidx = np.empty((h, w, kp), dtype=np.int32) if weights else None
    tw = np.empty((h, w, kp)) if weights else None
    tape = Tape(ctx)
    render_into(ctx, dscene, camera, cfg, tape, image, alpha, depth, tidx, tw, shard=shard)
    tape.host_scene = scene if isinstance(scene, GaussianScene) else None
    return ForwardResult(RenderBuffers(image, alpha, depth, tidx, tw), tape)


def render(scene, camera: Camera, cfg: SelectionConfig = SelectionConfig(), threads: int = 0, *,
           weights: bool = True, ctx: Optional[Context] = None) -> RenderBuffers:
    """``gvr::render`` (blender.cpp:141-144)."""
    return render_with_tape(scene, camera, cfg, threads, weights=weights, ctx=ctx).buffers


def scalar_loss_into(tape: Tape, target_image, target_alpha, w_image: float = 1.0, w_alpha: float = 1.0,
                     loss_out=None, d_image_out=None, d_alpha_out=None) -> None:
    """Low-level ``gvr_scalar_loss``: targets / outputs host or device; the
    upstream gradient is also kept in the tape for ``backward_into(tape, None, None)``."""
    ctx = tape.ctx
    with _stream_order(ctx, target_image, target_alpha, loss_out, d_image_out, d_alpha_out):
        ctx.check(ctx.lib.gvr_scalar_loss(ctx.handle, tape.handle, _ptr(target_image), _ptr(target_alpha),
                                          float(w_image), float(w_alpha), _ptr(loss_out), _ptr(d_image_out),
                                          _ptr(d_alpha_out)))


def scalar_loss(tape: Tape, loss: ScalarLoss, *, want_grads: bool = True):
    """``ScalarLoss::value`` evaluated on the device against the taped render.

    Returns ``(loss, d_image, d_alpha)`` (host arrays when ``want_grads``); the
    upstream gradient also stays in the tape for ``backward(tape, None, None)``."""
    ctx = tape.ctx
    h, w, kp, d = tape.shape()
    out = np.zeros(1)
    di = np.empty((h, w, max(d, 1))) if want_grads else None
    da = np.empty((h, w, 1)) if want_grads else None
    t_img = np.ascontiguousarray(loss.target_image, dtype=np.float64)  # kept alive across the call
    t_alpha = np.ascontiguousarray(loss.target_alpha, dtype=np.float64)
    ctx.check(ctx.lib.gvr_scalar_loss(ctx.handle, tape.handle, _ptr(t_img), _ptr(t_alpha), float(loss.w_image),
                                      float(loss.w_alpha), _ptr(out), _ptr(di), _ptr(da)))
    return float(out[0]), di, da


def backward_into(tape: Tape, d_image, d_alpha, flags: GradFlags = GradFlags(), d_center=None, d_inv_cov=None,
                  d_attr=None, d_rotation=None, d_translation=None, accumulate: bool = False) -> None:
    """Low-level backward: gradients written into caller buffers (host or device, any may
    be None); ``accumulate=True`` adds into device buffers (per-view sums of a fit)."""
    ctx = tape.ctx
    f = _lib.GvrGradFlags(int(bool(flags.through_transmittance)), int(bool(flags.through_density)))
    g = _lib.GvrGradients(_ptr(d_center), _ptr(d_inv_cov), _ptr(d_attr), _ptr(d_rotation), _ptr(d_translation))
    fn = ctx.lib.gvr_backward_accumulate if accumulate else ctx.lib.gvr_backward
    with _stream_order(ctx, d_image, d_alpha, d_center, d_inv_cov, d_attr, d_rotation, d_translation):
        ctx.check(fn(ctx.handle, tape.handle, _ptr(d_image), _ptr(d_alpha), ctypes.byref(f), ctypes.byref(g)))


def backward_packed_into(tape: Tape, d_image, d_alpha, flags: GradFlags, packed, d_rt) -> None:
    """``gvr_backward_packed``: per-kernel rows [d_center | d_inv_cov upper | d_attr]
    (device [K, 9 + D]) and d_rt = [d_rotation | d_translation] (device [12])."""
    ctx = tape.ctx
    f = _lib.GvrGradFlags(int(bool(flags.through_transmittance)), int(bool(flags.through_density)))
    with _stream_order(ctx, d_image, d_alpha, packed, d_rt):
        ctx.check(ctx.lib.gvr_backward_packed(ctx.handle, tape.handle, _ptr(d_image), _ptr(d_alpha),
                                              ctypes.byref(f), _ptr(packed), _ptr(d_rt)))


def unpack_gradients(packed, d_rt, D: int):
    """Split packed rows back into (d_center [K,3], d_inv_cov [K,3,3] symmetric,
    d_attr [K,D], d_rotation [3,3], d_translation [3]) (torch or numpy)."""
    c = packed[:, 0:3]
    u = packed[:, 3:9]
    rows = [[u[:, 0], u[:, 1], u[:, 2]], [u[:, 1], u[:, 3], u[:, 4]], [u[:, 2], u[:, 4], u[:, 5]]]
    try:
        import torch

        if isinstance(packed, torch.Tensor):
            inv = torch.stack([torch.stack(r, dim=1) for r in rows], dim=1)
            return c, inv, packed[:, 9:9 + D], d_rt[:9].reshape(3, 3), d_rt[9:12]
    except ImportError:
        pass
    inv = np.stack([np.stack(r, axis=1) for r in rows], axis=1)
    return c, inv, packed[:, 9:9 + D], d_rt[:9].reshape(3, 3), d_rt[9:12]


def adam_step(ctx: Context, params, grads, m, v, step: int, lr: float, beta1: float = 0.9, beta2: float = 0.999,
              eps: float = 1e-8, loss=None, diverged=None) -> None:
    """``AdamState::update`` (fit.cpp:20-42) on device tensors (FP64, same length).
    With ``loss`` (device FP64 scalar) and ``diverged`` (device int32 flag), the update
    follows fit_shape's divergence rule (fit.cpp:246-250): a non-finite loss skips it
    and latches the flag."""
    if loss is None:
        ctx.check(ctx.lib.gvr_adam_step(ctx.handle, _ptr(params), _ptr(grads), _ptr(m), _ptr(v), int(params.numel()),
                                        int(step), float(lr), float(beta1), float(beta2), float(eps)))
        return
    ctx.check(ctx.lib.gvr_adam_step_guarded(ctx.handle, _ptr(params), _ptr(grads), _ptr(m), _ptr(v),
                                            int(params.numel()), int(step), float(lr), float(beta1), float(beta2),
                                            float(eps), _ptr(loss), _ptr(diverged)))


def backward(tape, d_image, d_alpha, flags: GradFlags = GradFlags()) -> GradientBundle:
    """``gvr::backward`` (grad.cpp:49-199). ``tape`` may be a Tape or a ForwardResult.

    ``d_image`` must be [H, W, D] and ``d_alpha`` [H, W, 1] (reference shape rule,
    grad.cpp:58-63); pass both as None to use the upstream from :func:`scalar_loss`."""
    if isinstance(tape, ForwardResult):
        tape = tape.tape
    h, w, kp, d = tape.shape()
    if d_image is not None or d_alpha is not None:
        d_image = np.ascontiguousarray(d_image, dtype=np.float64) if isinstance(d_image, np.ndarray) else d_image
        d_alpha = np.ascontiguousarray(d_alpha, dtype=np.float64) if isinstance(d_alpha, np.ndarray) else d_alpha
        if isinstance(d_image, np.ndarray) and (d_image.ndim != 3 or d_image.shape != (h, w, d)):
            raise ValidationError("backward: d_image shape does not match the forward render")
        if isinstance(d_alpha, np.ndarray) and d_alpha.reshape(-1).shape[0] != h * w or (
            isinstance(d_alpha, np.ndarray) and d_alpha.ndim == 3 and d_alpha.shape[2] != 1
        ):
            raise ValidationError("backward: d_alpha shape does not match the forward render")
    k = tape.scene.K
    gb = GradientBundle(np.empty((k, 3)), np.empty((k, 3, 3)), np.empty((k, d)), np.empty((3, 3)), np.empty(3))
    backward_into(tape, d_image, d_alpha, flags, gb.d_center, gb.d_inv_cov, gb.d_attr if d > 0 else None,
                  gb.d_rotation, gb.d_translation)
    return gb


# ---------------------------------------------------------------- sampler + helpers


def _image3(x, what: str) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float64)
    if a.ndim == 2:
        a = a[..., None]
    if a.ndim != 3:
        raise ValidationError(f"{what} must be an H x W x C image")
    return a


def sample_attributes(observed, scene, camera: Camera, cfg: SelectionConfig = SelectionConfig(),
                      normalized: bool = False, threads: int = 0, *, ctx: Optional[Context] = None,
                      tape: Optional[Tape] = None) -> SampledAttributes:
    """``gvr::sample_attributes`` (sampler.cpp:11-51): weighted-mean inverse
    reconstruction alpha_k = sum_p W_pk phi_p / sum_p W_pk with the rendering
    weights. Pass ``tape`` (a render of the same scene/camera/cfg) to reuse it."""
    del threads
    ctx = ctx or (tape.ctx if tape is not None else default_context())
    obs = _image3(observed, "observed image")
    h, w, ch = obs.shape
    k = scene.K if isinstance(scene, DeviceScene) else scene.size
    attrs, support, masked = np.empty((k, ch)), np.empty(k), np.empty(k, dtype=np.uint8)
    if tape is not None:
        th, tw, _, _ = tape.shape()
        if (h, w) != (th, tw):
            raise ValidationError("observed image size does not match the camera")
        ctx.check(ctx.lib.gvr_tape_sample_attributes(ctx.handle, tape.handle, _ptr(obs), ch, int(bool(normalized)),
                                                     _ptr(attrs), _ptr(support), _ptr(masked)))
    else:
        dscene = _as_device_scene(scene, ctx)
        cam_c, sel_c = _camera_c(camera), _selection_c(cfg)
        ctx.check(ctx.lib.gvr_sample_attributes(ctx.handle, dscene.handle, ctypes.byref(cam_c), ctypes.byref(sel_c),
                                                _ptr(obs), h, w, ch, int(bool(normalized)), _ptr(attrs),
                                                _ptr(support), _ptr(masked)))
    return SampledAttributes(attrs, support, masked.astype(bool))


def resynthesize_scene(attrs: SampledAttributes, scene, ctx: Optional[Context] = None) -> DeviceScene:
    """Device scene with the sampled attributes (masked -> 0), sampler.cpp:53-63."""
    ctx = ctx or default_context()
    src = _as_device_scene(scene, ctx)
    a = np.ascontiguousarray(attrs.attrs, dtype=np.float64)
    if a.ndim == 1:
        a = a[:, None]
    m = np.ascontiguousarray(attrs.masked, dtype=np.uint8)
    n = a.shape[0]
    if m.shape[0] != n:
        raise ValidationError("sampled attribute count does not match the scene")
    dst = DeviceScene(ctx)
    ctx.check(ctx.lib.gvr_scene_resynthesize(ctx.handle, dst.handle, src.handle, n, a.shape[1], _ptr(a), _ptr(m)))
    dst.K, dst.D, dst.tau = src.K, a.shape[1], src.tau
    return dst


def resynthesize(attrs: SampledAttributes, scene, camera: Camera, cfg: SelectionConfig = SelectionConfig(),
                 threads: int = 0, *, ctx: Optional[Context] = None) -> RenderBuffers:
    """``gvr::resynthesize`` (sampler.cpp:53-66): render with the sampled attributes."""
    ctx = ctx or default_context()
    return render(resynthesize_scene(attrs, scene, ctx), camera, cfg, threads, ctx=ctx)


def transmittance_at(tape, t) -> np.ndarray:
    """``gvr::transmittance_at`` (blender.cpp:19-25) evaluated for every pixel of
    a taped render over that pixel's selected kernels, at depth ``t[H, W]``."""
    if isinstance(tape, ForwardResult):
        tape = tape.tape
    h, w, _, _ = tape.shape()
    tt = np.ascontiguousarray(t, dtype=np.float64).reshape(h, w)
    out = np.empty((h, w))
    tape.ctx.check(tape.ctx.lib.gvr_tape_transmittance(tape.ctx.handle, tape.handle, _ptr(tt), _ptr(out)))
    return out


def normalized_weights(tape, eps: float = 1e-8) -> np.ndarray:
    """``gvr::normalized_weights`` (blender.cpp:55-62) for every pixel: [H, W, K'],
    ascending (l, idx) like ``topk_idx``, 0 padded."""
    if isinstance(tape, ForwardResult):
        tape = tape.tape
    h, w, kp, _ = tape.shape()
    out = np.empty((h, w, kp))
    tape.ctx.check(tape.ctx.lib.gvr_tape_normalized_weights(tape.ctx.handle, tape.handle, float(eps), _ptr(out)))
    return out


def shade_lambert(normals, alpha, depth, camera: Camera, light_pos, light_color, *,
                  ctx: Optional[Context] = None) -> np.ndarray:
    """``gvr::shade_lambert`` (blender.cpp:146-172), same validation messages."""
    ctx = ctx or default_context()
    n = _image3(normals, "normals")
    al = _image3(alpha, "alpha")
    de = _image3(depth, "depth")
    if n.shape[2] != 3:
        raise ValidationError("shade_lambert expects a 3-channel normal image")
    if n.shape[:2] != al.shape[:2] or n.shape[:2] != de.shape[:2]:
        raise ValidationError("shade_lambert: buffer sizes do not match")
    h, w = n.shape[:2]
    cam = Camera(camera.rotation, camera.translation, camera.focal, camera.ox, camera.oy, h, w)
    out = np.empty((h, w, 3))
    lp = np.ascontiguousarray(light_pos, dtype=np.float64).reshape(3)
    lc = np.ascontiguousarray(light_color, dtype=np.float64).reshape(3)
    cam_c = _camera_c(cam)
    al1 = np.ascontiguousarray(al[..., :1])  # kept alive across the call
    de1 = np.ascontiguousarray(de[..., :1])
    ctx.check(ctx.lib.gvr_shade_lambert(ctx.handle, ctypes.byref(cam_c), _ptr(n), _ptr(al1), _ptr(de1), _ptr(lp),
                                        _ptr(lc), _ptr(out)))
    return out


# ---------------------------------------------------------------- multi-view batches (C3 / C5)


def _ptr_array(objs):
    arr = (ctypes.c_void_p * max(len(objs), 1))()
    for i, o in enumerate(objs):
        arr[i] = _ptr(o) if not isinstance(o, Tape) else o.handle.value
    return arr


def render_views_into(ctx: Context, dscene: DeviceScene, cameras, cfg: SelectionConfig, tapes, images=None,
                      alphas=None, depths=None, topk_idx=None, topk_w=None) -> None:
    """``gvr_render_views``: one render per camera, the views running concurrently
    on the context's worker streams. Output lists (host or device buffers, any
    may be None or contain None) are indexed like ``cameras``."""
    n = len(cameras)
    if len(tapes) != n:
        raise ValueError("one tape per view")
    cams = (_lib.GvrCamera * max(n, 1))(*[_camera_c(c) for c in cameras])
    pick = lambda lst, v: None if lst is None else lst[v]  # noqa: E731
    outs = (_lib.GvrRenderOutputs * max(n, 1))(*[
        _lib.GvrRenderOutputs(_ptr(pick(images, v)), _ptr(pick(alphas, v)), _ptr(pick(depths, v)),
                              _ptr(pick(topk_idx, v)), _ptr(pick(topk_w, v))) for v in range(n)])
    th = _ptr_array(tapes)
    sel_c = _selection_c(cfg)
    with _stream_order(ctx, images, alphas, depths, topk_idx, topk_w):
        ctx.check(ctx.lib.gvr_render_views(ctx.handle, dscene.handle, n, cams, ctypes.byref(sel_c), th, outs))
    for v, t in enumerate(tapes):
        t.scene, t.camera, t.cfg = dscene, cameras[v], cfg


def scalar_loss_views_into(ctx: Context, tapes, target_images, target_alphas, w_image: float = 1.0,
                           w_alpha: float = 1.0, losses=None) -> None:
    """``gvr_scalar_loss_views``: per-view ScalarLoss; ``losses`` [V] host or device (nullable)."""
    n = len(tapes)
    with _stream_order(ctx, target_images, target_alphas, losses):
        ctx.check(ctx.lib.gvr_scalar_loss_views(ctx.handle, n, _ptr_array(tapes), _ptr_array(target_images),
                                                _ptr_array(target_alphas), float(w_image), float(w_alpha),
                                                _ptr(losses)))


def backward_views_into(ctx: Context, tapes, flags: GradFlags = GradFlags(), outs=None, total=None) -> None:
    """``gvr_backward_views``: per-view gradients into ``outs`` (list of dicts of device
    tensors with keys d_center, d_inv_cov, d_attr, d_rotation, d_translation; entries
    may be missing) and / or their sum added into ``total`` (same dict form)."""
    n = len(tapes)

    def bundle(g):
        g = g or {}
        return _lib.GvrGradients(*[_ptr(g.get(k)) for k in ("d_center", "d_inv_cov", "d_attr", "d_rotation",
                                                               "d_translation")])

    f = _lib.GvrGradFlags(int(bool(flags.through_transmittance)), int(bool(flags.through_density)))
    o = (_lib.GvrGradients * max(n, 1))(*[bundle(outs[v]) for v in range(n)]) if outs is not None else None
    t = bundle(total) if total is not None else None
    with _stream_order(ctx, outs, total):
        ctx.check(ctx.lib.gvr_backward_views(ctx.handle, n, _ptr_array(tapes), ctypes.byref(f), o,
                                             ctypes.byref(t) if t is not None else None))
