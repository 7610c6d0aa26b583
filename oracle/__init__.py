"""CPU oracles for the render path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker / the timed CPU
reference. The product (``paper_2205_15401_b200``) never imports it.

Two oracles:

* ``port``  — ``oracle/gvr_oracle.c``, a plain-C FP64 restatement of the
  reference (each function cites proj/src file:line). Built by
  ``make -C oracle port`` (anywhere gcc exists, so also on the GPU box).
* ``ref``   — the reference itself, compiled unmodified from
  ``/root/reference/proj/src`` against ``oracle/shim`` (``make -C oracle ref``,
  dev container only; the prebuilt ``oracle/_ref/libgvr_ref.so`` travels).
  Pinned by the reference's own doctest suites (``make -C oracle check``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libgvr_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgvr_ref.so")

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class _CamC(ctypes.Structure):
    _fields_ = [
        ("rotation", ctypes.c_double * 9),
        ("translation", ctypes.c_double * 3),
        ("focal", ctypes.c_double),
        ("ox", ctypes.c_double),
        ("oy", ctypes.c_double),
        ("height", ctypes.c_int),
        ("width", ctypes.c_int),
    ]


class _SelC(ctypes.Structure):
    _fields_ = [
        ("eta", ctypes.c_double),
        ("k_prime", ctypes.c_int),
        ("coarse_enabled", ctypes.c_int),
        ("coarse_downsample", ctypes.c_int),
    ]


def _ptr(a: Optional[np.ndarray], kind=_dp):
    if a is None:
        return ctypes.cast(None, kind)
    return a.ctypes.data_as(kind)


def build_port() -> str:
    if not os.path.exists(PORT_SO) or os.path.getmtime(PORT_SO) < os.path.getmtime(os.path.join(HERE, "gvr_oracle.c")):
        subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    return PORT_SO


_port = None
_ref = None


def port_lib():
    global _port
    if _port is None:
        _port = ctypes.CDLL(build_port())
        _port.gvro_last_error.restype = ctypes.c_char_p
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref, needs /root/reference)")
        _ref = ctypes.CDLL(REF_SO)
        _ref.gvr_ref_last_error.restype = ctypes.c_char_p
    return _ref


def _scene_arrays(scene):
    c = np.ascontiguousarray(scene.centers, dtype=np.float64)
    s = np.ascontiguousarray(scene.inv_cov, dtype=np.float64)
    a = np.ascontiguousarray(scene.attr, dtype=np.float64)
    return c, s, a


def _cam_c(cam) -> _CamC:
    c = _CamC()
    c.rotation[:] = [float(x) for x in np.asarray(cam.rotation).reshape(9)]
    c.translation[:] = [float(x) for x in np.asarray(cam.translation).reshape(3)]
    c.focal, c.ox, c.oy = float(cam.focal), float(cam.ox), float(cam.oy)
    c.height, c.width = int(cam.height), int(cam.width)
    return c


def _sel_c(cfg) -> _SelC:
    return _SelC(float(cfg.eta), int(cfg.k_prime), int(bool(cfg.coarse_enabled)), int(cfg.coarse_downsample))


def _out_buffers(cam, d, kp):
    h, w = int(cam.height), int(cam.width)
    dc = max(d, 1)
    return dict(
        image=np.zeros((h, w, dc)),
        alpha=np.zeros((h, w, 1)),
        depth=np.zeros((h, w, 1)),
        topk_idx=np.full((h, w, kp), -1, dtype=np.int32),
        topk_w=np.zeros((h, w, kp)),
        topk_l=np.zeros((h, w, kp)),
        topk_q=np.zeros((h, w, kp)),
        topk_sigma=np.zeros((h, w, kp)),
    )


# ---------------------------------------------------------------- the C port


def port_render(scene, cam, cfg, threads: int = 0) -> dict:
    lib = port_lib()
    c, s, a = _scene_arrays(scene)
    out = _out_buffers(cam, scene.attr_dim(), int(cfg.k_prime))
    camc, selc = _cam_c(cam), _sel_c(cfg)
    rc = lib.gvro_render(
        scene.size, scene.attr_dim(), ctypes.c_double(scene.tau), _ptr(c), _ptr(s), _ptr(a),
        ctypes.byref(camc), ctypes.byref(selc), threads,
        _ptr(out["image"]), _ptr(out["alpha"]), _ptr(out["depth"]), _ptr(out["topk_idx"], _ip),
        _ptr(out["topk_w"]), _ptr(out["topk_l"]), _ptr(out["topk_q"]), _ptr(out["topk_sigma"]),
    )
    if rc:
        raise OracleError(rc, lib.gvro_last_error().decode())
    return out


def port_backward(scene, cam, cfg, d_image, d_alpha, through_transmittance=True, through_density=True,
                  threads: int = 0) -> dict:
    lib = port_lib()
    c, s, a = _scene_arrays(scene)
    k, d = scene.size, scene.attr_dim()
    g = dict(d_center=np.zeros((k, 3)), d_inv_cov=np.zeros((k, 3, 3)), d_attr=np.zeros((k, d)),
             d_rotation=np.zeros((3, 3)), d_translation=np.zeros(3))
    di = np.ascontiguousarray(d_image, dtype=np.float64)
    da = np.ascontiguousarray(d_alpha, dtype=np.float64)
    camc, selc = _cam_c(cam), _sel_c(cfg)
    rc = lib.gvro_backward(
        k, d, ctypes.c_double(scene.tau), _ptr(c), _ptr(s), _ptr(a), ctypes.byref(camc), ctypes.byref(selc),
        threads, _ptr(di), _ptr(da), int(through_transmittance), int(through_density),
        _ptr(g["d_center"]), _ptr(g["d_inv_cov"]), _ptr(g["d_attr"]), _ptr(g["d_rotation"]), _ptr(g["d_translation"]),
    )
    if rc:
        raise OracleError(rc, lib.gvro_last_error().decode())
    return g


def port_fwd_bwd_step(scene, cam, cfg, target_image, target_alpha, threads: int = 0):
    """C-port fwd+bwd step (render_with_tape -> ScalarLoss -> backward); returns (loss, d_center)."""
    lib = port_lib()
    c, s, a = _scene_arrays(scene)
    ti = np.ascontiguousarray(target_image, dtype=np.float64)
    ta = np.ascontiguousarray(target_alpha, dtype=np.float64)
    loss = ctypes.c_double(0.0)
    dc = np.zeros((scene.size, 3))
    camc, selc = _cam_c(cam), _sel_c(cfg)
    rc = lib.gvro_fwd_bwd_step(scene.size, scene.attr_dim(), ctypes.c_double(scene.tau), _ptr(c), _ptr(s), _ptr(a),
                               ctypes.byref(camc), ctypes.byref(selc), threads, _ptr(ti), _ptr(ta), ctypes.byref(loss),
                               _ptr(dc), ctypes.cast(None, _dp))
    if rc:
        raise OracleError(rc, lib.gvro_last_error().decode())
    return loss.value, dc


def port_coarse_boxes(scene, cam, cfg):
    lib = port_lib()
    c, s, a = _scene_arrays(scene)
    box = np.full((scene.size, 4), -1, dtype=np.int32)
    dropped = ctypes.c_int(0)
    camc, selc = _cam_c(cam), _sel_c(cfg)
    rc = lib.gvro_coarse_boxes(scene.size, scene.attr_dim(), ctypes.c_double(scene.tau), _ptr(c), _ptr(s), _ptr(a),
                               ctypes.byref(camc), ctypes.byref(selc), _ptr(box, _ip), ctypes.byref(dropped))
    if rc:
        raise OracleError(rc, lib.gvro_last_error().decode())
    return box, dropped.value


def _u8p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_ubyte))


def port_sample_attributes(scene, cam, cfg, observed, normalized=False, threads: int = 0):
    """C-port ``sample_attributes`` (sampler.cpp:11-51): (attrs [K,C], support [K], masked [K] bool)."""
    lib = port_lib()
    c, s, a = _scene_arrays(scene)
    obs = np.ascontiguousarray(observed, dtype=np.float64)
    ch = obs.shape[2] if obs.ndim == 3 else 1
    k = scene.size
    attrs, support, masked = np.zeros((k, ch)), np.zeros(k), np.zeros(k, dtype=np.uint8)
    camc, selc = _cam_c(cam), _sel_c(cfg)
    rc = lib.gvro_sample_attributes(k, scene.attr_dim(), ctypes.c_double(scene.tau), _ptr(c), _ptr(s), _ptr(a),
                                    ctypes.byref(camc), ctypes.byref(selc), threads, _ptr(obs), int(obs.shape[0]),
                                    int(obs.shape[1]), ch, int(bool(normalized)), _ptr(attrs), _ptr(support),
                                    _u8p(masked))
    if rc:
        raise OracleError(rc, lib.gvro_last_error().decode())
    return attrs, support, masked.astype(bool)


def port_pixel_helpers(scene, cam, cfg, t, eps=1e-8, threads: int = 0):
    """C-port per-pixel ``transmittance_at`` at depth t[p] and ``normalized_weights`` (blender.cpp:19-25, 55-62)."""
    lib = port_lib()
    c, s, a = _scene_arrays(scene)
    h, w, kp = int(cam.height), int(cam.width), int(cfg.k_prime)
    tt = np.ascontiguousarray(t, dtype=np.float64).reshape(h, w)
    trans, nw = np.zeros((h, w)), np.zeros((h, w, kp))
    camc, selc = _cam_c(cam), _sel_c(cfg)
    rc = lib.gvro_pixel_helpers(scene.size, scene.attr_dim(), ctypes.c_double(scene.tau), _ptr(c), _ptr(s), _ptr(a),
                                ctypes.byref(camc), ctypes.byref(selc), threads, _ptr(tt), _ptr(trans),
                                ctypes.c_double(eps), _ptr(nw))
    if rc:
        raise OracleError(rc, lib.gvro_last_error().decode())
    return trans, nw


def port_shade_lambert(cam, normals, alpha, depth, light_pos, light_color):
    """C-port ``shade_lambert`` (blender.cpp:146-172)."""
    lib = port_lib()
    h, w = int(cam.height), int(cam.width)
    n = np.ascontiguousarray(normals, dtype=np.float64)
    al = np.ascontiguousarray(alpha, dtype=np.float64)
    de = np.ascontiguousarray(depth, dtype=np.float64)
    lp = np.ascontiguousarray(light_pos, dtype=np.float64)
    lc = np.ascontiguousarray(light_color, dtype=np.float64)
    out = np.zeros((h, w, 3))
    camc = _cam_c(cam)
    lib.gvro_shade_lambert(ctypes.byref(camc), _ptr(n), _ptr(al), _ptr(de), _ptr(lp), _ptr(lc), _ptr(out))
    return out


# ---------------------------------------------------------------- the reference build


def _cam17(cam) -> np.ndarray:
    return np.concatenate([np.asarray(cam.rotation, dtype=np.float64).reshape(9),
                           np.asarray(cam.translation, dtype=np.float64).reshape(3),
                           [cam.focal, cam.ox, cam.oy, cam.height, cam.width]]).astype(np.float64)


def _ref_call(name, *args):
    lib = ref_lib()
    rc = getattr(lib, name)(*args)
    if rc:
        raise OracleError(rc, lib.gvr_ref_last_error().decode())


def ref_render(scene, cam, cfg, threads: int = 0) -> dict:
    c, s, a = _scene_arrays(scene)
    out = _out_buffers(cam, scene.attr_dim(), int(cfg.k_prime))
    c17 = _cam17(cam)
    _ref_call("gvr_ref_render", scene.size, scene.attr_dim(), ctypes.c_double(scene.tau), _ptr(c), _ptr(s), _ptr(a),
              _ptr(c17), ctypes.c_double(cfg.eta), int(cfg.k_prime), int(bool(cfg.coarse_enabled)),
              int(cfg.coarse_downsample), threads,
              _ptr(out["image"]), _ptr(out["alpha"]), _ptr(out["depth"]), _ptr(out["topk_idx"], _ip),
              _ptr(out["topk_w"]), _ptr(out["topk_l"]), _ptr(out["topk_q"]), _ptr(out["topk_sigma"]))
    return out


def ref_backward(scene, cam, cfg, d_image, d_alpha, through_transmittance=True, through_density=True,
                 threads: int = 0) -> dict:
    c, s, a = _scene_arrays(scene)
    k, d = scene.size, scene.attr_dim()
    g = dict(d_center=np.zeros((k, 3)), d_inv_cov=np.zeros((k, 3, 3)), d_attr=np.zeros((k, d)),
             d_rotation=np.zeros((3, 3)), d_translation=np.zeros(3))
    di = np.ascontiguousarray(d_image, dtype=np.float64)
    da = np.ascontiguousarray(d_alpha, dtype=np.float64)
    c17 = _cam17(cam)
    _ref_call("gvr_ref_backward", k, d, ctypes.c_double(scene.tau), _ptr(c), _ptr(s), _ptr(a), _ptr(c17),
              ctypes.c_double(cfg.eta), int(cfg.k_prime), int(bool(cfg.coarse_enabled)), int(cfg.coarse_downsample),
              threads, _ptr(di), _ptr(da), int(through_transmittance), int(through_density),
              _ptr(g["d_center"]), _ptr(g["d_inv_cov"]), _ptr(g["d_attr"]), _ptr(g["d_rotation"]),
              _ptr(g["d_translation"]))
    return g


def ref_fwd_bwd_step(scene, cam, cfg, target_image, target_alpha, threads: int = 0):
    """One reference fwd+bwd step (render_with_tape -> ScalarLoss -> backward)."""
    c, s, a = _scene_arrays(scene)
    ti = np.ascontiguousarray(target_image, dtype=np.float64)
    ta = np.ascontiguousarray(target_alpha, dtype=np.float64)
    loss = ctypes.c_double(0.0)
    dc = np.zeros((scene.size, 3))
    c17 = _cam17(cam)
    _ref_call("gvr_ref_fwd_bwd_step", scene.size, scene.attr_dim(), ctypes.c_double(scene.tau), _ptr(c), _ptr(s),
              _ptr(a), _ptr(c17), ctypes.c_double(cfg.eta), int(cfg.k_prime), int(bool(cfg.coarse_enabled)),
              int(cfg.coarse_downsample), threads, _ptr(ti), _ptr(ta), ctypes.byref(loss), _ptr(dc),
              ctypes.cast(None, _dp))
    return loss.value, dc


def ref_coarse_boxes(scene, cam, cfg):
    c, s, a = _scene_arrays(scene)
    box = np.full((scene.size, 4), -1, dtype=np.int32)
    dropped = ctypes.c_int(0)
    c17 = _cam17(cam)
    _ref_call("gvr_ref_coarse_boxes", scene.size, scene.attr_dim(), ctypes.c_double(scene.tau), _ptr(c), _ptr(s),
              _ptr(a), _ptr(c17), ctypes.c_double(cfg.eta), int(cfg.k_prime), int(cfg.coarse_downsample),
              _ptr(box, _ip), ctypes.byref(dropped))
    return box, dropped.value


def ref_work_counts(scene, cam, cfg, threads: int = 0):
    c, s, a = _scene_arrays(scene)
    counts = np.zeros(3)
    c17 = _cam17(cam)
    _ref_call("gvr_ref_work_counts", scene.size, scene.attr_dim(), ctypes.c_double(scene.tau), _ptr(c), _ptr(s),
              _ptr(a), _ptr(c17), ctypes.c_double(cfg.eta), int(cfg.k_prime), int(bool(cfg.coarse_enabled)),
              int(cfg.coarse_downsample), threads, _ptr(counts))
    return dict(C=counts[0], N1=counts[1], N2=counts[2])


def ref_make_bench_scene(n: int):
    lib = ref_lib()
    k, d, tau = ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
    null = ctypes.cast(None, _dp)
    _ref_call("gvr_ref_make_bench_scene", n, ctypes.byref(k), ctypes.byref(d), ctypes.byref(tau), null, null, null)
    c = np.zeros((k.value, 3))
    s = np.zeros((k.value, 3, 3))
    a = np.zeros((k.value, d.value))
    _ref_call("gvr_ref_make_bench_scene", n, ctypes.byref(k), ctypes.byref(d), ctypes.byref(tau), _ptr(c), _ptr(s),
              _ptr(a))
    del lib
    return c, s, a, tau.value


def ref_make_bench_camera(size: int) -> np.ndarray:
    c17 = np.zeros(17)
    _ref_call("gvr_ref_make_bench_camera", size, _ptr(c17))
    return c17


def ref_make_orbit_camera(azimuth, elevation, distance, target, height, width, focal) -> np.ndarray:
    c17 = np.zeros(17)
    t = np.asarray(target, dtype=np.float64)
    _ref_call("gvr_ref_make_orbit_camera", ctypes.c_double(azimuth), ctypes.c_double(elevation),
              ctypes.c_double(distance), _ptr(t), int(height), int(width), ctypes.c_double(focal), _ptr(c17))
    return c17


def ref_sample_attributes(scene, cam, cfg, observed, normalized=False, threads: int = 0):
    """Reference ``gvr::sample_attributes`` (sampler.cpp:11-51)."""
    c, s, a = _scene_arrays(scene)
    obs = np.ascontiguousarray(observed, dtype=np.float64)
    ch = obs.shape[2] if obs.ndim == 3 else 1
    k = scene.size
    attrs, support, masked = np.zeros((k, ch)), np.zeros(k), np.zeros(k, dtype=np.uint8)
    c17 = _cam17(cam)
    _ref_call("gvr_ref_sample_attributes", k, scene.attr_dim(), ctypes.c_double(scene.tau), _ptr(c), _ptr(s), _ptr(a),
              _ptr(c17), ctypes.c_double(cfg.eta), int(cfg.k_prime), int(bool(cfg.coarse_enabled)),
              int(cfg.coarse_downsample), threads, _ptr(obs), int(obs.shape[0]), int(obs.shape[1]), ch,
              int(bool(normalized)), _ptr(attrs), _ptr(support), _u8p(masked))
    return attrs, support, masked.astype(bool)


def ref_resynthesize(scene, cam, cfg, attrs, masked, threads: int = 0) -> dict:
    """Reference ``gvr::resynthesize`` (sampler.cpp:53-66): image, alpha, depth."""
    c, s, a = _scene_arrays(scene)
    at = np.ascontiguousarray(attrs, dtype=np.float64)
    mk = np.ascontiguousarray(masked, dtype=np.uint8)
    h, w = int(cam.height), int(cam.width)
    out = dict(image=np.zeros((h, w, max(at.shape[1], 1))), alpha=np.zeros((h, w, 1)), depth=np.zeros((h, w, 1)))
    c17 = _cam17(cam)
    _ref_call("gvr_ref_resynthesize", scene.size, scene.attr_dim(), ctypes.c_double(scene.tau), _ptr(c), _ptr(s),
              _ptr(a), _ptr(c17), ctypes.c_double(cfg.eta), int(cfg.k_prime), int(bool(cfg.coarse_enabled)),
              int(cfg.coarse_downsample), threads, int(at.shape[0]), int(at.shape[1]), _ptr(at), _u8p(mk),
              _ptr(out["image"]), _ptr(out["alpha"]), _ptr(out["depth"]))
    return out


def ref_pixel_helpers(scene, cam, cfg, t, eps=1e-8, threads: int = 0):
    """Reference per-pixel ``transmittance_at`` / ``normalized_weights`` (blender.cpp:19-25, 55-62)."""
    c, s, a = _scene_arrays(scene)
    h, w, kp = int(cam.height), int(cam.width), int(cfg.k_prime)
    tt = np.ascontiguousarray(t, dtype=np.float64).reshape(h, w)
    trans, nw = np.zeros((h, w)), np.zeros((h, w, kp))
    c17 = _cam17(cam)
    _ref_call("gvr_ref_pixel_helpers", scene.size, scene.attr_dim(), ctypes.c_double(scene.tau), _ptr(c), _ptr(s),
              _ptr(a), _ptr(c17), ctypes.c_double(cfg.eta), int(cfg.k_prime), int(bool(cfg.coarse_enabled)),
              int(cfg.coarse_downsample), threads, _ptr(tt), _ptr(trans), ctypes.c_double(eps), _ptr(nw))
    return trans, nw


def ref_shade_lambert(cam, normals, alpha, depth, light_pos, light_color):
    """Reference ``gvr::shade_lambert`` (blender.cpp:146-172)."""
    h, w = int(cam.height), int(cam.width)
    n = np.ascontiguousarray(normals, dtype=np.float64)
    al = np.ascontiguousarray(alpha, dtype=np.float64)
    de = np.ascontiguousarray(depth, dtype=np.float64)
    lp = np.ascontiguousarray(light_pos, dtype=np.float64)
    lc = np.ascontiguousarray(light_color, dtype=np.float64)
    out = np.zeros((h, w, 3))
    _ref_call("gvr_ref_shade_lambert", _ptr(_cam17(cam)), _ptr(n), _ptr(al), _ptr(de), _ptr(lp), _ptr(lc), _ptr(out))
    return out


def ref_shape_reg(edges, rest, centers):
    """Reference ShapeRegularizer::make + edge_reg / laplacian_reg (fit.cpp:44-113):
    (edge value, edge grad [N,3], laplacian value, laplacian grad [N,3])."""
    e = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 2)
    r = np.ascontiguousarray(rest, dtype=np.float64).reshape(-1, 3)
    c = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 3)
    vals, ge, gl = np.zeros(2), np.zeros_like(c), np.zeros_like(c)
    _ref_call("gvr_ref_shape_reg", r.shape[0], e.shape[0], _ptr(e, _ip), _ptr(r), _ptr(c), _ptr(vals), _ptr(ge), _ptr(gl))
    return vals[0], ge, vals[1], gl


def ref_view_transform(scene, cam):
    """Reference gvr::view_transform (scene.cpp:5-17): (centers [K,3], inv_cov [K,3,3])."""
    c, s, a = _scene_arrays(scene)
    oc, os_ = np.zeros((scene.size, 3)), np.zeros((scene.size, 3, 3))
    _ref_call("gvr_ref_view_transform", scene.size, scene.attr_dim(), ctypes.c_double(scene.tau), _ptr(c), _ptr(s),
              _ptr(a), _ptr(_cam17(cam)), _ptr(oc), _ptr(os_))
    return oc, os_
