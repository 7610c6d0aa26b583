"""ctypes binding of the C ABI (include/gvr_cuda.h) — no compute happens in Python.

The product path is: Python/C++ caller -> libgvr_cuda.so (C ABI) -> sm_100a kernels.
If the shared library is missing, importing the API fails loudly; there is no
CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GVR_LIB_PATH") or os.path.join(HERE, "libgvr_cuda.so")  # override: A/B builds

GVR_OK = 0
GVR_ERR_VALIDATION = 1
GVR_ERR_RUNTIME = 2

EXPORTED_SYMBOLS = (
    "gvr_context_create",
    "gvr_context_destroy",
    "gvr_last_error",
    "gvr_context_set_stream",
    "gvr_context_stream",
    "gvr_context_synchronize",
    "gvr_context_launch_count",
    "gvr_context_library_call_count",
    "gvr_context_enable_timing",
    "gvr_context_stage_times",
    "gvr_measure_pipe_peak",
    "gvr_context_set_prefilter_guard",
    "gvr_context_set_tile_capacity",
    "gvr_graph_begin",
    "gvr_graph_end",
    "gvr_graph_launch",
    "gvr_graph_destroy",
    "gvr_scene_create",
    "gvr_scene_destroy",
    "gvr_scene_set",
    "gvr_scene_size",
    "gvr_scene_attr_dim",
    "gvr_tape_create",
    "gvr_tape_destroy",
    "gvr_render",
    "gvr_render_shard",
    "gvr_tape_traced",
    "gvr_tape_shape",
    "gvr_scalar_loss",
    "gvr_backward",
    "gvr_backward_accumulate",
    "gvr_adam_step",
    "gvr_sample_attributes",
    "gvr_tape_sample_attributes",
    "gvr_scene_resynthesize",
    "gvr_tape_transmittance",
    "gvr_tape_normalized_weights",
    "gvr_shade_lambert",
    "gvr_render_views",
    "gvr_scalar_loss_views",
    "gvr_backward_views",
    "gvr_context_set_precise",
    "gvr_regularizer_create",
    "gvr_regularizer_destroy",
    "gvr_edge_reg",
    "gvr_laplacian_reg",
    "gvr_tape_cam_scene",
    "gvr_tape_dropped_behind_camera",
    "gvr_context_set_tile_profile",
    "gvr_scene_set_deferred",
    "gvr_camera_validate",
    "gvr_scene_check",
    "gvr_tape_tile_cycles",
    "gvr_tape_list_stats",
    "gvr_context_set_list_smem",
    "gvr_tape_check_finite",
    "gvr_adam_step_guarded",
    "gvr_trace_pairs",
    "gvr_view_transform",
    "gvr_pixel_rays",
    "gvr_coarse_select_boxes",
    "gvr_ray_sort",
    "gvr_blend_ray",
    "gvr_transmittance_ray",
    "gvr_normalized_weights_ray",
    "gvr_scalar_loss_buffers",
    "gvr_build_hash",
    "gvr_context_set_async",
    "gvr_backward_packed",
)


class GvrCamera(ctypes.Structure):
    _fields_ = [
        ("rotation", ctypes.c_double * 9),
        ("translation", ctypes.c_double * 3),
        ("focal", ctypes.c_double),
        ("ox", ctypes.c_double),
        ("oy", ctypes.c_double),
        ("height", ctypes.c_int32),
        ("width", ctypes.c_int32),
    ]


class GvrSelection(ctypes.Structure):
    _fields_ = [
        ("eta", ctypes.c_double),
        ("k_prime", ctypes.c_int32),
        ("coarse_enabled", ctypes.c_int32),
        ("coarse_downsample", ctypes.c_int32),
    ]


class GvrGradFlags(ctypes.Structure):
    _fields_ = [("through_transmittance", ctypes.c_int32), ("through_density", ctypes.c_int32)]


class GvrRenderOutputs(ctypes.Structure):
    _fields_ = [
        ("image", ctypes.c_void_p),
        ("alpha", ctypes.c_void_p),
        ("depth", ctypes.c_void_p),
        ("topk_idx", ctypes.c_void_p),
        ("topk_w", ctypes.c_void_p),
    ]


class GvrGradients(ctypes.Structure):
    _fields_ = [
        ("d_center", ctypes.c_void_p),
        ("d_inv_cov", ctypes.c_void_p),
        ("d_attr", ctypes.c_void_p),
        ("d_rotation", ctypes.c_void_p),
        ("d_translation", ctypes.c_void_p),
    ]


_lib = None


def load() -> ctypes.CDLL:
    """Load libgvr_cuda.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first (python -c 'import __graft_entry__ as g; g.build()')"
        )
    lib = ctypes.CDLL(LIB_PATH)
    lib.gvr_build_hash.restype = ctypes.c_char_p
    lib.gvr_build_hash.argtypes = []
    if "GVR_LIB_PATH" not in os.environ:  # A/B experiment builds are loaded on purpose
        from . import build as _build

        try:
            want = _build.source_hash()
        except OSError:  # sources not shipped next to the library
            want = None
        got = lib.gvr_build_hash().decode()
        if want is not None and got != want:
            raise ImportError(f"{LIB_PATH} was built from other sources (hash {got}, sources {want}): rebuild it "
                              "(python -c 'import __graft_entry__ as g; g.build()')")
    vp, i32, dp = ctypes.c_void_p, ctypes.c_int32, ctypes.c_double
    sig = {
        "gvr_context_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(vp)]),
        "gvr_context_destroy": (None, [vp]),
        "gvr_last_error": (ctypes.c_char_p, [vp]),
        "gvr_context_set_stream": (ctypes.c_int, [vp, vp]),
        "gvr_context_stream": (vp, [vp]),
        "gvr_context_synchronize": (ctypes.c_int, [vp]),
        "gvr_context_launch_count": (ctypes.c_int64, [vp]),
        "gvr_context_library_call_count": (ctypes.c_int64, [vp]),
        "gvr_context_enable_timing": (ctypes.c_int, [vp, ctypes.c_int]),
        "gvr_context_stage_times": (ctypes.c_int, [vp, vp, vp, ctypes.c_int]),
        "gvr_measure_pipe_peak": (ctypes.c_int, [vp, ctypes.c_int, ctypes.POINTER(dp)]),
        "gvr_context_set_prefilter_guard": (ctypes.c_int, [vp, dp]),
        "gvr_context_set_precise": (ctypes.c_int, [vp, ctypes.c_int]),
        "gvr_context_set_tile_capacity": (ctypes.c_int, [vp, ctypes.c_int]),
        "gvr_graph_begin": (ctypes.c_int, [vp]),
        "gvr_graph_end": (ctypes.c_int, [vp, ctypes.POINTER(vp)]),
        "gvr_graph_launch": (ctypes.c_int, [vp, vp]),
        "gvr_graph_destroy": (None, [vp]),
        "gvr_scene_create": (ctypes.c_int, [vp, ctypes.POINTER(vp)]),
        "gvr_scene_destroy": (None, [vp]),
        "gvr_scene_set": (ctypes.c_int, [vp, vp, i32, i32, dp, vp, vp, vp]),
        "gvr_scene_set_deferred": (ctypes.c_int, [vp, vp, i32, i32, dp, vp, vp, vp]),
        "gvr_scene_check": (ctypes.c_int, [vp, vp]),
        "gvr_camera_validate": (ctypes.c_int, [ctypes.POINTER(GvrCamera), ctypes.c_char_p, i32]),
        "gvr_scene_size": (i32, [vp]),
        "gvr_scene_attr_dim": (i32, [vp]),
        "gvr_tape_create": (ctypes.c_int, [vp, ctypes.POINTER(vp)]),
        "gvr_tape_destroy": (None, [vp]),
        "gvr_render": (ctypes.c_int, [vp, vp, ctypes.POINTER(GvrCamera), ctypes.POINTER(GvrSelection), vp,
                                      ctypes.POINTER(GvrRenderOutputs)]),
        "gvr_tape_traced": (ctypes.c_int, [vp, vp, vp, vp, vp, vp]),
        "gvr_tape_cam_scene": (ctypes.c_int, [vp, vp, vp, vp]),
        "gvr_tape_dropped_behind_camera": (ctypes.c_int, [vp, vp, ctypes.POINTER(i32)]),
        "gvr_context_set_tile_profile": (ctypes.c_int, [vp, ctypes.c_int]),
        "gvr_tape_tile_cycles": (ctypes.c_int, [vp, vp, vp, ctypes.c_int64]),
        "gvr_tape_list_stats": (ctypes.c_int, [vp, vp, vp]),
        "gvr_context_set_list_smem": (ctypes.c_int, [vp, ctypes.c_int]),
        "gvr_tape_check_finite": (ctypes.c_int, [vp, vp]),
        "gvr_context_set_async": (ctypes.c_int, [vp, ctypes.c_int]),
        "gvr_backward_packed": (ctypes.c_int, [vp, vp, vp, vp, ctypes.POINTER(GvrGradFlags), vp, vp]),
        "gvr_trace_pairs": (ctypes.c_int, [vp, ctypes.c_int64, vp, vp, vp, vp, vp, vp]),
        "gvr_view_transform": (ctypes.c_int, [vp, i32, vp, vp, ctypes.POINTER(GvrCamera), vp, vp]),
        "gvr_pixel_rays": (ctypes.c_int, [vp, ctypes.POINTER(GvrCamera), ctypes.c_int64, vp, vp, vp]),
        "gvr_coarse_select_boxes": (ctypes.c_int, [vp, i32, vp, vp, ctypes.POINTER(GvrCamera),
                                                   ctypes.POINTER(GvrSelection), vp, ctypes.POINTER(i32)]),
        "gvr_ray_sort": (ctypes.c_int, [vp, i32, vp, vp, vp, dp, vp, ctypes.POINTER(i32)]),
        "gvr_blend_ray": (ctypes.c_int, [vp, i32, vp, vp, vp, vp, dp, vp, vp, vp]),
        "gvr_transmittance_ray": (ctypes.c_int, [vp, i32, vp, vp, vp, dp, i32, vp, vp]),
        "gvr_normalized_weights_ray": (ctypes.c_int, [vp, i32, vp, dp, vp]),
        "gvr_scalar_loss_buffers": (ctypes.c_int, [vp, ctypes.c_int64, vp, vp, ctypes.c_int64, vp, vp, dp, dp, vp, vp,
                                                   vp]),
        "gvr_adam_step_guarded": (ctypes.c_int, [vp, vp, vp, vp, vp, ctypes.c_int64, ctypes.c_int64, dp, dp, dp, dp,
                                                 vp, vp]),
        "gvr_tape_shape": (ctypes.c_int, [vp, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32),
                                          ctypes.POINTER(i32)]),
        "gvr_scalar_loss": (ctypes.c_int, [vp, vp, vp, vp, dp, dp, vp, vp, vp]),
        "gvr_backward": (ctypes.c_int, [vp, vp, vp, vp, ctypes.POINTER(GvrGradFlags), ctypes.POINTER(GvrGradients)]),
        "gvr_backward_accumulate": (ctypes.c_int, [vp, vp, vp, vp, ctypes.POINTER(GvrGradFlags),
                                                   ctypes.POINTER(GvrGradients)]),
        "gvr_render_shard": (ctypes.c_int, [vp, vp, ctypes.POINTER(GvrCamera), ctypes.POINTER(GvrSelection), vp,
                                            ctypes.POINTER(GvrRenderOutputs), i32, i32]),
        "gvr_adam_step": (ctypes.c_int, [vp, vp, vp, vp, vp, ctypes.c_int64, ctypes.c_int64, dp, dp, dp, dp]),
        "gvr_sample_attributes": (ctypes.c_int, [vp, vp, ctypes.POINTER(GvrCamera), ctypes.POINTER(GvrSelection), vp,
                                                 i32, i32, i32, i32, vp, vp, vp]),
        "gvr_tape_sample_attributes": (ctypes.c_int, [vp, vp, vp, i32, i32, vp, vp, vp]),
        "gvr_scene_resynthesize": (ctypes.c_int, [vp, vp, vp, i32, i32, vp, vp]),
        "gvr_tape_transmittance": (ctypes.c_int, [vp, vp, vp, vp]),
        "gvr_tape_normalized_weights": (ctypes.c_int, [vp, vp, dp, vp]),
        "gvr_render_views": (ctypes.c_int, [vp, vp, i32, ctypes.POINTER(GvrCamera), ctypes.POINTER(GvrSelection),
                                            ctypes.POINTER(vp), ctypes.POINTER(GvrRenderOutputs)]),
        "gvr_scalar_loss_views": (ctypes.c_int, [vp, i32, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                                 dp, dp, vp]),
        "gvr_backward_views": (ctypes.c_int, [vp, i32, ctypes.POINTER(vp), ctypes.POINTER(GvrGradFlags),
                                              ctypes.POINTER(GvrGradients), ctypes.POINTER(GvrGradients)]),
        "gvr_regularizer_create": (ctypes.c_int, [vp, i32, i32, vp, vp, ctypes.POINTER(vp)]),
        "gvr_regularizer_destroy": (None, [vp]),
        "gvr_edge_reg": (ctypes.c_int, [vp, vp, vp, dp, vp, vp, i32]),
        "gvr_laplacian_reg": (ctypes.c_int, [vp, vp, vp, dp, vp, vp, i32]),
        "gvr_shade_lambert": (ctypes.c_int, [vp, ctypes.POINTER(GvrCamera), vp, vp, vp, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
