"""Data formats either side of the render path (reference: proj/include/gvr/scene_io.hpp,
image_io.hpp; proj/src/scene_io.cpp:53-157, image_io.cpp:124-190).

Scene: {"version": 1, "tau": t, "kernels": [{"center": [3], "inv_cov": [9 row-major], "attr": [D]}]}
Camera: {"version": 1, "R": [9 row-major], "T": [3], "F", "Ox", "Oy", "H", "W"}
Sampled attributes: {"version": 1, "attrs": [[D]...], "support": [K], "masked": [bool...]}
PFM: "PF" (3 channels) / "Pf" (1 channel), little-endian (scale -1.0), rows bottom-up, float32.

Writers go through a temporary file in the target directory and a rename
(``atomic_write_text``, scene_io.hpp:36); errors are ``ValidationError`` with the
reference's messages. JSON is written with 2-space indentation like the
reference's ``json::dump(2)``; numbers use Python's shortest round-trip repr,
so every double reads back bit-identically.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

from .types import Camera, GaussianScene, SampledAttributes, ValidationError


def atomic_write_text(path, content: str) -> None:
    """Write to ``path + ".tmp"`` then rename over ``path`` (scene_io.hpp:36)."""
    _atomic_write(path, content.encode())


def _atomic_write(path, data: bytes) -> None:
    path = os.fspath(path)
    tmp = path + ".tmp"
    try:
        with open(tmp, "wb") as f:
            f.write(data)
    except OSError:
        raise ValidationError(f"cannot write file: {tmp}") from None
    try:
        os.replace(tmp, path)
    except OSError as e:
        raise ValidationError(f"cannot move temp file onto {path}: {e.strerror}") from None


def _load(path):
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise ValidationError(f"cannot open file: {os.fspath(path)}") from None
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise ValidationError(f"invalid JSON in {os.fspath(path)}: {e}") from None
    if "version" in j and int(j["version"]) != 1:
        raise ValidationError(f"unsupported format version in {os.fspath(path)}")
    return j


def _dump(obj) -> str:
    return json.dumps(obj, indent=2) + "\n"


def load_scene_json(path) -> GaussianScene:
    """scene_io.cpp:53-74."""
    j = _load(path)
    ks = j["kernels"]
    for k in ks:
        if len(k["center"]) != 3 or len(k["inv_cov"]) != 9:
            raise ValidationError(f"bad kernel entry in {os.fspath(path)}")
    kernels = [(k["center"], np.asarray(k["inv_cov"], dtype=np.float64).reshape(3, 3), k["attr"]) for k in ks]
    return GaussianScene.from_kernels(kernels, float(j.get("tau", 1.0)))


def save_scene_json(scene: GaussianScene, path) -> None:
    """scene_io.cpp:76-92."""
    kernels = []
    for k in range(scene.size):
        kernels.append({"center": [float(v) for v in scene.centers[k]],
                        "inv_cov": [float(v) for v in np.asarray(scene.inv_cov[k]).reshape(9)],
                        "attr": [float(v) for v in scene.attr[k]]})
    atomic_write_text(path, _dump({"version": 1, "tau": float(scene.tau), "kernels": kernels}))


def validate_camera(camera: Camera) -> None:
    """``Camera::validate`` (types.cpp:44-63) through the library's host-side check
    (``gvr_camera_validate``: same code and messages as the render path; no device)."""
    from . import _lib
    from .render import _camera_c

    lib = _lib.load()
    msg = ctypes.create_string_buffer(256)
    c = _camera_c(camera)
    if lib.gvr_camera_validate(ctypes.byref(c), msg, len(msg)) != _lib.GVR_OK:
        raise ValidationError(msg.value.decode())


def load_camera_json(path) -> Camera:
    """scene_io.cpp:94-113 (validated like the reference's loader)."""
    j = _load(path)
    if len(j["R"]) != 9 or len(j["T"]) != 3:
        raise ValidationError(f"bad camera extrinsics in {os.fspath(path)}")
    cam = Camera(np.asarray(j["R"], dtype=np.float64).reshape(3, 3), np.asarray(j["T"], dtype=np.float64),
                 float(j["F"]), float(j["Ox"]), float(j["Oy"]), int(j["H"]), int(j["W"]))
    validate_camera(cam)
    return cam


def save_camera_json(camera: Camera, path) -> None:
    """scene_io.cpp:115-129."""
    atomic_write_text(path, _dump({
        "version": 1,
        "R": [float(v) for v in np.asarray(camera.rotation).reshape(9)],
        "T": [float(v) for v in np.asarray(camera.translation).reshape(3)],
        "F": float(camera.focal), "Ox": float(camera.ox), "Oy": float(camera.oy),
        "H": int(camera.height), "W": int(camera.width)}))


def load_attrs_json(path) -> SampledAttributes:
    """scene_io.cpp:131-145."""
    j = _load(path)
    attrs = [list(map(float, a)) for a in j["attrs"]]
    support = [float(v) for v in j["support"]]
    masked = [bool(v) for v in j["masked"]]
    if len(support) != len(attrs) or len(masked) != len(attrs):
        raise ValidationError(f"inconsistent attrs file: {os.fspath(path)}")
    d = len(attrs[0]) if attrs else 0
    return SampledAttributes(np.asarray(attrs, dtype=np.float64).reshape(len(attrs), d),
                             np.asarray(support, dtype=np.float64), np.asarray(masked, dtype=bool))


def save_attrs_json(attrs: SampledAttributes, path) -> None:
    """scene_io.cpp:147-158."""
    atomic_write_text(path, _dump({
        "version": 1,
        "attrs": [[float(v) for v in row] for row in np.asarray(attrs.attrs)],
        "support": [float(v) for v in np.asarray(attrs.support)],
        "masked": [bool(v) for v in np.asarray(attrs.masked)]}))


def write_pfm(image: np.ndarray, path) -> None:
    """image_io.cpp:124-157: [H, W, 1] -> "Pf", [H, W, 3] -> "PF"; float32, rows bottom-up."""
    img = np.asarray(image)
    if img.ndim == 2:
        img = img[:, :, None]
    if img.ndim != 3 or img.shape[2] not in (1, 3):
        raise ValidationError("write_pfm supports 1 or 3 channels")
    h, w, ch = img.shape
    header = f"{'PF' if ch == 3 else 'Pf'}\n{w} {h}\n-1.0\n".encode()
    body = np.ascontiguousarray(img[::-1].astype("<f4")).tobytes()
    _atomic_write(path, header + body)


def read_pfm(path) -> np.ndarray:
    """image_io.cpp:159-190: returns [H, W, C] float64 (C = 3 for "PF", 1 for "Pf")."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise ValidationError(f"cannot open file: {os.fspath(path)}") from None
    tokens, pos = [], 0
    while len(tokens) < 4:  # magic, width, height, scale separated by whitespace
        while pos < len(data) and data[pos:pos + 1].isspace():
            pos += 1
        start = pos
        while pos < len(data) and not data[pos:pos + 1].isspace():
            pos += 1
        if start == pos:
            break
        tokens.append(data[start:pos].decode("latin-1"))
    try:
        magic, w, h, scale = tokens[0], int(tokens[1]), int(tokens[2]), float(tokens[3])
    except (IndexError, ValueError):
        raise ValidationError(f"not a PFM file: {os.fspath(path)}") from None
    if magic not in ("PF", "Pf") or w <= 0 or h <= 0:
        raise ValidationError(f"not a PFM file: {os.fspath(path)}")
    if scale >= 0.0:
        raise ValidationError(f"big-endian PFM is not supported: {os.fspath(path)}")
    pos += 1  # the single whitespace after the scale
    ch = 3 if magic == "PF" else 1
    n = w * h * ch
    if len(data) - pos < 4 * n:
        raise ValidationError(f"truncated PFM data: {os.fspath(path)}")
    rows = np.frombuffer(data, dtype="<f4", count=n, offset=pos).reshape(h, w, ch)
    return rows[::-1].astype(np.float64)
