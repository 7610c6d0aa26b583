"""JSON scene / camera loading (reference format, proj/src/scene_io.cpp:53-129).

Scene: {"version": 1, "tau": t, "kernels": [{"center": [3], "inv_cov": [9 row-major], "attr": [D]}]}
Camera: {"version": 1, "R": [9 row-major], "T": [3], "F", "Ox", "Oy", "H", "W"}
Only what the tests need to read the reference's bundled fixtures.
"""
from __future__ import annotations

import json

import numpy as np

from .types import Camera, GaussianScene, ValidationError


def _load(path):
    with open(path) as f:
        j = json.load(f)
    if "version" in j and int(j["version"]) != 1:
        raise ValidationError(f"unsupported format version in {path}")
    return j


def load_scene_json(path) -> GaussianScene:
    j = _load(path)
    ks = j["kernels"]
    for k in ks:
        if len(k["center"]) != 3 or len(k["inv_cov"]) != 9:
            raise ValidationError(f"bad kernel entry in {path}")
    kernels = [(k["center"], np.asarray(k["inv_cov"], dtype=np.float64).reshape(3, 3), k["attr"]) for k in ks]
    return GaussianScene.from_kernels(kernels, float(j.get("tau", 1.0)))


def load_camera_json(path) -> Camera:
    j = _load(path)
    if len(j["R"]) != 9 or len(j["T"]) != 3:
        raise ValidationError(f"bad camera extrinsics in {path}")
    return Camera(np.asarray(j["R"], dtype=np.float64).reshape(3, 3), np.asarray(j["T"], dtype=np.float64),
                  float(j["F"]), float(j["Ox"]), float(j["Oy"]), int(j["H"]), int(j["W"]))
