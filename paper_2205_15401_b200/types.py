"""Data model of the render path, mirroring the reference's C++ types.

Reference: ``proj/include/gvr/types.hpp:19-93`` (GaussianKernel, GaussianScene,
Camera, Image, ValidationError), ``proj/include/gvr/tracer.hpp:18-25``
(SelectionConfig), ``proj/include/gvr/blender.hpp:18-25`` (RenderBuffers),
``proj/include/gvr/grad.hpp:13-54`` (GradientBundle, Tape, ForwardResult,
GradFlags, ScalarLoss).

The reference stores a vector of AoS Eigen kernels; here a scene is SoA numpy
FP64 arrays (``centers[K,3]``, ``inv_cov[K,3,3]`` row-major Sigma^-1,
``attr[K,D]``), which is exactly what the C ABI (include/gvr_cuda.h) uploads.
Images are ``[H, W, C]`` FP64 (channels interleaved, as ``gvr::Image``).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np


class ValidationError(RuntimeError):
    """``gvr::ValidationError`` (types.hpp:19-22): an input violates a precondition.

    Messages are identical to the reference's (e.g. ``"inv_cov is not
    positive-definite (kernel 3)"``)."""


@dataclass
class GaussianScene:
    """``gvr::GaussianScene`` (types.hpp:35-42) as SoA arrays."""

    centers: np.ndarray  # [K, 3] float64
    inv_cov: np.ndarray  # [K, 3, 3] float64 (Sigma^-1)
    attr: np.ndarray  # [K, D] float64
    tau: float = 1.0

    def __post_init__(self) -> None:
        self.centers = np.ascontiguousarray(np.asarray(self.centers, dtype=np.float64).reshape(-1, 3))
        k = self.centers.shape[0]
        self.inv_cov = np.ascontiguousarray(np.asarray(self.inv_cov, dtype=np.float64).reshape(k, 3, 3))
        attr = np.asarray(self.attr, dtype=np.float64)
        if attr.ndim == 1:
            attr = attr.reshape(k, -1) if k else attr.reshape(0, 0)
        self.attr = np.ascontiguousarray(attr)
        if self.attr.shape[0] != k:
            raise ValidationError("attribute dimension is not uniform (kernel 0)")
        self.tau = float(self.tau)

    @property
    def size(self) -> int:
        return int(self.centers.shape[0])

    def attr_dim(self) -> int:
        return int(self.attr.shape[1]) if self.size else 0

    def copy(self) -> "GaussianScene":
        return GaussianScene(self.centers.copy(), self.inv_cov.copy(), self.attr.copy(), self.tau)

    @staticmethod
    def from_kernels(kernels, tau: float = 1.0) -> "GaussianScene":
        """Build from a list of ``(center[3], inv_cov[3x3], attr[D])`` tuples;
        mixed attribute sizes raise like ``GaussianScene::validate``."""
        kernels = list(kernels)
        if not kernels:
            return GaussianScene(np.zeros((0, 3)), np.zeros((0, 3, 3)), np.zeros((0, 0)), tau)
        dim = len(kernels[0][2])
        for k, (_, _, a) in enumerate(kernels):
            if len(a) != dim:
                raise ValidationError(f"attribute dimension is not uniform (kernel {k})")
        return GaussianScene(
            np.array([c for c, _, _ in kernels], dtype=np.float64),
            np.array([s for _, s, _ in kernels], dtype=np.float64),
            np.array([a for _, _, a in kernels], dtype=np.float64).reshape(len(kernels), dim),
            tau,
        )


@dataclass
class Camera:
    """``gvr::Camera`` (types.hpp:46-56). Pixel (i, j) = (row, col); i pairs with Oy."""

    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))
    focal: float = 1.0
    ox: float = 0.0
    oy: float = 0.0
    height: int = 1
    width: int = 1

    def __post_init__(self) -> None:
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(3, 3)
        self.translation = np.asarray(self.translation, dtype=np.float64).reshape(3)

    def as_array(self) -> np.ndarray:
        """17 doubles: R (row-major) T focal ox oy height width."""
        return np.concatenate(
            [self.rotation.reshape(9), self.translation, [self.focal, self.ox, self.oy, self.height, self.width]]
        ).astype(np.float64)


@dataclass
class SelectionConfig:
    """``gvr::SelectionConfig`` (tracer.hpp:18-25)."""

    eta: float = 0.01
    k_prime: int = 20
    coarse_enabled: bool = True
    coarse_downsample: int = 8


@dataclass
class GradFlags:
    """``gvr::GradFlags`` (grad.hpp:46-49): ablation switches."""

    through_transmittance: bool = True
    through_density: bool = True


@dataclass
class RenderBuffers:
    """``gvr::RenderBuffers`` (blender.hpp:18-25).

    ``weight_store`` of the reference (per-pixel ``(index, W)`` lists ascending
    in ``(l, index)``) is the padded pair ``topk_idx[H, W, K']`` (int32, -1 pad)
    / ``topk_w[H, W, K']``; both are filled only when requested."""

    image: np.ndarray  # [H, W, max(D,1)]
    alpha: np.ndarray  # [H, W, 1]
    depth: np.ndarray  # [H, W, 1]
    topk_idx: Optional[np.ndarray] = None
    topk_w: Optional[np.ndarray] = None

    def weight_store(self, p: int):
        """Sparse list of pixel ``p`` (row-major), like ``weight_store[p]``."""
        if self.topk_idx is None:
            raise ValidationError("weight_store was not requested for this render")
        idx = self.topk_idx.reshape(-1, self.topk_idx.shape[-1])[p]
        w = self.topk_w.reshape(-1, self.topk_w.shape[-1])[p]
        n = int((idx >= 0).sum())
        return [(int(idx[s]), float(w[s])) for s in range(n)]


@dataclass
class GradientBundle:
    """``gvr::GradientBundle`` (grad.hpp:13-22), object-space gradients."""

    d_center: np.ndarray  # [K, 3]
    d_inv_cov: np.ndarray  # [K, 3, 3]
    d_attr: np.ndarray  # [K, D]
    d_rotation: np.ndarray  # [3, 3]
    d_translation: np.ndarray  # [3]


@dataclass
class ScalarLoss:
    """``gvr::ScalarLoss`` (grad.hpp:62-70, grad.cpp:201-216):
    L = 0.5 w_image |image - t|^2 + 0.5 w_alpha |alpha - t_alpha|^2."""

    target_image: np.ndarray
    target_alpha: np.ndarray
    w_image: float = 1.0
    w_alpha: float = 1.0


@dataclass
class SampledAttributes:
    """``gvr::SampledAttributes`` (sampler.hpp:8-15): per-kernel recovered
    attributes [K, D], support (sum of observed weights) [K], masked [K] bool."""

    attrs: np.ndarray
    support: np.ndarray
    masked: np.ndarray

    def masked_count(self) -> int:
        return int(np.count_nonzero(self.masked))


K_SUPPORT_EPS = 1e-8  # gvr::kSupportEps (sampler.hpp:18)
