"""Synthetic benchmark inputs, restated from the reference (host-side input generation only).

* ``make_bench_scene(N)``  = ``gvr::make_bench_scene`` (proj/src/bench.cpp:9-14):
  ``make_cuboid_scene((1,1,1), N, zeta=0.5, color (0.8,0.3,0.2), centre (0,0,4))``
  (shapes.cpp:108-116) -> ``make_box_mesh`` (shapes.cpp:57-106) ->
  ``mesh_to_gaussians`` (convert.cpp:90-130): one isotropic kernel per welded
  vertex, sigma = mean_edge^2 / (4 ln(1/zeta)), inv_cov = I / sigma.
* ``make_bench_camera(S)`` = bench.cpp:16-24 (R = I, T = 0, F = 1.6 S, Ox = Oy = (S-1)/2).
* ``make_orbit_camera``    = shapes.cpp:118-141.

Vectorised numpy with the reference's evaluation order; tests pin the outputs
against the reference build (tests/test_synthetic.py).
"""
from __future__ import annotations

import math

import numpy as np

from .types import Camera, GaussianScene


def make_box_mesh(size=(1.0, 1.0, 1.0), divisions: int = 1, center=(0.0, 0.0, 0.0)):
    """Welded box surface grid (shapes.cpp:57-106): returns (vertices[V,3], faces[F,3])."""
    n = int(divisions)
    if n < 1:
        raise ValueError("box divisions must be >= 1")
    size = np.asarray(size, dtype=np.float64)
    center = np.asarray(center, dtype=np.float64)
    p, q = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    corners_dudv = [(0, 0), (1, 0), (1, 1), (0, 1)]
    blocks = []
    for axis in range(3):
        u, v = (axis + 1) % 3, (axis + 2) % 3
        for side in range(2):
            c = np.zeros((n, n, 4, 3), dtype=np.int64)
            for ci, (du, dv) in enumerate(corners_dudv):
                c[:, :, ci, axis] = side * n
                c[:, :, ci, u] = p + du
                c[:, :, ci, v] = q + dv
            blocks.append(c)
    allc = np.stack(blocks)  # [6, n, n, 4, 3] in the reference's loop order
    flat = allc.reshape(-1, 3)
    base = n + 1
    keys = (flat[:, 0] * base + flat[:, 1]) * base + flat[:, 2]
    uniq, first, inverse = np.unique(keys, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")  # creation order = first occurrence
    rank = np.empty_like(order)
    rank[order] = np.arange(order.size)
    vid = rank[inverse].reshape(6, n, n, 4)
    ijk = flat[first[order]].astype(np.float64)
    verts = np.empty((ijk.shape[0], 3))
    for d in range(3):
        verts[:, d] = center[d] + (ijk[:, d] / n - 0.5) * size[d]
    faces = []
    for b in range(6):
        side = b % 2
        v00, v10, v11, v01 = (vid[b, :, :, i].reshape(-1) for i in range(4))
        if side == 1:
            f = np.stack([np.stack([v00, v10, v11], 1), np.stack([v00, v11, v01], 1)], 1)
        else:
            f = np.stack([np.stack([v00, v11, v10], 1), np.stack([v00, v01, v11], 1)], 1)
        faces.append(f.reshape(-1, 3))
    return verts, np.concatenate(faces)


def mesh_edges(faces) -> np.ndarray:
    """Unique undirected edges (a < b) in std::set order (convert.cpp:39-51): [E, 2] int32."""
    f = np.asarray(faces, dtype=np.int64)
    e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
    e = e[e[:, 0] != e[:, 1]]
    a = np.minimum(e[:, 0], e[:, 1])
    b = np.maximum(e[:, 0], e[:, 1])
    n = int(max(a.max(), b.max())) + 1 if len(a) else 1
    code = np.unique(a * n + b)
    return np.stack([code // n, code % n], 1).astype(np.int32)


def mesh_to_gaussians_isotropic(verts, faces, zeta: float, colors) -> GaussianScene:
    """``mesh_to_gaussians`` with flatten_rate = 1 (convert.cpp:90-130)."""
    nv = verts.shape[0]
    e = np.concatenate([faces[:, [0, 1]], faces[:, [1, 2]], faces[:, [2, 0]]])
    e = e[e[:, 0] != e[:, 1]]
    a = np.minimum(e[:, 0], e[:, 1])
    b = np.maximum(e[:, 0], e[:, 1])
    code = np.unique(a.astype(np.int64) * nv + b)  # std::set order
    a, b = code // nv, code % nv
    dv = verts[a] - verts[b]
    sq = dv * dv
    length = np.sqrt((sq[:, 0] + sq[:, 1]) + sq[:, 2])
    edge_sum = np.zeros(nv)
    edge_cnt = np.zeros(nv, dtype=np.int64)
    # sequential accumulation in edge order, a then b (convert.cpp:95-101)
    ab = np.stack([a, b], 1).reshape(-1)
    ll = np.repeat(length, 2)
    np.add.at(edge_sum, ab, ll)
    np.add.at(edge_cnt, ab, 1)
    if np.any(edge_cnt == 0):
        raise ValueError("vertex has no connected edges")
    mean_edge = edge_sum / edge_cnt
    sigma = mean_edge * mean_edge / (4.0 * math.log(1.0 / zeta))
    inv_cov = np.zeros((nv, 3, 3))
    for d in range(3):
        inv_cov[:, d, d] = 1.0 / sigma
    attr = np.broadcast_to(np.asarray(colors, dtype=np.float64), (nv, 3)).copy()
    return GaussianScene(verts.copy(), inv_cov, attr, 1.0)


def make_cuboid_scene(size, min_kernels: int, zeta: float, color, center) -> GaussianScene:
    """shapes.cpp:108-116: smallest div with 6 div^2 + 2 >= min_kernels."""
    div = 1
    while 6 * div * div + 2 < min_kernels:
        div += 1
    verts, faces = make_box_mesh(size, div, center)
    return mesh_to_gaussians_isotropic(verts, faces, zeta, color)


def make_bench_scene(kernel_count: int) -> GaussianScene:
    """bench.cpp:9-14."""
    return make_cuboid_scene((1.0, 1.0, 1.0), kernel_count, 0.5, (0.8, 0.3, 0.2), (0.0, 0.0, 4.0))


def make_bench_camera(image_size: int) -> Camera:
    """bench.cpp:16-24."""
    s = int(image_size)
    return Camera(np.eye(3), np.zeros(3), 1.6 * s, (s - 1) / 2.0, (s - 1) / 2.0, s, s)


def make_orbit_camera(azimuth: float, elevation: float, distance: float, target, height: int, width: int,
                      focal: float) -> Camera:
    """shapes.cpp:118-141."""
    target = np.asarray(target, dtype=np.float64)
    offset = np.array([distance * math.cos(elevation) * math.sin(azimuth), distance * math.sin(elevation),
                       -distance * math.cos(elevation) * math.cos(azimuth)])
    eye = target + offset

    def normalized(x):
        n = (x[0] * x[0] + x[1] * x[1]) + x[2] * x[2]
        return x / math.sqrt(n) if n > 0 else x

    forward = normalized(target - eye)
    up = np.array([0.0, 1.0, 0.0])
    if abs((forward[0] * up[0] + forward[1] * up[1]) + forward[2] * up[2]) > 0.999:
        up = np.array([0.0, 0.0, 1.0])

    def cross(x, y):
        return np.array([x[1] * y[2] - x[2] * y[1], x[2] * y[0] - x[0] * y[2], x[0] * y[1] - x[1] * y[0]])

    right = normalized(cross(up, forward))
    down = cross(right, forward)
    rot = np.stack([down, right, forward])
    t = -np.array([(rot[i, 0] * eye[0] + rot[i, 1] * eye[1]) + rot[i, 2] * eye[2] for i in range(3)])
    return Camera(rot, t, float(focal), (width - 1) / 2.0, (height - 1) / 2.0, int(height), int(width))
