"""Central-difference verification of the device backward.

Mirrors ``gvr::gradcheck`` (/root/reference/proj/src/grad.cpp:242-350) and its
report types (grad.hpp:67-82): parameter classes "center", "inv_cov", "attr"
and "pose" (camera axis-angle + translation); a direction is skipped (and
counted) when the selection sets change within +-h; the relative error is
|a - n| / max(|a| + |n|, 1e-6) with a 1e-7 zero floor (grad.cpp:235-238).
Every forward / loss / backward evaluation runs on the GPU through the C ABI;
this module only orchestrates the finite differences on the host, like the
reference's. The SO(3) chart helpers follow so3.cpp.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, Optional

import numpy as np

from .render import Context, DeviceScene, Tape, backward_into, default_context, render_into, scalar_loss_into
from .types import Camera, GaussianScene, ScalarLoss, SelectionConfig, ValidationError


def so3_hat(w) -> np.ndarray:
    """so3.cpp:7-13."""
    x, y, z = (float(v) for v in w)
    return np.array([[0.0, -z, y], [z, 0.0, -x], [-y, x, 0.0]])


def so3_exp(w) -> np.ndarray:
    """so3.cpp:15-24 (Rodrigues, second-order series below 1e-12)."""
    w = np.asarray(w, dtype=np.float64)
    theta = float(np.linalg.norm(w))
    k = so3_hat(w)
    if theta < 1e-12:
        return np.eye(3) + k + 0.5 * k @ k
    s = math.sin(theta) / theta
    c = (1.0 - math.cos(theta)) / (theta * theta)
    return np.eye(3) + s * k + c * (k @ k)


def so3_log(r) -> np.ndarray:
    """so3.cpp:26-46."""
    r = np.asarray(r, dtype=np.float64)
    cos_theta = min(max((np.trace(r) - 1.0) * 0.5, -1.0), 1.0)
    theta = math.acos(cos_theta)
    if theta < 1e-9:
        return 0.5 * np.array([r[2, 1] - r[1, 2], r[0, 2] - r[2, 0], r[1, 0] - r[0, 1]])
    if theta > math.pi - 1e-6:
        a = 0.5 * (r + np.eye(3))
        axis = np.sqrt(np.maximum(0.0, np.diag(a)))
        major = int(np.argmax(np.diag(a)))
        for i in range(3):
            if i != major and a[major, i] < 0.0:
                axis[i] = -axis[i]
        n = np.linalg.norm(axis)
        return np.zeros(3) if n < 1e-12 else theta * axis / n
    axis = np.array([r[2, 1] - r[1, 2], r[0, 2] - r[2, 0], r[1, 0] - r[0, 1]])
    return axis * (theta / (2.0 * math.sin(theta)))


def so3_exp_gradient(w, d_rotation) -> np.ndarray:
    """dL/dw of L(R(w)) given dL/dR (so3.cpp:48-65)."""
    w = np.asarray(w, dtype=np.float64)
    d_rotation = np.asarray(d_rotation, dtype=np.float64)
    theta2 = float(w @ w)
    r = so3_exp(w)
    grad = np.zeros(3)
    for i in range(3):
        e = np.zeros(3)
        e[i] = 1.0
        if theta2 < 1e-16:
            dr = so3_hat(e)
        else:
            v = np.cross(w, (np.eye(3) - r) @ e)
            dr = ((w[i] * so3_hat(w) + so3_hat(v)) / theta2) @ r
        grad[i] = float((d_rotation * dr).sum())
    return grad


@dataclass
class GradCheckEntry:
    """grad.hpp:67-73."""

    max_rel_err: float = 0.0
    checked: int = 0
    skipped_boundary: int = 0
    worst_analytic: float = 0.0
    worst_numeric: float = 0.0


@dataclass
class GradCheckReport:
    """grad.hpp:75-82."""

    per_class: Dict[str, GradCheckEntry] = field(default_factory=dict)
    max_rel_err: float = 0.0
    total_checked: int = 0
    total_skipped: int = 0

    def passed(self, tol: float) -> bool:
        return self.max_rel_err < tol


def _relative_error(analytic: float, numeric: float) -> float:
    """grad.cpp:235-238."""
    if abs(analytic) < 1e-7 and abs(numeric) < 1e-7:
        return 0.0
    return abs(analytic - numeric) / max(abs(analytic) + abs(numeric), 1e-6)


def gradcheck(scene: GaussianScene, camera: Camera, cfg: SelectionConfig, loss: ScalarLoss, h: float = 1e-4,
              tol: float = 1e-3, threads: int = 0, *, ctx: Optional[Context] = None) -> GradCheckReport:
    """``gvr::gradcheck`` (grad.cpp:242-350) with device renders."""
    del tol, threads  # the reference reports; the caller decides with passed(tol)
    ctx = ctx or default_context()
    h_img, w_img = int(camera.height), int(camera.width)
    kp = int(cfg.k_prime)
    t_img = np.ascontiguousarray(loss.target_image, dtype=np.float64)
    t_alpha = np.ascontiguousarray(loss.target_alpha, dtype=np.float64)
    omega0 = so3_log(camera.rotation)
    cam = Camera(so3_exp(omega0), camera.translation, camera.focal, camera.ox, camera.oy, h_img, w_img)

    dscene = DeviceScene(ctx)
    tape = Tape(ctx)
    sets = np.empty((h_img, w_img, kp), dtype=np.int32)
    lval = np.zeros(1)

    def forward(s: GaussianScene, c: Camera):
        """(loss, selection sets) or None when the perturbed inputs are invalid."""
        try:
            dscene.set(s)
            render_into(ctx, dscene, c, cfg, tape, topk_idx=sets)
            scalar_loss_into(tape, t_img, t_alpha, loss.w_image, loss.w_alpha, lval)
        except ValidationError:
            return None
        return float(lval[0]), sets.copy()

    # the finite differences need the forward to ~1e-15: verification mode for
    # the whole check (the analytic backward is the production one)
    ctx.set_precise(True)
    try:
        return _gradcheck(scene, cam, cfg, loss, h, ctx, forward, dscene, tape, omega0, h_img, w_img)
    finally:
        ctx.set_precise(False)


def _gradcheck(scene, cam, cfg, loss, h, ctx, forward, dscene, tape, omega0, h_img, w_img) -> GradCheckReport:
    base = forward(scene, cam)
    if base is None:
        raise ValidationError("gradcheck: the base scene does not render")
    base_sets = base[1]
    k, d = scene.size, scene.attr_dim()
    g_center, g_inv_cov, g_attr = np.empty((k, 3)), np.empty((k, 3, 3)), np.empty((k, d))
    g_rot, g_trans = np.empty((3, 3)), np.empty(3)
    backward_into(tape, None, None, d_center=g_center, d_inv_cov=g_inv_cov, d_attr=g_attr if d > 0 else None,
                  d_rotation=g_rot, d_translation=g_trans)

    report = GradCheckReport()

    def check(cls: str, analytic: float, apply, step: float) -> None:
        entry = report.per_class.setdefault(cls, GradCheckEntry())
        sp, cp = scene.copy(), Camera(cam.rotation.copy(), cam.translation.copy(), cam.focal, cam.ox, cam.oy,
                                      h_img, w_img)
        apply(sp, cp, step)
        plus = forward(sp, cp)
        sm, cm = scene.copy(), Camera(cam.rotation.copy(), cam.translation.copy(), cam.focal, cam.ox, cam.oy,
                                      h_img, w_img)
        apply(sm, cm, -step)
        minus = forward(sm, cm)
        if plus is None or minus is None or not np.array_equal(plus[1], base_sets) or \
                not np.array_equal(minus[1], base_sets):
            entry.skipped_boundary += 1
            report.total_skipped += 1
            return
        numeric = (plus[0] - minus[0]) / (2.0 * step)
        rel = _relative_error(analytic, numeric)
        entry.checked += 1
        report.total_checked += 1
        if rel > entry.max_rel_err:
            entry.max_rel_err, entry.worst_analytic, entry.worst_numeric = rel, analytic, numeric
        report.max_rel_err = max(report.max_rel_err, rel)

    for kk in range(k):
        for a in range(3):
            def f(s, c, eps, kk=kk, a=a):
                s.centers[kk, a] += eps
            check("center", float(g_center[kk, a]), f, h * max(1.0, abs(scene.centers[kk, a])))
        for i in range(3):
            for j in range(i, 3):
                analytic = float(g_inv_cov[kk, i, i]) if i == j else 2.0 * float(g_inv_cov[kk, i, j])

                def f(s, c, eps, kk=kk, i=i, j=j):
                    s.inv_cov[kk, i, j] += eps
                    if i != j:
                        s.inv_cov[kk, j, i] += eps
                check("inv_cov", analytic, f, h * max(1.0, abs(scene.inv_cov[kk, i, j])))
        for a in range(d):
            def f(s, c, eps, kk=kk, a=a):
                s.attr[kk, a] += eps
            check("attr", float(g_attr[kk, a]), f, h)

    d_omega = so3_exp_gradient(omega0, g_rot)
    for a in range(3):
        def f(s, c, eps, a=a):
            w = omega0.copy()
            w[a] += eps
            c.rotation = so3_exp(w)
        check("pose", float(d_omega[a]), f, h)
    for a in range(3):
        def f(s, c, eps, a=a):
            c.translation = c.translation.copy()
            c.translation[a] += eps
        check("pose", float(g_trans[a]), f, h * max(1.0, abs(cam.translation[a])))
    return report
