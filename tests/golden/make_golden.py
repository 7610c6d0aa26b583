"""Generate the golden vectors in tests/golden/*.npz from the REFERENCE build.

Run in the dev container (needs /root/reference and oracle/_ref/libgvr_ref.so,
i.e. ``make -C oracle ref``):  python tests/golden/make_golden.py

Each file holds the inputs (scene, camera, selection config, upstream
gradients) and the reference outputs of ``gvr::render_with_tape`` (image,
alpha, depth, weight_store as padded top-K idx/W, Tape::traced l/q/sigma) and
``gvr::backward`` (d_center, d_inv_cov, d_attr, d_rotation, d_translation).
Inputs come from the reference's own bundled fixtures
(/root/reference/proj/tests/data/*.json) and from deterministic synthetic
scenes (the reference's bench cuboid, seeded random anisotropic frustum scenes).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2205_15401_b200 import synthetic  # noqa: E402
from paper_2205_15401_b200.scene_io import load_camera_json, load_scene_json  # noqa: E402
from paper_2205_15401_b200.types import Camera, GaussianScene, SelectionConfig  # noqa: E402

DATA = "/root/reference/proj/tests/data"


def random_frustum_scene(seed: int, count: int, attr_dim: int = 3, lo: float = 2.0, hi: float = 30.0,
                         tau: float = 1.0) -> GaussianScene:
    """Analogue of fixtures::random_frustum_scene (proj/tests/fixtures.hpp:81-106) on numpy's RNG."""
    rng = np.random.default_rng(seed)
    centers = np.stack([rng.uniform(-1, 1, count), rng.uniform(-1, 1, count), rng.uniform(3, 6, count)], 1)
    inv = np.empty((count, 3, 3))
    for k in range(count):
        q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        if np.linalg.det(q) < 0:
            q[:, 0] = -q[:, 0]
        ev = rng.uniform(lo, hi, 3)
        m = q @ np.diag(ev) @ q.T
        inv[k] = 0.5 * (m + m.T)
    attr = rng.uniform(0, 1, (count, attr_dim))
    return GaussianScene(centers, inv, attr, tau)


def default_camera(size: int, focal: float) -> Camera:
    return Camera(np.eye(3), np.zeros(3), focal, (size - 1) / 2.0, (size - 1) / 2.0, size, size)


def save(name: str, scene: GaussianScene, cam: Camera, cfg: SelectionConfig, seed: int, traced: bool = True,
         flags=(True, True), extra=None) -> None:
    out = oracle.ref_render(scene, cam, cfg, threads=8)
    rng = np.random.default_rng(seed)
    h, w, d = cam.height, cam.width, scene.attr_dim()
    d_image = rng.uniform(-1, 1, (h, w, d))
    d_alpha = rng.uniform(-1, 1, (h, w, 1))
    g = oracle.ref_backward(scene, cam, cfg, d_image, d_alpha, flags[0], flags[1], threads=8)
    rec = dict(
        centers=scene.centers, inv_cov=scene.inv_cov, attr=scene.attr, tau=np.float64(scene.tau),
        camera=cam.as_array(), eta=np.float64(cfg.eta), k_prime=np.int32(cfg.k_prime),
        coarse=np.int32(cfg.coarse_enabled), ds=np.int32(cfg.coarse_downsample),
        through_transmittance=np.int32(flags[0]), through_density=np.int32(flags[1]),
        image=out["image"], alpha=out["alpha"], depth=out["depth"], topk_idx=out["topk_idx"], topk_w=out["topk_w"],
        d_image=d_image, d_alpha=d_alpha, **g,
    )
    if traced:
        rec.update(topk_l=out["topk_l"], topk_q=out["topk_q"], topk_sigma=out["topk_sigma"])
    if extra is not None:
        rec.update(extra(scene, cam, cfg, out, rng))
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **rec)
    n = (out["topk_idx"] >= 0).sum()
    print(f"{name}: K={scene.size} {h}x{w} selected entries={n} -> {os.path.getsize(path) / 1e3:.0f} kB")


def sampler_extra(scene, cam, cfg, out, rng) -> dict:
    """Reference outputs of the render-path helpers on the same inputs:
    sample_attributes (raw + normalized) of a noisy observation of the render,
    resynthesize with those attributes, per-pixel transmittance_at and
    normalized_weights, and shade_lambert of the rendered image as normals
    (proj/src/sampler.cpp:11-66, proj/src/blender.cpp:19-25, 55-62, 146-172)."""
    h, w = cam.height, cam.width
    observed = out["image"] + rng.uniform(-0.05, 0.05, out["image"].shape)
    sa, ss, sm = oracle.ref_sample_attributes(scene, cam, cfg, observed, False, threads=8)
    na, ns, nm = oracle.ref_sample_attributes(scene, cam, cfg, observed, True, threads=8)
    rs = oracle.ref_resynthesize(scene, cam, cfg, sa, sm, threads=8)
    t = out["depth"][..., 0] + rng.uniform(-0.3, 0.3, (h, w))
    trans, nw = oracle.ref_pixel_helpers(scene, cam, cfg, t, 1e-8, threads=8)
    light_pos, light_color = np.array([1.5, -1.0, 12.0]), np.array([1.0, 0.5, 0.25])
    shade = oracle.ref_shade_lambert(cam, out["image"], out["alpha"], out["depth"], light_pos, light_color)
    return dict(observed=observed, s_attrs=sa, s_support=ss, s_masked=sm, n_attrs=na, n_support=ns, n_masked=nm,
                resynth_image=rs["image"], resynth_alpha=rs["alpha"], t_query=t, trans_at=trans, norm_w=nw,
                light_pos=light_pos, light_color=light_color, shade=shade)


def main() -> None:
    cfg = SelectionConfig()
    save("test_scene", load_scene_json(f"{DATA}/test_scene.json"), load_camera_json(f"{DATA}/test_camera.json"), cfg, 1)
    save("gradcheck_scene", load_scene_json(f"{DATA}/gradcheck_scene.json"),
         load_camera_json(f"{DATA}/gradcheck_camera.json"), cfg, 2)
    save("texture_scene", load_scene_json(f"{DATA}/texture_scene.json"),
         load_camera_json(f"{DATA}/texture_camera.json"), cfg, 3)
    red = load_scene_json(f"{DATA}/part_red.json")
    blue = load_scene_json(f"{DATA}/part_blue.json")
    pair = GaussianScene(np.concatenate([red.centers, blue.centers]), np.concatenate([red.inv_cov, blue.inv_cov]),
                         np.concatenate([red.attr, blue.attr]), red.tau)
    save("fit_parts", pair, load_camera_json(f"{DATA}/fit_camera.json"), cfg, 4)
    # C1: the reference bench cuboid, 1k kernels at 128^2 (bench.cpp:9-24)
    save("bench_c1", synthetic.make_bench_scene(1000), synthetic.make_bench_camera(128), cfg, 5, traced=False)
    # seeded random anisotropic frustum scenes, selection variants from the reference tests
    rs = random_frustum_scene(11, 300, 3, 8.0, 120.0)
    save("random_coarse", rs, default_camera(64, 48.0), cfg, 6)
    save("random_nocoarse", rs, default_camera(64, 48.0), SelectionConfig(coarse_enabled=False), 7)
    save("random_ds5_kp4", rs, default_camera(61, 48.0), SelectionConfig(k_prime=4, coarse_downsample=5), 8)
    save("random_eta03_kp40", random_frustum_scene(12, 120, 2, 2.0, 60.0, tau=2.5), default_camera(47, 30.0),
         SelectionConfig(eta=0.3, k_prime=40), 9)
    rot = synthetic.make_orbit_camera(0.7, 0.3, 4.0, (0, 0, 4), 40, 56, 60.0)
    save("orbit_rect", synthetic.make_bench_scene(2000), rot, cfg, 10)
    save("blocked_t", rs, default_camera(64, 48.0), cfg, 11, flags=(False, True))
    save("blocked_rho", rs, default_camera(64, 48.0), cfg, 12, flags=(True, False))
    # sampler + helpers (sampler.cpp, blender.cpp helpers); a far kernel stays unobserved (masked)
    hs = random_frustum_scene(13, 200, 3, 8.0, 120.0)
    hs.centers[-1] = (0.0, 0.0, 300.0)
    save("sampler_random", hs, default_camera(48, 40.0), SelectionConfig(k_prime=12), 13, extra=sampler_extra)
    regularizer_golden()


def regularizer_golden() -> None:
    """fit.cpp:44-113 on the bench box mesh (divisions 6) with jittered centres."""
    verts, faces = synthetic.make_box_mesh((1.0, 1.0, 1.0), 6, (0.0, 0.0, 4.0))
    edges = synthetic.mesh_edges(faces)
    centers = verts + np.random.default_rng(14).normal(0.0, 0.01, verts.shape)
    ev, eg, lv, lg = oracle.ref_shape_reg(edges, verts, centers)
    path = os.path.join(HERE, "aux", "fit_regularizers.npz")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    np.savez_compressed(path, edges=edges, rest=verts, centers=centers, edge_value=ev, edge_grad=eg,
                        laplacian_value=lv, laplacian_grad=lg)
    print(f"fit_regularizers: V={len(verts)} E={len(edges)} edge={ev:.6e} laplacian={lv:.6e}")


if __name__ == "__main__":
    main()
