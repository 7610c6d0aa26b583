"""Small fwd+bwd (+ views, + sampler) for compute-sanitizer runs:
compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_smoke.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_15401_b200 as gvr
from paper_2205_15401_b200.types import SelectionConfig

ctx = gvr.Context()
scene = gvr.make_bench_scene(3000)
for size, kp in ((40, 20), (33, 40)):
    cam = gvr.make_orbit_camera(0.3, 0.3, 4.0, (0, 0, 4), size, size, 1.6 * size)
    fr = gvr.render_with_tape(scene, cam, SelectionConfig(k_prime=kp), ctx=ctx)
    rng = np.random.default_rng(0)
    g = gvr.backward(fr, fr.buffers.image - rng.uniform(0, 1, fr.buffers.image.shape),
                     fr.buffers.alpha - rng.uniform(0, 1, fr.buffers.alpha.shape))
    print(size, kp, float(np.abs(g.d_center).sum()))
ctx.set_tile_capacity(8)  # overflow path
fr = gvr.render_with_tape(scene, gvr.make_bench_camera(48), SelectionConfig(), ctx=ctx)
print("overflow", float(fr.buffers.image.sum()))
print("sanitize smoke ok")
