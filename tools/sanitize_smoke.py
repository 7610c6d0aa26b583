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
ctx.set_tile_capacity(0)
# repeated view on one tape (the last render's cycles order the tiles), async host buffers
import torch  # noqa: E402
c2 = gvr.Context()
c2.set_async(True)
ds = gvr.DeviceScene(c2).set(scene)
tp = gvr.Tape(c2)
cam = gvr.make_bench_camera(48)
img = torch.empty((48, 48, 3), dtype=torch.float64).pin_memory()
gc = torch.empty((scene.size, 3), dtype=torch.float64).pin_memory()
ti = torch.rand((48, 48, 3), dtype=torch.float64).pin_memory()
ta = torch.rand((48, 48, 1), dtype=torch.float64).pin_memory()
loss = torch.zeros(1, dtype=torch.float64).pin_memory()
for _ in range(3):
    gvr.render_into(c2, ds, cam, SelectionConfig(), tp, img)
    gvr.scalar_loss_into(tp, ti, ta, 1.0, 1.0, loss)
    gvr.backward_into(tp, None, None, gvr.GradFlags(), gc)
c2.synchronize()
print("async repeated view", float(loss[0]), float(gc.abs().sum()))
print("sanitize smoke ok")
