"""Scratch timing of the C2 fwd+bwd step (device-resident inputs)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2205_15401_b200 as gvr

ctx = gvr.default_context(0)
scene = gvr.make_bench_scene(100000)
cam = gvr.make_bench_camera(512)
cfg = gvr.SelectionConfig()
ds = gvr.DeviceScene(ctx).set(scene)
tape = gvr.Tape(ctx)
H = W = 512
dev = torch.device("cuda:0")
img = torch.empty((H, W, 3), dtype=torch.float64, device=dev)
al = torch.empty((H, W, 1), dtype=torch.float64, device=dev)
dp = torch.empty((H, W, 1), dtype=torch.float64, device=dev)
rng = np.random.default_rng(0)
ti = torch.tensor(rng.uniform(0, 1, (H, W, 3)), device=dev)
ta = torch.tensor(rng.uniform(0, 1, (H, W, 1)), device=dev)
loss_d = torch.zeros(1, dtype=torch.float64, device=dev)
grads = dict(d_center=torch.empty((ds.K, 3), dtype=torch.float64, device=dev),
             d_attr=torch.empty((ds.K, 3), dtype=torch.float64, device=dev))
import ctypes
from paper_2205_15401_b200.render import _ptr
def step():
    gvr.render_into(ctx, ds, cam, cfg, tape, img, al, dp)
    ctx.check(ctx.lib.gvr_scalar_loss(ctx.handle, tape.handle, _ptr(ti), _ptr(ta), 1.0, 1.0, _ptr(loss_d), None, None))
    gvr.backward_into(tape, None, None, gvr.GradFlags(), grads["d_center"], None, grads["d_attr"])
for _ in range(3): step()
ctx.synchronize()
for mode in ["fwd", "fwdbwd"]:
    n = 20
    ctx.synchronize(); t = time.perf_counter()
    for _ in range(n):
        if mode == "fwd": gvr.render_into(ctx, ds, cam, cfg, tape, img, al, dp)
        else: step()
    ctx.synchronize(); dt = (time.perf_counter() - t) / n
    print(f"{mode}: {dt*1e3:.3f} ms/step  {1/dt:.1f} renders/s", flush=True)
print("loss", loss_d.item(), "launches", ctx.launch_count)
