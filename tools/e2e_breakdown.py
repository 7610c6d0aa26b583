"""Where the end-to-end C2 step goes: PCIe bandwidth of pinned copies and the
time of each public call with host buffers (wall clock around synchronous calls)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2205_15401_b200 as gvr

dev = torch.device("cuda:0")
for mb in (12, 24):
    h = torch.empty(mb * 2**20 // 8, dtype=torch.float64).pin_memory()
    d = torch.empty_like(h, device=dev)
    for _ in range(3):
        d.copy_(h); h.copy_(d)
    torch.cuda.synchronize()
    t = time.perf_counter(); [d.copy_(h, non_blocking=True) for _ in range(10)]; torch.cuda.synchronize()
    h2d = 10 * mb * 2**20 / (time.perf_counter() - t) / 1e9
    t = time.perf_counter(); [h.copy_(d, non_blocking=True) for _ in range(10)]; torch.cuda.synchronize()
    d2h = 10 * mb * 2**20 / (time.perf_counter() - t) / 1e9
    print(f"pinned {mb} MB: H2D {h2d:.1f} GB/s  D2H {d2h:.1f} GB/s")

ctx = gvr.Context(0)
scene = gvr.make_bench_scene(100000); cam = gvr.make_bench_camera(512); cfg = gvr.SelectionConfig()
K = scene.size; H = W = 512
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
hc, hs, ha = pin(scene.centers), pin(scene.inv_cov), pin(scene.attr)
rng = np.random.default_rng(0)
hti, hta = pin(rng.uniform(0, 1, (H, W, 3))), pin(rng.uniform(0, 1, (H, W, 1)))
himg = torch.empty((H, W, 3), dtype=torch.float64).pin_memory()
hal = torch.empty((H, W, 1), dtype=torch.float64).pin_memory()
hdp = torch.empty((H, W, 1), dtype=torch.float64).pin_memory()
hl = torch.zeros(1, dtype=torch.float64).pin_memory()
hg = [torch.empty(s, dtype=torch.float64).pin_memory() for s in ((K, 3), (K, 3, 3), (K, 3), (3, 3), (3,))]
ds = gvr.DeviceScene(ctx); tp = gvr.Tape(ctx)
calls = {
    "scene_set": lambda: ds.set_raw(K, 3, scene.tau, hc, hs, ha),
    "render": lambda: gvr.render_into(ctx, ds, cam, cfg, tp, himg, hal, hdp),
    "loss": lambda: gvr.scalar_loss_into(tp, hti, hta, 1.0, 1.0, hl),
    "backward": lambda: gvr.backward_into(tp, None, None, gvr.GradFlags(), *hg),
}
for _ in range(3):
    for f in calls.values(): f()
ctx.synchronize()
acc = {k: 0.0 for k in calls}
n = 20
for _ in range(n):
    for k, f in calls.items():
        t = time.perf_counter(); f(); ctx.synchronize(); acc[k] += time.perf_counter() - t
tot = sum(acc.values()) / n
print("per call (ms):", {k: round(v / n * 1e3, 3) for k, v in acc.items()}, f"total {tot * 1e3:.3f} ms = {1 / tot:.0f} renders/s")
