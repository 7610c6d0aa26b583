"""Where the pipelined end-to-end C2 step is bound: pinned-copy bandwidth per
direction and both directions at once, then the e2e loop of bench.py
(measure_e2e) for several slot counts / step counts, with the scene uploaded
every step or once. Scratch experiment: python tools/e2e_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2205_15401_b200 as gvr  # noqa: E402

dev = torch.device("cuda:0")
mb = 22
h1 = torch.empty(mb * 2**20 // 8, dtype=torch.float64).pin_memory()
h2 = torch.empty_like(h1).pin_memory()
d1 = torch.empty_like(h1, device=dev)
d2 = torch.empty_like(h1, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d1.copy_(h1)
    h2.copy_(d2)
torch.cuda.synchronize()
n = 20
t = time.perf_counter()
with torch.cuda.stream(s1):
    for _ in range(n):
        d1.copy_(h1, non_blocking=True)
torch.cuda.synchronize()
h2d = n * mb * 2**20 / (time.perf_counter() - t) / 1e9
t = time.perf_counter()
with torch.cuda.stream(s2):
    for _ in range(n):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
d2h = n * mb * 2**20 / (time.perf_counter() - t) / 1e9
t = time.perf_counter()
with torch.cuda.stream(s1):
    for _ in range(n):
        d1.copy_(h1, non_blocking=True)
with torch.cuda.stream(s2):
    for _ in range(n):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
both = 2 * n * mb * 2**20 / (time.perf_counter() - t) / 1e9
print(f"pinned {mb} MB: H2D {h2d:.1f} GB/s, D2H {d2h:.1f} GB/s, both directions at once {both:.1f} GB/s total",
      flush=True)

scene = gvr.make_bench_scene(100000)
cam = gvr.make_bench_camera(512)
cfg = gvr.SelectionConfig()
K = scene.size
H = W = 512
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
h_c, h_s, h_a = pin(scene.centers), pin(scene.inv_cov), pin(scene.attr)
rng = np.random.default_rng(0)
h_ti, h_ta = pin(rng.uniform(0, 1, (H, W, 3))), pin(rng.uniform(0, 1, (H, W, 1)))


def run(ns, steps, upload_each, device_io=False):
    slots = []
    loc = dev if device_io else "cpu"
    mk = (lambda *shape: torch.empty(shape, dtype=torch.float64, device=dev)) if device_io else \
        (lambda *shape: torch.empty(shape, dtype=torch.float64).pin_memory())
    for _ in range(ns):
        c = gvr.Context(0)
        c.set_async(True)
        out = dict(img=mk(H, W, 3), alpha=mk(H, W, 1), depth=mk(H, W, 1), loss=mk(1), gc=mk(K, 3), gs=mk(K, 3, 3),
                   ga=mk(K, 3), gr=mk(3, 3), gt=mk(3), ti=h_ti.to(loc), ta=h_ta.to(loc))
        sc = gvr.DeviceScene(c)
        sc.set_raw(K, 3, scene.tau, h_c, h_s, h_a)
        slots.append((c, sc, gvr.Tape(c), out))

    def enqueue(slot):
        c, sc, tp, o = slot
        if upload_each:
            sc.set_raw(K, 3, scene.tau, h_c, h_s, h_a)
        gvr.render_into(c, sc, cam, cfg, tp, o["img"], o["alpha"], o["depth"])
        gvr.scalar_loss_into(tp, o["ti"], o["ta"], 1.0, 1.0, o["loss"])
        gvr.backward_into(tp, None, None, gvr.GradFlags(), o["gc"], o["gs"], o["ga"], o["gr"], o["gt"])

    def consume(slot):
        c, sc, tp, o = slot
        c.synchronize()
        sc.check()
        tp.check_finite()

    for i in range(2 * ns):
        enqueue(slots[i % ns])
        consume(slots[i % ns])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(steps):
        if i >= ns:
            consume(slots[i % ns])
        enqueue(slots[i % ns])
    for i in range(max(0, steps - ns), steps):
        consume(slots[i % ns])
    ms = (time.perf_counter() - t0) * 1e3 / steps
    print(f"slots {ns} steps {steps} scene upload {'every step' if upload_each else 'once'}"
          f"{' device buffers' if device_io else ''}: "
          f"{ms:.3f} ms/step = {1e3 / ms:.0f} renders/s", flush=True)


for ns in (1, 2, 4):
    run(ns, 200, False, device_io=True)
for ns, steps, up in [(4, 200, True), (4, 200, False), (6, 200, False)]:
    run(ns, steps, up)
