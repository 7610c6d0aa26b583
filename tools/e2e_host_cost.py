"""Host cost of one end-to-end C2 step in asynchronous host-buffer mode: the time
the Python caller spends issuing the step's C ABI calls (no waiting), against the
device + copy time of the step. usage: python tools/e2e_host_cost.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2205_15401_b200 as gvr  # noqa: E402
from paper_2205_15401_b200 import synthetic  # noqa: E402

scene = synthetic.make_bench_scene(100000)
cam = synthetic.make_bench_camera(512)
K, H = scene.size, 512
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
rng = np.random.default_rng(0)
h_c, h_s, h_a = pin(scene.centers), pin(scene.inv_cov), pin(scene.attr)
h_ti, h_ta = pin(rng.uniform(0, 1, (H, H, 3))), pin(rng.uniform(0, 1, (H, H, 1)))
c = gvr.Context(0)
c.set_async(True)
sc, tp = gvr.DeviceScene(c), gvr.Tape(c)
o = {k: torch.empty(s, dtype=torch.float64).pin_memory() for k, s in
     dict(img=(H, H, 3), a=(H, H, 1), d=(H, H, 1), l=(1,), gc=(K, 3), gs=(K, 3, 3), ga=(K, 3), gr=(3, 3), gt=(3,)).items()}


def enqueue():
    sc.set_raw(K, 3, scene.tau, h_c, h_s, h_a)
    gvr.render_into(c, sc, cam, gvr.SelectionConfig(), tp, o["img"], o["a"], o["d"])
    gvr.scalar_loss_into(tp, h_ti, h_ta, 1.0, 1.0, o["l"])
    gvr.backward_into(tp, None, None, gvr.GradFlags(), o["gc"], o["gs"], o["ga"], o["gr"], o["gt"])


for _ in range(3):
    enqueue()
    c.synchronize()
host, total = [], []
for _ in range(10):
    t0 = time.perf_counter()
    enqueue()
    t1 = time.perf_counter()
    c.synchronize()
    t2 = time.perf_counter()
    host.append(t1 - t0)
    total.append(t2 - t0)
print(f"host enqueue {1e3 * np.median(host):.3f} ms, enqueue + drain {1e3 * np.median(total):.3f} ms per step")
