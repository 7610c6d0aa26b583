"""Per-stage device times of one rank's C4 step (shard (0, n) of the 1024^2 /
1M-kernel view) on one GPU: what a rank of an n-GPU run computes, stage by stage.
usage: python tools/c4_shard_stages.py [n ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2205_15401_b200 as gvr  # noqa: E402
from paper_2205_15401_b200 import synthetic  # noqa: E402

ns = [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]
dev = torch.device("cuda:0")
ctx = gvr.Context(0)
stream = torch.cuda.ExternalStream(int(ctx.lib.gvr_context_stream(ctx.handle)), device=dev)
torch.cuda.set_stream(stream)
S = 1024
scene = synthetic.make_bench_scene(1_000_000)
cam = synthetic.make_bench_camera(S)
K = scene.size
ds = gvr.DeviceScene(ctx).set_raw(K, 3, scene.tau, torch.from_numpy(scene.centers).to(dev),
                                  torch.from_numpy(scene.inv_cov).to(dev), torch.from_numpy(scene.attr).to(dev))
tape = gvr.Tape(ctx)
rng = np.random.default_rng(4)
ti = torch.tensor(rng.uniform(0, 1, (S, S, 3)), device=dev)
ta = torch.tensor(rng.uniform(0, 1, (S, S, 1)), device=dev)
img = torch.empty((S, S, 3), dtype=torch.float64, device=dev)
loss = torch.zeros(1, dtype=torch.float64, device=dev)
packed = torch.zeros((K, 12), dtype=torch.float64, device=dev)
d_rt = torch.zeros(12, dtype=torch.float64, device=dev)
for n in ns:
    def step():
        gvr.render_into(ctx, ds, cam, gvr.SelectionConfig(), tape, img, shard=(0, n))
        gvr.scalar_loss_into(tape, ti, ta, 1.0, 1.0, loss)
        gvr.backward_packed_into(tape, None, None, gvr.GradFlags(), packed, d_rt)
    for _ in range(3):
        step()
    ctx.enable_timing(True)
    for _ in range(5):
        step()
    st = ctx.stage_times()
    ctx.enable_timing(False)
    print(n, {k: round(v[0] / 5 * 1e3, 1) for k, v in st.items() if v[1]})
