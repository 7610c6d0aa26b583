"""A few fwd + bwd steps of the bench workload on cuda:0 (for ncu launch lists):
python tools/one_step.py [n_kernels] [image_size] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2205_15401_b200 as gvr  # noqa: E402

NK = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
S = int(sys.argv[2]) if len(sys.argv) > 2 else 512
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
ctx = gvr.Context(0)
torch.cuda.set_stream(torch.cuda.ExternalStream(int(ctx.lib.gvr_context_stream(ctx.handle)), device="cuda:0"))
scene = gvr.make_bench_scene(NK)
cam = gvr.make_bench_camera(S)
ds = gvr.DeviceScene(ctx).set(scene)
tape = gvr.Tape(ctx)
dev = torch.device("cuda:0")
img = torch.empty((S, S, 3), dtype=torch.float64, device=dev)
al = torch.empty((S, S, 1), dtype=torch.float64, device=dev)
dp = torch.empty((S, S, 1), dtype=torch.float64, device=dev)
rng = np.random.default_rng(0)
ti = torch.tensor(rng.uniform(0, 1, (S, S, 3)), device=dev)
ta = torch.tensor(rng.uniform(0, 1, (S, S, 1)), device=dev)
loss = torch.zeros(1, dtype=torch.float64, device=dev)
gc = torch.empty((ds.K, 3), dtype=torch.float64, device=dev)
gs = torch.empty((ds.K, 3, 3), dtype=torch.float64, device=dev)
ga = torch.empty((ds.K, 3), dtype=torch.float64, device=dev)
for _ in range(steps):
    gvr.render_into(ctx, ds, cam, gvr.SelectionConfig(), tape, img, al, dp)
    gvr.scalar_loss_into(tape, ti, ta, 1.0, 1.0, loss)
    gvr.backward_into(tape, None, None, gvr.GradFlags(), gc, gs, ga)
ctx.synchronize()
print("loss", float(loss[0]))
