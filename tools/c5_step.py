"""A few C5 Fitter iterations (for ncu launch lists): python tools/c5_step.py [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2205_15401_b200 as gvr  # noqa: E402
from paper_2205_15401_b200 import synthetic  # noqa: E402
from paper_2205_15401_b200.fit import AdamConfig, Fitter, make_fit_views  # noqa: E402

ctx = gvr.Context(0)
target = synthetic.make_bench_scene(5e4)
views = make_fit_views(target, 32, 256, ctx=ctx)
start = synthetic.make_bench_scene(5e4)
fitter = Fitter(ctx, start, views, adam=AdamConfig(lr=0.002), device=torch.device("cuda:0"))
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    fitter.step()
print("loss", fitter.loss())
