"""Experiment: histogram of eligible candidates per 32-candidate batch of the select
kernel (build with -DGVR_SEL_STATS; GVR_LIB_PATH points at that build)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_15401_b200 as gvr
from paper_2205_15401_b200 import synthetic
from paper_2205_15401_b200.types import SelectionConfig
ctx = gvr.Context(); ctx.set_tile_profile(True)
ds = gvr.DeviceScene(ctx).set(synthetic.make_bench_scene(100000))
fr = gvr.render_with_tape(ds, synthetic.make_bench_camera(512), SelectionConfig(), ctx=ctx)
h = fr.tape.tile_cycles().ravel()[:66].astype(np.int64)
for name, hh in (("list empty", h[:33]), ("list non-empty", h[33:66])):
    tot = hh.sum(); ins = (hh * np.arange(33)).sum()
    print(f"{name}: batches {tot}, eligible {ins}, mean {ins / max(tot, 1):.2f}")
    print("  ", {i: int(c) for i, c in enumerate(hh) if c})
