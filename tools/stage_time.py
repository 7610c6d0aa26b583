"""Per-stage device times of the C2 fwd+bwd step for one or more library builds
(A/B experiments): python tools/stage_time.py build_ab/a.so build_ab/b.so ...
(GVR_NK / GVR_S select another bench scene size / image size, e.g. C4: 1000000 / 1024)
Each build runs in a fresh subprocess (GVR_LIB_PATH); prints ms per stage and per step,
plus a checksum of the outputs so that variants can be compared for equality."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import os, sys, json, numpy as np, torch
sys.path.insert(0, ROOT)
import paper_2205_15401_b200 as gvr
ctx = gvr.Context(0)
stream = torch.cuda.ExternalStream(int(ctx.lib.gvr_context_stream(ctx.handle)), device="cuda:0")
torch.cuda.set_stream(stream)
NK = int(os.environ.get("GVR_NK", "100000")); S = int(os.environ.get("GVR_S", "512"))
scene = gvr.make_bench_scene(NK); cam = gvr.make_bench_camera(S); cfg = gvr.SelectionConfig()
ds = gvr.DeviceScene(ctx).set(scene); tape = gvr.Tape(ctx)
dev = torch.device("cuda:0"); H = W = S
img = torch.empty((H, W, 3), dtype=torch.float64, device=dev)
al = torch.empty((H, W, 1), dtype=torch.float64, device=dev); dp = torch.empty((H, W, 1), dtype=torch.float64, device=dev)
rng = np.random.default_rng(0)
ti = torch.tensor(rng.uniform(0, 1, (H, W, 3)), device=dev); ta = torch.tensor(rng.uniform(0, 1, (H, W, 1)), device=dev)
loss = torch.zeros(1, dtype=torch.float64, device=dev)
gc = torch.empty((ds.K, 3), dtype=torch.float64, device=dev); gs = torch.empty((ds.K, 3, 3), dtype=torch.float64, device=dev)
ga = torch.empty((ds.K, 3), dtype=torch.float64, device=dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
def step():
    gvr.render_into(ctx, ds, cam, cfg, tape, img, al, dp)
    gvr.scalar_loss_into(tape, ti, ta, 1.0, 1.0, loss)
    gvr.backward_into(tape, None, None, gvr.GradFlags(), gc, gs, ga)
for _ in range(5): step()
torch.cuda.synchronize()
with ctx.capture() as g:
    step()
for _ in range(3): g.launch()
torch.cuda.synchronize()
n = 40
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
for a, b in ev:
    flush.zero_(); a.record(stream); g.launch(); b.record(stream)
torch.cuda.synchronize()
ms = sorted(a.elapsed_time(b) for a, b in ev)
ctx.enable_timing(True)
for _ in range(20):
    flush.zero_(); step()
torch.cuda.synchronize()
st = {k: v[0] / 20 for k, v in ctx.stage_times().items() if v[1]}
out = dict(step_ms_med=ms[n // 2], step_ms_mean=sum(ms) / n, stages=st, loss=float(loss.item()),
           img=float(img.sum().item()), gc=float(gc.abs().sum().item()), gs=float(gs.abs().sum().item()))
print("RESULT " + json.dumps(out))
'''

for lib in sys.argv[1:]:
    env = dict(os.environ, GVR_LIB_PATH=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", "ROOT=%r\n" % ROOT + CHILD], env=env, capture_output=True, text=True)
    line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
    if not line:
        print(lib, "FAILED", r.stderr[-2000:])
        continue
    d = json.loads(line[0][7:])
    st = " ".join(f"{k}={v * 1000:.1f}" for k, v in d["stages"].items())
    print(f"{os.path.basename(lib):<24} step {d['step_ms_med'] * 1000:.1f}us (mean {d['step_ms_mean'] * 1000:.1f})  "
          f"{st}  | loss {d['loss']:.9e} img {d['img']:.9e} gc {d['gc']:.9e} gs {d['gs']:.9e}", flush=True)
