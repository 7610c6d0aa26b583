"""Work counters of the benchmark workloads, taken from the REFERENCE build on
the same synthetic inputs (implementation independent):
C = sum_p |candidates(p)|, N1 = sum_p n_p, N2 = sum_p n_p^2.
Writes bench_workcounts.json (committed; bench.py reads it for the roofline)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle
from paper_2205_15401_b200 import synthetic
from paper_2205_15401_b200.types import SelectionConfig

out = {}
for name, n, size in [("C1", 1000, 128), ("C2", 100000, 512), ("C5_view", 50000, 256)]:
    scene = synthetic.make_bench_scene(n)
    cam = synthetic.make_bench_camera(size)
    wc = oracle.ref_work_counts(scene, cam, SelectionConfig(), threads=8)
    out[name] = dict(kernels=scene.size, image=size, C=int(wc["C"]), N1=int(wc["N1"]), N2=int(wc["N2"]),
                     source="oracle/_ref (reference build) gvr_ref_work_counts")
    print(name, out[name])
json.dump(out, open(os.path.join(ROOT, "bench_workcounts.json"), "w"), indent=1)
