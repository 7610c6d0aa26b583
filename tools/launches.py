"""Per-kernel device times from an ncu launch list (--metrics gpu__time_duration.sum --csv):
python tools/launches.py gpurun_out/launches.csv  -> the last launch of each kernel (us)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            agg.setdefault(d["Kernel Name"].split("(")[0], []).append(float(d["Metric Value"]))
for n, v in agg.items():
    print(f"{n[:60]:60s} n={len(v):3d} last={v[-1] / 1000:8.1f} us")
