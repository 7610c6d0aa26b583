"""Summarise a bench.py JSON line: python tools/bsum.py gpurun_out/bench.json"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value", round(d["value"], 1), "ms", round(d["ms_per_step"], 4), "e2e", d["e2e"] and round(d["e2e"]["value"], 1),
      "clocks", d["clocks"])
r = d["roofline"]
print("frac", round(r["frac"], 4), {k: round(v * 1000, 1) for k, v in r["stage_ms_per_step"].items()})
for c in ("c3", "c4", "c5"):
    if d.get(c):
        print(c, round(d[c]["value"], 1), d[c]["unit"], round(d[c]["ms_per_step"], 3), "ms")
if d.get("cpu_baseline"):
    print("cpu", d["cpu_baseline"]["value"])
