"""Per CUDA source line totals from an ncu mixed page
(ncu -i X --page source --csv --print-source cuda,sass): warp-stall samples and
warp-instructions of the SASS rows under each source line (inlined code is
attributed to the line it came from). usage: ncu_mixed.py page.csv [top]"""
import csv
import os
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
acc = defaultdict(lambda: [0, 0])
src = {}
cur_file, cur_line, hdr = "?", None, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = os.path.basename(r[1])
        continue
    if r and r[0] == "Line No":
        hdr = r
        S = 4
        I = 7
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur_line = f"{cur_file}:{r[0]}"
        src[cur_line] = r[1].strip()[:90]
        continue
    try:
        s, ins = int(r[S]), int(r[I])
    except ValueError:
        continue
    acc[cur_line][0] += s
    acc[cur_line][1] += ins
ts = sum(v[0] for v in acc.values())
ti = sum(v[1] for v in acc.values())
print(f"samples {ts}  warp-instructions {ti/1e6:.2f}M")
for k, (s, i) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/max(ts,1):5.1f}% smp {100*i/max(ti,1):5.1f}% ins {k:>20}: {src.get(k,'')}")
