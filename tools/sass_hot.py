"""Summarise an ncu SASS source page (ncu -i X --page source --csv --print-source sass):
stall totals and the hottest instructions by warp-stall samples.
usage: python tools/sass_hot.py page.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
data = rows[2:]
col = {h: i for i, h in enumerate(hdr)}
def num(r, name):
    try:
        return float(r[col[name]].replace(",", ""))
    except (ValueError, KeyError, IndexError):
        return 0.0
tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
inst = sum(num(r, "Instructions Executed") for r in data)
print(f"samples {tot:.0f}  warp instructions {inst:.0f}  sass lines {len(data)}")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
st = sorted(((sum(num(r, h) for r in data), h) for h in stalls), reverse=True)
print("stalls:", ", ".join(f"{h[6:]} {v / max(tot, 1):.1%}" for v, h in st if v > 0))
rank = sorted(data, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))
for r in rank[:top]:
    s = num(r, "Warp Stall Sampling (All Samples)")
    main = max(stalls, key=lambda h: num(r, h))
    print(f"{r[col['Address']]:>6} {s / max(tot, 1):6.2%} ex={num(r, 'Instructions Executed'):>9.0f} "
          f"thr={num(r, 'Avg. Threads Executed'):4.1f} {main[6:]:<14} {r[col['Source']][:70]}")
