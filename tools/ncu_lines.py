"""Summarise an ncu source page (--page source --csv --print-source cuda,sass):
per CUDA source line, warp-stall samples and warp-instructions executed.
usage: ncu_lines.py file.csv [top]"""
import csv, os, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
lines, cur, hdr = [], "?", None
tot_s = tot_i = 0
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = os.path.basename(r[1]); continue
    if r and r[0] == "Line No":
        hdr = r; S = hdr.index('Warp Stall Sampling (All Samples)'); I = hdr.index('Instructions Executed'); continue
    if hdr is None or len(r) < len(hdr) or not r[0]:
        continue
    try:
        s, ins = int(r[S]), int(r[I])
    except ValueError:
        continue
    lines.append((s, ins, f"{cur}:{r[0]}", r[1][:100])); tot_s += s; tot_i += ins
print(f"total samples {tot_s}  total warp-instructions {tot_i/1e6:.1f}M")
for s, ins, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100*s/max(tot_s,1):5.1f}% smp {100*ins/max(tot_i,1):5.1f}% ins  {ln:>22}: {src}")
