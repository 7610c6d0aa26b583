"""Attribute an ncu SASS source page to CUDA source lines.

usage: python tools/sass_lines.py <ncu sass csv> <cubin> <mangled kernel> [top]
The ncu rows are the kernel's SASS in program order; nvdisasm -gi of the same
cubin gives each instruction's (innermost) source line and the kernel-level line
it is inlined at. Prints warp-stall samples and executed instructions per line."""
import collections
import csv
import re
import subprocess
import sys

page, cubin, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(open(page)))
hdr = rows[1]
col = {h: i for i, h in enumerate(hdr)}
data = rows[2:]


def num(r, name):
    try:
        return float(r[col[name]].replace(",", ""))
    except (ValueError, KeyError, IndexError):
        return 0.0


dis = subprocess.run(["nvdisasm", "-c", "-gi", cubin], capture_output=True, text=True).stdout
sec = dis.split(f".text.{fn}:", 1)[1].split("//--------------------- .text.", 1)[0]
cur_inner, cur_outer = "?", "?"
lines = []
for ln in sec.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
    if m:
        f1 = m.group(1).rsplit("/", 1)[-1]
        cur_inner = f"{f1}:{m.group(2)}"
        cur_outer = f"{m.group(3).rsplit('/', 1)[-1]}:{m.group(4)}" if m.group(3) else cur_inner
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
        lines.append((cur_inner, cur_outer, ln.strip()))
if len(lines) != len(data):
    print(f"warning: {len(lines)} sass lines in cubin vs {len(data)} in the ncu page", file=sys.stderr)
tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data) or 1.0
by_inner = collections.defaultdict(lambda: [0.0, 0.0])
by_outer = collections.defaultdict(lambda: [0.0, 0.0])
for (inner, outer, _), r in zip(lines, data):
    s, e = num(r, "Warp Stall Sampling (All Samples)"), num(r, "Instructions Executed")
    by_inner[inner][0] += s
    by_inner[inner][1] += e
    by_outer[outer][0] += s
    by_outer[outer][1] += e
for title, d in (("kernel-level line", by_outer), ("innermost line", by_inner)):
    print(f"== by {title}: samples share, warp instructions")
    for k, (s, e) in sorted(d.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"  {k:<22} {s / tot:6.1%} {e:>12.0f}")
