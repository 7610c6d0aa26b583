"""Summarise a profiling session (tools/profile_round.sh output in gpurun_out/)
into profiles/: the per-launch list of one timed step, per-kernel ncu metrics of
the full captures, and profiles/ncu_traffic.json (DRAM bytes per launch, read by
bench.py's roofline.traffic).

usage: python tools/summarize_profiles.py <round-tag>
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
METRICS = [
    "gpu__time_duration.sum", "sm__cycles_active.avg", "sm__cycles_active.max", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__maximum_warps_per_active_cycle_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v.replace(",", "")) * scale


def launch_list(tag):
    path = os.path.join(OUT, "launches.csv")
    if not os.path.exists(path):
        return None
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    ks = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[h + 1:] if len(r) > vi]
    last = max(i for i, (k, _) in enumerate(ks) if "project_kernel" in k)
    if last > 0 and "clear_kernel" in ks[last - 1][0]:  # the render's first launch
        last -= 1
    step = [kv for kv in ks[last:] if "fma_peak" not in kv[0]]
    total = sum(v for _, v in step)
    lines = ["kernel,ns,share"]
    for k, v in step:
        lines.append(f"\"{k[:120]}\",{v:.0f},{v / total:.4f}")
    open(os.path.join(PROF, f"{tag}_launches_one_step.csv"), "w").write("\n".join(lines) + "\n")
    return step, total


def ncu_metrics(rep):
    if rep.endswith(".raw.csv"):  # exported on the GPU box (tools/profile_round.sh)
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, row = rows[0], rows[1], rows[2]
    res = {"kernel": row[hdr.index("Kernel Name")]}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            res[m] = (row[i], units[i])
    return res


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "round"
    os.makedirs(PROF, exist_ok=True)
    md = [f"# ncu summary — {tag}", ""]
    ll = launch_list(tag)
    if ll:
        step, total = ll
        md += [f"One timed C2 fwd+bwd step (ncu launch list, serialised, cold cache): {len(step)} launches, "
               f"{total / 1e3:.1f} us total.", "", "| kernel | us | share |", "|---|---|---|"]
        for k, v in step:
            md.append(f"| `{k.split('(')[0][:70]}` | {v / 1e3:.1f} | {100 * v / total:.1f}% |")
        md.append("")
    traffic = {}
    issue = {}
    for f in sorted(os.listdir(OUT)):
        if f.startswith("full_") and (f.endswith(".ncu-rep") or f.endswith(".raw.csv")):
            m = ncu_metrics(os.path.join(OUT, f))
            name = m["kernel"].split("(")[0].split("<")[0].replace("void ", "").replace("gvrk::", "")
            rb = to_bytes(*m["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in m else 0.0
            wb = to_bytes(*m["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in m else 0.0
            traffic[name] = rb + wb
            key = "smsp__issue_active.avg.pct_of_peak_sustained_active"
            if key in m:
                issue[name] = float(m[key][0].replace(",", ""))
            md += [f"## `{name}` (ncu --set full)", "", "| metric | value |", "|---|---|"]
            for k in METRICS:
                if k in m:
                    md.append(f"| {k} | {m[k][0]} {m[k][1]} |")
            md.append("")
    json.dump(traffic, open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)
    if issue:
        json.dump(issue, open(os.path.join(PROF, "ncu_issue.json"), "w"), indent=1)
    open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
