"""Summarise an .ncu-rep: headline metrics, pipe utilisation, top stall reasons,
and the instruction mix (python tools/ncu_summary.py file.ncu-rep)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = ("Duration", "Executed Ipc Active", "Issued Instructions", "Registers Per Thread", "Achieved Occupancy",
        "No Eligible", "Block Size", "Dynamic Shared Memory Per Block", "DRAM Throughput", "Memory Throughput",
        "L1/TEX Hit Rate", "Grid Size", "SM Frequency")
drows = list(csv.reader(io.StringIO(det)))
ni, ui, vi = (drows[0].index(x) for x in ("Metric Name", "Metric Unit", "Metric Value"))
for r in drows[1:]:
    if len(r) > vi and r[ni] in want:
        print(f"{r[ni]:34s} {r[vi]} {r[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2]
stalls, pipes = [], []
for h, v in zip(hdr, vals):
    try:
        f = float(v.replace(",", ""))
    except ValueError:
        continue
    if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
        stalls.append((f, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    if h.startswith("sm__inst_executed_pipe_") and h.endswith(".avg.pct_of_peak_sustained_active"):
        pipes.append((f, h[len("sm__inst_executed_pipe_"):-len(".avg.pct_of_peak_sustained_active")]))
    if h in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        print(f"{h:34s} {f}")
print("pipes (% of peak):", ", ".join(f"{n} {v:.1f}" for v, n in sorted(pipes, reverse=True)[:6]))
print("stalls (per issue):", ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)[:8]))
