"""Stall reasons per code region of a kernel, regions split at BAR.SYNC
(python tools/ncu_phase_stalls.py rep.ncu-rep [kernel-regex]).  For the exact
QC decoder the regions are: setup, CN phase, VN phase, outputs."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"]
if len(sys.argv) > 2:
    cmd += ["-k", f"regex:{sys.argv[2]}"]
text = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(text)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
src = hdr.index("Source")
ie = hdr.index("Instructions Executed")
reasons = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
segs = []
cur = None
for r in data:
    if cur is None:
        cur = {"n": 0, "instr": 0, "first": r[src].strip()[:40], "st": [0] * len(reasons)}
        segs.append(cur)
    cur["n"] += 1
    cur["instr"] += int(r[ie] or 0)
    for k, (i, _) in enumerate(reasons):
        cur["st"][k] += int(r[i] or 0)
    if "BAR.SYNC" in r[src]:
        cur = None
tot_i = sum(s["instr"] for s in segs) or 1
tot_s = sum(sum(s["st"]) for s in segs) or 1
for j, s in enumerate(segs):
    if s["instr"] * 100 < tot_i:
        continue
    top = sorted(zip(s["st"], [n for _, n in reasons]), reverse=True)[:6]
    print(f"region {j}: {s['n']} instrs, {100 * s['instr'] / tot_i:.1f}% executed, "
          f"{100 * sum(s['st']) / tot_s:.1f}% of stall samples; first: {s['first']}")
    print("   " + ", ".join(f"{n} {100 * v / max(1, sum(s['st'])):.0f}%" for v, n in top))
