"""Per-line instruction / stall shares of one kernel in an ncu report (source page):
    python tools/ncu_pix.py <rep> <kernel-regex> <units> [min_per_unit]
Prints the metrics summary and each CUDA line above min_per_unit warp-level
thread-instructions per unit (e.g. pixels)."""
import csv
import io
import subprocess
import sys

rep, kern, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
thr = float(sys.argv[4]) if len(sys.argv) > 4 else 3.0
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv", "-k", f"regex:{kern}"], capture_output=True,
                     text=True).stdout
want = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Executed Instructions", "No Eligible", "Eligible Warps Per Scheduler"]
r = list(csv.reader(io.StringIO(det)))
if r:
    h = r[0]
    for row in r[1:]:
        d = dict(zip(h, row))
        if d.get("Metric Name") in want:
            print(f"{d['Metric Name']}: {d['Metric Value']}")
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(x for x in rows if x and x[0] == "Line No")
ie = hdr.index("Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
cur, tot, tots, L = None, 0, 0, []
for x in rows:
    if x and x[0] == "File Path":
        cur = x[1].split("/")[-1]
        continue
    if x and x[0].isdigit() and len(x) == len(hdr):
        a, b = int(x[ie] or 0), int(x[ws] or 0)
        tot += a
        tots += b
        L.append((int(x[0]), cur, a, b, x[1][:72]))
print(f"total {tot * 32 / units:.1f} thread-inst per unit")
for ln, f, a, b, src in L:
    if a * 32 / units > thr or b / max(tots, 1) > 0.015:
        print(f"{f[:12]:12s} {ln:5d} {a * 32 / units:7.1f} {100 * b / max(tots, 1):5.1f}%  {src}")
