"""Instruction / stall shares of an ncu report per source region.
    python tools/ncu_regions.py <report> <kernel-regex> <file> <npx> marker1 marker2 ...
Each marker is a substring of a line in <file> or a line number "L<n>";
regions run between markers."""
import csv
import io
import re
import subprocess
import sys

rep, kern, fname, npx = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
marks = sys.argv[5:]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
cur, hdr, data = None, None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        ii = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        data.append((int(r[ii] or 0), int(r[si] or 0), cur, int(r[0])))
tot = sum(d[0] for d in data) or 1
tots = sum(d[1] for d in data) or 1
src = open(fname).read().splitlines()
base = fname.split("/")[-1]
pos = []
for m in marks:
    if re.fullmatch(r"L\d+", m):  # a line number
        ln = int(m[1:])
    else:
        ln = next((i + 1 for i, l in enumerate(src) if m in l), None)
    pos.append((m[:24], ln))
pos.append(("<end>", len(src) + 1))
print(f"total {tot * 32 / npx:.1f} thread-inst/px")
for (n, a), (_, b) in zip(pos, pos[1:]):
    if a is None:
        continue
    s = sum(d[0] for d in data if d[2] == base and a <= d[3] < b)
    ss = sum(d[1] for d in data if d[2] == base and a <= d[3] < b)
    print(f"{n:26s} inst {100 * s / tot:5.1f}% ({s * 32 / npx:7.1f}/px)  stall {100 * ss / tots:5.1f}%")
other = sum(d[0] for d in data if d[2] != base)
print(f"other files {other * 32 / npx:.1f}/px")
