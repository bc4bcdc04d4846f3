"""Stall reasons per source region from an ncu report (source page, SASS
correlated): python tools/ncu_stalls.py <rep> <kernel-regex> <file> marker1 ...
A marker is a substring of a source line or a line number "L<n>"."""
import csv
import io
import re
import subprocess
import sys

rep, kern, fname = sys.argv[1], sys.argv[2], sys.argv[3]
marks = sys.argv[4:]
src = open(fname).read().splitlines()
starts = []
for m in marks:
    ln = int(m[1:]) if re.fullmatch(r"L\d+", m) else next(i + 1 for i, l in enumerate(src) if m in l)
    starts.append((ln, m))
starts.sort()
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
base = fname.split("/")[-1]
cur, hdr = None, None
agg = {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit() or cur != base or "stall_wait" not in hdr:
        continue
    ln = int(r[0])
    reg = "pre"
    for s_, m in starts:
        if ln >= s_:
            reg = m[:40]
    d = agg.setdefault(reg, {})
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                d[h[6:]] = d.get(h[6:], 0) + int(r[i] or 0)
            except ValueError:
                pass
tot = sum(sum(v.values()) for v in agg.values()) or 1
for reg, d in agg.items():
    s = sum(d.values())
    top = sorted(d.items(), key=lambda kv: -kv[1])[:6]
    print(f"{reg:42s} {100 * s / tot:5.1f}%  " + "  ".join(f"{k}:{100 * v / tot:.1f}" for k, v in top))
