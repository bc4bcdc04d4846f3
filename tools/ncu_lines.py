"""Per-CUDA-line instruction and stall-sample shares from an ncu report:
    python tools/ncu_lines.py <report> <kernel-regex> [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
fname, hdr, data = "?", None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        ii = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            data.append((int(r[ii] or 0), int(r[si] or 0), f"{fname}:{r[0]}", r[1].strip()[:90]))
        except ValueError:
            pass
tot = sum(d[0] for d in data) or 1
tots = sum(d[1] for d in data) or 1
print(f"total warp-inst {tot}  stall samples {tots}")
for d in sorted(data, key=lambda x: -x[1])[:top]:
    print(f"{100 * d[0] / tot:5.1f}% inst {100 * d[1] / tots:5.1f}% smpl  {d[2]}: {d[3]}")
