"""DRAM traffic per kernel launch (dram__bytes_read.sum + dram__bytes_write.sum)
from an `ncu --set full` report -> profiles/traffic.json (bytes, per launch),
and warp instructions per launch (smsp__inst_executed.sum) ->
profiles/instructions.json (bench.py's issue-rate view).
    python tools/ncu_traffic.py <report.ncu-rep> [out.json]"""
import csv
import io
import json
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
rep = sys.argv[1]
out_path = sys.argv[2] if len(sys.argv) > 2 else "profiles/traffic.json"
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, units = rows[0], rows[1]
ki = h.index("Kernel Name")
ri, wi = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
ti = h.index("gpu__time_duration.sum")
ii = h.index("smsp__inst_executed.sum")
out = {}
for row in rows[2:]:
    name = row[ki].split("(")[0].split("::")[-1].split("<")[0]
    b = float(row[ri]) * UNIT[units[ri]] + float(row[wi]) * UNIT[units[wi]]
    out.setdefault(name, {"dram_bytes_per_launch": b, "ncu_us": float(row[ti]),
                          "warp_inst_per_launch": float(row[ii].replace(",", ""))})
print(json.dumps(out, indent=1))
json.dump({k: v["dram_bytes_per_launch"] for k, v in out.items()}, open(out_path, "w"), indent=1)
inst_path = out_path.replace("traffic.json", "instructions.json")
json.dump({k: v["warp_inst_per_launch"] for k, v in out.items()}, open(inst_path, "w"), indent=1)
