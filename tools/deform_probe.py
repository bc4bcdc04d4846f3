"""k_canvas_deform timing: min over repeated ping-pong passes of an n x n
canvas through a smooth canvas-wide field (bench.py canvas_lattice).
    python tools/deform_probe.py [n]"""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
from paper_2103_07414_b200 import mosaic as M

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
ctx = M.Context(0)
ctx.set_stream(st.cuda_stream)
a, q, alpha = bench.canvas_lattice(n)
disp = torch.empty((n, n, 2), dtype=torch.float32, device=dev)
M.node_field_device((0.0, 0.0, n, n), torch.from_numpy(a).to(dev), torch.from_numpy(q).to(dev), alpha, disp, None,
                    ctx=ctx)
r = bench.deform_numbers(ctx, st, n, disp, 6451.2)
print(json.dumps({"ms": r["ms"], "frac": r["roofline_k_canvas_deform"]["frac"]}))
