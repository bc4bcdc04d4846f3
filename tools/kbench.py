"""Development: per-kernel average times (library CUDA-event profiling) of the
C2 step, for comparing variants: NRM_B200_VARIANT=<name> python tools/kbench.py"""
import json
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2103_07414_b200 import mosaic as M
from paper_2103_07414_b200 import workload as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
wl = W.frame_workload(cfg)
dev = torch.device("cuda", 0)
s = torch.cuda.Stream(dev)
torch.cuda.set_stream(s)
ctx = M.Context(0)
ctx.set_stream(s.cuda_stream)
poly = M.invert_frame_boundary(wl.frame_w, wl.frame_h, wl.anchors, wl.warps, wl.params.alpha, ctx=ctx)
cv = M.Canvas(ctx)
cv.ensure_contains(wl.canvas_rect)
e = wl.emdq
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
frame_t, anc, war = T(wl.frame), T(wl.anchors), T(wl.warps)
apts, loc, prob, act = T(e.apts), T(e.locals_), T(e.probs), T(e.active)
disp = torch.empty((wl.frame_h, wl.frame_w, 2), dtype=torch.float32, device=dev)
unc = torch.empty((wl.frame_h, wl.frame_w), dtype=torch.float32, device=dev)
st = torch.zeros(4, dtype=torch.int64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def step():
    M.emdq_field_device((0.0, 0.0, wl.frame_w, wl.frame_h), apts, loc, prob, act, wl.params.alpha, wl.params.beta,
                        disp, unc, 16, ctx=ctx)
    M.blend_frame_device(cv, frame_t, wl.frame_w, wl.frame_h, 3, anc, war, wl.params.alpha, poly, st)


for _ in range(5):
    step()
ctx.profile(True)
for _ in range(steps):
    flush.zero_()
    step()
torch.cuda.synchronize()
kt = ctx.kernel_times()
d0 = disp.double().sum().item()
print(json.dumps({"variant": os.environ.get("NRM_B200_VARIANT", "main"), "exc": ctx.exceptions(),
                  "us": {k: round(1e3 * v[0] / max(v[1], 1), 2) for k, v in kt.items()},
                  "checksum": d0}))
