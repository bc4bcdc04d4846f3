"""Development: the C2 step's two chains alone and overlapped (device time per
step, CUDA events, L2 flushed between steps): K3 = dense EMDQ field on a
high-priority stream, K1 = blend on a second stream."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2103_07414_b200 import mosaic as M
from paper_2103_07414_b200 import workload as W

wl = W.frame_workload("c2")
dev = torch.device("cuda", 0)
sa = torch.cuda.Stream(dev, priority=-1)
sb = torch.cuda.Stream(dev)
ctx_a, ctx_b = M.Context(0), M.Context(0)
ctx_a.set_stream(sa.cuda_stream)
ctx_b.set_stream(sb.cuda_stream)
poly = M.invert_frame_boundary(wl.frame_w, wl.frame_h, wl.anchors, wl.warps, wl.params.alpha, ctx=ctx_a)
cv = M.Canvas(ctx_b)
cv.ensure_contains(wl.canvas_rect)
e = wl.emdq
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
frame_t, anc, war = T(wl.frame), T(wl.anchors), T(wl.warps)
apts, loc, prob, act = T(e.apts), T(e.locals_), T(e.probs), T(e.active)
disp = torch.empty((wl.frame_h, wl.frame_w, 2), dtype=torch.float32, device=dev)
unc = torch.empty((wl.frame_h, wl.frame_w), dtype=torch.float32, device=dev)
st = torch.zeros(4, dtype=torch.int64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def run(k3, k1, n=200):
    ts = []
    for i in range(n + 10):
        with torch.cuda.stream(sa):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(sa)
            sb.wait_event(e0)
            if k3:
                M.emdq_field_device((0.0, 0.0, wl.frame_w, wl.frame_h), apts, loc, prob, act, wl.params.alpha,
                                    wl.params.beta, disp, unc, 16, ctx=ctx_a)
            if k1:
                M.blend_frame_device(cv, frame_t, wl.frame_w, wl.frame_h, 3, anc, war, wl.params.alpha, poly, st)
            eb = torch.cuda.Event()
            eb.record(sb)
            sa.wait_event(eb)
            e1.record(sa)
        if i >= 10:
            ts.append((e0, e1))
    torch.cuda.synchronize()
    return np.median([a.elapsed_time(b) for a, b in ts]) * 1e3


for name, k3, k1 in (("K3 alone", 1, 0), ("K1 alone", 0, 1), ("both", 1, 1)):
    print(f"{name:9s} {run(k3, k1):7.1f} us/step")
