"""Per-rank work of bench.py's weak-scaling step at G GPUs, on one GPU: one
EMDQ field (K3) plus G frame blends into band 0 of G (K1; the G frames lie in
disjoint canvas lanes and go through one batched blend call), streams as in
the bench. Estimates the per-rank step time without the collectives.
    python tools/rank_emulation.py [G ...]"""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2103_07414_b200 import mosaic as M
from paper_2103_07414_b200 import workload as W

Gs = [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]
wl = W.frame_workload("c2")
dev = torch.device("cuda", 0)
e = wl.emdq
fw, fh, alpha, beta = wl.frame_w, wl.frame_h, wl.params.alpha, wl.params.beta
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
for G in Gs:
    sa, sb = torch.cuda.Stream(dev, priority=-1), torch.cuda.Stream(dev)
    ctx, ctx_b = M.Context(0), M.Context(0)
    ctx.set_stream(sa.cuda_stream)
    ctx_b.set_stream(sb.cuda_stream)
    p0 = M.invert_frame_boundary(fw, fh, wl.anchors, wl.warps, alpha, ctx=ctx)
    lane_w = float(np.ceil(p0[:, 0].max() - p0[:, 0].min()) + 64.0)  # bench.py: frames in disjoint lanes
    shifts = [k * lane_w for k in range(G)]
    anc = [T(wl.anchors + np.array([s, 0.0])) for s in shifts]
    war = [T(W.shifted_warps(wl.warps, s, 0.0)) for s in shifts]
    polys = [M.invert_frame_boundary(fw, fh, wl.anchors + np.array([s, 0.0]), W.shifted_warps(wl.warps, s, 0.0),
                                     alpha, ctx=ctx) for s in shifts]
    cv = M.Canvas(ctx_b)
    r = wl.canvas_rect
    cv.reserve((r[0], r[1], r[2] + shifts[-1], r[3]))
    cv.set_band(0, G)
    frame_t = T(wl.frame)
    apts, loc, prob, act = T(e.apts), T(e.locals_), T(e.probs), T(e.active)
    disp = torch.empty((fh, fw, 2), dtype=torch.float32, device=dev)
    unc = torch.empty((fh, fw), dtype=torch.float32, device=dev)
    st = torch.zeros((G, 4), dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        e0 = torch.cuda.Event()
        e0.record(sa)
        sb.wait_event(e0)
        M.emdq_field_device((0.0, 0.0, fw, fh), apts, loc, prob, act, alpha, beta, disp, unc, 16, ctx=ctx)
        if G == 1:
            M.blend_frame_device(cv, frame_t, fw, fh, 3, anc[0], war[0], alpha, polys[0], st[0])
        else:
            M.blend_frames_device(cv, [frame_t] * G, fw, fh, 3, anc, war, alpha, polys, st)
        e1 = torch.cuda.Event()
        e1.record(sb)
        sa.wait_event(e1)

    for _ in range(10):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(200):
        with torch.cuda.stream(sa):
            flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(sa)
        step()
        b.record(sa)
        ts.append((a, b))
    torch.cuda.synchronize()
    ms = sorted(x.elapsed_time(y) for x, y in ts)[len(ts) // 2]
    # serialised per-kernel times of one rank's step (library CUDA events)
    ctx.profile(True)
    ctx_b.profile(True)
    for _ in range(20):
        step()
    torch.cuda.synchronize()
    kt = {k: round(1e3 * v[0] / 20, 1) for k, v in {**ctx.kernel_times(), **ctx_b.kernel_times()}.items()}
    ctx.profile(False)
    ctx_b.profile(False)
    print(json.dumps({"G": G, "per_rank_step_ms": ms, "rank_frames_per_s": G / (ms * 1e-3),
                      "kernel_us_per_step": kt}), flush=True)
