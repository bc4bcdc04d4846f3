"""Development: e2e pipelining variants of the bench's host-API step (fields in
flight on their own contexts, blends inline or on their own thread)."""
import collections
import ctypes as C
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2103_07414_b200 import mosaic as M
from paper_2103_07414_b200 import workload as W

dev = torch.device("cuda", 0)
wl = W.frame_workload("c2")
e = wl.emdq
fw, fh = wl.frame_w, wl.frame_h
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
h_frame = pin(wl.frame)
h_anc, h_war = pin(wl.anchors), pin(wl.warps)
h_apts, h_loc, h_prob, h_act = pin(e.apts), pin(e.locals_), pin(e.probs), pin(e.active)
g = M.Grid(0.0, 0.0, fw, fh)
ctx_b = M.Context(0)
lib = ctx_b._lib
poly = np.ascontiguousarray(M.invert_frame_boundary(fw, fh, wl.anchors, wl.warps, wl.params.alpha, ctx=ctx_b))
cv = M.Canvas(ctx_b)
cv.ensure_contains(wl.canvas_rect)
alpha, beta = wl.params.alpha, wl.params.beta


def blend():
    s = M.BlendStats()
    M.check(lib.nrm_blend_frame(cv.handle, h_frame.ctypes.data, fw, fh, 3, h_anc.ctypes.data, h_war.ctypes.data,
                                len(h_anc), alpha, poly.ctypes.data, len(poly), C.byref(s)))


def run(nfl, mode, N=300):
    ctxs = [M.Context(0) for _ in range(nfl)]
    for c_ in ctxs:
        c_.set_stream(torch.cuda.Stream(dev, priority=-1).cuda_stream)
    outs = [(torch.empty((fh, fw, 2), dtype=torch.float32).pin_memory().numpy(),
             torch.empty((fh, fw), dtype=torch.float32).pin_memory().numpy()) for _ in range(nfl)]

    def fld(k):
        c_, (d_, u_) = ctxs[k], outs[k]
        M.check(lib.nrm_emdq_field(c_.handle, C.byref(g), h_apts.ctypes.data, h_loc.ctypes.data, h_prob.ctypes.data,
                                   len(h_apts), h_act.ctypes.data, len(h_act), alpha, 16, beta, d_.ctypes.data,
                                   u_.ctypes.data))
    pl = ThreadPoolExecutor(nfl)
    for warm in (True, False):
        n = 20 if warm else N
        pend = collections.deque()
        bt = None
        if mode == "thread":
            bt = threading.Thread(target=lambda: [blend() for _ in range(n)])
        t0 = time.perf_counter()
        if bt:
            bt.start()
        for i in range(n):
            if len(pend) == nfl:
                pend.popleft().result()
            pend.append(pl.submit(fld, i % nfl))
            if mode == "inline":
                blend()
        while pend:
            pend.popleft().result()
        if bt:
            bt.join()
        dt = (time.perf_counter() - t0) / n
    pl.shutdown()
    return dt


for mode in ("inline", "thread", "none"):
    for nfl in (2, 3, 4):
        dt = run(nfl, mode)
        print(f"blend {mode:6s} fields in flight {nfl}: {dt * 1e3:.3f} ms/frame = {fw * fh / dt / 1e6:.0f} Mpix/s")
