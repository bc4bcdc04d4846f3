"""Development: where the end-to-end (host-pointer) step spends its time."""
import ctypes as C
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2103_07414_b200 import mosaic as M
from paper_2103_07414_b200 import workload as W

dev = torch.device("cuda", 0)


def tm(fn, n=50):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


for mb in (6, 25, 100):
    nb = mb << 20
    h = torch.empty(nb, dtype=torch.uint8).pin_memory()
    d = torch.empty(nb, dtype=torch.uint8, device=dev)
    t_d2h = tm(lambda: h.copy_(d, non_blocking=True))
    t_h2d = tm(lambda: d.copy_(h, non_blocking=True))
    print(f"{mb} MiB: D2H {t_d2h:.3f} ms ({nb / t_d2h / 1e6:.1f} GB/s)  H2D {t_h2d:.3f} ms ({nb / t_h2d / 1e6:.1f} GB/s)")

wl = W.frame_workload("c2")
e = wl.emdq
ctx = M.Context(0)
ctx_b = M.Context(0)
lib = ctx._lib
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
fw, fh = wl.frame_w, wl.frame_h
h_frame = pin(wl.frame)
h_anc, h_war = pin(wl.anchors), pin(wl.warps)
h_apts, h_loc, h_prob, h_act = pin(e.apts), pin(e.locals_), pin(e.probs), pin(e.active)
h_disp = torch.empty((fh, fw, 2), dtype=torch.float32).pin_memory().numpy()
h_unc = torch.empty((fh, fw), dtype=torch.float32).pin_memory().numpy()
g = M.Grid(0.0, 0.0, fw, fh)
poly = np.ascontiguousarray(M.invert_frame_boundary(fw, fh, wl.anchors, wl.warps, wl.params.alpha, ctx=ctx))
cv = M.Canvas(ctx_b)
cv.ensure_contains(wl.canvas_rect)
alpha, beta = wl.params.alpha, wl.params.beta


def field(disp=True, unc=True):
    M.check(lib.nrm_emdq_field(ctx.handle, C.byref(g), h_apts.ctypes.data, h_loc.ctypes.data, h_prob.ctypes.data,
                               len(h_apts), h_act.ctypes.data, len(h_act), alpha, 16, beta,
                               h_disp.ctypes.data if disp else None, h_unc.ctypes.data if unc else None))


def blend():
    s = M.BlendStats()
    M.check(lib.nrm_blend_frame(cv.handle, h_frame.ctypes.data, fw, fh, 3, h_anc.ctypes.data, h_war.ctypes.data,
                                len(h_anc), alpha, poly.ctypes.data, len(poly), C.byref(s)))


T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
d_apts, d_loc, d_prob, d_act = T(e.apts), T(e.locals_), T(e.probs), T(e.active)
d_disp = torch.empty((fh, fw, 2), dtype=torch.float32, device=dev)
d_unc = torch.empty((fh, fw), dtype=torch.float32, device=dev)


def field_dev():
    M.emdq_field_device((0.0, 0.0, fw, fh), d_apts, d_loc, d_prob, d_act, alpha, beta, d_disp, d_unc, 16, ctx=ctx)
    ctx.synchronize()


print(f"field device     {tm(field_dev):.3f} ms")
print(f"field (disp+unc) {tm(field):.3f} ms")
print(f"field (disp)     {tm(lambda: field(True, False)):.3f} ms")
print(f"field (no out)   {tm(lambda: field(False, False)):.3f} ms")
print(f"blend            {tm(blend):.3f} ms")
from concurrent.futures import ThreadPoolExecutor  # noqa: E402
pool = ThreadPoolExecutor(1)


def both():
    f = pool.submit(field)
    blend()
    f.result()


print(f"field || blend   {tm(both):.3f} ms")


# per-call durations while running in parallel
durs = {"field": [], "blend": []}


def timed(name, fn):
    def run():
        t0 = time.perf_counter()
        fn()
        durs[name].append((t0, time.perf_counter()))
    return run


tf, tb = timed("field", field), timed("blend", blend)
for _ in range(30):
    f = pool.submit(tf)
    tb()
    f.result()
import statistics as S  # noqa: E402
for k, v in durs.items():
    print(k, "median ms", round(S.median([(b - a) * 1e3 for a, b in v[5:]]), 3))
st = [min(durs["field"][i][0], durs["blend"][i][0]) for i in range(30)]
off = [(durs["blend"][i][0] - durs["field"][i][0]) * 1e3 for i in range(30)]
print("blend start - field start (ms) median", round(S.median(off[5:]), 3))
print(f"field || field-dev {tm(lambda: (pool.submit(field_dev), blend())):.3f}")

# ---- fields in flight (own contexts + pinned outputs), with and without the blend
import collections  # noqa: E402
for nfl in (1, 2, 3):
    ctxs = [ctx] + [M.Context(0) for _ in range(nfl - 1)]
    outs = [(h_disp, h_unc)] + [(torch.empty((fh, fw, 2), dtype=torch.float32).pin_memory().numpy(),
                                 torch.empty((fh, fw), dtype=torch.float32).pin_memory().numpy())
                                for _ in range(nfl - 1)]

    def fld(k):
        c_, (d_, u_) = ctxs[k], outs[k]
        M.check(lib.nrm_emdq_field(c_.handle, C.byref(g), h_apts.ctypes.data, h_loc.ctypes.data, h_prob.ctypes.data,
                                   len(h_apts), h_act.ctypes.data, len(h_act), alpha, 16, beta, d_.ctypes.data,
                                   u_.ctypes.data))
    pl = ThreadPoolExecutor(nfl)
    for with_blend in (False, True):
        pend = collections.deque()
        t0 = time.perf_counter()
        N = 200
        for i in range(N):
            if len(pend) == nfl:
                pend.popleft().result()
            pend.append(pl.submit(fld, i % nfl))
            if with_blend:
                blend()
        while pend:
            pend.popleft().result()
        dt = (time.perf_counter() - t0) / N
        print(f"fields in flight {nfl}, blend {with_blend}: {dt * 1e3:.3f} ms/frame, {1 / dt:.0f} frames/s")
