import sys, numpy as np
sys.path.insert(0, '.')
from paper_2103_07414_b200 import mosaic as M, workload as W
from oracle.oracle import Oracle
O = Oracle()
ctx = M.Context(0)
for name in ("c2", "c4"):
    wl = W.frame_workload(name)
    # the node field on the canvas region the frame maps from (reference coords)
    poly = M.invert_frame_boundary(wl.frame_w, wl.frame_h, wl.anchors, wl.warps, wl.params.alpha, ctx=ctx)
    x0, y0 = np.floor(poly.min(0)).astype(int); x1, y1 = np.ceil(poly.max(0)).astype(int)
    h = min(y1 - y0, 600)
    grid = (float(x0), float(y0 + (y1 - y0) // 2 - h // 2), int(x1 - x0), int(h))
    d, s = M.node_field(grid, wl.anchors, wl.warps, wl.params.alpha, ctx=ctx)
    od, os_ = O.node_field_grid(grid, wl.anchors, wl.warps, wl.params.alpha)
    m = os_.astype(bool)
    err = np.abs(d.astype(np.float64) - od)[m]
    print(name, grid, "max err px", err.max(), "p99.99", np.quantile(err, 0.9999), "exceptions", ctx.exceptions())
