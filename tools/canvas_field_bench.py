"""Canvas-wide node field (K2) with a canvas-covering node lattice -- the
'blending-bound field over the canvas' of BASELINE configs[3]/[4]:
time per pass and Gpx/s, and oracle parity on sampled windows.
    python tools/canvas_field_bench.py [canvas_px ...]"""
import json
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2103_07414_b200 import mosaic as M
from paper_2103_07414_b200 import workload as W

sizes = [int(a) for a in sys.argv[1:]] or [16384, 32768]
dev = torch.device("cuda", 0)
ctx = M.Context(0)
s_ = torch.cuda.Stream(dev)
ctx.set_stream(s_.cuda_stream)
torch.cuda.set_stream(s_)
for n in sizes:
    sp = W.scaled_params(3840, 2160)  # C4/C5 frame scale: hex 480 px, alpha 3.125e-6
    rect = (0.0, 0.0, float(n), float(n))
    anchors = W.hex_lattice(rect, sp.hex_spacing)
    rng = np.random.default_rng(5)
    warps = np.tile(np.array([1.0, 1.0, 0.0, 0.0, 0.0]), (len(anchors), 1))
    ang = rng.uniform(-0.02, 0.02, len(anchors))
    warps[:, 0] = rng.uniform(0.99, 1.01, len(anchors))
    warps[:, 1], warps[:, 2] = np.cos(ang / 2), np.sin(ang / 2)
    warps[:, 3:5] = rng.normal(0, 4.0, (len(anchors), 2))
    a_t = torch.from_numpy(anchors).to(dev)
    q_t = torch.from_numpy(warps).to(dev)
    rows = 8192 if n > 16384 else n  # 32768^2 runs as 4 bands of 8192 rows (disp buffer 2 GB)
    disp = torch.empty((rows, n, 2), dtype=torch.float32, device=dev)
    sup = torch.empty((rows, n), dtype=torch.uint8, device=dev)
    M.node_field_device((0.0, 0.0, n, rows), a_t, q_t, sp.alpha, disp, sup, ctx=ctx)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.profile(True)
    e0.record(s_)
    for y0 in range(0, n, rows):
        M.node_field_device((0.0, float(y0), n, rows), a_t, q_t, sp.alpha, disp, sup, ctx=ctx)
    e1.record(s_)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    kt = {k: round(v[0], 3) for k, v in ctx.kernel_times().items()}
    ctx.profile(False)
    out = {"canvas": n, "nodes": len(anchors), "ms_profiled": ms, "gpx_per_s": n * n / (ms * 1e-3) / 1e9,
           "kernel_ms": kt, "exceptions": ctx.exceptions()}
    # parity on windows of the last band against the oracle
    try:
        from oracle.oracle import Oracle
        O = Oracle()
        y0 = n - rows
        d = disp.cpu().numpy()
        su = sup.cpu().numpy()
        err = 0.0
        for (wx, wy) in ((0, 0), (n // 2, rows // 2), (n - 128, rows - 128)):
            od, osu = O.node_field_grid((float(wx), float(y0 + wy), 128, 128), anchors, warps, sp.alpha)
            assert np.array_equal(su[wy:wy + 128, wx:wx + 128].astype(bool), osu.astype(bool))
            m = osu.astype(bool)
            err = max(err, float(np.abs(d[wy:wy + 128, wx:wx + 128][m] - od[m]).max()))
        out["max_disp_err_px_vs_oracle"] = err
    except Exception as ex:  # noqa: BLE001
        out["oracle"] = repr(ex)
    print(json.dumps(out), flush=True)
