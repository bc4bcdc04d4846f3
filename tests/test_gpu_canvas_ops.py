"""Canvas plumbing on the GPU:

* canvases taller than the 65,535-block grid limit (render, download, upload,
  occupancy) -- the reference renders any size (mosaic.hpp:301-331);
* the exception queue never loses a pixel: with a 16-slot queue the spilled
  deferrals are resolved by the exact pass's scan, and blends, node fields and
  batched blends are bit-identical to the default queue;
* banded canvas deformation (north_star extension): N block-cyclic bands on
  one device exchange their halo rows (dist.halo_plan + pack/unpack), deform
  their own stripes, and reassemble to the single-canvas deformation bit for
  bit; both deformation paths (ping-pong pass, region scratch) match the
  oracle restatement;
* dist.BandedMosaic runs on torch's current stream: its stats and render
  equal blend_frame / render;
* K1's canvas tile staged by TMA tensor maps (the default) and by cp.async
  (NRM_B200_NO_TMA) gives the same bits, single and batched blends;
* the binned supertile scan of large candidate sets keeps its bin counts
  clean across calls with different grid sizes."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def split_polys(g):
    out, o = [], 0
    for n in g["npoly"]:
        out.append(g["polys"][o:o + n])
        o += n
    return out


def test_tall_canvas_beyond_grid_y_limit(nrm, ctx, golden):
    g = golden("blend_first_frame")
    cv = nrm.Canvas(ctx)
    # a vertical scan: 256 px wide, 70,000 rows (> 65,535)
    cv.ensure_contains((0.0, -69000.0, 200.0, 999.0))
    assert cv.height() > 65535
    rng = np.random.default_rng(3)
    band = rng.random((64, cv.width(), 3))
    wts = rng.integers(1, 31, (64, cv.width())).astype(np.uint8)
    y_last = cv.height() - 64
    cv.write(0, y_last, band, wts)  # upload past row 65,535
    col, wt = cv.read(0, y_last, cv.width(), 64)
    assert np.array_equal(wt, wts)
    assert np.array_equal(col, band.astype(np.float32).astype(np.float64))
    assert cv.occupied_count() == int((wts > 0).sum())
    img, org = nrm.render(cv, crop=True)
    assert img.shape[0] == 64 and org[1] == cv.origin_offset()[1] + y_last
    full, _ = nrm.render(cv, crop=False)
    assert full.shape[0] == cv.height() and (full[y_last:, :, 3] == 255).all() and not full[:y_last, :, 3].any()


@pytest.fixture()
def tiny_queue(ctx):
    ctx.set_exception_capacity(16)
    yield
    ctx.set_exception_capacity(0)


def _blend_all(nrm, ctx, g, polys, band=None):
    cv = nrm.Canvas(ctx)
    if band:
        cv.set_band(*band)
    st = [nrm.blend_frame(cv, g["frame"], g["anchors"], g["warps"][k], float(g["alpha"]), p).as_tuple()
          for k, p in enumerate(polys)]
    col, wt = cv.read()
    return st, col, wt


@pytest.mark.parametrize("case", ["blend_c1_seq", "blend_gray_rotated"])
def test_spilled_exceptions_are_resolved(nrm, ctx, golden, case):
    g = golden(case)
    polys = split_polys(g) if "npoly" in g else [g["polys"]] * len(g["warps"])
    ref = _blend_all(nrm, ctx, g, polys)
    before = ctx.spilled_launches()
    ctx.set_exception_capacity(1)
    try:
        got = _blend_all(nrm, ctx, g, polys)
        band = _blend_all(nrm, ctx, g, polys, band=(1, 3))
    finally:
        ctx.set_exception_capacity(0)
    if case == "blend_gray_rotated":  # whole tiles take the exact tier
        assert ctx.spilled_launches() > before, "the tiny queue never overflowed: the test does not reach the scan"
    assert got[0] == ref[0]
    assert np.array_equal(got[2], ref[2]) and np.array_equal(got[1], ref[1])
    mask = band[2] > 0
    assert np.array_equal(band[2][mask], ref[2][mask]) and np.array_equal(band[1][mask], ref[1][mask])


def test_spilled_exceptions_node_field(nrm, ctx, oracle):
    rng = np.random.default_rng(5)
    n = 60
    anchors = rng.uniform(-300, 500, (n, 2))
    ang = rng.uniform(-np.pi, np.pi, n)  # hemisphere flips: whole tiles take the exact tier
    warps = np.stack([rng.uniform(0.8, 1.2, n), np.cos(ang / 2), np.sin(ang / 2),
                      rng.normal(0, 20, n), rng.normal(0, 20, n)], 1)
    grid = (-100.25, -50.5, 300, 200)
    d0, s0 = nrm.node_field(grid, anchors, warps, 4e-4, ctx=ctx)
    before = ctx.spilled_launches()
    ctx.set_exception_capacity(16)
    try:
        d1, s1 = nrm.node_field(grid, anchors, warps, 4e-4, ctx=ctx)
    finally:
        ctx.set_exception_capacity(0)
    assert ctx.spilled_launches() > before
    assert np.array_equal(s0, s1) and np.array_equal(d0, d1)
    assert not np.isnan(d1).any()
    od, osup = oracle.node_field_grid(grid, anchors, warps, 4e-4)
    assert np.array_equal(s1.astype(bool), osup.astype(bool))


def test_spilled_exceptions_batched_blend(nrm, ctx):
    import importlib.util
    from pathlib import Path
    spec = importlib.util.spec_from_file_location("_batch", Path(__file__).with_name("test_gpu_batch.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    run = mod.run
    a = run(nrm, ctx, None, 4, 800.0, batched=True)
    ctx.set_exception_capacity(16)
    try:
        b = run(nrm, ctx, None, 4, 800.0, batched=True)
        c = run(nrm, ctx, (1, 2), 4, 800.0, batched=True)
    finally:
        ctx.set_exception_capacity(0)
    d = run(nrm, ctx, (1, 2), 4, 800.0, batched=True)
    for x, y in ((a, b), (d, c)):
        assert np.array_equal(x[0], y[0]) and np.array_equal(x[2], y[2]) and np.array_equal(x[1], y[1])


def _seq_canvas(nrm, ctx, g, band=None):
    cv = nrm.Canvas(ctx)
    if band:
        cv.set_band(*band)
    for k, p in enumerate(split_polys(g)):
        nrm.blend_frame(cv, g["frame"], g["anchors"], g["warps"][k], float(g["alpha"]), p)
    return cv


@pytest.mark.parametrize("region", ["canvas", "small"])
def test_deform_paths_match_oracle(nrm, ctx, oracle, golden, region):
    g = golden("blend_c1_seq")
    cv = _seq_canvas(nrm, ctx, g)
    col0, wt0 = cv.read()
    H, Wd = wt0.shape
    ox, oy = cv.origin_offset()
    ocv = oracle.canvas()
    ocv.ensure_contains((ox, oy, ox + Wd - 1, oy + H - 1))
    ocv.set_arrays(col0.astype(np.float32).astype(np.float64), wt0)
    if region == "canvas":   # >= 1/4 of the canvas: ping-pong pass
        x, y, w, h = 0, 0, Wd, H
    else:                     # region scratch + commit
        x, y, w, h = 301, 222, 517, 389
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    d = np.stack([3.5 * np.sin(xx / 97.0) + 0.25 * np.cos(yy / 41.0),
                  -2.25 * np.cos(yy / 83.0) + 0.125 * np.sin(xx / 29.0)], -1).astype(np.float32)
    cv.deform(d, x, y)
    ocv.deform(x, y, w, h, d)
    col1, wt1 = cv.read()
    ocol, owt = ocv.arrays()
    assert np.array_equal(wt1, owt)
    assert np.array_equal(col1.astype(np.float64), ocol)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_banded_deformation_with_halo_is_bitwise_identical(nrm, ctx, golden, world):
    """N ranks emulated on one device (no kernel waits on another): blend into
    banded canvases, exchange halo rows through pack/unpack, deform twice,
    reassemble; equals the single canvas bit for bit."""
    import torch
    from paper_2103_07414_b200 import dist as D
    g = golden("blend_c1_seq")
    full = _seq_canvas(nrm, ctx, g)
    H, Wd = full.height(), full.width()
    _, oy = full.origin_offset()
    dev = torch.device("cuda", 0)
    yy, xx = np.mgrid[0:H, 0:Wd].astype(np.float64)
    fields = [np.stack([2.0 * np.sin(xx / 71.0), 11.5 * np.cos(yy / 57.0) + 0.5 * np.sin(xx / 13.0)], -1),
              np.stack([-1.25 * np.cos(yy / 33.0), -6.75 * np.sin(xx / 91.0)], -1)]
    bands = [_seq_canvas(nrm, ctx, g, band=(r, world)) for r in range(world)]
    for d in fields:
        d32 = np.ascontiguousarray(d, np.float32)
        dt = torch.from_numpy(d32).to(dev)
        torch.cuda.synchronize()
        full.deform(dt)
        halo = int(np.ceil(np.abs(d32[..., 1]).max())) + 1
        plan = D.halo_plan(int(oy), H, world, halo)
        sent = 0
        for q in range(world):
            for r in range(world):
                rows = plan[q][r]
                if len(rows):
                    buf = torch.empty(len(rows) * 13 * Wd, dtype=torch.uint8, device=dev)
                    bands[r].pack_rows(rows, buf)
                    bands[q].unpack_rows(rows, buf)
                    sent += len(rows)
        assert sent > 0
        for cv in bands:
            cv.deform(dt)
    ctx.synchronize()
    fcol, fwt = full.read()
    fimg, _ = nrm.render(full)
    ren = np.zeros(fimg.shape, np.int64)
    for r, cv in enumerate(bands):
        mask = D.owned_rows_mask(int(oy), H, r, world)
        col, wt = cv.read()
        assert np.array_equal(wt[mask], fwt[mask]), r
        assert np.array_equal(col[mask], fcol[mask]), r
        img, _ = nrm.render(cv)
        ren += img
    assert np.array_equal(ren, fimg.astype(np.int64))


def test_banded_mosaic_runs_on_torchs_stream(nrm, golden):
    import torch
    from paper_2103_07414_b200 import dist as D
    g = golden("blend_c1_seq")
    polys = split_polys(g)
    dev = torch.device("cuda", 0)
    bm = D.BandedMosaic(0, 1, 0)
    cur = torch.cuda.current_stream(dev).cuda_stream
    assert bm.ctx.stream() == (cur or 1)  # torch's default stream is cudaStreamLegacy at the ABI
    ref = nrm.Canvas(nrm.Context(0))
    fh, fw = g["frame"].shape[:2]
    ch = g["frame"].shape[2] if g["frame"].ndim == 3 else 1
    for k, p in enumerate(polys):
        # inputs produced by torch on its stream right before the blend
        f = torch.from_numpy(np.ascontiguousarray(g["frame"])).to(dev, non_blocking=True)
        a = torch.from_numpy(np.ascontiguousarray(g["anchors"])).to(dev, non_blocking=True)
        w = torch.from_numpy(np.ascontiguousarray(g["warps"][k])).to(dev, non_blocking=True)
        st = torch.full((4,), -1, dtype=torch.int64, device=dev)
        bm.blend(f, fw, fh, ch, a, w, float(g["alpha"]), p, st)
        got = tuple(int(v) for v in st.cpu())
        exp = nrm.blend_frame(ref, g["frame"], g["anchors"], g["warps"][k], float(g["alpha"]), p).as_tuple()
        assert got == exp
    img, org = bm.render(crop=True)
    rimg, rorg = nrm.render(ref, crop=True)
    assert np.array_equal(img, rimg) and tuple(org) == tuple(rorg)


def test_banded_node_field_is_bitwise_identical(nrm, ctx):
    """The canvas-wide field split into block-cyclic stripes (one call per
    rank): the ranks' rows together are the single field bit for bit."""
    import torch
    from paper_2103_07414_b200 import workload as W
    from paper_2103_07414_b200 import dist as D
    sp = W.scaled_params(1920, 1080)
    x0, y0, w, h = -512, -333, 2304, 1500
    anchors = W.hex_lattice((x0, y0, x0 + w, y0 + h), sp.hex_spacing)
    rng = np.random.default_rng(9)
    warps = np.tile(np.array([1.0, 1.0, 0.0, 0.0, 0.0]), (len(anchors), 1))
    ang = rng.uniform(-0.05, 0.05, len(anchors))
    warps[:, 0] = rng.uniform(0.995, 1.005, len(anchors))
    warps[:, 1], warps[:, 2] = np.cos(ang / 2), np.sin(ang / 2)
    warps[:, 3:5] = rng.normal(0, 3.0, (len(anchors), 2))
    dev = torch.device("cuda", 0)
    a_t, q_t = torch.from_numpy(anchors).to(dev), torch.from_numpy(warps).to(dev)
    grid = (float(x0), float(y0), w, h)
    d_full = torch.zeros((h, w, 2), dtype=torch.float32, device=dev)
    s_full = torch.zeros((h, w), dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    nrm.node_field_band_device(grid, a_t, q_t, sp.alpha, d_full, s_full, 0, 1, ctx=ctx)
    d_rel = torch.zeros_like(d_full)
    nrm.node_field_device(grid, a_t, q_t, sp.alpha, d_rel, None, ctx=ctx)
    ctx.synchronize()
    assert (d_rel - d_full).abs().max().item() <= 1e-3  # other tiling, same field
    for world in (2, 3):
        d_b = torch.full((h, w, 2), float("nan"), dtype=torch.float32, device=dev)
        s_b = torch.full((h, w), 7, dtype=torch.uint8, device=dev)
        torch.cuda.synchronize()
        for r in range(world):
            nrm.node_field_band_device(grid, a_t, q_t, sp.alpha, d_b, s_b, r, world, ctx=ctx)
        ctx.synchronize()
        assert torch.equal(d_b, d_full) and torch.equal(s_b, s_full)
        # a single rank writes only its own rows
        d_1 = torch.full((h, w, 2), float("nan"), dtype=torch.float32, device=dev)
        torch.cuda.synchronize()
        nrm.node_field_band_device(grid, a_t, q_t, sp.alpha, d_1, s_b, 1, world, ctx=ctx)
        ctx.synchronize()
        mask = torch.from_numpy(D.owned_rows_mask(y0, h, 1, world)).to(dev)
        assert torch.equal(d_1[mask], d_full[mask]) and torch.isnan(d_1[~mask]).all()


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_emdq_exact_queue_matches_inline_exact_bitwise(nrm, ctx, name):
    """The dense EMDQ field queues single near-tie pixels for the warp-parallel
    exact pass (k_emdq_exceptions). With a one-slot queue every pixel but one
    runs the thread-per-pixel exact tier inside k_pixels instead; both must
    give the same bits (the inline tier is the one pinned to the reference)."""
    from paper_2103_07414_b200 import workload as W
    wl = W.frame_workload(name)
    e = wl.emdq
    grid = (0.0, 0.0, wl.frame_w, wl.frame_h)
    args = (grid, e.apts, e.locals_, e.probs, e.active, wl.params.alpha, wl.params.beta, 16)
    d0, u0 = nrm.emdq_field(*args, ctx=ctx)
    n_exact = ctx.exceptions()[1]
    assert n_exact > 1, "no exact-tier pixels: the test does not reach the queue"
    ctx.set_exception_capacity(1)
    try:
        d1, u1 = nrm.emdq_field(*args, ctx=ctx)
    finally:
        ctx.set_exception_capacity(0)
    assert ctx.exceptions()[1] == n_exact
    assert np.array_equal(d0.view(np.uint32), d1.view(np.uint32))
    assert np.array_equal(u0.view(np.uint32), u1.view(np.uint32))


def _large_emdq_case(seed, w, h):
    rng = np.random.default_rng(seed)
    m = 6000
    apts = np.stack([rng.uniform(-80, w + 80, m), rng.uniform(-80, h + 80, m)], 1)
    apts[:60] += rng.choice([-1.0, 1.0], (60, 2)) * rng.uniform(500, 3000, (60, 2))  # margin cells
    ang = rng.uniform(-0.05, 0.05, m)
    loc = np.zeros((m, 5))
    loc[:, 0] = rng.uniform(0.9, 1.1, m)
    loc[:, 1], loc[:, 2] = np.cos(ang / 2), np.sin(ang / 2)
    loc[:, 3:5] = rng.normal(0, 6.0, (m, 2))
    probs = rng.uniform(0, 1, m)
    active = np.sort(rng.choice(m, 5000, replace=False)).astype(np.int32)
    return (0.0, 0.0, w, h), apts, loc, probs, active, 5e-4, 5e-4, 16


def test_binned_supertile_scan_mixed_grid_sizes(nrm, ctx, oracle):
    """Large candidate sets take the binned supertile scan (persistent-zero
    bin counts). A large grid, then a small one, then the large one again
    must give the same bits for the large grid, and rows of both match the
    oracle."""
    big = _large_emdq_case(11, 1400, 900)
    small = _large_emdq_case(12, 300, 200)
    d0, u0 = nrm.emdq_field(*big, ctx=ctx)
    ds, us = nrm.emdq_field(*small, ctx=ctx)
    d1, u1 = nrm.emdq_field(*big, ctx=ctx)
    assert np.array_equal(d0.view(np.uint32), d1.view(np.uint32))
    assert np.array_equal(u0.view(np.uint32), u1.view(np.uint32))
    for args, d, u in ((big, d0, u0), (small, ds, us)):
        grid, apts, loc, probs, active, alpha, beta, S = args
        h = int(grid[3])
        for j in (0, h // 2, h - 1):
            od, ou = oracle.emdq_field_grid(grid, apts, loc, probs, active, alpha, beta, S, rows=(j, j + 1), fast=True)
            assert np.abs(d[j] - od[j]).max() <= 1e-3
            assert np.abs(u[j] / ou[j] - 1).max() <= 1e-6


_NO_TMA_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2103_07414_b200 import mosaic as nrm
g = dict(np.load(sys.argv[2]))
ctx = nrm.Context(0)
cv = nrm.Canvas(ctx)
polys, o = [], 0
for n in g["npoly"]:
    polys.append(g["polys"][o:o + n])
    o += n
st = [nrm.blend_frame(cv, g["frame"], g["anchors"], g["warps"][k], float(g["alpha"]), p).as_tuple()
      for k, p in enumerate(polys)]
col, wt = cv.read()
np.savez(sys.argv[3], st=np.array(st), col=col, wt=wt)
"""


@pytest.mark.parametrize("case", ["blend_c1_seq", "blend_gray_rotated"])
def test_canvas_staging_tma_matches_cp_async(nrm, ctx, golden, tmp_path, case):
    """The same blends with K1's canvas tile staged by cp.async (a fresh
    process with NRM_B200_NO_TMA set) are bit-identical to the TMA path."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    g = golden(case)
    polys = split_polys(g) if "npoly" in g else [g["polys"]] * len(g["warps"])
    inp = tmp_path / "in.npz"
    np.savez(inp, frame=g["frame"], anchors=g["anchors"], warps=g["warps"], alpha=g["alpha"],
             polys=np.concatenate(polys), npoly=np.array([len(p) for p in polys]))
    ref = _blend_all(nrm, ctx, g, polys)
    out = tmp_path / "out.npz"
    env = dict(os.environ, NRM_B200_NO_TMA="1")
    root = str(Path(__file__).resolve().parents[1])
    r = subprocess.run([sys.executable, "-c", _NO_TMA_SCRIPT, root, str(inp), str(out)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = np.load(out)
    assert [tuple(x) for x in got["st"].tolist()] == [tuple(x) for x in ref[0]]
    assert np.array_equal(got["wt"], ref[2]) and np.array_equal(got["col"], ref[1])
