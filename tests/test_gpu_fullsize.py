"""GPU parity at BASELINE.json's full sizes (configs[1] = C2, configs[3] = C4,
configs[4] = C5).

The oracle (the C restatement, pinned to the reference by the golden tests)
runs the same inputs:
  * C2 and C4 blend_frame in full: BlendStats and the weight plane must match
    exactly, colour to 1e-3, the rendered mosaic to +-1 level;
  * K1's own field: a ramp frame (R = x mod 256, G = y mod 256) blended into
    a fresh canvas turns each blended colour into the frame position K1
    computed (c * 255 = position mod 256, to ~2e-5 px); it must be within
    1e-3 px of the oracle's pixel_warp position at every blended pixel;
  * the C2 / C4 / C5 dense EMDQ field at EVERY frame pixel (1920x1080 with
    1,600 candidates; 3840x2160 with 8,000 and with 25,000): displacement
    <= 1e-3 px, uncertainty <= 1e-6 relative (checker: the oracle's grid-kNN
    variant, bit-identical to its full scan and to the reference golden);
  * the C4 node field (K2) on windows, and the C5 canvas-wide K2 (32768^2
    canvas, 5,707-node lattice, one launch over the whole canvas) on windows
    at the corners, edges and centre.
Inputs come from workload.py (synthetic frames and matches with a known
smooth deformation, as the bench uses)."""
import numpy as np
import pytest

from paper_2103_07414_b200 import workload as W

pytestmark = pytest.mark.gpu

DISP_TOL = 1e-3
COLOR_TOL = 1e-3


@pytest.fixture(scope="module")
def c2():
    return W.frame_workload("c2")


def test_c2_blend_frame_full_matches_oracle(nrm, ctx, oracle, c2):
    wl = c2
    poly = nrm.invert_frame_boundary(wl.frame_w, wl.frame_h, wl.anchors, wl.warps, wl.params.alpha, ctx=ctx)
    cv = nrm.Canvas(ctx)
    st = nrm.blend_frame(cv, wl.frame, wl.anchors, wl.warps, wl.params.alpha, poly).as_tuple()
    ocv = oracle.canvas()
    ost = oracle.blend_frame(ocv, wl.frame, wl.anchors, wl.warps, wl.params.alpha, poly)
    assert tuple(st) == ost, (st, ost)
    assert ost[1] > 2_000_000
    ox, oy, w, h = ocv.info()
    assert (cv.origin_offset(), cv.width(), cv.height()) == ((ox, oy), w, h)
    col, wt = cv.read()
    ocol, owt = ocv.arrays()
    assert np.array_equal(wt, owt)
    assert np.abs(col.astype(np.float64) - ocol).max() <= COLOR_TOL
    img, org = nrm.render(cv, crop=True)
    oimg, oorg = oracle.render(ocv, crop=True)
    assert org == oorg and img.shape == oimg.shape
    assert np.abs(img.astype(np.int16) - oimg.astype(np.int16)).max() <= 1


@pytest.fixture(scope="module")
def c4():
    return W.frame_workload("c4")


@pytest.mark.parametrize("name", ["c2", "c4", "c5"])
def test_emdq_field_full_frame_matches_oracle(nrm, ctx, oracle, c2, c4, name):
    wl = {"c2": c2, "c4": c4}.get(name) or W.frame_workload(name)
    e = wl.emdq
    grid = (0.0, 0.0, wl.frame_w, wl.frame_h)
    disp, unc = nrm.emdq_field(grid, e.apts, e.locals_, e.probs, e.active, wl.params.alpha, wl.params.beta, 16,
                               ctx=ctx)
    assert np.isfinite(disp).all() and np.isfinite(unc).all()
    od, ou = oracle.emdq_field_grid(grid, e.apts, e.locals_, e.probs, e.active, wl.params.alpha, wl.params.beta,
                                    16, fast=True)
    err = np.abs(disp - od).max()
    assert err <= DISP_TOL, (name, err)
    rel = np.abs(unc / ou - 1).max()
    assert rel <= 1e-6, (name, rel)
    assert len(e.active) >= {"c2": 1500, "c4": 7500, "c5": 24000}[name]


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_k1_frame_positions_match_oracle(nrm, ctx, oracle, c2, c4, name):
    """K1's field, read back through the blend itself (see module doc)."""
    wl = {"c2": c2, "c4": c4}[name]
    ramp = W.ramp_frame(wl.frame_w, wl.frame_h)
    poly = nrm.invert_frame_boundary(wl.frame_w, wl.frame_h, wl.anchors, wl.warps, wl.params.alpha, ctx=ctx)
    cv = nrm.Canvas(ctx)
    st = nrm.blend_frame(cv, ramp, wl.anchors, wl.warps, wl.params.alpha, poly).as_tuple()
    col, wt = cv.read()
    ox, oy = cv.origin_offset()
    ys, xs = np.nonzero(wt)
    y0, y1, x0, x1 = ys.min(), ys.max() + 1, xs.min(), xs.max() + 1
    od, osup = oracle.node_field_grid((ox + x0, oy + y0, int(x1 - x0), int(y1 - y0)), wl.anchors, wl.warps,
                                      wl.params.alpha)
    m = wt[y0:y1, x0:x1] > 0
    assert m.sum() == st[1] and osup[m].all()
    gx, gy = np.meshgrid(ox + np.arange(x0, x1), oy + np.arange(y0, y1))
    fx = (gx + od[..., 0])[m]  # the oracle's frame position of each blended pixel
    fy = (gy + od[..., 1])[m]
    c = col[y0:y1, x0:x1][m]
    worst = 0.0
    for pos, val in ((fx, c[:, 0]), (fy, c[:, 1])):
        r = np.mod(pos, 256.0)
        ok = (r > 1.0) & (r < 254.0)  # away from the ramp's wrap (bilinear across 255 -> 0)
        assert ok.mean() > 0.95
        worst = max(worst, float(np.abs(val[ok] * 255.0 - r[ok]).max()))
    assert worst <= DISP_TOL + 1e-4, worst


def test_c4_node_field_windows_match_oracle(nrm, ctx, oracle, c4):
    wl = c4
    for (x0, y0) in ((1792.0, 976.0), (0.0, 0.0), (3584.0, 1904.0)):
        grid = (x0, y0, 256, 256)
        disp, sup = nrm.node_field(grid, wl.anchors, wl.warps, wl.params.alpha, ctx=ctx)
        od, osup = oracle.node_field_grid(grid, wl.anchors, wl.warps, wl.params.alpha)
        assert np.array_equal(sup.astype(bool), osup.astype(bool))
        m = osup.astype(bool)
        assert np.abs(disp[m] - od[m]).max() <= DISP_TOL


def test_c4_blend_frame_full_matches_oracle(nrm, ctx, oracle, c4):
    """configs[3] frame size: one 3840 x 2160 frame into a fresh canvas with its
    frame lattice, in full (about 9 M footprint pixels)."""
    wl = c4
    poly = nrm.invert_frame_boundary(wl.frame_w, wl.frame_h, wl.anchors, wl.warps, wl.params.alpha, ctx=ctx)
    cv = nrm.Canvas(ctx)
    st = nrm.blend_frame(cv, wl.frame, wl.anchors, wl.warps, wl.params.alpha, poly).as_tuple()
    ocv = oracle.canvas()
    ost = oracle.blend_frame(ocv, wl.frame, wl.anchors, wl.warps, wl.params.alpha, poly)
    assert tuple(st) == ost, (st, ost)
    assert ost[1] > 8_000_000
    col, wt = cv.read()
    ocol, owt = ocv.arrays()
    assert np.array_equal(wt, owt)
    assert np.abs(col.astype(np.float64) - ocol).max() <= COLOR_TOL
    img, org = nrm.render(cv, crop=True)
    oimg, oorg = oracle.render(ocv, crop=True)
    assert org == oorg and img.shape == oimg.shape
    assert np.abs(img.astype(np.int16) - oimg.astype(np.int16)).max() <= 1


def test_c5_canvas_wide_node_field_windows(nrm, ctx, oracle):
    """configs[4]: the blending-bound field over a 32768^2 canvas with the
    canvas-covering hex lattice of the 4K frame scale (5,707 nodes), as ONE
    node-field launch over the whole canvas (prefilter chunking included);
    windows at the corners, edges and centre against the oracle."""
    import torch
    sp = W.scaled_params(3840, 2160)
    n = 32768
    anchors = W.hex_lattice((0.0, 0.0, float(n), float(n)), sp.hex_spacing)
    assert len(anchors) > 5000
    rng = np.random.default_rng(5)
    warps = np.tile(np.array([1.0, 1.0, 0.0, 0.0, 0.0]), (len(anchors), 1))
    ang = rng.uniform(-0.02, 0.02, len(anchors))
    warps[:, 0] = rng.uniform(0.99, 1.01, len(anchors))
    warps[:, 1], warps[:, 2] = np.cos(ang / 2), np.sin(ang / 2)
    warps[:, 3:5] = rng.normal(0, 4.0, (len(anchors), 2))
    dev = torch.device("cuda", 0)
    a_t = torch.from_numpy(anchors).to(dev)
    q_t = torch.from_numpy(warps).to(dev)
    disp = torch.empty((n, n, 2), dtype=torch.float32, device=dev)  # 8.6 GB
    sup = torch.empty((n, n), dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    nrm.node_field_device((0.0, 0.0, n, n), a_t, q_t, sp.alpha, disp, sup, ctx=ctx)
    ctx.synchronize()
    win = 96
    spots = [(0, 0), (n - win, 0), (0, n - win), (n - win, n - win), (n // 2, n // 2), (n // 2, 0),
             (0, n // 2), (12345, 23456), (31000, 17000)]
    for (x0, y0) in spots:
        d = disp[y0:y0 + win, x0:x0 + win].cpu().numpy()
        s_ = sup[y0:y0 + win, x0:x0 + win].cpu().numpy()
        od, osu = oracle.node_field_grid((float(x0), float(y0), win, win), anchors, warps, sp.alpha)
        assert np.array_equal(s_.astype(bool), osu.astype(bool)), (x0, y0)
        m = osu.astype(bool)
        if m.any():
            assert np.abs(d[m] - od[m]).max() <= DISP_TOL, (x0, y0)
    del disp, sup
    torch.cuda.empty_cache()
