"""GPU parity at BASELINE.json's full sizes (configs[1] = C2, configs[3] = C4).

The oracle (the C restatement, pinned to the reference by the golden tests)
runs the same inputs:
  * C2 and C4 blend_frame in full: BlendStats and the weight plane must match
    exactly, colour to 1e-3, the rendered mosaic to +-1 level;
  * C2 / C4 dense EMDQ field on bands of rows spread over the frame (top,
    middle, bottom): displacement <= 1e-3 px, uncertainty <= 1e-6 relative;
  * C4 node field (K2) on windows at the frame centre and corner.
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


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_emdq_field_full_size_rows_match_oracle(nrm, ctx, oracle, name):
    wl = W.frame_workload(name)
    e = wl.emdq
    grid = (0.0, 0.0, wl.frame_w, wl.frame_h)
    disp, unc = nrm.emdq_field(grid, e.apts, e.locals_, e.probs, e.active, wl.params.alpha, wl.params.beta, 16,
                               ctx=ctx)
    assert np.isfinite(disp).all() and np.isfinite(unc).all()
    h = wl.frame_h
    rows = 8 if name == "c2" else 4
    for r0 in (0, h // 2 - rows // 2, h - rows):
        od, ou = oracle.emdq_field_grid(grid, e.apts, e.locals_, e.probs, e.active, wl.params.alpha,
                                        wl.params.beta, 16, rows=(r0, r0 + rows))
        err = np.abs(disp[r0:r0 + rows] - od[r0:r0 + rows]).max()
        assert err <= DISP_TOL, (name, r0, err)
        rel = np.abs(unc[r0:r0 + rows] / ou[r0:r0 + rows] - 1).max()
        assert rel <= 1e-6, (name, r0, rel)


def test_c4_node_field_windows_match_oracle(nrm, ctx, oracle):
    wl = W.frame_workload("c4")
    for (x0, y0) in ((1792.0, 976.0), (0.0, 0.0), (3584.0, 1904.0)):
        grid = (x0, y0, 256, 256)
        disp, sup = nrm.node_field(grid, wl.anchors, wl.warps, wl.params.alpha, ctx=ctx)
        od, osup = oracle.node_field_grid(grid, wl.anchors, wl.warps, wl.params.alpha)
        assert np.array_equal(sup.astype(bool), osup.astype(bool))
        m = osup.astype(bool)
        assert np.abs(disp[m] - od[m]).max() <= DISP_TOL


def test_c4_blend_frame_full_matches_oracle(nrm, ctx, oracle):
    """configs[3] frame size: one 3840 x 2160 frame into a fresh canvas with its
    frame lattice, in full (about 9 M footprint pixels)."""
    wl = W.frame_workload("c4")
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
