"""Extension (north_star "deforming the existing canvas with bilinear
sampling", no reference counterpart): nrm_canvas_deform.

* d == 0 is a bit-exact no-op on a real mosaic (golden two-frame sequence);
* an integer translation moves occupied pixels exactly;
* a smooth sub-pixel deformation (the node field of the C1 lattice, shrunk)
  matches the C restatement (oracle orc_canvas_deform) bit for bit: both run
  the same unfused FP64 arithmetic on float32 canvas values."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def split_polys(g):
    out, o = [], 0
    for n in g["npoly"]:
        out.append(g["polys"][o:o + n])
        o += n
    return out


@pytest.fixture()
def mosaic(nrm, ctx, golden):
    g = golden("blend_c1_seq")
    cv = nrm.Canvas(ctx)
    for k, poly in enumerate(split_polys(g)):
        nrm.blend_frame(cv, g["frame"], g["anchors"], g["warps"][k], float(g["alpha"]), poly)
    return cv, g


def test_zero_deformation_is_a_bitwise_noop(nrm, mosaic):
    cv, _ = mosaic
    col0, wt0 = cv.read()
    h, w = wt0.shape
    cv.deform(np.zeros((h, w, 2), np.float32))
    col1, wt1 = cv.read()
    assert np.array_equal(wt0, wt1) and np.array_equal(col0, col1)


def test_integer_translation_moves_pixels_exactly(nrm, mosaic):
    cv, _ = mosaic
    col0, wt0 = cv.read()
    h, w = wt0.shape
    y0, x0, hh, ww = 100, 120, 300, 400
    d = np.zeros((hh, ww, 2), np.float32)
    d[..., 0], d[..., 1] = 7.0, -3.0
    cv.deform(d, x0, y0)
    col1, wt1 = cv.read()
    src = (slice(y0 - 3, y0 - 3 + hh), slice(x0 + 7, x0 + 7 + ww))
    dst = (slice(y0, y0 + hh), slice(x0, x0 + ww))
    assert np.array_equal(wt1[dst], wt0[src])
    assert np.array_equal(col1[dst], col0[src])
    # outside the rectangle nothing moved
    mask = np.ones((h, w), bool)
    mask[dst] = False
    assert np.array_equal(wt1[mask], wt0[mask]) and np.array_equal(col1[mask], col0[mask])


def test_smooth_deformation_matches_oracle(nrm, ctx, oracle, mosaic):
    cv, g = mosaic
    col0, wt0 = cv.read()
    h, w = wt0.shape
    ox, oy = cv.origin_offset()
    # the oracle canvas starts from the same float32 values
    ocv = oracle.canvas()
    ocv.ensure_contains((ox, oy, ox + w - 1, oy + h - 1))
    assert ocv.info() == (int(ox), int(oy), w, h)
    ocv.set_arrays(col0.astype(np.float32).astype(np.float64), wt0)
    # a smooth field with sub-pixel and multi-pixel parts
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    d = np.stack([3.5 * np.sin(xx / 97.0) + 0.25 * np.cos(yy / 41.0),
                  -2.25 * np.cos(yy / 83.0) + 0.125 * np.sin(xx / 29.0)], -1).astype(np.float32)
    cv.deform(d)
    ocv.deform(0, 0, w, h, d)
    col1, wt1 = cv.read()
    ocol, owt = ocv.arrays()
    assert np.array_equal(wt1, owt)
    assert np.array_equal(col1.astype(np.float64), ocol)
    assert (wt1 > 0).sum() > 0.9 * (wt0 > 0).sum()
