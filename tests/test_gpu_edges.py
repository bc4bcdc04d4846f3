"""Edge cases and error behaviour of the scattered-point EMDQ (E-step), the
weighted blend and the canvas deformation, against the oracle (which the
golden tests pin to the reference) where a value is defined, and against the
reference's exception rules where it is not (std::invalid_argument ->
NRM_EINVAL -> ValueError in Python)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _c1(golden):
    g = golden("emdq_c1")
    return g["apts"], g["locals"], g["probs"], g["active"], float(g["alpha"]), float(g["beta"])


def test_points_support_larger_than_candidates(nrm, ctx, oracle, golden):
    """kk = min(support, |active|) (fieldest.hpp:88): 5 candidates, support 16."""
    ap, lo, pr, act, alpha, beta = _c1(golden)
    act5 = act[:5]
    q = np.array([[100.0, 80.0], [600.0, 400.0], [-1000.0, 5000.0]])
    w, pred, unc, st = nrm.emdq_points(q, ap, lo, pr, act5, alpha, beta, 16, ctx=ctx)
    assert (st == 0).all()
    for k in range(len(q)):
        ow = oracle.blend_local(lo, ap, pr, act5, q[k, 0], q[k, 1], alpha, 16)
        assert np.array_equal(w[k], ow)
        assert unc[k] == oracle.node_uncertainty(q[k, 0], q[k, 1], ap[act5], beta)


def test_points_far_and_coincident_queries(nrm, ctx, oracle, golden):
    """Queries far outside the candidates' hull (the d2min rescaling keeps the
    weights finite, fieldest.hpp:71-74) and exactly on a candidate."""
    ap, lo, pr, act, alpha, beta = _c1(golden)
    q = np.array([[1e5, -3e4], [ap[act[7], 0], ap[act[7], 1]], [-2e5, 2e5]])
    w, _, unc, st = nrm.emdq_points(q, ap, lo, pr, act, alpha, beta, 16, ctx=ctx)
    assert (st == 0).all()
    for k in range(len(q)):
        assert np.array_equal(w[k], oracle.blend_local(lo, ap, pr, act, q[k, 0], q[k, 1], alpha, 16))
    assert unc[1] == 1.0  # node_uncertainty at an inlier: exp(0)


def test_points_exclusion_of_every_candidate(nrm, ctx, golden):
    """A lone candidate excluded -> status 1 (the E-step's others.empty())."""
    ap, lo, pr, act, alpha, beta = _c1(golden)
    j = int(act[3])
    w, pred, _, st = nrm.emdq_points(ap[[j]], ap, lo, pr, act[3:4], alpha, beta, 16,
                                     exclude=np.array([j], np.int32), ctx=ctx)
    assert st.tolist() == [1]
    assert (w == 0).all() and (pred == 0).all()


def test_points_reject_bad_arguments(nrm, ctx, golden):
    ap, lo, pr, act, alpha, beta = _c1(golden)
    q = np.array([[1.0, 2.0]])
    with pytest.raises(ValueError):  # active index out of range
        nrm.emdq_points(q, ap, lo, pr, np.array([len(ap)], np.int32), alpha, beta, 16, ctx=ctx)
    with pytest.raises(ValueError):  # support outside [1, 32]
        nrm.emdq_points(q, ap, lo, pr, act, alpha, beta, 33, ctx=ctx)
    with pytest.raises(ValueError):  # beta <= 0 with uncertainty requested (fieldest.hpp:46)
        nrm.emdq_points(q, ap, lo, pr, act, alpha, 0.0, 16, ctx=ctx)
    with pytest.raises(ValueError):  # non-finite query
        nrm.emdq_points(np.array([[np.nan, 1.0]]), ap, lo, pr, act, alpha, beta, 16, ctx=ctx)
    # an empty query set is fine
    w, _, _, st = nrm.emdq_points(np.zeros((0, 2)), ap, lo, pr, act, alpha, beta, 16, ctx=ctx)
    assert w.shape == (0, 5)


def test_weighted_blend_clamps_low_or_invalid_uncertainty(nrm, ctx, golden):
    """u < 1 or NaN counts as u = 1 (confidence 1): the reference rule."""
    g = golden("blend_c1")
    poly = g["polys"][: g["npoly"][0]]
    h, w = g["frame"].shape[:2]
    low = np.full((h, w), 0.25, np.float32)
    low[::7, ::5] = np.nan
    a, b = nrm.Canvas(ctx), nrm.Canvas(ctx)
    nrm.blend_frame(a, g["frame"], g["anchors"], g["warps"][0], float(g["alpha"]), poly)
    nrm.blend_frame(b, g["frame"], g["anchors"], g["warps"][0], float(g["alpha"]), poly, unc=low)
    ca, wa = a.read()
    cb, wb = b.read()
    assert np.array_equal(wa, wb)
    # NaN taps poison only the bilinear sample of their neighbourhood; away
    # from them the result is the reference rule exactly
    assert np.abs(ca - cb).max() <= 1e-3


def test_weighted_blend_rejects_shape_and_null(nrm, ctx, golden):
    g = golden("blend_c1")
    poly = g["polys"][: g["npoly"][0]]
    cv = nrm.Canvas(ctx)
    with pytest.raises(ValueError):
        nrm.blend_frame(cv, g["frame"], g["anchors"], g["warps"][0], float(g["alpha"]), poly,
                        unc=np.ones((10, 10), np.float32))


def test_deform_edges(nrm, ctx, golden):
    """Sources beyond the canvas leave pixels unoccupied; bad regions are
    rejected (also on banded canvases)."""
    g = golden("blend_c1")
    poly = g["polys"][: g["npoly"][0]]
    cv = nrm.Canvas(ctx)
    nrm.blend_frame(cv, g["frame"], g["anchors"], g["warps"][0], float(g["alpha"]), poly)
    _, wt0 = cv.read()
    h, w = wt0.shape
    d = np.zeros((h, w, 2), np.float32)
    d[..., 0] = 1e6  # everything samples outside
    cv.deform(d)
    _, wt1 = cv.read()
    assert (wt1 == 0).all()
    with pytest.raises(ValueError):
        cv.deform(np.zeros((10, 10, 2), np.float32), x=w - 5, y=0)  # region outside the canvas
    # banded canvases deform their own stripes (halo rows: dist.exchange_halo)
    banded = nrm.Canvas(ctx)
    banded.ensure_contains((0.0, 0.0, 300.0, 300.0))
    banded.set_band(0, 2)
    banded.deform(np.zeros((8, 8, 2), np.float32))
    with pytest.raises(ValueError):
        banded.deform(np.zeros((8, 8, 2), np.float32), x=-1)


def test_rgba_frame_ignores_alpha(nrm, ctx, oracle, golden):
    """ImageU8 with 4 channels: sample_bilinear_rgb reads RGB and ignores
    alpha (image.hpp:78-92). An RGBA copy of the golden frame must give the
    same canvas as the RGB frame, on the GPU and in the oracle."""
    g = golden("blend_c1")
    poly = g["polys"][: g["npoly"][0]]
    rgb = g["frame"]
    rng = np.random.default_rng(4)
    rgba = np.concatenate([rgb, rng.integers(0, 256, rgb.shape[:2] + (1,), dtype=np.uint8)], axis=2)
    a, b = nrm.Canvas(ctx), nrm.Canvas(ctx)
    sa = nrm.blend_frame(a, rgb, g["anchors"], g["warps"][0], float(g["alpha"]), poly).as_tuple()
    sb = nrm.blend_frame(b, rgba, g["anchors"], g["warps"][0], float(g["alpha"]), poly).as_tuple()
    assert sa == sb
    ca, wa = a.read()
    cb, wb = b.read()
    assert np.array_equal(wa, wb) and np.array_equal(ca, cb)
    oa, ob = oracle.canvas(), oracle.canvas()
    assert oracle.blend_frame(oa, rgb, g["anchors"], g["warps"][0], float(g["alpha"]), poly) == \
        oracle.blend_frame(ob, rgba, g["anchors"], g["warps"][0], float(g["alpha"]), poly)
    assert np.array_equal(oa.arrays()[0], ob.arrays()[0])
