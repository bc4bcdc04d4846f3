"""Extension (north_star "uncertainty-weighted blending"; SURVEY Appendix A.2,
no reference counterpart): nrm_blend_frame_weighted.

* u == 1 everywhere must be the reference rule bit for bit (same canvas as
  nrm_blend_frame, same BlendStats);
* with a real uncertainty map (the EMDQ field's own per-pixel uncertainty on
  the frame grid) the GPU matches the C restatement of the same rule
  (oracle/nrm_oracle.c: orc_blend_frame_weighted): BlendStats and weights
  exact, colour within 1e-3, as for the reference rule."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

COLOR_TOL = 1e-3


def split_polys(g):
    out, o = [], 0
    for n in g["npoly"]:
        out.append(g["polys"][o:o + n])
        o += n
    return out


def test_uniform_uncertainty_is_the_reference_rule(nrm, ctx, golden):
    g = golden("blend_c1_seq")
    polys = split_polys(g)
    h, w = g["frame"].shape[:2]
    ones = np.ones((h, w), np.float32)
    a, b = nrm.Canvas(ctx), nrm.Canvas(ctx)
    for k, poly in enumerate(polys):
        sa = nrm.blend_frame(a, g["frame"], g["anchors"], g["warps"][k], float(g["alpha"]), poly).as_tuple()
        sb = nrm.blend_frame(b, g["frame"], g["anchors"], g["warps"][k], float(g["alpha"]), poly,
                             unc=ones).as_tuple()
        assert sa == sb
    ca, wa = a.read()
    cb, wb = b.read()
    assert np.array_equal(wa, wb)
    assert np.array_equal(ca, cb)


def test_weighted_blend_matches_oracle(nrm, ctx, oracle, golden):
    from paper_2103_07414_b200 import workload as W
    g = golden("blend_c1_seq")
    e = golden("emdq_c1")
    polys = split_polys(g)
    h, w = g["frame"].shape[:2]
    # the EMDQ field's own per-pixel uncertainty on the frame grid (>= 1)
    _, unc = nrm.emdq_field((0.0, 0.0, w, h), e["apts"], e["locals"], e["probs"], e["active"], float(e["alpha"]),
                            float(e["beta"]) * 40.0, 16, ctx=ctx)
    assert unc.min() >= 1.0 and unc.max() > 2.0
    cv, ocv = nrm.Canvas(ctx), oracle.canvas()
    for k, poly in enumerate(polys):
        st = nrm.blend_frame(cv, g["frame"], g["anchors"], g["warps"][k], float(g["alpha"]), poly,
                             unc=unc).as_tuple()
        ost = oracle.blend_frame_weighted(ocv, g["frame"], g["anchors"], g["warps"][k], float(g["alpha"]), poly,
                                          unc)
        assert st == ost
    col, wt = cv.read()
    ocol, owt = ocv.arrays()
    assert np.array_equal(wt, owt)
    assert np.abs(col.astype(np.float64) - ocol).max() <= COLOR_TOL
    # and the weighting did something: differs from the reference rule
    ref = oracle.canvas()
    for k, poly in enumerate(polys):
        oracle.blend_frame(ref, g["frame"], g["anchors"], g["warps"][k], float(g["alpha"]), poly)
    rcol, _ = ref.arrays()
    assert np.abs(rcol - ocol).max() > 1e-2
    del W


def test_weighted_device_variant(nrm, ctx, golden):
    import torch
    g = golden("blend_c1")
    polys = split_polys(g)
    h, w = g["frame"].shape[:2]
    rng = np.random.default_rng(1)
    unc = (1.0 + 3.0 * rng.random((h, w))).astype(np.float32)
    dev = torch.device("cuda", 0)
    a, b = nrm.Canvas(ctx), nrm.Canvas(ctx)
    sa = nrm.blend_frame(a, g["frame"], g["anchors"], g["warps"][0], float(g["alpha"]), polys[0], unc=unc)
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
    st = torch.zeros(4, dtype=torch.int64, device=dev)
    nrm.blend_frame_device(b, T(g["frame"]), w, h, 3, T(g["anchors"]), T(g["warps"][0]), float(g["alpha"]),
                           polys[0], st, unc_t=T(unc))
    ctx.synchronize()
    assert tuple(st.cpu().tolist()) == sa.as_tuple()
    ca, wa = a.read()
    cb, wb = b.read()
    assert np.array_equal(wa, wb) and np.array_equal(ca, cb)


@pytest.mark.parametrize("off", [0.0, 21000.0])
def test_node_variance_field_matches_oracle(nrm, ctx, oracle, off):
    """Dense Engine::blended_variance_at (slam.hpp:703-714):
    within 1e-6 of max |var| of the reference formula (oracle, pinned to the
    reference by test_variance_field_restates_the_reference)."""
    rng = np.random.default_rng(12)
    n = 73
    pos = rng.uniform(-50, 700, (n, 2)) + off
    var = rng.uniform(0.0, 40.0, n)
    grid = (off - 3.5, off + 2.0, 640, 480)
    v = nrm.variance_field(grid, pos, var, 8.265e-5, ctx=ctx)
    ov = oracle.variance_field(grid, pos, var, 8.265e-5)
    assert np.abs(v - ov).max() <= 1e-6 * var.max()


def test_blend_weighted_by_node_variance(nrm, ctx, oracle):
    """The node-variance map as the uncertainty of the weighted blend:
    u = 1 + v / 4 at the frame's own node positions (the SLAM engine's
    current positions), against the oracle's weighted blend with the same map."""
    from paper_2103_07414_b200 import workload as W
    wl = W.frame_workload("c1")
    rng = np.random.default_rng(3)
    var = rng.uniform(0.0, 20.0, len(wl.anchors))
    pos = np.stack([W._apply_warps(wl.warps[i:i + 1], wl.anchors[i:i + 1])[0] for i in range(len(wl.anchors))])
    v = nrm.variance_field((0.0, 0.0, wl.frame_w, wl.frame_h), pos, var, wl.params.alpha, ctx=ctx)
    unc = (1.0 + v / 4.0).astype(np.float32)
    assert unc.max() > 2.0
    poly = nrm.invert_frame_boundary(wl.frame_w, wl.frame_h, wl.anchors, wl.warps, wl.params.alpha, ctx=ctx)
    cv, ocv = nrm.Canvas(ctx), oracle.canvas()
    for k in range(2):
        st = nrm.blend_frame(cv, wl.frame, wl.anchors, wl.warps, wl.params.alpha, poly, unc=unc).as_tuple()
        ost = oracle.blend_frame_weighted(ocv, wl.frame, wl.anchors, wl.warps, wl.params.alpha, poly, unc)
        assert st == ost
    col, wt = cv.read()
    ocol, owt = ocv.arrays()
    assert np.array_equal(wt, owt)
    assert np.abs(col.astype(np.float64) - ocol).max() <= 1e-3
