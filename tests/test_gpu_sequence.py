"""BASELINE configs[2]: a frame sequence mosaicked with uncertainty blending.

* C3 at C1 frame size (the oracle finishes in seconds): 24 frames along a
  serpentine scan with overlapping footprints. Each is blended with the
  uncertainty-weighted rule (the EMDQ field's per-pixel uncertainty of the
  frame) and compared with the C restatement: per-frame BlendStats and the
  weight plane exact, colour within 1e-3.
* C3 at full size (200 1080p frames into an 8192^2 canvas) against the
  REFERENCE (golden c3_sequence.npz from oracle/_ref, oracle/make_golden.py):
  every frame's BlendStats and the final weight plane exact, colour within
  1e-3 and the rendered mosaic within +-1 level at 200k sampled pixels --
  through blend_frame and through the weighted extension with u == 1;
* the same sequence via size-independent properties: the weighted rule with
  u == 1 equals the reference rule bit for bit over the whole sequence, and 4
  block-cyclic bands assemble to the single canvas bit for bit."""
import numpy as np
import pytest

from paper_2103_07414_b200 import workload as W

pytestmark = pytest.mark.gpu

COLOR_TOL = 1e-3


def sequence(wl, n, canvas):
    offs = W.scan_offsets(n, wl.frame_w, wl.frame_h, canvas)
    frames = [wl.frame, np.ascontiguousarray(wl.frame[::-1])]
    out = []
    for k, (tx, ty) in enumerate(offs):
        out.append((frames[k % 2], wl.anchors + np.array([tx, ty]), W.shifted_warps(wl.warps, tx, ty)))
    return out


def test_c3_small_sequence_weighted_matches_oracle(nrm, ctx, oracle):
    wl = W.frame_workload("c1")
    e = wl.emdq
    _, unc = nrm.emdq_field((0.0, 0.0, wl.frame_w, wl.frame_h), e.apts, e.locals_, e.probs, e.active,
                            wl.params.alpha, wl.params.beta * 20.0, 16, ctx=ctx)
    assert unc.max() > 1.5
    cv, ocv = nrm.Canvas(ctx), oracle.canvas()
    for frame, anchors, warps in sequence(wl, 24, 2048):
        poly = nrm.invert_frame_boundary(wl.frame_w, wl.frame_h, anchors, warps, wl.params.alpha, ctx=ctx)
        st = nrm.blend_frame(cv, frame, anchors, warps, wl.params.alpha, poly, unc=unc).as_tuple()
        ost = oracle.blend_frame_weighted(ocv, frame, anchors, warps, wl.params.alpha, poly, unc)
        assert st == ost
    ox, oy, w, h = ocv.info()
    assert (cv.origin_offset(), cv.width(), cv.height()) == ((ox, oy), w, h)
    col, wt = cv.read()
    ocol, owt = ocv.arrays()
    assert np.array_equal(wt, owt)
    assert np.abs(col.astype(np.float64) - ocol).max() <= COLOR_TOL
    assert (wt > 1).sum() > 0.3 * (wt > 0).sum()  # the footprints overlap


@pytest.mark.parametrize("weighted", [False, True])
def test_c3_full_sequence_matches_reference(nrm, ctx, golden, weighted):
    import hashlib
    import torch
    g = golden("c3_sequence")
    wl = W.frame_workload("c2")
    assert hashlib.sha256(np.ascontiguousarray(wl.frame).tobytes()).hexdigest() == str(g["frame_sha"]), \
        "the synthetic C2 frame differs from the one the golden was made with"
    fw, fh, alpha = wl.frame_w, wl.frame_h, float(g["alpha"])
    assert np.array_equal(W.scan_offsets(len(g["offsets"]), fw, fh, wl.canvas), g["offsets"])
    dev = torch.device("cuda", 0)
    frames_t = [torch.from_numpy(np.ascontiguousarray(f)).to(dev) for f in (wl.frame, wl.frame[::-1])]
    ones_t = torch.ones((fh, fw), dtype=torch.float32, device=dev) if weighted else None
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
    cv = nrm.Canvas(ctx)
    st = torch.zeros((len(g["offsets"]), 4), dtype=torch.int64, device=dev)
    torch.cuda.synchronize()
    for k, (tx, ty) in enumerate(g["offsets"]):
        anchors = g["anchors"] + np.array([tx, ty])
        warps = W.shifted_warps(g["warps"], tx, ty)
        poly = nrm.invert_frame_boundary(fw, fh, anchors, warps, alpha, ctx=ctx)
        a_t, q_t = T(anchors), T(warps)
        torch.cuda.synchronize()
        nrm.blend_frame_device(cv, frames_t[k % 2], fw, fh, 3, a_t, q_t, alpha, poly, st[k], unc_t=ones_t)
    ctx.synchronize()
    assert np.array_equal(st.cpu().numpy(), g["stats"]), "per-frame BlendStats differ from the reference"
    ox, oy = cv.origin_offset()
    assert (int(ox), int(oy), cv.width(), cv.height()) == tuple(int(v) for v in g["info"])
    col, wt = cv.read()
    assert hashlib.sha256(wt.tobytes()).hexdigest() == str(g["weight_sha"]), "weight plane differs"
    xs, ys = g["sample_xy"][:, 0], g["sample_xy"][:, 1]
    assert np.abs(col[ys, xs].astype(np.float64) - g["sample_color"]).max() <= COLOR_TOL
    del col
    img, _ = nrm.render(cv, crop=False)
    assert np.abs(img[ys, xs].astype(np.int16) - g["sample_render"].astype(np.int16)).max() <= 1
    assert int((img[..., 3] > 0).sum()) == int(g["occupied"])


def _planes_equal(a, b, rows=512):
    """Bitwise equality of two canvases, downloaded in row chunks."""
    assert (a.origin_offset(), a.width(), a.height()) == (b.origin_offset(), b.width(), b.height())
    for y in range(0, a.height(), rows):
        h = min(rows, a.height() - y)
        ca, wa = a.read(0, y, a.width(), h)
        cb, wb = b.read(0, y, b.width(), h)
        if not (np.array_equal(wa, wb) and np.array_equal(ca, cb)):
            return False
    return True


def test_c3_full_sequence_properties(nrm, ctx):
    import torch
    from paper_2103_07414_b200 import dist as D
    wl = W.frame_workload("c2")
    seq = sequence(wl, 200, wl.canvas)
    dev = torch.device("cuda", 0)
    fw, fh, alpha = wl.frame_w, wl.frame_h, wl.params.alpha
    frames_t = [torch.from_numpy(f).to(dev) for f in (seq[0][0], seq[1][0])]
    ones_t = torch.ones((fh, fw), dtype=torch.float32, device=dev)
    polys = [nrm.invert_frame_boundary(fw, fh, a, q, alpha, ctx=ctx) for _, a, q in seq]
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
    nodes = [(T(a), T(q)) for _, a, q in seq]

    def run(band=None, unc_t=None):
        cv = nrm.Canvas(ctx)
        cv.reserve(wl.canvas_rect)
        if band is not None:
            cv.set_band(*band)
        st = torch.zeros((len(seq), 4), dtype=torch.int64, device=dev)
        for k in range(len(seq)):
            nrm.blend_frame_device(cv, frames_t[k % 2], fw, fh, 3, nodes[k][0], nodes[k][1], alpha, polys[k],
                                   st[k], unc_t=unc_t)
        ctx.synchronize()
        return cv, st.cpu().numpy()

    ref, st_ref = run()
    assert st_ref[:, 1].sum() > 200 * 1_500_000
    wtd, st_w = run(unc_t=ones_t)
    assert np.array_equal(st_ref, st_w)
    assert _planes_equal(ref, wtd)
    del wtd
    # block-cyclic bands: each band canvas holds its own stripes; together they
    # are the single canvas, and the band stats add up to the single stats
    bands = [run(band=(r, 4)) for r in range(4)]
    assert np.array_equal(sum(b[1][:, 1:] for b in bands), st_ref[:, 1:])
    ox, oy = ref.origin_offset()
    for y in range(0, ref.height(), 512):
        h = min(512, ref.height() - y)
        c0, w0 = ref.read(0, y, ref.width(), h)
        mask = [D.owned_rows_mask(int(oy) + y, h, r, 4) for r in range(4)]
        for r, (cvb, _) in enumerate(bands):
            cb, wb = cvb.read(0, y, ref.width(), h)
            assert np.array_equal(wb[mask[r]], w0[mask[r]])
            assert np.array_equal(cb[mask[r]], c0[mask[r]])
