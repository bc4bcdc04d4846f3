"""GPU: several frames per call (nrm_blend_frames_device, the multi-GPU
weak-scaling step's per-rank blends). Frames with pairwise disjoint
footprints go through one batched planner / field / exception launch; the
canvas, the weights and every frame's BlendStats must equal the frame-by-frame
blend_frame calls bit for bit, on whole and banded canvases. Overlapping
frames fall back to frame-by-frame blending with the same results."""
import numpy as np
import pytest

from paper_2103_07414_b200 import workload as W

pytestmark = pytest.mark.gpu


def frames_setup(nrm, ctx, shift_x, G):
    import torch
    wl = W.frame_workload("c1")
    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    anc = [wl.anchors + np.array([k * shift_x, 0.0]) for k in range(G)]
    war = [W.shifted_warps(wl.warps, k * shift_x, 0.0) for k in range(G)]
    polys = [nrm.invert_frame_boundary(wl.frame_w, wl.frame_h, a, q, wl.params.alpha, ctx=ctx)
             for a, q in zip(anc, war)]
    return wl, T(wl.frame), [T(a) for a in anc], [T(q) for q in war], polys, dev


def run(nrm, ctx, band, G, shift_x, batched):
    import torch
    wl, fr, anc, war, polys, dev = frames_setup(nrm, ctx, shift_x, G)
    cv = nrm.Canvas(ctx)
    if band is not None:
        cv.set_band(*band)
    st = torch.zeros((G, 4), dtype=torch.int64, device=dev)
    if batched:
        nrm.blend_frames_device(cv, [fr] * G, wl.frame_w, wl.frame_h, 3, anc, war, wl.params.alpha, polys, st)
    else:
        for k in range(G):
            nrm.blend_frame_device(cv, fr, wl.frame_w, wl.frame_h, 3, anc[k], war[k], wl.params.alpha, polys[k],
                                   st[k])
    ctx.synchronize()
    col, wt = cv.read()
    return st.cpu().numpy(), col, wt, (cv.origin_offset(), cv.width(), cv.height())


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("band", [None, (0, 2), (1, 4)])
def test_batched_disjoint_frames_equal_sequential(nrm, ctx, G, band):
    shift = 800.0  # the C1 footprint spans about 710 px: pairwise disjoint footprints
    a = run(nrm, ctx, band, G, shift, batched=True)
    b = run(nrm, ctx, band, G, shift, batched=False)
    assert np.array_equal(a[0], b[0])
    assert a[3] == b[3]
    assert np.array_equal(a[2], b[2])
    assert np.array_equal(a[1], b[1])
    assert (a[0][:, 1] > 0).all() if band is None else True


def test_batch_takes_one_launch_per_stage(nrm, ctx):
    import torch
    wl, fr, anc, war, polys, dev = frames_setup(nrm, ctx, 800.0, 8)
    cv = nrm.Canvas(ctx)
    st = torch.zeros((8, 4), dtype=torch.int64, device=dev)
    cv.ensure_contains((-100.0, -100.0, 8 * 800.0, 600.0))
    ctx.synchronize()
    n0 = ctx.launch_count()
    nrm.blend_frames_device(cv, [fr] * 8, wl.frame_w, wl.frame_h, 3, anc, war, wl.params.alpha, polys, st)
    ctx.synchronize()
    assert ctx.launch_count() - n0 == 4  # frame textures, planner, field, exception pass for all 8 frames
    assert (st[:, 1] > 0).all()


def test_overlapping_frames_fall_back_in_order(nrm, ctx):
    a = run(nrm, ctx, None, 4, 200.0, batched=True)  # overlapping footprints: order matters
    b = run(nrm, ctx, None, 4, 200.0, batched=False)
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[2], b[2])
    assert np.array_equal(a[1], b[1])
    assert (a[2] >= 2).any()  # the frames really overlap
