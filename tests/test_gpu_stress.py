"""Canvas-scale randomized parity and adversarial stress of the fast tiers'
routing margins (k_nodefield.cu kCutLo/kCutHi/kBoundMargin, k_emdq.cu
d2_tol; DESIGN.md §5 derives them).

At reference coordinates of 8k-32k px an FP32 ulp is 1e-3 to 4e-3 px, which
is where a fast tier that took absolute coordinates would mis-decide. Every
case here is compared with the oracle (pinned to the reference by the golden
tests), with the parity bars of tests/test_gpu_parity.py: BlendStats, weight
planes and supports exact, fields <= 1e-3 px, colour <= 1e-3, render +-1.

Adversarial inputs put many pixels exactly ON a decision:
* node weights exactly at the 1e-6 cutoff (mosaic.hpp:250): integer anchors,
  integer pixels and alpha = -ln(1e-6) / R2 with R2 = 5525, which has 48
  lattice representations x^2 + y^2 = R2, so 48 pixels per node sit on the
  cutoff (and their neighbours within one FP64 ulp of it);
* frame positions exactly on the frame edges (mosaic.hpp:271): integer
  translations of the identity warp;
* kNN-16 membership decided by exact (d2, j) ties (fieldest.hpp:82-85):
  candidates on an integer lattice (with duplicates) queried at integer
  pixels, with wildly different local warps so a wrong member shows."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
N = int(os.environ.get("NRM_FUZZ_SEEDS", "8"))
DISP_TOL = 1e-3
COLOR_TOL = 1e-3
R2 = 5525
ALPHA_CUT = -np.log(1e-6) / R2


def big_offset(rng):
    return rng.uniform(8000, 32000, 2) * rng.choice([-1.0, 1.0], 2)


def random_warps(rng, n, rot=np.pi, scale=(0.5, 2.0), trans=40.0):
    ang = rng.uniform(-rot, rot, n)
    q = np.zeros((n, 5))
    q[:, 0] = rng.uniform(*scale, n)
    q[:, 1], q[:, 2] = np.cos(ang / 2), np.sin(ang / 2)
    q[:, 3:5] = rng.normal(0, trans, (n, 2))
    return q


def conjugated(warps, t):
    """x -> W(x - t) + t: a warp defined around the origin moved to canvas
    coordinates around t, displacements unchanged (the canvas-wide fields of
    configs[3]/[4] are near-identity at any position)."""
    from paper_2103_07414_b200 import workload as W
    q = W.shifted_warps(warps, t[0], t[1])
    w_, z_, s_ = q[:, 1], q[:, 2], q[:, 0]
    # output + t: translation 2 M d grows by t / s  ->  d += M^T t / (2 s)
    q[:, 3] += (w_ * t[0] + z_ * t[1]) / (2 * s_)
    q[:, 4] += (-z_ * t[0] + w_ * t[1]) / (2 * s_)
    return q


def field_tol(ref):
    """1e-3 px plus half an FP32 ulp of the value: displacements are returned
    as float32 (nrm_node_field / nrm_emdq_field), whose ulp exceeds 1e-3 px
    beyond 8192 px of displacement."""
    return DISP_TOL + 0.5 * np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)


def compare_blends(nrm, ctx, oracle, frame, seq, alpha):
    """seq: [(anchors, warps)]; blends each with its own footprint on a GPU and
    an oracle canvas and compares everything."""
    fh, fw = frame.shape[:2]
    cv, ocv = nrm.Canvas(ctx), oracle.canvas()
    for anchors, warps in seq:
        poly = nrm.invert_frame_boundary(fw, fh, anchors, warps, alpha, ctx=ctx)
        st = nrm.blend_frame(cv, frame, anchors, warps, alpha, poly).as_tuple()
        ost = oracle.blend_frame(ocv, frame, anchors, warps, alpha, poly)
        assert st == ost, (st, ost)
    assert (cv.origin_offset(), cv.width(), cv.height()) == (tuple(map(float, ocv.info()[:2])),) + ocv.info()[2:]
    col, wt = cv.read()
    ocol, owt = ocv.arrays()
    assert np.array_equal(wt, owt)
    assert np.abs(col.astype(np.float64) - ocol).max() <= COLOR_TOL
    img, org = nrm.render(cv, crop=True)
    oimg, oorg = oracle.render(ocv, crop=True)
    assert org == oorg and np.abs(img.astype(int) - oimg.astype(int)).max() <= 1
    return ost


# ---- canvas-scale randomized ------------------------------------------------
@pytest.mark.parametrize("seed", range(N))
def test_canvas_scale_node_field(nrm, ctx, oracle, seed):
    rng = np.random.default_rng(500 + seed)
    off = big_offset(rng)
    n = int(rng.integers(1, 120))
    x0, y0 = off[0] + rng.uniform(-50, 50), off[1] + rng.uniform(-50, 50)
    if seed % 2:
        x0, y0 = np.floor(x0) + 0.5, np.floor(y0) + 0.25
    w, h = int(rng.integers(40, 220)), int(rng.integers(30, 160))
    anchors = np.stack([rng.uniform(x0 - 200, x0 + w + 200, n), rng.uniform(y0 - 200, y0 + h + 200, n)], 1)
    warps = random_warps(rng, n, rot=np.pi if seed % 3 == 0 else 0.3, scale=(0.9, 1.1) if seed % 2 else (0.5, 2.0))
    if seed % 4 != 3:  # near-identity at the offset; seed % 4 == 3: raw warps (displacements of 1e4-1e5 px)
        warps = conjugated(warps, off)
    alpha = float(rng.uniform(2e-5, 2e-3))
    grid = (float(x0), float(y0), w, h)
    disp, sup = nrm.node_field(grid, anchors, warps, alpha, ctx=ctx)
    od, osup = oracle.node_field_grid(grid, anchors, warps, alpha)
    assert np.array_equal(sup.astype(bool), osup.astype(bool))
    m = osup.astype(bool)
    if m.any():
        assert (np.abs(disp[m] - od[m]) <= field_tol(od[m])).all()


@pytest.mark.parametrize("seed", range(max(1, 3 * N // 4)))
def test_canvas_scale_blend_sequence(nrm, ctx, oracle, seed):
    from paper_2103_07414_b200 import workload as W
    rng = np.random.default_rng(600 + seed)
    fw, fh = int(rng.integers(60, 200)), int(rng.integers(50, 150))
    ch = (1, 3, 4)[seed % 3]
    frame = rng.integers(0, 256, (fh, fw, ch), dtype=np.uint8)
    if ch == 1:
        frame = frame[:, :, 0]
    base = W.hex_lattice((0.0, 0.0, float(fw), float(fh)), float(rng.uniform(15, 60)))
    alpha = float(rng.uniform(3e-4, 3e-3))
    off = big_offset(rng)
    seq = []
    for k in range(3):
        warps = random_warps(rng, len(base), rot=0.25 if seed % 2 else 0.05, scale=(0.9, 1.15), trans=6.0)
        warps[:, 3:5] += rng.normal(0, 20.0, 2)
        # the same canvas->frame map, moved to canvas coordinates around `off`
        seq.append((base + off, W.shifted_warps(warps, off[0], off[1])))
    compare_blends(nrm, ctx, oracle, frame, seq, alpha)


@pytest.mark.parametrize("seed", range(N))
def test_canvas_scale_emdq(nrm, ctx, oracle, seed):
    rng = np.random.default_rng(700 + seed)
    off = big_offset(rng)
    m = int(rng.integers(20, 400))
    w, h = int(rng.integers(40, 200)), int(rng.integers(30, 150))
    x0, y0 = float(off[0]), float(off[1])
    if seed % 3 == 0:
        centres = np.stack([rng.uniform(x0, x0 + w, 5), rng.uniform(y0, y0 + h, 5)], 1)
        apts = centres[rng.integers(0, 5, m)] + rng.normal(0, 3.0, (m, 2))
    else:
        apts = np.stack([rng.uniform(x0 - 50, x0 + w + 50, m), rng.uniform(y0 - 50, y0 + h + 50, m)], 1)
    if seed % 4 == 1:
        apts[1::7] = apts[0::7][: len(apts[1::7])]
    locals_ = random_warps(rng, m, rot=np.pi if seed % 2 else 0.2, scale=(0.8, 1.25), trans=10.0)
    if seed % 4 != 3:
        locals_ = conjugated(locals_, off)
    probs = rng.uniform(0, 1, m)
    probs[rng.random(m) < 0.2] = 0.0
    active = np.sort(rng.choice(m, int(rng.integers(1, m + 1)), replace=False)).astype(np.int32)
    support = int((1, 4, 16, 32)[seed % 4])
    alpha, beta = float(rng.uniform(1e-4, 5e-3)), float(rng.uniform(1e-4, 5e-3))
    grid = (x0, y0, w, h)
    disp, unc = nrm.emdq_field(grid, apts, locals_, probs, active, alpha, beta, support, ctx=ctx)
    od, ou = oracle.emdq_field_grid(grid, apts, locals_, probs, active, alpha, beta, support, fast=True)
    fin = np.isfinite(od).all(-1)
    assert np.array_equal(np.isfinite(disp).all(-1), fin)
    if fin.any():
        assert (np.abs(disp[fin] - od[fin]) <= field_tol(od[fin])).all()
    assert np.abs(unc / ou - 1).max() <= 1e-6


# ---- adversarial: decisions exactly on the margins -----------------------------
def cutoff_ring_count():
    k = int(np.sqrt(R2))
    return sum(1 for x in range(-k, k + 1) for y in range(-k, k + 1) if x * x + y * y == R2)


@pytest.mark.parametrize("seed", range(4))
def test_weights_exactly_at_the_cutoff(nrm, ctx, oracle, seed):
    """Node field and blend where many pixels carry a node weight of exactly
    exp(-ln 1e-6) ~ 1e-6 (the reference's `w <= 1e-6` decides them by the last
    bit of its FP64 exp)."""
    assert cutoff_ring_count() == 48
    rng = np.random.default_rng(800 + seed)
    off = np.floor(big_offset(rng)) if seed else np.zeros(2)
    n = 6
    # integer anchors, sparse enough that each ring's pixels see few other nodes
    anchors = off + np.stack([rng.integers(0, 400, n), rng.integers(0, 300, n)], 1).astype(np.float64)
    warps = conjugated(random_warps(rng, n, rot=0.2, scale=(0.95, 1.05), trans=3.0), off)
    grid = (float(off[0] - 80), float(off[1] - 80), 560, 460)
    disp, sup = nrm.node_field(grid, anchors, warps, ALPHA_CUT, ctx=ctx)
    od, osup = oracle.node_field_grid(grid, anchors, warps, ALPHA_CUT)
    assert np.array_equal(sup.astype(bool), osup.astype(bool))
    m = osup.astype(bool)
    assert np.abs(disp[m] - od[m]).max() <= DISP_TOL
    # pixels whose only node sits exactly on the cutoff: support is decided there
    gx, gy = np.meshgrid(grid[0] + np.arange(grid[2]), grid[1] + np.arange(grid[3]))
    d2 = (gx[..., None] - anchors[:, 0]) ** 2 + (gy[..., None] - anchors[:, 1]) ** 2
    on_ring = (d2 == R2).any(-1)
    assert on_ring.sum() >= 48
    # and the mosaic update over the same nodes (frame = the node region,
    # identity warps moved to the canvas-scale offset)
    from paper_2103_07414_b200 import workload as W
    fw, fh = 400, 300
    frame = rng.integers(0, 256, (fh, fw, 3), dtype=np.uint8)
    q = np.tile(np.array([1.0, 1.0, 0.0, 0.0, 0.0]), (n, 1))
    seq = [(anchors, W.shifted_warps(q, off[0], off[1]))]
    ost = compare_blends(nrm, ctx, oracle, frame, seq, ALPHA_CUT)
    assert ost[2] > 0  # some pixels lack support: the cutoff is inside the footprint


@pytest.mark.parametrize("seed", range(4))
def test_frame_positions_exactly_on_the_frame_edges(nrm, ctx, oracle, seed):
    """Identity warps with integer translations put whole pixel rows and
    columns exactly on x = 0, x = W-1, y = 0, y = H-1 (mosaic.hpp:271-274),
    at canvas-scale coordinates."""
    from paper_2103_07414_b200 import workload as W
    rng = np.random.default_rng(900 + seed)
    fw, fh = int(rng.integers(80, 200)), int(rng.integers(60, 150))
    frame = rng.integers(0, 256, (fh, fw, 3), dtype=np.uint8)
    base = W.hex_lattice((0.0, 0.0, float(fw), float(fh)), 40.0)
    alpha = 1e-3
    off = np.floor(big_offset(rng)) if seed else np.zeros(2)
    seq = []
    for k in range(3):
        q = np.tile(np.array([1.0, 1.0, 0.0, 0.0, 0.0]), (len(base), 1))
        t = rng.integers(-30, 30, 2).astype(np.float64)
        q = W.shifted_warps(q, -t[0], -t[1])  # x -> x + t
        seq.append((base + off, W.shifted_warps(q, off[0], off[1])))
    ost = compare_blends(nrm, ctx, oracle, frame, seq, alpha)
    assert ost[3] > 0


@pytest.mark.parametrize("seed", range(4))
def test_knn_membership_by_exact_ties(nrm, ctx, oracle, seed):
    """Candidates on an integer lattice (plus exact duplicates) queried at
    integer pixels: the 16th / 17th keys tie in d2 at most pixels and the
    index decides (fieldest.hpp:82-85). Local warps differ by tens of pixels,
    so a wrong member would move the field far beyond 1e-3 px."""
    rng = np.random.default_rng(1000 + seed)
    off = np.floor(big_offset(rng)) if seed else np.zeros(2)
    gx, gy = np.meshgrid(np.arange(0, 120, 6.0), np.arange(0, 90, 6.0))
    apts = np.stack([gx.ravel(), gy.ravel()], 1) + off
    dup = rng.choice(len(apts), len(apts) // 5, replace=False)
    apts = np.concatenate([apts, apts[dup]])
    perm = rng.permutation(len(apts))
    apts = apts[perm]
    m = len(apts)
    locals_ = conjugated(random_warps(rng, m, rot=0.3, scale=(0.9, 1.1), trans=30.0), off)
    probs = rng.uniform(0.2, 1, m)
    active = np.sort(rng.choice(m, int(0.9 * m), replace=False)).astype(np.int32)
    grid = (float(off[0] - 3), float(off[1] - 3), 126, 96)
    for support in (16, 5):
        disp, unc = nrm.emdq_field(grid, apts, locals_, probs, active, 2e-3, 1e-3, support, ctx=ctx)
        od, ou = oracle.emdq_field_grid(grid, apts, locals_, probs, active, 2e-3, 1e-3, support)
        assert np.abs(disp - od).max() <= DISP_TOL
        assert np.abs(unc / ou - 1).max() <= 1e-6
    exact = ctx.exceptions()[1]
    assert exact > 0  # the ties were routed to the exact tier
