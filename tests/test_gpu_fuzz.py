"""Seeded randomized parity against the oracle (which the golden tests pin to
the reference), over the corners the fixed workloads do not reach:

* warps with rotations up to +-pi, so tiles span hemisphere flips and take
  the exact tier; scales 0.5-2; sparse and dense lattices; grids at negative
  and fractional origins;
* blends of 1-, 3- and 4-channel frames through arbitrary warps, with the
  frame boundary polygon from invert_frame_boundary;
* EMDQ candidate sets with clustered points, near-duplicate distances,
  probabilities down to 0 (the 1e-6 floor), support 1..32 and small active
  subsets.

Tolerances are the parity bars of tests/test_gpu_parity.py: exact for
integers and decisions, <= 1e-3 px for fields, <= 1e-3 colour, <= 1e-6
relative uncertainty; the scattered-point EMDQ is bit-exact."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
N = int(os.environ.get("NRM_FUZZ_SEEDS", "8"))  # wider sweeps: NRM_FUZZ_SEEDS=200

DISP_TOL = 1e-3
COLOR_TOL = 1e-3


def random_warps(rng, n, rot=np.pi, scale=(0.5, 2.0), trans=40.0):
    ang = rng.uniform(-rot, rot, n)
    q = np.zeros((n, 5))
    q[:, 0] = rng.uniform(*scale, n)
    q[:, 1], q[:, 2] = np.cos(ang / 2), np.sin(ang / 2)
    q[:, 3:5] = rng.normal(0, trans, (n, 2))
    return q


@pytest.mark.parametrize("seed", range(N))
def test_fuzz_node_field(nrm, ctx, oracle, seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 120))
    x0, y0 = float(rng.uniform(-500, 500)), float(rng.uniform(-500, 500))
    if seed % 2:
        x0, y0 = np.floor(x0) + 0.5, np.floor(y0) + 0.25  # fractional grid origin
    w, h = int(rng.integers(40, 220)), int(rng.integers(30, 160))
    anchors = np.stack([rng.uniform(x0 - 200, x0 + w + 200, n), rng.uniform(y0 - 200, y0 + h + 200, n)], 1)
    rot = np.pi if seed % 3 == 0 else 0.3
    warps = random_warps(rng, n, rot=rot, scale=(0.9, 1.1) if seed % 2 else (0.5, 2.0))
    alpha = float(rng.uniform(2e-5, 2e-3))
    grid = (x0, y0, w, h)
    disp, sup = nrm.node_field(grid, anchors, warps, alpha, ctx=ctx)
    od, osup = oracle.node_field_grid(grid, anchors, warps, alpha)
    assert np.array_equal(sup.astype(bool), osup.astype(bool))
    m = osup.astype(bool)
    if m.any():
        assert np.abs(disp[m] - od[m]).max() <= DISP_TOL


@pytest.mark.parametrize("seed", range(max(1, 3 * N // 4)))
def test_fuzz_blend_sequence(nrm, ctx, oracle, seed):
    from paper_2103_07414_b200 import workload as W
    rng = np.random.default_rng(200 + seed)
    fw, fh = int(rng.integers(60, 200)), int(rng.integers(50, 150))
    ch = (1, 3, 4)[seed % 3]
    frame = rng.integers(0, 256, (fh, fw, ch), dtype=np.uint8)
    if ch == 1:
        frame = frame[:, :, 0]
    anchors = W.hex_lattice((0.0, 0.0, float(fw), float(fh)), float(rng.uniform(15, 60)))
    alpha = float(rng.uniform(3e-4, 3e-3))
    cv, ocv = nrm.Canvas(ctx), oracle.canvas()
    for k in range(3):
        warps = random_warps(rng, len(anchors), rot=0.25 if seed % 2 else 0.05, scale=(0.9, 1.15), trans=6.0)
        warps[:, 3:5] += rng.normal(0, 20.0, 2)  # a common shift per frame
        poly = nrm.invert_frame_boundary(fw, fh, anchors, warps, alpha, ctx=ctx)
        st = nrm.blend_frame(cv, frame, anchors, warps, alpha, poly).as_tuple()
        ost = oracle.blend_frame(ocv, frame, anchors, warps, alpha, poly)
        assert st == ost, (k, st, ost)
    col, wt = cv.read()
    ocol, owt = ocv.arrays()
    assert np.array_equal(wt, owt)
    assert np.abs(col.astype(np.float64) - ocol).max() <= COLOR_TOL
    img, org = nrm.render(cv, crop=True)
    oimg, oorg = oracle.render(ocv, crop=True)
    assert org == oorg and np.abs(img.astype(int) - oimg.astype(int)).max() <= 1


@pytest.mark.parametrize("seed", range(N))
def test_fuzz_emdq(nrm, ctx, oracle, seed):
    rng = np.random.default_rng(300 + seed)
    m = int(rng.integers(20, 400))
    w, h = int(rng.integers(40, 200)), int(rng.integers(30, 150))
    x0, y0 = float(rng.uniform(-300, 300)), float(rng.uniform(-300, 300))
    if seed % 3 == 0:  # clustered points: many near-equal distances
        centres = np.stack([rng.uniform(x0, x0 + w, 5), rng.uniform(y0, y0 + h, 5)], 1)
        apts = centres[rng.integers(0, 5, m)] + rng.normal(0, 3.0, (m, 2))
    else:
        apts = np.stack([rng.uniform(x0 - 50, x0 + w + 50, m), rng.uniform(y0 - 50, y0 + h + 50, m)], 1)
    if seed % 4 == 1:  # exact duplicates of some points: ties broken by index
        apts[1::7] = apts[0::7][: len(apts[1::7])]
    locals_ = random_warps(rng, m, rot=np.pi if seed % 2 else 0.2, scale=(0.8, 1.25), trans=10.0)
    probs = rng.uniform(0, 1, m)
    probs[rng.random(m) < 0.2] = 0.0
    active = np.sort(rng.choice(m, int(rng.integers(1, m + 1)), replace=False)).astype(np.int32)
    support = int((1, 4, 16, 32)[seed % 4])
    alpha, beta = float(rng.uniform(1e-4, 5e-3)), float(rng.uniform(1e-4, 5e-3))
    grid = (x0, y0, w, h)
    disp, unc = nrm.emdq_field(grid, apts, locals_, probs, active, alpha, beta, support, ctx=ctx)
    od, ou = oracle.emdq_field_grid(grid, apts, locals_, probs, active, alpha, beta, support)
    fin = np.isfinite(od).all(-1)
    assert np.array_equal(np.isfinite(disp).all(-1), fin)
    if fin.any():
        assert np.abs(disp[fin] - od[fin]).max() <= DISP_TOL
    assert np.abs(unc / ou - 1).max() <= 1e-6
    # scattered points, with leave-one-out, bit-exact
    q = apts[active[: min(len(active), 40)]]
    ex = active[: len(q)]
    wq, _, _, st = nrm.emdq_points(q, apts, locals_, probs, active, alpha, beta, support, exclude=ex, ctx=ctx)
    for k in range(len(q)):
        others = active[active != ex[k]]
        if len(others) == 0:
            assert st[k] == 1
            continue
        assert st[k] == 0
        assert np.array_equal(wq[k], oracle.blend_local(locals_, apts, probs, others, q[k, 0], q[k, 1], alpha,
                                                        support))
