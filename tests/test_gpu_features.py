"""GPU parity of the sparse front end: to_gray,
detect_features and match_features (features.hpp:58-254, image.hpp:63-75) on
the B200 against the reference's golden vectors and the C restatement.

Every output is compared bit for bit: keypoint positions and responses,
descriptors (FP32 bits), the keypoint order, the matches and their scores."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN_CASES = ["self", "translate", "noise", "tiny", "scene_rgb"]


def textured(w, h, seed, passes=2):
    """Box-blurred random bytes (the shape of test_features.cpp:14-32)."""
    rng = np.random.default_rng(seed)
    a = rng.integers(0, 256, (h, w)).astype(np.int32)
    for _ in range(passes):
        b = a.copy()
        s = sum(a[1 + dy:h - 1 + dy, 1 + dx:w - 1 + dx] for dy in (-1, 0, 1) for dx in (-1, 0, 1))
        b[1:-1, 1:-1] = s // 9
        a = b
    return a.astype(np.uint8)


def same_features(got, want):
    (k1, d1), (k2, d2) = got, want
    assert k1.shape == k2.shape, (k1.shape, k2.shape)
    assert np.array_equal(k1, k2)
    assert np.array_equal(d1.view(np.uint32), d2.view(np.uint32))


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_features_match_reference_golden(nrm, ctx, golden, case):
    g = golden("features")
    ka, da = nrm.detect_features(g[f"{case}_a"], ctx=ctx)
    kb, db = nrm.detect_features(g[f"{case}_b"], ctx=ctx)
    same_features((ka, da), (g[f"{case}_kpa"], g[f"{case}_da"]))
    same_features((kb, db), (g[f"{case}_kpb"], g[f"{case}_db"]))
    for key in g:
        if key.startswith(f"{case}_m"):
            ratio = int(key[len(case) + 2:]) / 100.0
            assert np.array_equal(nrm.match_features(ka, da, kb, db, ratio, ctx=ctx), g[key]), key


def test_gray_input_equals_image_input(nrm, ctx, oracle):
    im = textured(300, 220, 5)
    gray = oracle.to_gray(im)
    same_features(nrm.detect_features(gray, ctx=ctx), nrm.detect_features(im, ctx=ctx))


def test_fullsize_frames_match_oracle(nrm, ctx, oracle):
    """Two 1080p RGB frames of the C2 workload's synthetic scene."""
    from paper_2103_07414_b200 import workload as W
    wl = W.frame_workload("c2")
    a = wl.frame
    b = np.roll(a, (7, -12), axis=(0, 1))
    ga, gb = oracle.to_gray(a), oracle.to_gray(b)
    want_a, want_b = oracle.detect_features(ga), oracle.detect_features(gb)
    got_a, got_b = nrm.detect_features(a, ctx=ctx), nrm.detect_features(b, ctx=ctx)
    same_features(got_a, want_a)
    same_features(got_b, want_b)
    assert len(got_a[0]) == 800
    m = nrm.match_features(*got_a, *got_b, 0.8, ctx=ctx)
    assert np.array_equal(m, oracle.match_features(*want_a, *want_b, 0.8))
    assert len(m) > 100


@pytest.mark.parametrize("cfg", [dict(nms_radius=0), dict(nms_radius=1), dict(nms_radius=10),
                                 dict(max_features=1), dict(max_features=37), dict(max_features=5000),
                                 dict(quality=0.0), dict(quality=0.2), dict(quality=0.9)])
def test_detector_config_variants(nrm, ctx, oracle, cfg):
    im = textured(400, 300, 11, passes=1)
    args = dict(max_features=800, quality=0.005, nms_radius=4)
    args.update(cfg)
    g = oracle.to_gray(im)
    same_features(nrm.detect_features(im, ctx=ctx, **args), oracle.detect_features(g, **args))


def test_tied_responses_take_the_global_sort(nrm, ctx, oracle):
    """A periodic pattern gives thousands of maxima with the same response:
    more than 2048 survive the radix select, so the selection falls back to
    the global bitonic sort. The order among ties is by (y, x, raster)."""
    tile = np.zeros((12, 12), np.uint8)
    tile[3:9, 3:9] = 200
    im = np.tile(tile, (90, 100))  # 1080 x 1200
    g = oracle.to_gray(im)
    want = oracle.detect_features(g, max_features=800)
    got = nrm.detect_features(im, max_features=800, ctx=ctx)
    same_features(got, want)
    assert len(np.unique(want[0][:, 2])) < 10  # heavily tied


@pytest.mark.parametrize("ch", [1, 3, 4])
def test_channel_layouts(nrm, ctx, oracle, ch):
    rng = np.random.default_rng(ch)
    im = rng.integers(0, 256, (160, 200, ch), dtype=np.uint8)
    for _ in range(2):  # smooth every channel a little
        im[1:-1, 1:-1] = ((im[:-2, 1:-1].astype(int) + im[2:, 1:-1] + im[1:-1, :-2] + im[1:-1, 2:]) // 4)
    g = oracle.to_gray(im)
    same_features(nrm.detect_features(im, ctx=ctx), oracle.detect_features(g))


def test_edge_cases(nrm, ctx, oracle):
    # smaller than 2 * margin + 1 = 21 px: no features (features.hpp:144)
    k, d = nrm.detect_features(textured(20, 40, 1), ctx=ctx)
    assert len(k) == 0 and d.shape == (0, 64)
    im = textured(21, 21, 2)
    same_features(nrm.detect_features(im, ctx=ctx), oracle.detect_features(oracle.to_gray(im)))
    # constant image: max response 0 -> nothing (features.hpp:151)
    assert len(nrm.detect_features(np.full((64, 64), 77, np.uint8), ctx=ctx)[0]) == 0
    # matching needs na > 0 and nb >= 2 (features.hpp:211)
    ka, da = nrm.detect_features(textured(120, 100, 3), ctx=ctx)
    assert len(nrm.match_features(ka, da, ka[:1], da[:1], ctx=ctx)) == 0
    assert len(nrm.match_features(ka[:0], da[:0], ka, da, ctx=ctx)) == 0
    two = nrm.match_features(ka, da, ka[:2], da[:2], 0.8, ctx=ctx)
    assert np.array_equal(two, oracle.match_features(ka, da, ka[:2], da[:2], 0.8))
    # bad arguments fail loudly
    with pytest.raises(ValueError):
        nrm.detect_features(np.zeros((40, 40, 2), np.uint8), ctx=ctx)
    with pytest.raises(ValueError):
        nrm.detect_features(textured(60, 60, 4), nms_radius=11, ctx=ctx)


def test_device_api_and_determinism(nrm, ctx):
    import torch
    im = textured(640, 480, 9)
    b = np.roll(im, 5, axis=1)
    ka, da = nrm.detect_features(im, ctx=ctx)
    kb, db = nrm.detect_features(b, ctx=ctx)
    dev = torch.device("cuda", 0)
    cap = 800
    kp_a, ds_a = torch.zeros((cap, 3), dtype=torch.float64, device=dev), torch.zeros((cap, 64), device=dev)
    kp_b, ds_b = torch.zeros((cap, 3), dtype=torch.float64, device=dev), torch.zeros((cap, 64), device=dev)
    na, nb = torch.zeros(1, dtype=torch.int32, device=dev), torch.zeros(1, dtype=torch.int32, device=dev)
    ia = torch.from_numpy(np.ascontiguousarray(im)).to(dev)
    ib = torch.from_numpy(np.ascontiguousarray(b)).to(dev)
    nrm.detect_features_device(ia, 640, 480, 1, kp_a, ds_a, na, ctx=ctx)
    nrm.detect_features_device(ib, 640, 480, 1, kp_b, ds_b, nb, ctx=ctx)
    ctx.synchronize()
    n_a, n_b = int(na.item()), int(nb.item())
    same_features((kp_a[:n_a].cpu().numpy(), ds_a[:n_a].cpu().numpy()), (ka, da))
    same_features((kp_b[:n_b].cpu().numpy(), ds_b[:n_b].cpu().numpy()), (kb, db))
    out = torch.zeros((n_a, 5), dtype=torch.float64, device=dev)
    nm = torch.zeros(1, dtype=torch.int32, device=dev)
    nrm.match_features_device(kp_a, ds_a, n_a, kp_b, ds_b, n_b, 0.8, out, nm, ctx=ctx)
    ctx.synchronize()
    m_host = nrm.match_features(ka, da, kb, db, 0.8, ctx=ctx)
    assert np.array_equal(out[:int(nm.item())].cpu().numpy(), m_host)
    # run-to-run determinism
    same_features(nrm.detect_features(im, ctx=ctx), (ka, da))
    assert np.array_equal(nrm.match_features(ka, da, kb, db, 0.8, ctx=ctx), m_host)
