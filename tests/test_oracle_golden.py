"""CPU: the C restatement (oracle/) must reproduce the reference's golden
vectors (tests/golden, produced by the real reference via oracle/_ref and
oracle/make_golden.py) bit for bit. This pins the oracle the GPU parity
tests compare against."""
import hashlib

import numpy as np
import pytest

BLEND_CASES = ["first_frame", "repeated_constant", "translated", "deformed", "weight_cap", "gray_rotated",
               "c1", "c1_seq"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def split_polys(g):
    out, o = [], 0
    for n in g["npoly"]:
        out.append(g["polys"][o:o + n])
        o += n
    return out


def test_pixel_warp_known_answers(oracle, golden):
    g = golden("pixel_warp")
    # test_mosaic.cpp:39-49 SingleNodeDominates
    w = oracle.pixel_warp(100, 100, g["single_anchors"], g["single_warps"], 2e-4)
    assert w[0] == 1.5
    assert np.array_equal(w, g["single_out"])
    got = oracle.warp_apply(w, 7, 9)
    want = oracle.warp_apply(g["single_warps"][0], 7, 9)
    assert np.abs(got - want).max() < 1e-12
    # test_mosaic.cpp:67-76 MidpointOfTwoTranslationsAverages
    a = np.array([[100.0, 100.0], [140.0, 100.0]])
    q = np.array([[1.0, 1.0, 0.0, 0.0, 0.0], [1.0, 1.0, 0.0, 1.0, 0.0]])
    w = oracle.pixel_warp(120, 100, a, q, 2e-4)
    assert np.abs(oracle.warp_apply(w, 120, 100) - [121.0, 100.0]).max() < 1e-12
    # test_mosaic.cpp:78-82 NoSupportFarFromNodes
    assert oracle.pixel_warp(1e4, 1e4, np.array([[0.0, 0.0]]), np.array([[1.0, 1, 0, 0, 0]]), 2e-4) is None


def test_pixel_warp_matches_reference_bitwise(oracle, golden):
    g = golden("pixel_warp")
    for (x, y), want, ok in zip(g["points"], g["out"], g["valid"]):
        got = oracle.pixel_warp(x, y, g["anchors"], g["warps"], float(g["alpha"]))
        assert (got is not None) == bool(ok)
        if ok:
            assert np.array_equal(got, want)


def test_invert_frame_boundary_matches_reference_bitwise(oracle, golden):
    g = golden("invert_boundary")
    poly = oracle.invert_frame_boundary(int(g["fw"]), int(g["fh"]), g["anchors"], g["warps"], float(g["alpha"]))
    assert np.array_equal(poly, g["poly"])


@pytest.mark.parametrize("case", BLEND_CASES)
def test_blend_frame_matches_reference_bitwise(oracle, golden, case):
    g = golden(f"blend_{case}")
    cv = oracle.canvas()
    for k, poly in enumerate(split_polys(g)):
        st = oracle.blend_frame(cv, g["frame"], g["anchors"], g["warps"][k], float(g["alpha"]), poly)
        assert st == tuple(g["stats"][k])
    assert tuple(cv.info()) == tuple(g["canvas_info"])
    col, wt = cv.arrays()
    assert sha(col) == str(g["color_sha"])
    assert sha(wt) == str(g["weight_sha"])
    img, org = oracle.render(cv, crop=True)
    assert sha(img) == str(g["render_crop_sha"])
    assert org == tuple(g["crop_origin"])
    full, _ = oracle.render(cv, crop=False)
    assert sha(full) == str(g["render_full_sha"])


def test_blend_frame_reference_test_semantics(oracle, golden):
    """The reference's own BlendFrame assertions (test_mosaic.cpp:84-224)."""
    g = golden("blend_first_frame")
    assert tuple(g["stats"][0])[1] == 320 * 200                      # FirstFrameInsertsExactly
    img = g["render_crop"]
    assert img.shape == (200, 320, 4) and np.array_equal(img[..., :3], g["frame"])
    g = golden("blend_repeated_constant")                             # capped weight 30
    assert int(g["weight"].max()) == 30
    g = golden("blend_weight_cap")
    assert int(g["weight"].max()) <= 30
    g = golden("blend_translated")                                    # overlap weight 2
    assert int(g["weight"].max()) == 2 and g["render_crop"].shape[1] == 256 + 100


def test_empty_inputs_give_empty_stats(oracle):
    cv = oracle.canvas()
    a = np.array([[0.0, 0.0]])
    q = np.array([[1.0, 1, 0, 0, 0]])
    assert oracle.blend_frame(cv, np.zeros((0, 0, 3), np.uint8), a, q, 2e-4, [[0, 0], [1, 0], [1, 1]]) == (0, 0, 0, 0)
    assert oracle.blend_frame(cv, np.zeros((8, 8, 3), np.uint8), a, q, 2e-4, [[0, 0], [1, 0]]) == (0, 0, 0, 0)
    assert cv.info()[2] == 0  # canvas untouched (mosaic.hpp:201)
    img, _ = oracle.render(cv, crop=True)
    assert img.shape[:2] == (0, 0)


def test_node_uncertainty_known_answers(oracle):
    """test_fieldest.cpp:184-214."""
    assert oracle.node_uncertainty(100, 100, [[100, 100]], 3e-3) == 1.0
    assert abs(oracle.node_uncertainty(100, 100, [[110, 100]], 3e-3) - 1.3498588075760032) < 1e-12
    assert oracle.node_uncertainty(100, 100, [[105, 100], [150, 100]], 3e-3) == np.exp(3e-3 * 25.0)
    assert np.isnan(oracle.node_uncertainty(0, 0, np.zeros((0, 2)), 3e-3))
    prev = 0.0
    for d in range(0, 401, 20):
        u = oracle.node_uncertainty(d, 0, [[0, 0]], 3e-3)
        assert u >= prev and u >= 1.0
        prev = u


def test_emdq_points_match_reference_bitwise(oracle, golden):
    g = golden("emdq_c1")
    for (x, y), want, wu in zip(g["qpts"], g["qout"], g["qunc"]):
        got = oracle.blend_local(g["locals"], g["apts"], g["probs"], g["active"], x, y, float(g["alpha"]))
        assert np.array_equal(got, want)
        assert oracle.node_uncertainty(x, y, g["apts"][g["active"]], float(g["beta"])) == wu
    # node increments of the reference's estimate_field = blend_local at the anchors
    for a, inc in zip(g["node_anchors"], g["node_inc"]):
        got = oracle.blend_local(g["locals"], g["apts"], g["probs"], g["active"], a[0], a[1], float(g["alpha"]))
        assert np.array_equal(got, inc)


def test_emdq_grid_matches_reference(oracle, golden):
    g = golden("emdq_c1")
    x0, y0, w, h = g["grid"]
    disp, unc = oracle.emdq_field_grid((x0, y0, int(w), int(h)), g["apts"], g["locals"], g["probs"], g["active"],
                                       float(g["alpha"]), float(g["beta"]))
    assert sha(disp) == str(g["disp_sha"])
    assert sha(unc) == str(g["unc_sha"])


def test_emdq_edge_cases_match_reference(oracle, golden):
    g = golden("emdq_edge")
    x0, y0, w, h = g["grid"]
    grid = (x0, y0, int(w), int(h))
    d, u = oracle.emdq_field_grid(grid, g["apts"], g["locals"], g["probs"], g["small_active"], float(g["alpha"]),
                                  float(g["beta"]))
    assert np.array_equal(d, g["disp_small"]) and np.array_equal(u, g["unc_small"])
    d, u = oracle.emdq_field_grid(grid, g["apts"], g["locals"], g["probs"], g["active"], float(g["alpha"]),
                                  float(g["beta"]), support=4)
    assert np.array_equal(d, g["disp_s4"]) and np.array_equal(u, g["unc_s4"])


def test_oracle_estep_matches_reference(oracle, golden):
    """The C restatement's blend_local over active minus j reproduces the
    reference's E-step (fieldest.hpp:195-209) bit for bit."""
    g = golden("emdq_estep")
    c1 = golden("emdq_c1")
    for name in ("c1", "few"):
        act = g[f"{name}_active"]
        for j in range(0, len(c1["apts"]), 7):
            others = act[act != j]
            w = oracle.blend_local(c1["locals"], c1["apts"], c1["probs"], others, *c1["apts"][j],
                                   float(c1["alpha"]), 16)
            assert np.array_equal(w, g[f"{name}_warps"][j]), (name, j)
            assert np.array_equal(oracle.warp_apply(w, *c1["apts"][j]), g[f"{name}_pred"][j]), (name, j)


def test_oracle_weighted_blend_with_unit_uncertainty_is_reference(oracle, golden):
    """Extension rule: u == 1 everywhere reproduces the reference update bit for bit."""
    g = golden("blend_c1")
    poly = g["polys"][: g["npoly"][0]]
    h, w = g["frame"].shape[:2]
    a, b = oracle.canvas(), oracle.canvas()
    sa = oracle.blend_frame(a, g["frame"], g["anchors"], g["warps"][0], float(g["alpha"]), poly)
    sb = oracle.blend_frame_weighted(b, g["frame"], g["anchors"], g["warps"][0], float(g["alpha"]), poly,
                                     np.ones((h, w), np.float32))
    assert sa == sb
    ca, wa = a.arrays()
    cb, wb = b.arrays()
    assert np.array_equal(wa, wb) and np.array_equal(ca, cb)


FEATURE_CASES = ["self", "translate", "noise", "tiny", "scene_rgb"]


@pytest.mark.parametrize("case", FEATURE_CASES)
def test_oracle_features_match_reference_bitwise(oracle, golden, case):
    """to_gray / detect_features / match_features (features.hpp) of the C
    restatement against the reference on its own detector-test fixtures."""
    g = golden("features")
    ga, gb = oracle.to_gray(g[f"{case}_a"]), oracle.to_gray(g[f"{case}_b"])
    assert sha(ga) == str(g[f"{case}_ga_sha"]) and sha(gb) == str(g[f"{case}_gb_sha"])
    ka, da = oracle.detect_features(ga)
    kb, db = oracle.detect_features(gb)
    assert np.array_equal(ka, g[f"{case}_kpa"]) and np.array_equal(kb, g[f"{case}_kpb"])
    assert np.array_equal(da.view(np.uint32), g[f"{case}_da"].view(np.uint32))
    assert np.array_equal(db.view(np.uint32), g[f"{case}_db"].view(np.uint32))
    for key in g:
        if key.startswith(f"{case}_m"):
            ratio = int(key[len(case) + 2:]) / 100.0
            assert np.array_equal(oracle.match_features(ka, da, kb, db, ratio), g[key]), key


def test_features_reference_test_semantics(golden):
    """The reference's detector tests (test_features.cpp:48-127) on the golden
    outputs: self-matches have zero displacement, a 10-px wrap translation is
    recovered by >= 80 % of the matches, noise gives few matches, a tiny image
    none, and stricter ratios give fewer matches."""
    g = golden("features")
    m = g["self_m80"]
    assert len(m) > 20 and np.array_equal(m[:, 0:2], m[:, 2:4])
    assert ((m[:, 4] >= 0) & (m[:, 4] <= 1)).all()
    t = g["translate_m80"]
    good = ((np.abs(t[:, 2] - t[:, 0] - 10) <= 1) & (np.abs(t[:, 3] - t[:, 1]) <= 1)).sum()
    assert len(t) > 30 and good >= 0.8 * len(t)
    assert len(g["noise_m80"]) < min(len(g["noise_kpa"]), len(g["noise_kpb"])) // 5 + 5
    assert len(g["tiny_kpa"]) == 0 and len(g["tiny_m80"]) == 0
    assert len(g["translate_m60"]) <= len(g["translate_m80"]) <= len(g["translate_m95"])


def test_fast_emdq_grid_reproduces_the_reference_golden(oracle, golden):
    """orc_emdq_field_grid_fast (grid kNN + OpenMP rows), the checker the
    full-frame C2/C4/C5 GPU tests use, reproduces the reference's dense C1
    field bit for bit (golden SHA from oracle/_ref)."""
    g = golden("emdq_c1")
    x0, y0, w, h = g["grid"]
    disp, unc = oracle.emdq_field_grid((x0, y0, int(w), int(h)), g["apts"], g["locals"], g["probs"], g["active"],
                                       float(g["alpha"]), float(g["beta"]), 16, fast=True)
    assert sha(disp) == str(g["disp_sha"])
    assert sha(unc) == str(g["unc_sha"])


@pytest.mark.parametrize("seed", range(6))
def test_fast_emdq_grid_equals_full_scan(oracle, seed):
    """Clustered / duplicated candidates (index tie-breaks), queries far outside
    the candidates' box, support 1..32, canvas-scale coordinates: the grid
    search selects the same keys in the same order as the full scan."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 300))
    m = n + 5
    off = np.array([0.0, 0.0]) if seed % 3 == 0 else rng.uniform(8000, 32000, 2) * rng.choice([-1, 1], 2)
    apts = np.round(rng.normal(0, 60, (m, 2)) * 4) / 4 + off
    if seed % 2:
        apts[: n // 2] = apts[n // 2: 2 * (n // 2)]  # exact duplicates: (d2, j) ties
    loc = np.zeros((m, 5))
    ang = rng.uniform(-3, 3, m)
    loc[:, 0] = rng.uniform(0.5, 2, m)
    loc[:, 1], loc[:, 2] = np.cos(ang / 2), np.sin(ang / 2)
    loc[:, 3:] = rng.normal(0, 5, (m, 2))
    pr = rng.uniform(0, 1, m)
    pr[::7] = 0.0
    act = np.sort(rng.choice(m, n, replace=False)).astype(np.int32)
    grid = (off[0] - 300.5, off[1] - 200.25, 257, 181)
    for sup in (1, 7, 16, 32):
        a = oracle.emdq_field_grid(grid, apts, loc, pr, act, 1e-3, 2e-3, sup)
        b = oracle.emdq_field_grid(grid, apts, loc, pr, act, 1e-3, 2e-3, sup, fast=True)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), sup


def test_variance_field_restates_the_reference():
    """orc_variance_field = Engine::blended_variance_at (slam.hpp:703-714),
    called on the reference itself (oracle/_ref), bit for bit."""
    from oracle import oracle as orc
    if not orc.reference_available():
        pytest.skip("oracle/_ref not built (reference tree absent)")
    O, R = orc.Oracle(), orc.Reference()
    rng = np.random.default_rng(4)
    for off, n in ((0.0, 70), (23000.0, 5), (-9000.5, 160)):
        pos = rng.uniform(-100, 700, (n, 2)) + off
        var = rng.uniform(0, 50, n)
        grid = (off - 20.5, off + 10.25, 37, 23)
        a = O.variance_field(grid, pos, var, 2e-4)
        gx, gy = np.meshgrid(grid[0] + np.arange(grid[2]), grid[1] + np.arange(grid[3]))
        b = R.blended_variance_at(np.stack([gx.ravel(), gy.ravel()], 1), pos, var, 2e-4).reshape(a.shape)
        assert np.array_equal(a, b)
