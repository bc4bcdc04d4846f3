"""CPU: the drop-in header compiles against the REAL reference types (the
reference's geometry/dualquat/image headers) with a call sequence shaped like
the reference CLI's (tools/main.cpp:174-176, 229-230, 268). Skipped where the
reference tree is absent (the GPU box)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/proj")

SRC = r'''
#include "nrmosaic_b200/mosaic.hpp"
using namespace nrmosaic;
int run(const ImageU8& frame, std::span<const Vec2> anchors, std::span<const WarpFunction> warps, double alpha) {
    Canvas canvas;
    const auto poly = invert_frame_boundary(frame.width, frame.height, anchors, warps, alpha);
    const BlendStats s = blend_frame(canvas, frame, anchors, warps, alpha, poly, 8);
    Vec2 origin;
    const ImageU8 mosaic = render(canvas, true, &origin);
    const auto w = pixel_warp(Vec2{1.0, 2.0}, anchors, warps, alpha);
    return static_cast<int>(s.blended_pixels) + mosaic.width + (w ? 1 : 0) + canvas.weight(0, 0);
}
'''


@pytest.mark.skipif(not (REF / "include" / "nrmosaic" / "mosaic.hpp").exists(), reason="reference tree absent")
def test_shim_compiles_against_reference_types(tmp_path):
    src = tmp_path / "dropin.cpp"
    src.write_text(SRC)
    cmd = ["g++", "-std=c++20", "-fsyntax-only", "-include", "algorithm", "-include", "memory",
           f"-I{ROOT / 'include'}", f"-I{ROOT / 'oracle' / 'stub'}", f"-I{REF / 'include'}", str(src)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


SRC_FEATURES = r'''
#include "nrmosaic_b200/features.hpp"
using namespace nrmosaic;
// the front end as the reference CLI runs it (tools/main.cpp:169-216, 367-377)
std::size_t run(const ImageU8& a, const ImageU8& b, const std::string& path) {
    DetectorConfig cfg;
    cfg.workers = 8;
    const FrameFeatures fa = detect_features(to_gray(a), cfg);
    const FrameFeatures fb = detect_features(b, cfg);
    const auto m = match_features(fa, fb, cfg.ratio_test, cfg.workers);
    save_matches(path, detect_and_match(a, b, cfg));
    return m.size() + load_matches(path).size() + fa.descriptors.size();
}
'''


@pytest.mark.skipif(not (REF / "include" / "nrmosaic" / "image.hpp").exists(), reason="reference tree absent")
def test_features_shim_compiles_against_reference_types(tmp_path):
    src = tmp_path / "dropin_features.cpp"
    src.write_text(SRC_FEATURES)
    cmd = ["g++", "-std=c++20", "-fsyntax-only", "-include", "algorithm", "-include", "memory",
           f"-I{ROOT / 'include'}", f"-I{ROOT / 'oracle' / 'stub'}", f"-I{REF / 'include'}", str(src)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


SRC_PRODUCTION = r'''
// the reference CLI's include set (tools/main.cpp:15-19 minus the json/CLI11
// parts): slam.hpp re-includes nrmosaic/mosaic.hpp (slam.hpp:16) and
// nrmosaic/features.hpp (slam.hpp:13)
#include "nrmosaic/config.hpp"
#include "nrmosaic/mosaic.hpp"
#include "nrmosaic/slam.hpp"
#include "nrmosaic/synth.hpp"
using namespace nrmosaic;
#ifndef NRM_B200_H
#error "the override did not take effect: nrmosaic/mosaic.hpp is not the B200 drop-in"
#endif
int run(const SyntheticScene& scene) {
    Config cfg;
    const auto params = make_engine_params(cfg, scene.spec().width, scene.spec().height);
    const DetectorConfig det = make_detector_config(cfg);
    Engine engine(params);
    Canvas canvas;
    const ImageU8 f0 = scene.render_frame(0, 1);
    engine.initialize(detect_features(to_gray(f0), det), f0.width, f0.height);
    const BlendStats s = blend_frame(canvas, f0, engine.graph().anchors(), engine.graph().warps(), params.alpha,
                                     engine.last_footprint(), 8);
    Vec2 origin;
    return static_cast<int>(s.blended_pixels) + render(canvas, true, &origin).width;
}
'''


@pytest.mark.skipif(not (REF / "include" / "nrmosaic" / "slam.hpp").exists(), reason="reference tree absent")
def test_override_compiles_the_reference_include_set(tmp_path):
    """The production callers include both nrmosaic/mosaic.hpp and
    nrmosaic/slam.hpp; with -Iinclude/override both resolve to the B200
    drop-in without redefinition errors."""
    src = tmp_path / "production.cpp"
    src.write_text(SRC_PRODUCTION)
    cmd = ["g++", "-std=c++20", "-fsyntax-only", "-include", "algorithm", "-include", "memory",
           f"-I{ROOT / 'include' / 'override'}", f"-I{ROOT / 'include'}", f"-I{ROOT / 'oracle' / 'stub'}",
           f"-I{REF / 'include'}", str(src)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_match_files_round_trip_in_the_reference_format(tmp_path):
    """save_matches / load_matches of the shim write the reference's format
    (features.hpp:272-305): a '# ax ay bx by score' header, %.17g fields."""
    src = tmp_path / "mf.cpp"
    src.write_text(r'''
#include "nrmosaic_b200/features.hpp"
#include <cstdio>
using namespace nrmosaic;
int main(int argc, char** argv) {
    std::vector<MatchPair> m(2);
    m[0].point_a = Vec2{0.1, -2.5}; m[0].point_b = Vec2{1e-300, 123456.789012345678}; m[0].score = 0.3333333333333333;
    m[1].point_a = Vec2{-0.0, 7.0}; m[1].point_b = Vec2{1.0 / 3.0, 2.0 / 3.0}; m[1].score = 1.0;
    save_matches(argv[1], m);
    const auto r = load_matches(argv[1]);
    bool ok = r.size() == 2;
    for (std::size_t i = 0; ok && i < 2; ++i)
        ok = r[i].point_a.x == m[i].point_a.x && r[i].point_a.y == m[i].point_a.y && r[i].point_b.x == m[i].point_b.x &&
             r[i].point_b.y == m[i].point_b.y && r[i].score == m[i].score;
    try { load_matches(argv[2]); ok = false; } catch (const std::runtime_error& e) { std::printf("%s\n", e.what()); }
    return ok ? 0 : 1;
}
''')
    exe = tmp_path / "mf"
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-DNRM_B200_STANDALONE_TYPES", f"-I{ROOT / 'include'}", str(src),
                        "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    bad = tmp_path / "bad.txt"
    bad.write_text("# header\n\n1 2 3 4 5\n1 2 3 4\n")
    r = subprocess.run([str(exe), str(tmp_path / "m.txt"), str(bad)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip() == f"{bad}:4: expected 5 fields 'ax ay bx by score'"
    lines = (tmp_path / "m.txt").read_text().splitlines()
    want = ["# ax ay bx by score"] + ["%.17g %.17g %.17g %.17g %.17g" % v for v in
                                      [(0.1, -2.5, 1e-300, 123456.789012345678, 0.3333333333333333),
                                       (-0.0, 7.0, 1.0 / 3.0, 2.0 / 3.0, 1.0)]]
    assert lines == want
