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
