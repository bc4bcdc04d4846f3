// pipeline_dump.cpp -- TEST INFRASTRUCTURE: the reference's production call
// sequence (tools/main.cpp run_mosaic: detect -> match -> Engine::process_frame
// -> blend_frame every blend_stride-th tracked frame -> render(crop)), driven
// by the reference's own synthetic scene (synth.hpp SyntheticScene), written
// against the reference's public API only.
//
// Built twice from this one source:
//   oracle/_ref/pipeline_ref      -- the reference headers as they are (CPU)
//   tests/cpp/pipeline_b200       -- -Iinclude/override: every
//                                    "nrmosaic/mosaic.hpp" (this file's,
//                                    slam.hpp:16's) is the B200 drop-in
// and the two dumps are compared (tests/test_gpu_dropin.py): identical
// per-frame status, BlendStats and node trajectories, mosaic within +-1.
//
// usage: pipeline_dump <out.bin> [scan|outback] [frames] [workers] [width height]
// Output (little endian): "NRMP" u32 version=1, i32 frames, then per frame
// i32 status (FrameStatus: 0 tracked, 1 loop closed, 2 lost), i32 blended (0/1),
// i64[4] BlendStats, i32 nodes, f64[nodes][2] positions; then the mosaic:
// i32 w, i32 h, f64 origin x, f64 origin y, u8[h][w][4].
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "nrmosaic/config.hpp"
#include "nrmosaic/features.hpp"
#include "nrmosaic/mosaic.hpp"
#include "nrmosaic/slam.hpp"
#include "nrmosaic/synth.hpp"

using namespace nrmosaic;

namespace {
template <class T>
void put(std::FILE* f, const T& v) {
    std::fwrite(&v, sizeof(T), 1, f);
}
}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s out.bin [scan|outback] [frames] [workers]\n", argv[0]);
        return 2;
    }
    SceneSpec spec;
    spec.path = argc > 2 ? argv[2] : "scan";
    spec.path_extent = 240.0;
    if (argc > 3) spec.frames = std::atoi(argv[3]);
    const int workers = argc > 4 ? std::atoi(argv[4]) : 8;
    if (argc > 6) {  // other resolutions: the scene scales like the reference's Config (config.hpp:144-157)
        spec.width = std::atoi(argv[5]);
        spec.height = std::atoi(argv[6]);
        const double s = (spec.width / 480.0 + spec.height / 270.0) / 2.0;
        spec.max_displacement *= s;
        spec.bump_radius *= s;
        spec.path_extent *= s;
    }
    const SyntheticScene scene = SyntheticScene::build(spec);

    Config cfg;
    cfg.workers = workers;
    const Engine::Params params = make_engine_params(cfg, spec.width, spec.height);
    DetectorConfig det = make_detector_config(cfg);
    det.workers = workers;

    std::FILE* out = std::fopen(argv[1], "wb");
    if (!out) return 3;
    std::fwrite("NRMP", 1, 4, out);
    put(out, std::uint32_t{1});
    put(out, std::int32_t{spec.frames});

    Engine engine(params);
    Canvas canvas;
    auto dump = [&](int status, const BlendStats* bs) {
        put(out, std::int32_t{status});
        put(out, std::int32_t{bs ? 1 : 0});
        const BlendStats z{};
        const BlendStats& s = bs ? *bs : z;
        put(out, s.footprint_pixels);
        put(out, s.blended_pixels);
        put(out, s.skipped_no_support);
        put(out, s.skipped_out_of_frame);
        const auto pos = engine.graph().positions();
        put(out, std::int32_t(pos.size()));
        for (const Vec2& p : pos) {
            put(out, p.x);
            put(out, p.y);
        }
    };
    for (int t = 0; t < spec.frames; ++t) {
        const ImageU8 frame = scene.render_frame(t, workers);
        const FrameFeatures cur = detect_features(to_gray(frame), det);
        if (t == 0) {
            engine.initialize(cur, frame.width, frame.height);
            const BlendStats bs = blend_frame(canvas, frame, engine.graph().anchors(), engine.graph().warps(),
                                              params.alpha, engine.last_footprint(), workers);
            dump(0, &bs);
            continue;
        }
        const auto matches = match_features(engine.previous_features(), cur, det.ratio_test, workers);
        const FrameReport rep = engine.process_frame(cur, matches, [&](const KeyFrame& kf) {
            return match_features(kf.features, cur, det.ratio_test, workers);
        });
        const int status = static_cast<int>(rep.status);
        if (rep.status != FrameStatus::Lost && t % cfg.blend_stride == 0) {
            const BlendStats bs = blend_frame(canvas, frame, engine.graph().anchors(), engine.graph().warps(),
                                              params.alpha, engine.last_footprint(), workers);
            dump(status, &bs);
        } else {
            dump(status, nullptr);
        }
    }
    Vec2 origin;
    const ImageU8 mosaic = render(canvas, true, &origin);
    put(out, std::int32_t{mosaic.width});
    put(out, std::int32_t{mosaic.height});
    put(out, origin.x);
    put(out, origin.y);
    std::fwrite(mosaic.data.data(), 1, mosaic.data.size(), out);
    std::fclose(out);
    std::printf("frames %d mosaic %dx%d\n", spec.frames, mosaic.width, mosaic.height);
    return 0;
}
