// snapshot_dump.cpp -- TEST INFRASTRUCTURE: records node states with the
// reference's own writers (snapshot.hpp:17-44 write_snapshot, 80-104
// TrajectoryWriter) while running the reference pipeline (the run_mosaic call
// sequence of tools/main.cpp on the reference's synthetic scene), plus the
// frames and footprints of the blended frames, for the replay fixtures
// (oracle/make_golden.py replay_case; paper_2103_07414_b200/replay.py reads
// them). Built against the unmodified reference headers (oracle/Makefile).
//
// usage: snapshot_dump <outdir> <frames> [scan|outback] [scene_frames]
//   the scene is built for scene_frames (default 200, the camera path spans
//   the scene's frames) and the first <frames> of it are run
//   <outdir>/snapshot_<t>.json   write_snapshot after frame t (blended frames)
//   <outdir>/frame_<t>.rgb       the frame (w*h*3 bytes), footprint_<t>.txt
//   <outdir>/trajectory.jsonl    TrajectoryWriter lines, every frame
#include <cstdio>
#include <string>

#include "nrmosaic/config.hpp"
#include "nrmosaic/features.hpp"
#include "nrmosaic/mosaic.hpp"
#include "nrmosaic/slam.hpp"
#include "nrmosaic/snapshot.hpp"
#include "nrmosaic/synth.hpp"

using namespace nrmosaic;

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    const std::string dir = argv[1];
    SceneSpec spec;
    const int run_frames = std::atoi(argv[2]);
    spec.frames = argc > 4 ? std::atoi(argv[4]) : 200;
    spec.path = argc > 3 ? argv[3] : "scan";
    spec.path_extent = 240.0;
    const SyntheticScene scene = SyntheticScene::build(spec);
    Config cfg;
    cfg.workers = 8;
    const Engine::Params params = make_engine_params(cfg, spec.width, spec.height);
    DetectorConfig det = make_detector_config(cfg);
    det.workers = 8;
    Engine engine(params);
    TrajectoryWriter traj(dir + "/trajectory.jsonl");
    auto record = [&](int t, const ImageU8& frame) {
        write_snapshot(dir + "/snapshot_" + std::to_string(t) + ".json", engine.graph());
        std::FILE* f = std::fopen((dir + "/frame_" + std::to_string(t) + ".rgb").c_str(), "wb");
        std::fwrite(frame.data.data(), 1, frame.data.size(), f);
        std::fclose(f);
        f = std::fopen((dir + "/footprint_" + std::to_string(t) + ".txt").c_str(), "w");
        for (const Vec2& p : engine.last_footprint()) std::fprintf(f, "%.17g %.17g\n", p.x, p.y);
        std::fclose(f);
    };
    for (int t = 0; t < run_frames; ++t) {
        const ImageU8 frame = scene.render_frame(t, 8);
        const FrameFeatures cur = detect_features(to_gray(frame), det);
        if (t == 0) {
            engine.initialize(cur, frame.width, frame.height);
            traj.append(0, FrameStatus::Tracked, engine.graph());
            record(0, frame);
            continue;
        }
        const auto matches = match_features(engine.previous_features(), cur, det.ratio_test, 8);
        const FrameReport rep = engine.process_frame(cur, matches, [&](const KeyFrame& kf) {
            return match_features(kf.features, cur, det.ratio_test, 8);
        });
        traj.append(t, rep.status, engine.graph());
        if (rep.status != FrameStatus::Lost && t % cfg.blend_stride == 0) record(t, frame);
    }
    std::printf("%d %d\n", spec.width, spec.height);
    return 0;
}
