// nrmosaic_b200/features.hpp -- drop-in replacement for the reference's
// nrmosaic/features.hpp (proj/include/nrmosaic/features.hpp) backed by the
// B200 C ABI (include/nrm_b200.h, libnrm_b200.so). SURVEY §8f NEXT #4.
//
// Callers (tools/main.cpp:169-216, 367-377; acceptance.cpp:369-383;
// slam.hpp:13) switch by replacing
//     #include "nrmosaic/features.hpp"
// with
//     #include "nrmosaic_b200/features.hpp"
// and linking -lnrm_b200. Same names, members and results:
//   Keypoint, MatchPair, DetectorConfig, FrameFeatures  (features.hpp:19-50)
//   detect_features(const ImageF&, const DetectorConfig&)  (features.hpp:140)
//   detect_features(const ImageU8&, const DetectorConfig&) -- to_gray fused
//       on the GPU; equals detect_features(to_gray(image), cfg)
//   match_features(a, b, ratio, workers)                (features.hpp:208)
//   detect_and_match(a, b, cfg)                         (features.hpp:258)
//   save_matches / load_matches (plain host text I/O)   (features.hpp:272-305)
// Every keypoint, descriptor, match and score is bit-identical to the
// reference's (tests/test_gpu_features.py). `workers` is accepted for
// signature compatibility and ignored.
//
// ImageU8 / ImageF / Vec2 come from the reference's image.hpp / geometry.hpp
// unless NRM_B200_STANDALONE_TYPES is defined (see nrmosaic_b200/mosaic.hpp).
#pragma once

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "nrmosaic_b200/mosaic.hpp"

#ifdef NRM_B200_STANDALONE_TYPES
namespace nrmosaic {
struct ImageF {
    int width = 0, height = 0;
    std::vector<float> data;
};
}  // namespace nrmosaic
#endif

namespace nrmosaic {

struct Keypoint {
    Vec2 position;
    double response = 0.0;
};

struct MatchPair {
    Vec2 point_a;
    Vec2 point_b;
    double score = 0.0;  // descriptor similarity in [0, 1]
};

struct DetectorConfig {
    int max_features = 800;
    double quality_level = 0.005;
    int nms_radius = 4;
    double ratio_test = 0.8;
    int workers = 1;  // accepted, unused (the GPU does the work)
};

struct FrameFeatures {
    static constexpr int kDescriptorDim = 64;
    std::vector<Keypoint> keypoints;
    std::vector<float> descriptors;  // row i belongs to keypoints[i]

    const float* descriptor(std::size_t i) const { return descriptors.data() + i * kDescriptorDim; }
    std::size_t size() const { return keypoints.size(); }
};

namespace b200 {
inline nrm_detector_config detector_config(const DetectorConfig& c) {
    return nrm_detector_config{c.max_features, c.quality_level, c.nms_radius, c.ratio_test};
}
inline FrameFeatures unpack_features(const std::vector<double>& kp, std::vector<float>& desc, int n) {
    FrameFeatures f;
    f.keypoints.resize(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) f.keypoints[i] = Keypoint{Vec2{kp[3 * i], kp[3 * i + 1]}, kp[3 * i + 2]};
    desc.resize(static_cast<std::size_t>(n) * FrameFeatures::kDescriptorDim);
    f.descriptors = std::move(desc);
    return f;
}
}  // namespace b200

/// detect_features (features.hpp:140-205) on an FP32 gray image.
inline FrameFeatures detect_features(const ImageF& gray, const DetectorConfig& cfg) {
    const auto c = b200::detector_config(cfg);
    const std::size_t cap = static_cast<std::size_t>(cfg.max_features > 0 ? cfg.max_features : 0);
    std::vector<double> kp(3 * cap + 3);
    std::vector<float> desc(FrameFeatures::kDescriptorDim * cap + FrameFeatures::kDescriptorDim);
    int n = 0;
    b200::check(nrm_detect_features_gray(b200::context(), gray.data.data(), gray.width, gray.height, &c, kp.data(),
                                         desc.data(), &n));
    return b200::unpack_features(kp, desc, n);
}

/// detect_features(to_gray(image), cfg) with to_gray on the GPU.
inline FrameFeatures detect_features(const ImageU8& image, const DetectorConfig& cfg) {
    const auto c = b200::detector_config(cfg);
    const std::size_t cap = static_cast<std::size_t>(cfg.max_features > 0 ? cfg.max_features : 0);
    std::vector<double> kp(3 * cap + 3);
    std::vector<float> desc(FrameFeatures::kDescriptorDim * cap + FrameFeatures::kDescriptorDim);
    int n = 0;
    b200::check(nrm_detect_features(b200::context(), image.data.data(), image.width, image.height,
                                    image.channels ? image.channels : 1, &c, kp.data(), desc.data(), &n));
    return b200::unpack_features(kp, desc, n);
}

/// match_features (features.hpp:208-254).
inline std::vector<MatchPair> match_features(const FrameFeatures& a, const FrameFeatures& b, double ratio,
                                             int /*workers*/ = 1) {
    std::vector<MatchPair> out;
    if (a.size() == 0 || b.size() < 2) return out;
    auto pack = [](const FrameFeatures& f) {
        std::vector<double> kp(3 * f.size());
        for (std::size_t i = 0; i < f.size(); ++i) {
            kp[3 * i] = f.keypoints[i].position.x;
            kp[3 * i + 1] = f.keypoints[i].position.y;
            kp[3 * i + 2] = f.keypoints[i].response;
        }
        return kp;
    };
    const auto ka = pack(a), kb = pack(b);
    std::vector<double> rows(5 * a.size());
    int n = 0;
    b200::check(nrm_match_features(b200::context(), ka.data(), a.descriptors.data(), static_cast<int>(a.size()),
                                   kb.data(), b.descriptors.data(), static_cast<int>(b.size()), ratio, rows.data(),
                                   &n));
    out.resize(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i)
        out[i] = MatchPair{Vec2{rows[5 * i], rows[5 * i + 1]}, Vec2{rows[5 * i + 2], rows[5 * i + 3]}, rows[5 * i + 4]};
    return out;
}

/// detect_and_match (features.hpp:258-265).
inline std::vector<MatchPair> detect_and_match(const ImageU8& image_a, const ImageU8& image_b,
                                               const DetectorConfig& cfg) {
    if (image_a.channels != image_b.channels)
        throw std::invalid_argument("detect_and_match: mismatched channel layouts");
    const FrameFeatures fa = detect_features(image_a, cfg);
    const FrameFeatures fb = detect_features(image_b, cfg);
    return match_features(fa, fb, cfg.ratio_test, cfg.workers);
}

/// Match files: the reference's text format (features.hpp:272-305) -- one
/// match per line "ax ay bx by score" at 17 significant digits (so doubles
/// round-trip), '#' comment lines, the same error text for malformed lines --
/// so files written by either implementation load in the other.
inline void save_matches(const std::string& path, const std::vector<MatchPair>& matches) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot write " + path);
    std::ostringstream text;
    text.precision(17);  // default float field at precision 17 == printf %.17g
    text << "# ax ay bx by score\n";
    for (const MatchPair& m : matches)
        text << m.point_a.x << ' ' << m.point_a.y << ' ' << m.point_b.x << ' ' << m.point_b.y << ' ' << m.score
             << '\n';
    out << text.str();
}

inline std::vector<MatchPair> load_matches(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path);
    std::vector<MatchPair> result;
    std::string row;
    int number = 0;
    while (std::getline(in, row)) {
        ++number;
        // tokens separated by blanks; a row of blanks or starting with '#' is skipped
        std::vector<double> vals;
        const char* c = row.c_str();
        bool bad = false;
        while (true) {
            while (*c == ' ' || *c == '\t' || *c == '\r') ++c;
            if (!*c) break;
            if (vals.empty() && *c == '#') break;
            char* end = nullptr;
            const double v = std::strtod(c, &end);
            if (end == c || (*end && *end != ' ' && *end != '\t' && *end != '\r')) {
                bad = true;
                break;
            }
            vals.push_back(v);
            c = end;
        }
        if (vals.empty() && !bad) continue;
        if (bad || vals.size() != 5)
            throw std::runtime_error(path + ":" + std::to_string(number) + ": expected 5 fields 'ax ay bx by score'");
        MatchPair m;
        m.point_a = Vec2{vals[0], vals[1]};
        m.point_b = Vec2{vals[2], vals[3]};
        m.score = vals[4];
        result.push_back(m);
    }
    return result;
}

}  // namespace nrmosaic
