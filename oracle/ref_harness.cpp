// ref_harness.cpp -- TEST INFRASTRUCTURE: a C-linkage shim over the REAL
// reference headers (/root/reference/proj/include, read in place, never
// copied). Built by oracle/Makefile into oracle/_ref/libnrm_ref.so with a
// declaration-only png.h stub (oracle/stub). Used to
//   * generate golden vectors (oracle/make_golden.py -> tests/golden/),
//   * pin the C restatement (oracle/nrm_oracle.c) bit-for-bit,
//   * time the reference CPU path for bench.py (cpu_baseline, --impl reference).
// Nothing in the product links it.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

// Engine::blended_variance_at (slam.hpp:703-714) is private; the checker
// ref_blended_variance_at calls it on a default Engine (test infrastructure
// only). The standard headers the reference uses come first, unaffected.
#include <algorithm>
#include <array>
#include <atomic>
#include <filesystem>
#include <fstream>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <numeric>
#include <optional>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <utility>
#define private public
#include "nrmosaic/config.hpp"
#include "nrmosaic/features.hpp"
#include "nrmosaic/fieldest.hpp"
#include "nrmosaic/mosaic.hpp"
#include "nrmosaic/slam.hpp"
#include "nrmosaic/synth.hpp"
#undef private
#include "oracles.hpp"

using namespace nrmosaic;

namespace {

std::vector<Vec2> to_vec2(const double* p, int n) {
    std::vector<Vec2> v(n > 0 ? n : 0);
    for (int i = 0; i < n; ++i) v[i] = {p[2 * i], p[2 * i + 1]};
    return v;
}

std::vector<WarpFunction> to_warps(const double* p, int n) {
    std::vector<WarpFunction> v(n > 0 ? n : 0);
    for (int i = 0; i < n; ++i) v[i] = {p[5 * i], {p[5 * i + 1], p[5 * i + 2], p[5 * i + 3], p[5 * i + 4]}};
    return v;
}

void put_warp(const WarpFunction& w, double* out5) {
    out5[0] = w.scale;
    out5[1] = w.dq.w;
    out5[2] = w.dq.z;
    out5[3] = w.dq.dx;
    out5[4] = w.dq.dy;
}

ImageU8 to_image(const std::uint8_t* data, int w, int h, int ch) {
    ImageU8 im;
    if (w <= 0 || h <= 0) return im;
    im = ImageU8::make(w, h, ch);
    std::memcpy(im.data.data(), data, static_cast<std::size_t>(w) * h * ch);
    return im;
}

}  // namespace

extern "C" {

int ref_pixel_warp(double x, double y, const double* anchors, const double* warps, int n,
                   double alpha, double* out5) {
    const auto a = to_vec2(anchors, n);
    const auto w = to_warps(warps, n);
    const auto r = pixel_warp({x, y}, a, w, alpha);
    if (!r) return 0;
    put_warp(*r, out5);
    return 1;
}

void* ref_canvas_new() { return new Canvas(); }
void ref_canvas_free(void* c) { delete static_cast<Canvas*>(c); }

void ref_canvas_ensure_contains(void* c, double x0, double y0, double x1, double y1) {
    static_cast<Canvas*>(c)->ensure_contains({x0, y0, x1, y1});
}

void ref_canvas_info(void* cv, std::int64_t* ox, std::int64_t* oy, int* w, int* h) {
    const Canvas& c = *static_cast<Canvas*>(cv);
    *ox = static_cast<std::int64_t>(c.origin_offset().x);
    *oy = static_cast<std::int64_t>(c.origin_offset().y);
    *w = c.width();
    *h = c.height();
}

// Copies out the full color (h*w*3 doubles) and weight (h*w) planes.
void ref_canvas_read(void* cv, double* color, std::uint8_t* weight) {
    const Canvas& c = *static_cast<Canvas*>(cv);
    for (int y = 0; y < c.height(); ++y)
        for (int x = 0; x < c.width(); ++x) {
            const double* px = c.color(x, y);
            const std::size_t o = static_cast<std::size_t>(y) * c.width() + x;
            if (color) {
                color[o * 3] = px[0];
                color[o * 3 + 1] = px[1];
                color[o * 3 + 2] = px[2];
            }
            if (weight) weight[o] = c.weight(x, y);
        }
}

int ref_blend_frame(void* cv, const std::uint8_t* frame, int fw, int fh, int ch,
                    const double* anchors, const double* warps, int n, double alpha,
                    const double* poly, int npoly, int workers, std::int64_t* stats) {
    const ImageU8 im = to_image(frame, fw, fh, ch);
    const auto a = to_vec2(anchors, n);
    const auto w = to_warps(warps, n);
    const auto p = to_vec2(poly, npoly);
    const BlendStats s = blend_frame(*static_cast<Canvas*>(cv), im, a, w, alpha, p, workers);
    stats[0] = s.footprint_pixels;
    stats[1] = s.blended_pixels;
    stats[2] = s.skipped_no_support;
    stats[3] = s.skipped_out_of_frame;
    return 0;
}

void ref_render(void* cv, int crop, std::uint8_t* out, int* out_w, int* out_h, double* origin2) {
    Vec2 org;
    const ImageU8 im = render(*static_cast<Canvas*>(cv), crop != 0, &org);
    *out_w = im.width;
    *out_h = im.height;
    if (origin2) {
        origin2[0] = org.x;
        origin2[1] = org.y;
    }
    if (out && !im.empty()) std::memcpy(out, im.data.data(), im.data.size());
}

int ref_invert_frame_boundary(int fw, int fh, const double* anchors, const double* warps, int n,
                              double alpha, double step, double* poly, int cap) {
    const auto a = to_vec2(anchors, n);
    const auto w = to_warps(warps, n);
    const auto p = invert_frame_boundary(fw, fh, a, w, alpha, step);
    for (int i = 0; i < static_cast<int>(p.size()) && i < cap; ++i) {
        poly[2 * i] = p[i].x;
        poly[2 * i + 1] = p[i].y;
    }
    return static_cast<int>(p.size());
}

int ref_blend_local(const double* locals, const double* apts, const double* probs,
                    const std::int32_t* active, int nactive, double qx, double qy, double alpha,
                    int support, int m_total, double* out5) {
    const auto l = to_warps(locals, m_total);
    const auto a = to_vec2(apts, m_total);
    const std::vector<double> p(probs, probs + m_total);
    const std::vector<int> act(active, active + nactive);
    put_warp(detail::blend_local(l, a, p, act, {qx, qy}, alpha, support), out5);
    return 0;
}

double ref_node_uncertainty(double qx, double qy, const double* pts, int m, double beta) {
    return node_uncertainty({qx, qy}, to_vec2(pts, m), beta);
}

// Dense EMDQ field + uncertainty over rows [row_begin, row_end) of a w x h
// grid at (x0 + i, y0 + j), with the reference's own row-parallel runner
// (parallel.hpp) -- the CPU baseline of SURVEY §8d.
void ref_emdq_field_grid(double x0, double y0, int w, int h, const double* apts,
                         const double* locals, const double* probs, const std::int32_t* active,
                         int nactive, int m_total, double alpha, int support, double beta,
                         int workers, int row_begin, int row_end, double* disp, double* unc) {
    const auto l = to_warps(locals, m_total);
    const auto a = to_vec2(apts, m_total);
    const std::vector<double> p(probs, probs + m_total);
    const std::vector<int> act(active, active + nactive);
    std::vector<Vec2> pts;
    for (int j : act) pts.push_back(a[j]);
    if (row_begin < 0) row_begin = 0;
    if (row_end < 0 || row_end > h) row_end = h;
    const std::size_t rows = static_cast<std::size_t>(row_end - row_begin);
    parallel_for(rows, workers, [&](std::size_t r0, std::size_t r1) {
        for (std::size_t r = r0; r < r1; ++r) {
            const int j = row_begin + static_cast<int>(r);
            for (int i = 0; i < w; ++i) {
                const Vec2 q{x0 + i, y0 + j};
                const WarpFunction f = detail::blend_local(l, a, p, act, q, alpha, support);
                const Vec2 y = f.apply(q);
                const std::size_t o = static_cast<std::size_t>(j) * w + i;
                if (disp) {
                    disp[2 * o] = y.x - q.x;
                    disp[2 * o + 1] = y.y - q.y;
                }
                if (unc) unc[o] = node_uncertainty(q, pts, beta);
            }
        }
    }, 1);
}

// Hex lattice covering a w x h rect (slam.hpp:270, as test_mosaic.cpp:24-31).
int ref_rect_lattice(double x0, double y0, double x1, double y1, double spacing, double alpha,
                     double* anchors, int cap) {
    NodeGraph g;
    g.hex_spacing = spacing;
    insert_nodes(g, CoverageRegion::from_rect({x0, y0, x1, y1}), alpha);
    const auto a = g.anchors();
    for (int i = 0; i < static_cast<int>(a.size()) && i < cap; ++i) {
        anchors[2 * i] = a[i].x;
        anchors[2 * i + 1] = a[i].y;
    }
    return static_cast<int>(a.size());
}

// Acceptance-style synthetic matches (acceptance.cpp:276-308 pattern),
// scaled by s: global similarity + 3 Gaussian bumps, inliers uniform over the
// frame, outliers uniform random pairs. out_a/out_b: (n_in+n_out) x 2.
void ref_synth_matches(int fw, int fh, double s, int n_in, int n_out, std::uint64_t seed,
                       double* out_a, double* out_b) {
    test::RandomGen gen(seed);
    const Similarity2 global{gen.uniform(0.95, 1.05), gen.uniform(-0.1, 0.1),
                             {gen.uniform(-10 * s, 10 * s), gen.uniform(-10 * s, 10 * s)}};
    struct Bump { Vec2 c, d; double rho; };
    std::vector<Bump> bumps;
    for (int b = 0; b < 3; ++b)
        bumps.push_back({{gen.uniform(0, fw), gen.uniform(0, fh)},
                         {gen.uniform(-12 * s, 12 * s), gen.uniform(-12 * s, 12 * s)},
                         gen.uniform(70 * s, 120 * s)});
    auto truth = [&](const Vec2& p) {
        Vec2 out = global.apply(p);
        for (const auto& b : bumps) out += std::exp(-dist2(p, b.c) / (2 * b.rho * b.rho)) * b.d;
        return out;
    };
    const double m = 5 * s;
    int k = 0;
    for (int i = 0; i < n_in; ++i, ++k) {
        const Vec2 a{gen.uniform(m, fw - m), gen.uniform(m, fh - m)};
        const Vec2 b = truth(a);
        out_a[2 * k] = a.x; out_a[2 * k + 1] = a.y;
        out_b[2 * k] = b.x; out_b[2 * k + 1] = b.y;
    }
    for (int i = 0; i < n_out; ++i, ++k) {
        out_a[2 * k] = gen.uniform(m, fw - m); out_a[2 * k + 1] = gen.uniform(m, fh - m);
        out_b[2 * k] = gen.uniform(m, fw - m); out_b[2 * k + 1] = gen.uniform(m, fh - m);
    }
}

// estimate_field (fieldest.hpp:112) followed by the exact locals
// reconstruction of SURVEY §8c. Outputs (all sized by n matches):
//   locals[n*5] (identity for non-inliers), probs[n], inlier[n];
//   node_inc[nn*5] = est.node_increments, node_unc[nn].
// Returns the inlier count, or -1 when estimation fails.
int ref_estimate_locals(const double* pa, const double* pb, int n, const double* node_anchors,
                        int nn, double alpha, double beta, double inlier_threshold, int knn,
                        int seed_trials, std::uint64_t seed, int workers, double* locals,
                        double* probs, std::uint8_t* inlier, double* node_inc, double* node_unc) {
    std::vector<MatchPair> m(n);
    for (int i = 0; i < n; ++i) m[i] = {{pa[2 * i], pa[2 * i + 1]}, {pb[2 * i], pb[2 * i + 1]}, 1.0};
    const auto anchors = to_vec2(node_anchors, nn);
    FieldParams fp;
    fp.alpha = alpha;
    fp.beta = beta;
    fp.inlier_threshold = inlier_threshold;
    fp.knn = knn;
    fp.seed_trials = seed_trials;
    fp.seed = seed;
    fp.workers = workers;
    const auto est = estimate_field(m, anchors, fp);
    if (!est) return -1;
    std::vector<Vec2> apts(n), bpts(n);
    for (int i = 0; i < n; ++i) {
        apts[i] = m[i].point_a;
        bpts[i] = m[i].point_b;
    }
    std::vector<int> inl;
    for (int j = 0; j < n; ++j) {
        inlier[j] = est->inlier_flags[j];
        if (est->inlier_flags[j]) inl.push_back(j);
    }
    const double tau = inlier_threshold;
    const double sigma_em2 = 0.25 * tau * tau;
    std::vector<int> nbrs;
    for (int j = 0; j < n; ++j) {
        probs[j] = std::exp(-est->match_residuals[j] / (2.0 * sigma_em2));
        WarpFunction loc = WarpFunction::identity();
        if (est->inlier_flags[j]) {
            detail::knn_indices(apts, inl, j, apts[j], knn, nbrs);
            std::vector<Vec2> src{apts[j]}, dst{bpts[j]};
            for (int q : nbrs) { src.push_back(apts[q]); dst.push_back(bpts[q]); }
            const auto sim = fit_similarity(src, dst);
            if (sim && sim->scale > 0.05 && sim->scale < 20.0)
                loc = WarpFunction::from_similarity(*sim);
            else
                loc = {1.0, DualQuat2::from_translation(bpts[j] - apts[j])};
        }
        put_warp(loc, &locals[5 * j]);
    }
    for (int i = 0; i < nn; ++i) {
        put_warp(est->node_increments[i], &node_inc[5 * i]);
        node_unc[i] = est->node_uncertainties[i];
    }
    return est->inlier_count;
}

// The EM E-step's leave-one-out prediction (fieldest.hpp:195-209) for every
// match j over the candidate set `active`, using the reference's own
// detail::blend_local and WarpFunction::apply: warps[n*5] (zeros when no
// other candidate remains), pred[n*2] (bpts[j] in that case, as the
// reference does), empty[n] = 1 for that case.
void ref_estep_loo(const double* apts, const double* bpts, const double* locals, const double* probs,
                   int n, const std::int32_t* active, int nactive, double alpha, int support, int workers,
                   int j_begin, int j_end, double* warps, double* pred, std::uint8_t* empty) {
    const auto l = to_warps(locals, n);
    const auto a = to_vec2(apts, n);
    const std::vector<double> p(probs, probs + n);
    if (j_begin < 0) j_begin = 0;
    if (j_end < 0 || j_end > n) j_end = n;
    // the reference's own runner and grain for this loop (fieldest.hpp:197)
    parallel_for(static_cast<std::size_t>(j_end - j_begin), workers, [&](std::size_t i0, std::size_t i1) {
        std::vector<int> others;
        for (std::size_t ii = i0; ii < i1; ++ii) {
            const int j = j_begin + static_cast<int>(ii);
            others.clear();
            for (int k = 0; k < nactive; ++k)
                if (active[k] != j) others.push_back(active[k]);
            empty[j] = others.empty() ? 1 : 0;
            if (others.empty()) {
                for (int c = 0; c < 5; ++c) warps[5 * j + c] = 0.0;
                pred[2 * j] = bpts[2 * j];
                pred[2 * j + 1] = bpts[2 * j + 1];
                continue;
            }
            const WarpFunction f = detail::blend_local(l, a, p, others, a[j], alpha, support);
            put_warp(f, &warps[5 * j]);
            const Vec2 y = f.apply(a[j]);
            pred[2 * j] = y.x;
            pred[2 * j + 1] = y.y;
        }
    }, 16);
}

// warp_update (dualquat.hpp:181-190)
void ref_warp_update(const double* old5, const double* delta5, double* out5) {
    const auto o = to_warps(old5, 1);
    const auto d = to_warps(delta5, 1);
    put_warp(warp_update(o[0], d[0]), out5);
}

// SyntheticScene::render_frame (synth.hpp:204-220): RGB8 frame t.
int ref_scene_render(int width, int height, int frames, std::uint64_t seed, int num_bumps,
                     double max_disp, double bump_radius, double path_extent, int t, int workers,
                     std::uint8_t* out) {
    SceneSpec spec;
    spec.width = width;
    spec.height = height;
    spec.frames = frames;
    spec.seed = seed;
    spec.num_bumps = num_bumps;
    spec.max_displacement = max_disp;
    spec.bump_radius = bump_radius;
    spec.path_extent = path_extent;
    const auto scene = SyntheticScene::build(spec);
    const ImageU8 f = scene.render_frame(t, workers);
    std::memcpy(out, f.data.data(), f.data.size());
    return 0;
}

// Wall-clock of one blend_frame on a fresh canvas pre-sized to `pre` (x0,y0,x1,y1).
double ref_time_blend_frame(const std::uint8_t* frame, int fw, int fh, int ch,
                            const double* anchors, const double* warps, int n, double alpha,
                            const double* poly, int npoly, const double* pre, int workers,
                            std::int64_t* stats) {
    Canvas c;
    c.ensure_contains({pre[0], pre[1], pre[2], pre[3]});
    const ImageU8 im = to_image(frame, fw, fh, ch);
    const auto a = to_vec2(anchors, n);
    const auto w = to_warps(warps, n);
    const auto p = to_vec2(poly, npoly);
    const auto t0 = std::chrono::steady_clock::now();
    const BlendStats s = blend_frame(c, im, a, w, alpha, p, workers);
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (stats) {
        stats[0] = s.footprint_pixels;
        stats[1] = s.blended_pixels;
        stats[2] = s.skipped_no_support;
        stats[3] = s.skipped_out_of_frame;
    }
    return dt;
}

// ---- sparse front end (features.hpp) ----------------

// The fixture image of the reference's detector tests (test_features.cpp:14-32):
// uniform random bytes from std::mt19937_64(seed), then two 3 x 3 box means
// over the interior with integer division. Gray, 1 channel.
void ref_textured_image(int w, int h, std::uint64_t seed, std::uint8_t* out) {
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<int> dist(0, 255);
    std::vector<std::uint8_t> a(static_cast<std::size_t>(w) * h);
    for (auto& p : a) p = static_cast<std::uint8_t>(dist(rng));
    for (int pass = 0; pass < 2; ++pass) {
        std::vector<std::uint8_t> b = a;
        for (int y = 1; y + 1 < h; ++y)
            for (int x = 1; x + 1 < w; ++x) {
                int s = 0;
                for (int v = -1; v <= 1; ++v)
                    for (int u = -1; u <= 1; ++u) s += a[static_cast<std::size_t>(y + v) * w + (x + u)];
                b[static_cast<std::size_t>(y) * w + x] = static_cast<std::uint8_t>(s / 9);
            }
        a.swap(b);
    }
    std::memcpy(out, a.data(), a.size());
}

// to_gray (image.hpp:63-75)
void ref_to_gray(const std::uint8_t* im, int w, int h, int ch, float* out) {
    const ImageF g = to_gray(to_image(im, w, h, ch));
    if (!g.data.empty()) std::memcpy(out, g.data.data(), g.data.size() * sizeof(float));
}

static int put_features(const FrameFeatures& f, double* kp, float* desc, int cap) {
    const int n = static_cast<int>(f.size());
    for (int i = 0; i < n && i < cap; ++i) {
        kp[3 * i] = f.keypoints[i].position.x;
        kp[3 * i + 1] = f.keypoints[i].position.y;
        kp[3 * i + 2] = f.keypoints[i].response;
        std::memcpy(desc + 64 * static_cast<std::size_t>(i), f.descriptor(i), 64 * sizeof(float));
    }
    return n;
}

static FrameFeatures to_features(const double* kp, const float* desc, int n) {
    FrameFeatures f;
    f.keypoints.resize(n);
    for (int i = 0; i < n; ++i) f.keypoints[i] = {{kp[3 * i], kp[3 * i + 1]}, kp[3 * i + 2]};
    f.descriptors.assign(desc, desc + 64 * static_cast<std::size_t>(n));
    return f;
}

// detect_features (features.hpp:140-205) on an FP32 gray image.
int ref_detect_features(const float* gray, int w, int h, int max_features, double quality, int nms_radius,
                        int workers, double* kp, float* desc, int cap) {
    ImageF g = ImageF::make(w, h);
    std::memcpy(g.data.data(), gray, g.data.size() * sizeof(float));
    DetectorConfig cfg;
    cfg.max_features = max_features;
    cfg.quality_level = quality;
    cfg.nms_radius = nms_radius;
    cfg.workers = workers;
    return put_features(detect_features(g, cfg), kp, desc, cap);
}

// match_features (features.hpp:208-254): rows (ax, ay, bx, by, score).
int ref_match_features(const double* kp_a, const float* desc_a, int na, const double* kp_b, const float* desc_b,
                       int nb, double ratio, int workers, double* out, int cap) {
    const auto m = match_features(to_features(kp_a, desc_a, na), to_features(kp_b, desc_b, nb), ratio, workers);
    const int n = static_cast<int>(m.size());
    for (int i = 0; i < n && i < cap; ++i) {
        out[5 * i] = m[i].point_a.x;
        out[5 * i + 1] = m[i].point_a.y;
        out[5 * i + 2] = m[i].point_b.x;
        out[5 * i + 3] = m[i].point_b.y;
        out[5 * i + 4] = m[i].score;
    }
    return n;
}

// Wall-clock of the reference's front end for one frame pair as its callers
// run it (main.cpp:198-202): to_gray + detect_features on frame b, then
// match_features against a's features, with `workers` threads.
double ref_time_detect_match(const std::uint8_t* img_b, int w, int h, int ch, const double* kp_a,
                             const float* desc_a, int na, int max_features, double quality, int nms_radius,
                             double ratio, int workers, int* counts2) {
    const ImageU8 im = to_image(img_b, w, h, ch);
    const FrameFeatures fa = to_features(kp_a, desc_a, na);
    DetectorConfig cfg;
    cfg.max_features = max_features;
    cfg.quality_level = quality;
    cfg.nms_radius = nms_radius;
    cfg.workers = workers;
    const auto t0 = std::chrono::steady_clock::now();
    const FrameFeatures fb = detect_features(to_gray(im), cfg);
    const auto m = match_features(fa, fb, ratio, workers);
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (counts2) {
        counts2[0] = static_cast<int>(fb.size());
        counts2[1] = static_cast<int>(m.size());
    }
    return dt;
}

/* Engine::blended_variance_at (slam.hpp:703-714) at npts points. */
void ref_blended_variance_at(const double* pts, int npts, const double* pos, const double* var, int n, double alpha,
                             double* out) {
    Engine::Params prm;
    prm.alpha = alpha;
    Engine eng(prm);
    std::vector<Vec2> p(n);
    for (int i = 0; i < n; ++i) p[i] = Vec2{pos[2 * i], pos[2 * i + 1]};
    const std::span<const Vec2> ps(p);
    const std::span<const double> vs(var, (size_t)n);
    for (int k = 0; k < npts; ++k) out[k] = eng.blended_variance_at(Vec2{pts[2 * k], pts[2 * k + 1]}, ps, vs);
}

}  // extern "C"
