// nrmosaic_b200/mosaic.hpp -- drop-in replacement for the reference's
// nrmosaic/mosaic.hpp (proj/include/nrmosaic/mosaic.hpp) backed by the
// B200 C ABI (include/nrm_b200.h, libnrm_b200.so).
//
// Existing callers (tools/main.cpp:174-176, 229-230, 268; the acceptance
// harness acceptance.cpp:371-387) switch by replacing
//     #include "nrmosaic/mosaic.hpp"
// with
//     #include "nrmosaic_b200/mosaic.hpp"
// and linking -lnrm_b200. Same names, signatures, exceptions and
// std::optional returns:
//   pixel_warp            (mosaic.hpp:22)   -> std::optional<WarpFunction>
//   invert_frame_boundary (mosaic.hpp:58)   -> std::vector<Vec2>
//   Canvas                (mosaic.hpp:100)  kWeightCap, kTile, empty, width, height,
//                                           origin_offset, color, weight, weight_ref,
//                                           occupied, occupied_count, ensure_contains
//   BlendStats            (mosaic.hpp:184)
//   blend_frame           (mosaic.hpp:196)
//   render                (mosaic.hpp:301)
// plus the dense EMDQ field (detail::blend_local + node_uncertainty at every
// pixel of a grid, fieldest.hpp:44-97) as dense_emdq_field(), and
// blend_local at scattered points for the EM loop of estimate_field (the
// E-step's leave-one-out, fieldest.hpp:195-209, and the final field,
// fieldest.hpp:263-270) as blend_local_points().
//
// Canvas pixels live in HBM. Canvas::color()/weight() read through a host
// mirror kept per 256 x 256 tile and downloaded lazily after GPU updates;
// writes through color()/weight_ref() mark their tile dirty and are uploaded
// before the next GPU operation on that canvas (the explicit sync SURVEY §7
// calls for).
//
// Production callers that include both nrmosaic/mosaic.hpp and
// nrmosaic/slam.hpp (which includes nrmosaic/mosaic.hpp itself, slam.hpp:16)
// switch with an include path instead of an edit: -Iinclude/override ahead
// of the reference's include directory makes every "nrmosaic/mosaic.hpp"
// resolve to include/override/nrmosaic/mosaic.hpp, which forwards here.
//
// Types: by default Vec2, Rect, DualQuat2, WarpFunction and ImageU8 come
// from the reference headers (nrmosaic/geometry.hpp, dualquat.hpp,
// image.hpp) so the rest of a caller's code is untouched. Define
// NRM_B200_STANDALONE_TYPES to use minimal layout-compatible stand-ins
// instead (for builds without the reference tree).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>
#include <algorithm>

#include "nrm_b200.h"

#ifndef NRM_B200_STANDALONE_TYPES
#include "nrmosaic/dualquat.hpp"
#include "nrmosaic/geometry.hpp"
#include "nrmosaic/image.hpp"
#else
namespace nrmosaic {
struct Vec2 {
    double x = 0.0, y = 0.0;
    Vec2() = default;
    constexpr Vec2(double x_, double y_) : x(x_), y(y_) {}
    Vec2 operator+(const Vec2& o) const { return {x + o.x, y + o.y}; }
    Vec2 operator-(const Vec2& o) const { return {x - o.x, y - o.y}; }
};
struct Rect {
    double x0 = 0.0, y0 = 0.0, x1 = 0.0, y1 = 0.0;
    static Rect of_size(double w, double h) { return {0.0, 0.0, w, h}; }
};
struct DualQuat2 {
    double w = 1.0, z = 0.0, dx = 0.0, dy = 0.0;
    static DualQuat2 from_translation(const Vec2& t) { return {1.0, 0.0, 0.5 * t.x, 0.5 * t.y}; }
    static DualQuat2 from_rigid(double angle, const Vec2& t) {
        DualQuat2 q;
        q.w = std::cos(0.5 * angle);
        q.z = std::sin(0.5 * angle);
        q.dx = 0.5 * (t.x * q.w + t.y * q.z);
        q.dy = 0.5 * (-t.x * q.z + t.y * q.w);
        return q;
    }
    Vec2 apply(const Vec2& p) const {
        const double c = w * w - z * z, s = 2.0 * w * z;
        return {c * p.x - s * p.y + 2.0 * (dx * w - dy * z), s * p.x + c * p.y + 2.0 * (dx * z + dy * w)};
    }
};
struct WarpFunction {
    double scale = 1.0;
    DualQuat2 dq;
    static WarpFunction identity() { return {}; }
    Vec2 apply(const Vec2& p) const {
        const Vec2 q = dq.apply(p);
        return {q.x * scale, q.y * scale};
    }
};
struct ImageU8 {
    int width = 0, height = 0, channels = 0;
    std::vector<std::uint8_t> data;
    static ImageU8 make(int w, int h, int c, std::uint8_t fill = 0) {
        ImageU8 im;
        im.width = w;
        im.height = h;
        im.channels = c;
        im.data.assign(static_cast<std::size_t>(w) * h * c, fill);
        return im;
    }
    bool empty() const { return width == 0 || height == 0; }
    std::uint8_t& at(int x, int y, int c) { return data[(static_cast<std::size_t>(y) * width + x) * channels + c]; }
    std::uint8_t at(int x, int y, int c) const {
        return data[(static_cast<std::size_t>(y) * width + x) * channels + c];
    }
};
}  // namespace nrmosaic
#endif

namespace nrmosaic {

constexpr double kPixelWeightCutoff = 1e-6;  // mosaic.hpp:16

namespace b200 {

// Maps C ABI status codes onto the reference's exception types.
inline void check(int rc) {
    if (rc == NRM_OK) return;
    const std::string msg = nrm_last_error();
    if (rc == NRM_EINVAL || rc == NRM_EDEGENERATE) throw std::invalid_argument(msg);
    throw std::runtime_error("nrm_b200: " + msg);
}

// One context per process (device from NRM_B200_DEVICE, default 0).
inline nrm_ctx* context() {
    struct Holder {
        nrm_ctx* c = nullptr;
        Holder() {
            const char* d = std::getenv("NRM_B200_DEVICE");
            check(nrm_ctx_create(d ? std::atoi(d) : 0, &c));
        }
        ~Holder() { nrm_ctx_destroy(c); }
    };
    static Holder h;
    return h.c;
}

inline std::vector<double> pack_points(std::span<const Vec2> pts) {
    std::vector<double> v(pts.size() * 2);
    for (std::size_t i = 0; i < pts.size(); ++i) {
        v[2 * i] = pts[i].x;
        v[2 * i + 1] = pts[i].y;
    }
    return v;
}

inline std::vector<double> pack_warps(std::span<const WarpFunction> w) {
    std::vector<double> v(w.size() * 5);
    for (std::size_t i = 0; i < w.size(); ++i) {
        v[5 * i] = w[i].scale;
        v[5 * i + 1] = w[i].dq.w;
        v[5 * i + 2] = w[i].dq.z;
        v[5 * i + 3] = w[i].dq.dx;
        v[5 * i + 4] = w[i].dq.dy;
    }
    return v;
}

inline WarpFunction unpack_warp(const double* p) {
    WarpFunction w;
    w.scale = p[0];
    w.dq.w = p[1];
    w.dq.z = p[2];
    w.dq.dx = p[3];
    w.dq.dy = p[4];
    return w;
}

}  // namespace b200

/// pixel_warp (mosaic.hpp:22-51), evaluated on the GPU in the exact tier.
inline std::optional<WarpFunction> pixel_warp(const Vec2& x_ref, std::span<const Vec2> anchors,
                                              std::span<const WarpFunction> warps, double alpha) {
    if (anchors.size() != warps.size()) throw std::invalid_argument("pixel_warp: size mismatch");
    const double p[2] = {x_ref.x, x_ref.y};
    const auto a = b200::pack_points(anchors);
    const auto w = b200::pack_warps(warps);
    double out[5];
    std::uint8_t valid = 0;
    b200::check(nrm_pixel_warp(b200::context(), p, 1, a.data(), w.data(), static_cast<int>(anchors.size()), alpha,
                               out, &valid));
    if (!valid) return std::nullopt;
    return b200::unpack_warp(out);
}

/// invert_frame_boundary (mosaic.hpp:58-96), one GPU thread per boundary sample.
inline std::vector<Vec2> invert_frame_boundary(int frame_w, int frame_h, std::span<const Vec2> anchors,
                                               std::span<const WarpFunction> warps, double alpha,
                                               double step = 8.0) {
    const auto a = b200::pack_points(anchors);
    const auto w = b200::pack_warps(warps);
    int n = 0;
    b200::check(nrm_invert_frame_boundary(b200::context(), frame_w, frame_h, a.data(), w.data(),
                                          static_cast<int>(anchors.size()), alpha, step, nullptr, 0, &n));
    std::vector<double> poly(static_cast<std::size_t>(n) * 2);
    b200::check(nrm_invert_frame_boundary(b200::context(), frame_w, frame_h, a.data(), w.data(),
                                          static_cast<int>(anchors.size()), alpha, step, poly.data(), n, &n));
    std::vector<Vec2> out(n);
    for (int i = 0; i < n; ++i) out[i] = Vec2{poly[2 * i], poly[2 * i + 1]};
    return out;
}

/// Canvas (mosaic.hpp:100-182), HBM-resident.
///
/// color()/weight()/weight_ref() go through a host mirror kept per 256 x 256
/// canvas tile (Canvas::kTile): the first access to a tile after a GPU update
/// downloads that tile only (1.6 MB), writes mark it dirty, and dirty tiles
/// are uploaded before the next GPU operation on the canvas. Returned
/// pointers stay valid until the next GPU operation or ensure_contains, like
/// the reference's until its next reallocation.
class Canvas {
public:
    static constexpr int kWeightCap = 30;
    static constexpr int kTile = 256;

    Canvas() { b200::check(nrm_canvas_create(b200::context(), &h_)); }
    ~Canvas() {
        if (h_) nrm_canvas_destroy(h_);
    }
    Canvas(const Canvas&) = delete;
    Canvas& operator=(const Canvas&) = delete;
    Canvas(Canvas&& o) noexcept { *this = std::move(o); }
    Canvas& operator=(Canvas&& o) noexcept {
        std::swap(h_, o.h_);
        std::swap(tiles_, o.tiles_);
        return *this;
    }

    bool empty() const { return width() == 0; }
    int width() const { return info().w; }
    int height() const { return info().h; }
    /// Reference-frame coordinate of canvas pixel (0, 0).
    Vec2 origin_offset() const {
        const Info i = info();
        return {static_cast<double>(i.ox), static_cast<double>(i.oy)};
    }

    double* color(int x, int y) {
        Tile& t = tile(x, y);
        t.dirty = true;
        return &t.color[t.offset(x, y) * 3];
    }
    const double* color(int x, int y) const {
        const Tile& t = tile(x, y);
        return &t.color[t.offset(x, y) * 3];
    }
    std::uint8_t weight(int x, int y) const {
        const Tile& t = tile(x, y);
        return t.weight[t.offset(x, y)];
    }
    std::uint8_t& weight_ref(int x, int y) {
        Tile& t = tile(x, y);
        t.dirty = true;
        return t.weight[t.offset(x, y)];
    }
    bool occupied(int x, int y) const { return weight(x, y) > 0; }
    std::int64_t occupied_count() const {
        push();
        std::int64_t n = 0;
        b200::check(nrm_canvas_occupied_count(h_, &n));
        return n;
    }
    /// Grows the canvas (tile-aligned) so the reference-frame rectangle fits.
    void ensure_contains(const Rect& r) {
        push();
        b200::check(nrm_canvas_ensure_contains(h_, r.x0, r.y0, r.x1, r.y1));
        tiles_.clear();  // canvas coordinates may have shifted
    }

    /// B200 extensions: pre-allocate HBM for a region; band for multi-GPU.
    void reserve(const Rect& r) { b200::check(nrm_canvas_reserve(h_, r.x0, r.y0, r.x1, r.y1)); }
    void set_band(int rank, int count) { b200::check(nrm_canvas_set_band(h_, rank, count)); }
    /// The C handle, after uploading host edits (call before any GPU operation).
    nrm_canvas* handle() const {
        push();
        return h_;
    }
    /// Drops the host mirror (after a GPU update of the canvas).
    void invalidate_mirror() { tiles_.clear(); }

private:
    struct Info {
        std::int64_t ox, oy;
        int w, h;
    };
    struct Tile {
        int x0 = 0, y0 = 0, w = 0, h = 0;
        bool dirty = false;
        std::vector<double> color;
        std::vector<std::uint8_t> weight;
        std::size_t offset(int x, int y) const {
            return static_cast<std::size_t>(y - y0) * static_cast<std::size_t>(w) + static_cast<std::size_t>(x - x0);
        }
    };
    Info info() const {
        Info i{};
        b200::check(nrm_canvas_info(h_, &i.ox, &i.oy, &i.w, &i.h));
        return i;
    }
    Tile& tile(int x, int y) const {
        const Info i = info();
        if (x < 0 || y < 0 || x >= i.w || y >= i.h) throw std::out_of_range("Canvas: pixel outside the canvas");
        const std::int64_t tx = x / kTile, ty = y / kTile;
        const std::int64_t key = ty * ((i.w + kTile - 1) / kTile) + tx;
        auto it = tiles_.find(key);
        if (it != tiles_.end()) return it->second;
        Tile t;
        t.x0 = static_cast<int>(tx * kTile);
        t.y0 = static_cast<int>(ty * kTile);
        t.w = std::min(kTile, i.w - t.x0);
        t.h = std::min(kTile, i.h - t.y0);
        t.color.assign(static_cast<std::size_t>(t.w) * t.h * 3, 0.0);
        t.weight.assign(static_cast<std::size_t>(t.w) * t.h, 0);
        b200::check(nrm_canvas_download(h_, t.x0, t.y0, t.w, t.h, t.color.data(), t.weight.data()));
        return tiles_.emplace(key, std::move(t)).first->second;
    }
    void push() const {
        for (auto& [key, t] : tiles_) {
            (void)key;
            if (!t.dirty) continue;
            b200::check(nrm_canvas_upload(h_, t.x0, t.y0, t.w, t.h, t.color.data(), t.weight.data()));
            t.dirty = false;
        }
    }

    nrm_canvas* h_ = nullptr;
    mutable std::unordered_map<std::int64_t, Tile> tiles_;
};

struct BlendStats {
    std::int64_t footprint_pixels = 0;
    std::int64_t blended_pixels = 0;
    std::int64_t skipped_no_support = 0;
    std::int64_t skipped_out_of_frame = 0;
};

/// blend_frame (mosaic.hpp:196-296). `workers` is accepted for signature
/// compatibility; the GPU grid replaces the host thread pool.
inline BlendStats blend_frame(Canvas& canvas, const ImageU8& frame, std::span<const Vec2> anchors,
                              std::span<const WarpFunction> warps, double alpha,
                              std::span<const Vec2> footprint_polygon, int workers) {
    (void)workers;
    if (anchors.size() != warps.size()) throw std::invalid_argument("blend_frame: size mismatch");
    const auto a = b200::pack_points(anchors);
    const auto w = b200::pack_warps(warps);
    const auto p = b200::pack_points(footprint_polygon);
    nrm_blend_stats s{};
    b200::check(nrm_blend_frame(canvas.handle(), frame.data.data(), frame.width, frame.height,
                                frame.channels ? frame.channels : 3, a.data(), w.data(),
                                static_cast<int>(anchors.size()), alpha, p.data(),
                                static_cast<int>(footprint_polygon.size()), &s));
    canvas.invalidate_mirror();
    return {s.footprint_pixels, s.blended_pixels, s.skipped_no_support, s.skipped_out_of_frame};
}

/// Extension (north_star "uncertainty-weighted blending", no reference
/// counterpart): blend_frame whose update step is scaled by the confidence
/// 1 / max(u, 1) of a frame-aligned uncertainty map (e.g. dense_emdq_field's
/// `unc`); u == 1 everywhere is blend_frame bit for bit. See nrm_b200.h.
inline BlendStats blend_frame_weighted(Canvas& canvas, const ImageU8& frame, std::span<const Vec2> anchors,
                                       std::span<const WarpFunction> warps, double alpha,
                                       std::span<const Vec2> footprint_polygon, std::span<const float> unc) {
    if (anchors.size() != warps.size()) throw std::invalid_argument("blend_frame: size mismatch");
    if (unc.size() != static_cast<std::size_t>(frame.width) * static_cast<std::size_t>(frame.height))
        throw std::invalid_argument("blend_frame_weighted: uncertainty map must match the frame");
    const auto a = b200::pack_points(anchors);
    const auto w = b200::pack_warps(warps);
    const auto p = b200::pack_points(footprint_polygon);
    nrm_blend_stats s{};
    b200::check(nrm_blend_frame_weighted(canvas.handle(), frame.data.data(), frame.width, frame.height,
                                         frame.channels ? frame.channels : 3, a.data(), w.data(),
                                         static_cast<int>(anchors.size()), alpha, p.data(),
                                         static_cast<int>(footprint_polygon.size()), unc.data(), &s));
    canvas.invalidate_mirror();
    return {s.footprint_pixels, s.blended_pixels, s.skipped_no_support, s.skipped_out_of_frame};
}

/// Extension (north_star "deforming the existing canvas", no reference
/// counterpart): new(p) = old(p + d(p)) over the canvas rectangle
/// [x, x+w) x [y, y+h); disp holds h*w (dx, dy) pairs in canvas pixels.
/// d == 0 is a bit-exact no-op. See nrm_canvas_deform.
inline void deform_canvas(Canvas& canvas, int x, int y, int w, int h, std::span<const float> disp) {
    if (disp.size() != static_cast<std::size_t>(w) * static_cast<std::size_t>(h) * 2)
        throw std::invalid_argument("deform_canvas: displacement field must hold w * h * 2 floats");
    b200::check(nrm_canvas_deform(canvas.handle(), x, y, w, h, disp.data()));  // handle() pushes host edits
    canvas.invalidate_mirror();
}

/// save_png (image.hpp:160-192) with the parallel band encoder of
/// nrm_save_png: ImageU8 with 1 / 3 / 4 channels -> 8-bit PNG. For the
/// render() of a canvas-wide mosaic (up to 4 GiB of RGBA) the bands are
/// deflated on all host cores. Throws std::runtime_error on I/O failure.
inline void save_png_parallel(const std::string& path, const ImageU8& im, int threads = 0, int level = 6) {
    const int rc = nrm_save_png(path.c_str(), im.data.data(), im.width, im.height, im.channels, level, threads);
    if (rc == NRM_EINVAL && im.channels != 1 && im.channels != 3 && im.channels != 4)
        throw std::runtime_error("unsupported channel count");
    if (rc != NRM_OK) throw std::runtime_error(std::string("nrm_b200: ") + nrm_last_error());
}

/// Engine::blended_variance_at (slam.hpp:703-714) at every pixel (x0 + i, y0 + j)
/// of a w x h grid: the node-variance map (node current positions and
/// variances), a per-pixel uncertainty source for blend_frame_weighted
/// (e.g. unc = 1 + v / v0). out receives w * h floats.
inline void blended_variance_field(double x0, double y0, int w, int h, std::span<const Vec2> positions,
                                   std::span<const double> variances, double alpha, float* out) {
    if (positions.size() != variances.size()) throw std::invalid_argument("blended_variance_field: size mismatch");
    const auto p = b200::pack_points(positions);
    const nrm_grid g{x0, y0, w, h};
    b200::check(nrm_variance_field(b200::context(), &g, p.data(), variances.data(),
                                   static_cast<int>(positions.size()), alpha, out));
}

/// render (mosaic.hpp:301-331).
inline ImageU8 render(const Canvas& canvas, bool crop = false, Vec2* crop_origin = nullptr) {
    int w = 0, h = 0;
    double org[2] = {0.0, 0.0};
    b200::check(nrm_render(canvas.handle(), crop ? 1 : 0, nullptr, &w, &h, org));
    if (crop_origin) *crop_origin = Vec2{org[0], org[1]};
    if (w == 0 || h == 0) return ImageU8{};
    ImageU8 out = ImageU8::make(w, h, 4);
    b200::check(nrm_render(canvas.handle(), crop ? 1 : 0, out.data.data(), &w, &h, org));
    return out;
}

/// Dense EMDQ field: detail::blend_local (fieldest.hpp:75-97) applied at every
/// pixel (x0 + i, y0 + j) of a w x h grid plus node_uncertainty
/// (fieldest.hpp:44-52). disp receives w*h*2 floats (warp(p) - p), unc w*h.
inline void dense_emdq_field(double x0, double y0, int w, int h, std::span<const Vec2> apts,
                             std::span<const WarpFunction> locals, std::span<const double> probs,
                             std::span<const int> active, double alpha, int support, double beta, float* disp,
                             float* unc) {
    if (apts.size() != locals.size() || apts.size() != probs.size())
        throw std::invalid_argument("dense_emdq_field: size mismatch");
    const auto a = b200::pack_points(apts);
    const auto l = b200::pack_warps(locals);
    std::vector<std::int32_t> act(active.begin(), active.end());
    const nrm_grid g{x0, y0, w, h};
    b200::check(nrm_emdq_field(b200::context(), &g, a.data(), l.data(), probs.data(), static_cast<int>(apts.size()),
                               act.data(), static_cast<int>(act.size()), alpha, support, beta, disp, unc));
}

/// detail::blend_local (fieldest.hpp:75-97) at every query point, bit-identical
/// to the reference (GPU exact tier). exclude[k] (empty span: none) is a match
/// index left out of query k's candidates: the E-step passes the match points
/// and exclude[j] = j, i.e. `others` = active minus j (fieldest.hpp:197-206).
/// Returns nullopt where no candidate remains (the E-step then uses bpts[j]);
/// throws std::invalid_argument where dq_blend would (dualquat.hpp:137-146).
/// Optional outputs: pred[k] = warp.apply(q[k]); unc[k] = node_uncertainty
/// over the same candidates (fieldest.hpp:44-52, needs beta > 0).
inline std::vector<std::optional<WarpFunction>> blend_local_points(
    std::span<const Vec2> queries, std::span<const int> exclude, std::span<const WarpFunction> locals,
    std::span<const Vec2> apts, std::span<const double> probs, std::span<const int> active, double alpha,
    int support, std::vector<Vec2>* pred = nullptr, std::vector<double>* unc = nullptr, double beta = 1.0) {
    if (apts.size() != locals.size() || apts.size() != probs.size())
        throw std::invalid_argument("blend_local_points: size mismatch");
    if (!exclude.empty() && exclude.size() != queries.size())
        throw std::invalid_argument("blend_local_points: exclude must be empty or one per query");
    const std::size_t n = queries.size();
    std::vector<std::optional<WarpFunction>> out(n);
    if (n == 0) return out;
    const auto q = b200::pack_points(queries);
    const auto a = b200::pack_points(apts);
    const auto l = b200::pack_warps(locals);
    std::vector<std::int32_t> act(active.begin(), active.end());
    std::vector<std::int32_t> ex(exclude.begin(), exclude.end());
    std::vector<double> w(5 * n), pr(pred ? 2 * n : 0), un(unc ? n : 0);
    std::vector<std::int32_t> st(n);
    b200::check(nrm_emdq_points(b200::context(), q.data(), ex.empty() ? nullptr : ex.data(), static_cast<int>(n),
                                a.data(), l.data(), probs.data(), static_cast<int>(apts.size()), act.data(),
                                static_cast<int>(act.size()), alpha, support, beta, w.data(),
                                pred ? pr.data() : nullptr, unc ? un.data() : nullptr, st.data()));
    if (pred) pred->assign(n, Vec2{});
    for (std::size_t k = 0; k < n; ++k) {
        if (st[k] == 2) throw std::invalid_argument("dq_blend: all weights are zero or degenerate blend");
        if (st[k] == 0) out[k] = b200::unpack_warp(&w[5 * k]);
        if (pred) (*pred)[k] = Vec2{pr[2 * k], pr[2 * k + 1]};
    }
    if (unc) *unc = std::move(un);
    return out;
}

}  // namespace nrmosaic
