// nrm_internal.h -- host-side objects behind the C ABI and the kernel
// launch interfaces shared between translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "nrm_b200.h"

namespace nrm {

// Grow-only device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes);
    void release();
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

struct PinnedBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes);
    void release();
};

// Per-context kernel timing (nrm_ctx_profile): a CUDA event is recorded on the
// launching stream before every kernel and after every profiled API call; a
// kernel's time is the interval to the next event.
struct Prof {
    bool on = false;
    std::vector<cudaEvent_t> ev;
    std::vector<const char*> name;
    size_t used = 0;
};

constexpr int kFrameSlots = 16;  // frames of a batched blend (nrm_blend_frames_device)

// Records a timing mark for the context of the current API call (no-op
// unless that context has profiling enabled).
void prof_mark(const char* name, cudaStream_t st);

}  // namespace nrm

struct nrm_ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    int64_t launches = 0;
    int num_sms = 148;
    int64_t exc_cap_override = 0;  // nrm_ctx_set_exception_capacity (tests); 0 = default sizing
    // scratch (grow-only)
    nrm::DevBuf emdq_cell_cnt;  // K3 candidate bin counts (zeroed on allocation, kept zero by k_bin_scan)
    nrm::DevBuf emdq_cells;     // K3 candidate bins: starts, cursors, indices
    nrm::DevBuf frame_raw, anchors, warps, exc, misc, stats, pts, locals, probs,
        active, out_a, out_b, tiles, feat, feat_io, batch, halo,
        frame_rgba;  // K1: RGBA8 copies of the blended frames (texture storage, one slot per frame)
    // texture objects over the frame_rgba slots, rebuilt when a slot's storage
    // or the frame shape changes
    unsigned long long ftex[nrm::kFrameSlots] = {};
    const void* ftex_ptr[nrm::kFrameSlots] = {};
    int ftex_w[nrm::kFrameSlots] = {}, ftex_h[nrm::kFrameSlots] = {};
    size_t ftex_pitch[nrm::kFrameSlots] = {};
    nrm::PinnedBuf staging, staging_out;
    nrm::Prof prof;
};

struct nrm_canvas {
    nrm_ctx* ctx = nullptr;
    // logical canvas: reference bookkeeping (mosaic.hpp:176-181)
    int64_t origin_x = 0, origin_y = 0;
    int width = 0, height = 0;
    // physical device storage: cap_w x cap_h pixels whose (0,0) is the
    // absolute reference coordinate (phys_x0, phys_y0); SoA planes.
    int64_t phys_x0 = 0, phys_y0 = 0;
    int cap_w = 0, cap_h = 0;
    float* r = nullptr;
    float* g = nullptr;
    float* b = nullptr;
    uint8_t* w = nullptr;
    // alternate planes of the same physical extent for the ping-pong canvas
    // deformation (allocated on first use, dropped when the canvas grows)
    float* ar = nullptr;
    float* ag = nullptr;
    float* ab = nullptr;
    uint8_t* aw = nullptr;
    // reservation (absolute, tile-aligned), 0-size when none
    int64_t res_x0 = 0, res_y0 = 0, res_x1 = 0, res_y1 = 0;
    int band_rank = 0, band_count = 1;
};

namespace nrm {

// Makes `c` the profiled context of this thread for the scope of an API call
// and closes the call with an end mark.
struct ProfScope {
    nrm_ctx* prev;
    explicit ProfScope(nrm_ctx* c);
    ~ProfScope();
};

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

// ---- launches (k_nodefield.cu) ----------------------------------------
struct FieldGrid {
    double gx, gy;      // coordinate of index (0, 0)
    int i0, j0, i1, j1; // valid index range, inclusive
};

struct NodeFieldLaunch {
    // K1: TMA tensor maps of the canvas planes R, G, B (FP32) and W (u8), box
    // 32 x 32 (one K1 CTA's canvas tile); `ctm_ok` 0: cp.async staging instead
    alignas(64) CUtensorMap ctm[4];
    int ctm_ok = 0;
    // inputs
    const uint8_t* frame = nullptr;  // ImageU8 layout: h x w x fch, fch in {1, 3, 4}
    int fw = 0, fh = 0, fch = 3;
    // the same frame as an RGBA8 texture (normalised reads; 0: none): the fast
    // tier's bilinear sample is three 2 x 2 gathers (tex2Dgather) instead of
    // twelve byte loads and conversions
    unsigned long long ftex = 0;
    // when set, the first k_nf_plan launch appends conversion CTAs that write
    // the frame's RGBA8 rows (pitch frgba_pitch) the texture reads
    uint8_t* frgba = nullptr;
    size_t frgba_pitch = 0;
    // optional (extension): frame-aligned per-pixel
    // uncertainty (fw x fh, node_uncertainty >= 1); the blend's update step is
    // scaled by the confidence 1 / max(u, 1) sampled bilinearly at the frame
    // position. Null (or u == 1 everywhere) is the reference rule bit for bit.
    const float* unc = nullptr;
    const double* anchors = nullptr;
    const double* warps = nullptr;
    int n = 0;
    double alpha = 0.0;
    FieldGrid grid{};
    // BLEND mode: canvas planes (index (i, j) == absolute reference pixel)
    float* R = nullptr;
    float* G = nullptr;
    float* B = nullptr;
    uint8_t* W = nullptr;
    long long pitch = 0;
    int phys_x0 = 0, phys_y0 = 0;
    int band_rank = 0, band_count = 1;
    // FIELD mode outputs (row-major over the valid range)
    float2* disp = nullptr;
    uint8_t* support = nullptr;
    // Persistent per-context state, zero between calls (the exception pass
    // restores it): acc[0..2] = blended, no_support, out_of_frame partial sums.
    unsigned long long* acc = nullptr;
    // BLEND mode: final BlendStats (int64[4]) written by the exception pass
    unsigned long long* stats_out = nullptr;
    unsigned long long footprint = 0;
    // exception queue (count persistent-zero, reset by the exception pass)
    int2* exc = nullptr;
    unsigned* exc_count = nullptr;
    unsigned exc_cap = 0;
    unsigned* exc_overflow = nullptr;  // launches whose queue overflowed (diagnostics, accumulated)
    unsigned* exc_last = nullptr;      // pixels the last exception pass resolved (diagnostics)
    unsigned* exc_done = nullptr;      // finished exception CTAs (persistent-zero)
    void* plans = nullptr;             // tile-plan scratch (node_field_plan_bytes(n))
    // Per launch chunk (chunk_rows launch tile rows each): index-ordered
    // lists of the nodes that can reach the chunk, written by k_nf_prefilter
    // (lists == null: every chunk scans all n nodes).
    int* lists = nullptr;              // [nchunks][col_groups][lstride]
    int* lcounts = nullptr;            // [nchunks][col_groups]
    int lstride = 0, chunk_rows = 1;
    int col_groups = 1;                // tile-column groups of NF_GROUP_TILES per chunk
    int tile_j0 = 0, band_s1 = 0;      // launch-row <-> tile-row mapping (exact pass)
};
size_t node_field_scratch_bytes(const NodeFieldLaunch& L);

// mode 0 = blend into canvas, 1 = node field (disp/support)
cudaError_t launch_node_field(const NodeFieldLaunch& L, int mode, cudaStream_t st, int64_t* launches);
// ImageU8 frames (fch 3 or 4) -> RGBA8 rows of `pitch` bytes, frame k into
// out + k * slot_bytes (K1's frame textures); one launch for all frames.
struct FrameSet {
    const uint8_t* f[kFrameSlots];
};
cudaError_t launch_frame_rgba(const FrameSet& fs, int nf, int fw, int fh, int fch, uint8_t* out, size_t pitch,
                              size_t slot_bytes, cudaStream_t st, int64_t* launches);
// Blends of several frames whose footprints are pairwise disjoint, in one
// planner / field / exception launch each (reference rule, frame lattices of
// fewer than 257 nodes, all tiles in one plan chunk; otherwise
// cudaErrorNotSupported and the caller blends frame by frame). Each Ls[f]
// carries its own exception queue, counters and stats_out.
size_t node_field_batch_scratch_bytes(int nf);
cudaError_t launch_node_field_batch(const NodeFieldLaunch* Ls, int nf, void* scratch, cudaStream_t st,
                                    int64_t* launches);
cudaError_t launch_pixel_warp_points(const double* pts, int npts, const double* anchors,
                                     const double* warps, int n, double alpha, double* out,
                                     uint8_t* valid, cudaStream_t st, int64_t* launches);
cudaError_t launch_invert_boundary(int fw, int fh, const double* anchors, const double* warps,
                                   int n, double alpha, double step, double* poly, int nsamples,
                                   cudaStream_t st, int64_t* launches);

cudaError_t launch_selftest_libm(const double* x, const double* y, int n, double* ex, double* hy,
                                 cudaStream_t st, int64_t* launches);

cudaError_t run_peak_probe(int which, int num_sms, int iters, float* scratch, cudaStream_t st,
                           float* ms, int64_t* launches);

// ---- k_emdq.cu ------------------------------------------------------------
struct EmdqLaunch {
    FieldGrid grid{};
    const double* apts = nullptr;     // m_total x 2
    const double* locals = nullptr;   // m_total x 5
    const double* probs = nullptr;    // m_total
    const int32_t* active = nullptr;  // nactive
    int m_total = 0, nactive = 0;
    double alpha = 0.0, beta = 0.0;
    int support = 16;
    float2* disp = nullptr;
    float* unc = nullptr;
    unsigned* exact_count = nullptr;  // pixels that took the exact tier (diagnostics, accumulated)
    // exact-tier queue of the dense field (k_pixels -> k_emdq_exceptions),
    // carved from the scratch by launch_emdq_field
    int2* exq = nullptr;
    unsigned* exq_count = nullptr;
    unsigned exq_cap = 0;
    int64_t exq_cap_override = 0;  // nrm_ctx_set_exception_capacity (tests); 0 = default sizing
    // large candidate sets: the candidates binned into 64 px cells (the
    // supertile grid plus a margin ring), so k_super scans only the cells
    // near each supertile. cell_cnt: per-cell counts, persistent-zero (its
    // own buffer: a call with fewer cells must not leave data where a later
    // call with more cells counts); cells: start[nc + 1] | cursor[nc] | index[N]
    int* cell_cnt = nullptr;
    int* cells = nullptr;
    // scratch: gathered candidates (SoA, nactive each)
    double* cx = nullptr;
    double* cy = nullptr;
    double* cl = nullptr;   // nactive x 5 (scale, w, z, dx, dy)
    double* cp = nullptr;   // max(prob, 1e-6)
};
cudaError_t launch_emdq_field(const EmdqLaunch& L, cudaStream_t st, int64_t* launches);
// binning buffers for a call (0, 0: no binning at this size)
void emdq_cell_bytes(int nactive, const FieldGrid& g, size_t* count_bytes, size_t* bin_bytes);
size_t emdq_scratch_bytes(int nactive, const FieldGrid& g, bool tile_plans = true);
// Scattered queries (EM E-step / final field): L.grid is a grid covering the
// queries (only its supertile geometry is used); exact tier throughout.
struct PointsLaunch {
    const double* q = nullptr;
    const int32_t* excl = nullptr;
    int nq = 0;
    double* warps = nullptr;
    double* pred = nullptr;
    double* unc = nullptr;
    int32_t* status = nullptr;
    bool full_scan = false;  // every query scans all candidates (very spread-out queries)
};
cudaError_t launch_emdq_points(const EmdqLaunch& L, const PointsLaunch& P, cudaStream_t st, int64_t* launches);
// Device-side bounding box of nq points -> out4 = {minx, miny, maxx, maxy}.
cudaError_t launch_points_bbox(const double* q, int nq, double* out4, cudaStream_t st, int64_t* launches);

// ---- k_variance.cu (Engine::blended_variance_at, slam.hpp:703-714, per pixel) ----
cudaError_t launch_variance_field(double x0, double y0, int w, int h, const double* pos, const double* var, int n,
                                  double alpha, float* out, cudaStream_t st, int64_t* launches);

// ---- k_canvas.cu ----------------------------------------------------------
cudaError_t launch_render(const nrm_canvas* cv, int x, int y, int w, int h, uint8_t* out,
                          cudaStream_t st, int64_t* launches);
// Extension: canvas deformation new(p) = old(p + d(p)) over a logical
// region. Regions of a quarter of the canvas or more run one ping-pong pass
// over the canvas into the alternate planes (swapped in afterwards); smaller
// ones use `scratch` (13 B per region pixel) and a copy-back.
bool deform_uses_ping_pong(const nrm_canvas* cv, int w, int h);
cudaError_t launch_canvas_deform(nrm_canvas* cv, int x, int y, int w, int h, const float2* disp, float* scratch,
                                 cudaStream_t st, int64_t* launches);
// Halo rows of banded canvases: rows (logical canvas rows, device int array)
// packed as {R, G, B float32, W uint8} x canvas width per row (13 w bytes).
cudaError_t launch_rows_pack(const nrm_canvas* cv, const int* d_rows, int nrows, void* d_buf, cudaStream_t st,
                             int64_t* launches);
cudaError_t launch_rows_unpack(nrm_canvas* cv, const int* d_rows, int nrows, const void* d_buf, cudaStream_t st,
                               int64_t* launches);
cudaError_t launch_occupied(const nrm_canvas* cv, unsigned long long* count, int* bbox4,
                            cudaStream_t st, int64_t* launches);
cudaError_t launch_canvas_read(const nrm_canvas* cv, int x, int y, int w, int h, double* rgb,
                               uint8_t* weight, cudaStream_t st, int64_t* launches);
cudaError_t launch_canvas_write(nrm_canvas* cv, int x, int y, int w, int h, const double* rgb,
                                const uint8_t* weight, cudaStream_t st, int64_t* launches);


// ---- k_features.cu -------------------------------------
struct FeatLaunch {
    const uint8_t* image = nullptr;  // ImageU8 layout, or null when gray_in is set
    const float* gray_in = nullptr;  // ImageF gray (detect_features' own input)
    int w = 0, h = 0, ch = 1;
    int max_features = 800, nms_radius = 4;
    float quality = 0.005f;          // static_cast<float>(quality_level) (features.hpp:150)
    double* kp = nullptr;            // [max_features][3]: x, y, response
    float* desc = nullptr;           // [max_features][64]
    int* status = nullptr;           // device int[2]: [0] keypoints
    void* scratch = nullptr;         // features_scratch_bytes
};
size_t features_cand_cap(int w, int h, int r);
size_t features_scratch_bytes(int w, int h, int r, int kmax);
cudaError_t launch_detect_features(const FeatLaunch& F, cudaStream_t st, int64_t* launches);
struct MatchLaunch {
    const double* kp_a = nullptr;
    const float* desc_a = nullptr;
    int na = 0;
    const double* kp_b = nullptr;
    const float* desc_b = nullptr;
    int nb = 0;
    double ratio = 0.8;
    double* out = nullptr;  // [na][5]: ax, ay, bx, by, score
    int* nout = nullptr;    // device int
    void* scratch = nullptr;
};
size_t match_scratch_bytes(int na, int nb);
cudaError_t launch_match_features(const MatchLaunch& M, cudaStream_t st, int64_t* launches);

}  // namespace nrm
