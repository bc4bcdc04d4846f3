/*
 * nrm_b200.h -- C ABI of the B200-native dense per-pixel stage of the
 * real-time non-rigid mosaicking pipeline (arXiv 2103.07414).
 *
 * This is the drop-in boundary for the reference's header-only C++ API
 * (namespace nrmosaic, /root/reference/proj/include/nrmosaic). Each entry
 * point names the reference function it replaces (file:line). The C++ shim
 * include/nrmosaic_b200/mosaic.hpp maps these back onto the reference's
 * signatures, exceptions and std::optional so existing callers recompile
 * unchanged.
 *
 * Conventions
 *   - Every function returns NRM_OK (0) or an NRM_E* code; never throws.
 *     nrm_last_error() gives a thread-local message for the last failure.
 *   - Host-pointer entry points copy inputs to the device with
 *     cudaMemcpyAsync on the context stream (fast from pinned host memory;
 *     pageable memory goes through the driver's own staging) and block until
 *     results are on the host.
 *   - *_device entry points take device pointers, enqueue on the context's
 *     stream and return without synchronising.
 *   - Array layouts:
 *       points / anchors : double[n][2]  (x, y)          -- Vec2 (geometry.hpp:12)
 *       warps / locals   : double[n][5]  (scale, w, z, dx, dy)
 *                                         -- WarpFunction{scale, DualQuat2{w,z,dx,dy}}
 *                                            (dualquat.hpp:97-107, 22-26)
 *       frame            : uint8[h][w][ch], ch in {1, 3, 4} -- ImageU8 (image.hpp:21-43)
 *       canvas colour    : double[h][w][3] in [0,1], weight uint8[h][w]
 *                                         -- Canvas (mosaic.hpp:100-182)
 *   - One context = one CUDA device + one stream; a context is used by one
 *     host thread at a time (the reference's single coordinator thread,
 *     SPEC.md:438). Several contexts may coexist.
 *   - Multi-GPU: one process per GPU, each with its own context. A canvas
 *     can be restricted to block-cyclic 64-row stripes (nrm_canvas_set_band);
 *     control points and frames are replicated by the caller (NCCL).
 */
#ifndef NRM_B200_H
#define NRM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NRM_ABI_VERSION 1

enum {
    NRM_OK = 0,
    NRM_EINVAL = 1,      /* bad argument (reference: std::invalid_argument)        */
    NRM_ENOSUPPORT = 2,  /* no node carries weight (reference: std::nullopt)       */
    NRM_EDEGENERATE = 3, /* DualQuat2 real part < 1e-300 (dualquat.hpp:49-50)      */
    NRM_ECUDA = 4,       /* CUDA runtime / launch failure                          */
    NRM_ENOMEM = 5,      /* device or pinned allocation failed                     */
    NRM_ESTATE = 6       /* object used from the wrong context / after destroy     */
};

typedef struct nrm_ctx nrm_ctx;
typedef struct nrm_canvas nrm_canvas;

/* BlendStats (mosaic.hpp:184-189). */
typedef struct nrm_blend_stats {
    int64_t footprint_pixels;
    int64_t blended_pixels;
    int64_t skipped_no_support;
    int64_t skipped_out_of_frame;
} nrm_blend_stats;

/* Query grid for the dense fields: pixel (i, j) is the reference-frame
 * coordinate (x0 + i, y0 + j), 0 <= i < width, 0 <= j < height. */
typedef struct nrm_grid {
    double x0, y0;
    int width, height;
} nrm_grid;

/* ---- library / context ------------------------------------------------ */
int nrm_abi_version(void);
const char *nrm_last_error(void);

/* Creates a context on CUDA device `device` with its own non-blocking stream.
 * Device scratch grows on first use and is kept until nrm_ctx_destroy.
 * Blends and node fields plan in chunks of 8,192 tiles, about 200 MB. Dense
 * EMDQ fields plan in chunks of 32,768 tiles, 128 MB plus the candidate
 * arrays. Both sizes fit a 4K frame into one launch chunk. */
int nrm_ctx_create(int device, nrm_ctx **out);
int nrm_ctx_destroy(nrm_ctx *ctx);
/* Enqueue subsequent work on an external cudaStream_t (NULL = own stream;
 * the legacy default stream is cudaStreamLegacy, (void *)0x1). */
int nrm_ctx_set_stream(nrm_ctx *ctx, void *cuda_stream);
void *nrm_ctx_stream(nrm_ctx *ctx);
int nrm_ctx_synchronize(nrm_ctx *ctx);
/* Number of kernels this context has launched so far. */
int nrm_ctx_launch_count(nrm_ctx *ctx, int64_t *out);

/* ---- Canvas (mosaic.hpp:100-182) ------------------------------------- */
/* Empty canvas (Canvas::Canvas(), mosaic.hpp:100). Storage lives in HBM:
 * float32 R/G/B planes + uint8 weight plane. */
int nrm_canvas_create(nrm_ctx *ctx, nrm_canvas **out);
int nrm_canvas_destroy(nrm_canvas *cv);
/* Pre-allocates device storage so growth inside rect never reallocates.
 * Does not change the logical canvas (origin/width/height). */
int nrm_canvas_reserve(nrm_canvas *cv, double x0, double y0, double x1, double y1);
/* Canvas::ensure_contains (mosaic.hpp:131-174): identical origin/size
 * bookkeeping (256-px tile alignment); existing pixels preserved exactly. */
int nrm_canvas_ensure_contains(nrm_canvas *cv, double x0, double y0, double x1, double y1);
/* origin_offset() (mosaic.hpp:109), width(), height(). */
int nrm_canvas_info(const nrm_canvas *cv, int64_t *origin_x, int64_t *origin_y, int *width,
                    int *height);
/* Restrict this canvas (this rank) to block-cyclic stripes of 64 reference
 * rows: rows with floor(y / 64) mod count == rank. count = 1: whole canvas. */
int nrm_canvas_set_band(nrm_canvas *cv, int rank, int count);
/* Reads canvas-pixel rectangle [x, x+w) x [y, y+h) (canvas coordinates, as
 * Canvas::color(x, y) / weight(x, y), mosaic.hpp:111-120) into host arrays.
 * Either output may be NULL. */
int nrm_canvas_download(nrm_canvas *cv, int x, int y, int w, int h, double *rgb,
                        uint8_t *weight);
/* Writes a rectangle (Canvas::color(x,y)[k] = ..., weight_ref(x,y) = ...). */
int nrm_canvas_upload(nrm_canvas *cv, int x, int y, int w, int h, const double *rgb,
                      const uint8_t *weight);
/* Extension (north_star "deforming the existing canvas with bilinear
 * sampling"; no reference counterpart): over the canvas
 * rectangle [x, x+w) x [y, y+h), new(p) = old(p + d(p)) with d = disp[h][w][2]
 * in canvas pixels (e.g. a dense field from nrm_node_field / nrm_emdq_field).
 * Bilinear in FP64 over the occupied taps (weights renormalised), weight of
 * the nearest occupied tap; sources outside the canvas or without occupied
 * taps leave the pixel unoccupied. d == 0 is a bit-exact no-op.
 * On a banded canvas (nrm_canvas_set_band) only the rows this rank owns are
 * deformed; their sources must be current, i.e. rows within ceil(max |d_y|)+1
 * of an owned row that other ranks own must first be brought in with
 * nrm_canvas_pack_rows_device / nrm_canvas_unpack_rows_device (the halo
 * exchange, paper_2103_07414_b200/dist.py). Regions of a quarter of the canvas
 * or more run as one ping-pong pass over the canvas (a second set of planes
 * is allocated on first use). */
int nrm_canvas_deform(nrm_canvas *cv, int x, int y, int w, int h, const float *disp);
int nrm_canvas_deform_device(nrm_canvas *cv, int x, int y, int w, int h, const float *d_disp);
/* Halo rows of banded canvases: rows[nrows] (host array of
 * logical canvas rows) across the full canvas width, packed into / unpacked
 * from device memory d_buf as 13 * width bytes per row (R, G, B float32
 * planes, then the uint8 weight). Asynchronous on the context stream. */
int nrm_canvas_pack_rows_device(nrm_canvas *cv, const int *rows, int nrows, void *d_buf);
int nrm_canvas_unpack_rows_device(nrm_canvas *cv, const int *rows, int nrows, const void *d_buf);
/* Canvas::occupied_count (mosaic.hpp:123-127). */
int nrm_canvas_occupied_count(nrm_canvas *cv, int64_t *out);

/* ---- blend_frame (mosaic.hpp:196-296) -------------------------------- */
/* Blends one frame into the canvas. anchors[n][2] are the node anchors in
 * reference coordinates, warps[n][5] their WarpFunctions, alpha the Gaussian
 * coefficient, poly[npoly][2] the footprint polygon (reference coords).
 * Returns the reference's BlendStats; an empty frame or npoly < 3 gives
 * all-zero stats (mosaic.hpp:201). Blocks until done. */
int nrm_blend_frame(nrm_canvas *cv, const uint8_t *frame, int fw, int fh, int ch,
                    const double *anchors, const double *warps, int n, double alpha,
                    const double *poly, int npoly, nrm_blend_stats *out);
/* Device-resident variant: d_frame, d_anchors, d_warps are device pointers,
 * poly stays on the host (it only sets the bounding box). Stats are written
 * to d_stats (int64[4], device) in enqueue order. Asynchronous. */
int nrm_blend_frame_device(nrm_canvas *cv, const uint8_t *d_frame, int fw, int fh, int ch,
                           const double *d_anchors, const double *d_warps, int n, double alpha,
                           const double *poly, int npoly, int64_t *d_stats);

/* Extension (north_star "uncertainty-weighted blending"; no reference
 * counterpart): blend_frame with a frame-aligned
 * per-pixel uncertainty map unc[fh][fw] (node_uncertainty values, >= 1, e.g.
 * the `unc` output of nrm_emdq_field on the frame grid). At a blended pixel
 * the confidence cf = 1 / max(u, 1), u sampled bilinearly at the frame
 * position, scales the update:
 *   colour <- ((w + 1 - cf) colour + cf rgb / 255) / (w + 1),  w <- min(w + 1, 30).
 * With u == 1 everywhere this is the reference rule (mosaic.hpp:278-282) bit
 * for bit. BlendStats and the weight plane are unchanged by the map. */
int nrm_blend_frame_weighted(nrm_canvas *canvas, const uint8_t *frame, int fw, int fh, int ch,
                             const double *anchors, const double *warps, int n, double alpha,
                             const double *poly, int npoly, const float *unc, nrm_blend_stats *out);
int nrm_blend_frame_weighted_device(nrm_canvas *canvas, const uint8_t *d_frame, int fw, int fh, int ch,
                                    const double *d_anchors, const double *d_warps, int n, double alpha,
                                    const double *poly, int npoly, const float *d_unc, int64_t *d_stats);

/* ---- render (mosaic.hpp:301-331) -------------------------------------- */
/* RGBA8 raster of the canvas; alpha 255 where weight > 0. With crop, the
 * bounding box of occupied pixels. Call with out == NULL to get the size
 * (0 x 0 when empty) and crop origin, then with an out_w*out_h*4 buffer. */
int nrm_render(nrm_canvas *cv, int crop, uint8_t *out, int *out_w, int *out_h,
               double *crop_origin2);
/* Renders canvas rectangle [x, x+w) x [y, y+h) into device memory d_out
 * (w*h*4 bytes); rows this rank does not own are written as zeros, so a
 * SUM-reduce over ranks assembles the banded canvas. Asynchronous. */
int nrm_render_device(nrm_canvas *cv, int x, int y, int w, int h, uint8_t *d_out);
/* Occupied bounding box (canvas coords) of the pixels this rank owns;
 * returns x1 < x0 when nothing is occupied. */
int nrm_canvas_occupied_bbox(nrm_canvas *cv, int *x0, int *y0, int *x1, int *y1);

/* ---- PNG output (image.hpp:160-192 save_png) --------
 * Writes image[h][w][channels] (1: gray, 3: RGB, 4: RGBA, as save_png) as an
 * 8-bit non-interlaced PNG, deflating bands of scanlines on `threads` host
 * threads (<= 0: all cores) at zlib `level` (-1 default, 0..9). Host only,
 * needs no device. E.g. the RGBA of nrm_render. */
int nrm_save_png(const char *path, const uint8_t *image, int w, int h, int channels, int level,
                 int threads);

/* ---- node field: pixel_warp (mosaic.hpp:22-51) ------------------------ */
/* pixel_warp at npts arbitrary points (exact FP64 path). out_warps[npts][5];
 * valid[i] = 0 where the reference returns nullopt. */
int nrm_pixel_warp(nrm_ctx *ctx, const double *points, int npts, const double *anchors,
                   const double *warps, int n, double alpha, double *out_warps, uint8_t *valid);
/* Dense node field on a grid: disp[j][i] = pixel_warp(p)(p) - p (float2),
 * support[j][i] = 1, or (0, 0) / 0 where nullopt. Either output may be NULL. */
int nrm_node_field(nrm_ctx *ctx, const nrm_grid *grid, const double *anchors,
                   const double *warps, int n, double alpha, float *disp, uint8_t *support);
int nrm_node_field_device(nrm_ctx *ctx, const nrm_grid *grid, const double *d_anchors,
                          const double *d_warps, int n, double alpha, float *d_disp,
                          uint8_t *d_support);

/* The dense node field restricted to the block-cyclic 64-row stripes of
 * rank band_rank of band_count (nrm_canvas_set_band's rule on absolute rows):
 * only those rows of d_disp / d_support are written. The grid origin must be
 * integral; its planning tiles are anchored to absolute reference pixels like
 * the canvas's, so the ranks' rows together are bit-identical to the
 * band_count = 1 call for any band count (the canvas-wide field of a
 * multi-GPU canvas deformation). Values agree with
 * nrm_node_field_device to the field tolerance. */
int nrm_node_field_band_device(nrm_ctx *ctx, const nrm_grid *grid, const double *d_anchors,
                               const double *d_warps, int n, double alpha, float *d_disp,
                               uint8_t *d_support, int band_rank, int band_count);

/* ---- node variance field: Engine::blended_variance_at (slam.hpp:703-714) --
 * at every grid pixel: out[j][i] = sum_k w_k var_k / sum_k w_k with
 * w_k = exp(-alpha (|pos_k - p|^2 - d2min(p))) over all n nodes (their
 * current positions pos[n][2], variances var[n]); 0 without nodes. A per-pixel
 * uncertainty source for nrm_blend_frame_weighted. Values
 * agree with the reference's FP64 formula to 1e-6 of max |var|. O(n) per
 * pixel (no cutoff, like the reference): frame lattices. */
int nrm_variance_field(nrm_ctx *ctx, const nrm_grid *grid, const double *positions,
                       const double *variances, int n, double alpha, float *out);
int nrm_variance_field_device(nrm_ctx *ctx, const nrm_grid *grid, const double *d_positions,
                              const double *d_variances, int n, double alpha, float *d_out);

/* ---- footprint: invert_frame_boundary (mosaic.hpp:58-96) -------------- */
/* Writes up to cap points to poly[cap][2]; *npoly = the full polygon size. */
int nrm_invert_frame_boundary(nrm_ctx *ctx, int fw, int fh, const double *anchors,
                              const double *warps, int n, double alpha, double step,
                              double *poly, int cap, int *npoly);

/* ---- EMDQ field: detail::blend_local (fieldest.hpp:75-97) + node_uncertainty
 *      (fieldest.hpp:44-52) at every grid pixel ---------------------------- */
/* apts[m_total][2], locals[m_total][5], probs[m_total]: the estimator's
 * per-match arrays; active[nactive]: the candidate indices (the inliers).
 * disp[j][i] = blend_local(p)(p) - p (float2), unc[j][i] =
 * node_uncertainty(p, apts[active], beta). support = FieldParams::blend_support
 * (fieldest.hpp:26, 1..32). Either output may be NULL. */
int nrm_emdq_field(nrm_ctx *ctx, const nrm_grid *grid, const double *apts, const double *locals,
                   const double *probs, int m_total, const int32_t *active, int nactive,
                   double alpha, int support, double beta, float *disp, float *unc);
int nrm_emdq_field_device(nrm_ctx *ctx, const nrm_grid *grid, const double *d_apts,
                          const double *d_locals, const double *d_probs, int m_total,
                          const int32_t *d_active, int nactive, double alpha, int support,
                          double beta, float *d_disp, float *d_unc);

/* ---- EMDQ at scattered points: the EM E-step and the final field --------
 * detail::blend_local (fieldest.hpp:75-97) at nq query points q[nq][2], in
 * the exact tier (FP64, the reference's operation order and libm: results
 * are bit-identical to the reference's). exclude[k] (or NULL: none) is an
 * original match index left out of query k's candidates: the E-step's
 * leave-one-out residual passes q = apts, exclude[j] = j over the matches
 * (fieldest.hpp:195-209); the final field passes the node anchors and no
 * exclusion (fieldest.hpp:263-270). Outputs (each may be NULL):
 *   warps[nq][5] = blend_local(q) as {scale, w, z, dx, dy},
 *   pred[nq][2]  = blend_local(q).apply(q),
 *   unc[nq]      = bounded_exp(beta * d2min) over the same candidates
 *                  (node_uncertainty, fieldest.hpp:44-52; beta > 0),
 *   status[nq]   = 0 ok, 1 no candidate left (the E-step's `others.empty()`),
 *                  2 dq_blend would throw (no positive weight / degenerate).
 * Non-zero status leaves warps/pred zero and unc as computed. */
int nrm_emdq_points(nrm_ctx *ctx, const double *q, const int32_t *exclude, int nq,
                    const double *apts, const double *locals, const double *probs, int m_total,
                    const int32_t *active, int nactive, double alpha, int support, double beta,
                    double *warps, double *pred, double *unc, int32_t *status);
int nrm_emdq_points_device(nrm_ctx *ctx, const double *d_q, const int32_t *d_exclude, int nq,
                           const double *d_apts, const double *d_locals, const double *d_probs,
                           int m_total, const int32_t *d_active, int nactive, double alpha,
                           int support, double beta, double *d_warps, double *d_pred,
                           double *d_unc, int32_t *d_status);

/* blend_frame for nf frames of one size, in order, on device pointers (the
 * multi-GPU weak-scaling step blends several frames per rank). Frames whose
 * footprint windows are pairwise disjoint go through one planner, one field
 * and one exception launch for all of them (up to 16 frames); otherwise (or
 * for node lattices of 257+ nodes) the frames are blended one by one. Results are identical to
 * nf nrm_blend_frame_device calls. d_stats: int64[nf][4] on the device. */
int nrm_blend_frames_device(nrm_canvas *canvas, int nf, const uint8_t *const *d_frames, int fw, int fh,
                            int ch, const double *const *d_anchors, const double *const *d_warps,
                            const int *n, double alpha, const double *const *polys, const int *npoly,
                            int64_t *d_stats);

/* ---- sparse front end -------------------------------
 * Corner detection and ratio-test matching before the EM, bit-identical to
 * the reference (features.hpp). */
/* DetectorConfig (features.hpp:30-36); `workers` has no meaning here. */
typedef struct nrm_detector_config {
    int max_features;      /* 800 */
    double quality_level;  /* 0.005: fraction of the maximum corner response */
    int nms_radius;        /* 4 */
    double ratio_test;     /* 0.8: used by nrm_match_features callers */
} nrm_detector_config;

/* detect_features(to_gray(image), cfg) (features.hpp:140-205,
 * image.hpp:63-75). Keypoints in the reference's order (response desc, y, x),
 * at most cfg->max_features: kp = double[n][3] (x, y, response), desc =
 * float[n][64] (FrameFeatures::descriptors). Both arrays must hold
 * cfg->max_features rows; *n receives the count. An image smaller than
 * 2 * 10 + 1 px in either direction, or without a positive response, gives 0
 * keypoints, as in the reference. */
int nrm_detect_features(nrm_ctx *ctx, const uint8_t *image, int w, int h, int ch,
                        const nrm_detector_config *cfg, double *kp, float *desc, int *n);
/* The same on an FP32 gray image (ImageF, detect_features' own input). */
int nrm_detect_features_gray(nrm_ctx *ctx, const float *gray, int w, int h,
                             const nrm_detector_config *cfg, double *kp, float *desc, int *n);
/* Device pointers; d_n is a device int. Enqueued on the context stream;
 * returns without synchronising. */
int nrm_detect_features_device(nrm_ctx *ctx, const uint8_t *d_image, int w, int h, int ch,
                               const nrm_detector_config *cfg, double *d_kp, float *d_desc,
                               int *d_n);

/* match_features(a, b, ratio) (features.hpp:208-254): for every keypoint of
 * a (in order) whose nearest descriptor in b passes the ratio test, one row
 * (ax, ay, bx, by, score) of `out` (double[na][5]); *n receives the count.
 * nb < 2 or na == 0 gives no matches. kp_* use the nrm_detect_features
 * layout (x, y, response). */
int nrm_match_features(nrm_ctx *ctx, const double *kp_a, const float *desc_a, int na,
                       const double *kp_b, const float *desc_b, int nb, double ratio,
                       double *out, int *n);
int nrm_match_features_device(nrm_ctx *ctx, const double *d_kp_a, const float *d_desc_a, int na,
                              const double *d_kp_b, const float *d_desc_b, int nb,
                              double ratio, double *d_out, int *d_n);

/* ---- kernel timing -------------------------------------------------------
 * With profiling on, a CUDA event is recorded on the context stream before
 * every kernel and at the end of every compute call; a kernel's time is the
 * interval to the next event. nrm_ctx_profile(ctx, 1) clears and enables,
 * 0 disables. nrm_ctx_profile_read returns per-kernel totals: names joined
 * by '\n' into `names`, total ms and launch counts (up to cap entries). */
int nrm_ctx_profile(nrm_ctx *ctx, int enable);
int nrm_ctx_profile_read(nrm_ctx *ctx, char *names, int names_len, double *ms, int64_t *counts,
                         int cap, int *n);

/* ---- pure host planning (no CUDA device needed) --------------------------
 * The host-side bookkeeping the entry points above perform, exposed for
 * testing and for multi-GPU orchestration. */
/* Canvas::ensure_contains (mosaic.hpp:131-174): logical canvas after growth. */
int nrm_plan_ensure_contains(int64_t origin_x, int64_t origin_y, int width, int height, double x0,
                             double y0, double x1, double y1, int64_t *new_origin_x,
                             int64_t *new_origin_y, int *new_width, int *new_height);
/* blend_frame's pixel window (mosaic.hpp:203-213) on a canvas whose origin
 * (after ensure_contains) is (origin_x, origin_y): inclusive canvas-pixel
 * bbox {px0, py0, px1, py1} of polygon_bbox(poly).expanded(4) and its pixel
 * count (BlendStats::footprint_pixels). */
int nrm_plan_footprint(const double *poly, int npoly, int64_t origin_x, int64_t origin_y,
                       int64_t *bbox4, int64_t *footprint);
/* 1 if absolute reference row `abs_row` belongs to band `rank` of `count`
 * (block-cyclic 64-row stripes, nrm_canvas_set_band). */
int nrm_band_owns_row(int64_t abs_row, int rank, int count);

/* ---- diagnostics ---------------------------------------------------------
 * Evaluates the exact tier's exp / hypot emulation (nrm_libm.cuh) on the
 * device so tests can check it bit-for-bit against the host libm. */
int nrm_selftest_libm(nrm_ctx *ctx, const double *x, const double *y, int n, double *exp_out,
                      double *hypot_out);
/* Margin-classified exceptions of the last calls on this context (parity
 * reporting): pixels the last blend_frame / node_field exception pass resolved
 * in the exact tier, and pixels of the last emdq_field that took the exact
 * tier. Synchronises the context stream. */
int nrm_ctx_exceptions(nrm_ctx *ctx, int64_t *blend_exceptions, int64_t *emdq_exact);
/* Exception-queue slots per launch (0 = default: 1/64 of the launch's
 * pixels, at least 2^18, for the node field and the blend; 1/32, at least
 * 2^16, for the EMDQ field). Deferred pixels past the capacity are never
 * lost: the node field and the blend mark them in the output and resolve
 * them by a scan in the exact pass, the EMDQ field resolves them in place,
 * so results do not depend on this value (tests force tiny queues with it). */
int nrm_ctx_set_exception_capacity(nrm_ctx *ctx, int64_t slots);
/* Number of launches on this context whose exception queue overflowed into
 * the scan path (diagnostics; synchronises the context stream). */
int nrm_ctx_spilled_launches(nrm_ctx *ctx, int64_t *out);
/* Measured pipe throughput on this device, lane-operations per second:
 * which = 0: FP32 FFMA, which = 1: MUFU.EX2 (roofline denominators). */
int nrm_selftest_peak(nrm_ctx *ctx, int which, double *ops_per_s);

#ifdef __cplusplus
}
#endif
#endif /* NRM_B200_H */
