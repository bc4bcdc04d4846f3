/*
 * nrm_oracle.h -- CPU restatement of the reference's dense per-pixel stage.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker for the CUDA product
 * in paper_2103_07414_b200/. Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it. The product
 * never links or calls it.
 *
 * Every function restates one reference function in plain C99, in the same
 * floating-point operation order (FP64, no contraction), so its results are
 * bit-identical to the reference built with g++ on x86-64. Pinned against
 * golden vectors produced by the real reference (oracle/_ref, see
 * oracle/make_golden.py and tests/test_oracle_golden.py).
 *
 * Array layouts (shared with include/nrm_b200.h):
 *   points / anchors : double[n][2]            (x, y)
 *   warps / locals   : double[n][5]            (scale, w, z, dx, dy)
 *   frame            : uint8[h][w][ch], ch in {1,3,4}
 *   stats            : int64[4] = footprint, blended, no_support, out_of_frame
 */
#ifndef NRM_ORACLE_H
#define NRM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Reference Canvas (mosaic.hpp:100-182): tile-aligned, FP64 RGB + u8 weight. */
typedef struct orc_canvas {
    int64_t origin_x, origin_y;
    int width, height;
    double *color;     /* [height][width][3] */
    uint8_t *weight;   /* [height][width]    */
} orc_canvas;

orc_canvas *orc_canvas_new(void);
void orc_canvas_free(orc_canvas *c);
/* Canvas::ensure_contains (mosaic.hpp:131-174). Returns 0, or -1 on OOM. */
int orc_canvas_ensure_contains(orc_canvas *c, double x0, double y0, double x1, double y1);
void orc_canvas_info(const orc_canvas *c, int64_t *ox, int64_t *oy, int *w, int *h);
double *orc_canvas_color(orc_canvas *c);
uint8_t *orc_canvas_weight(orc_canvas *c);

/* pixel_warp (mosaic.hpp:22-51). Returns 1 with out5 = {scale,w,z,dx,dy}, or 0 (nullopt). */
int orc_pixel_warp(double x, double y, const double *anchors, const double *warps, int n,
                   double alpha, double *out5);

/* WarpFunction::apply (dualquat.hpp:107, 75-80). */
void orc_warp_apply(const double *warp5, double px, double py, double *out2);

/* blend_frame (mosaic.hpp:196-296). stats: int64[4]. Returns 0 or -1 on OOM. */
int orc_blend_frame(orc_canvas *c, const uint8_t *frame, int fw, int fh, int ch,
                    const double *anchors, const double *warps, int n, double alpha,
                    const double *poly, int npoly, int64_t *stats);
/* blend_frame restricted to block-cyclic 64-row stripes (nrm_canvas_set_band). */
int orc_blend_frame_band(orc_canvas *cv, const uint8_t *frame, int fw, int fh, int ch,
                         const double *anchors, const double *warps, int n, double alpha,
                         const double *poly, int npoly, int band_rank, int band_count, int64_t *stats);

/* render (mosaic.hpp:301-331). Two-phase: call with out == NULL to get the size
 * (out_w, out_h; 0x0 when empty) and crop origin; then with a w*h*4 buffer. */
/* Extension (no reference counterpart): uncertainty-weighted blend_frame,
 * unc[fh][fw] frame-aligned; see nrm_blend_frame_weighted. */
int orc_blend_frame_weighted(orc_canvas *c, const uint8_t *frame, int fw, int fh, int ch,
                             const double *anchors, const double *warps, int n, double alpha,
                             const double *poly, int npoly, const float *unc, int64_t *stats);
/* Extension (no reference counterpart): new(p) = old(p + d(p)) over the
 * canvas rectangle [x, x+w) x [y, y+h), d = disp[h][w][2]; colours are read
 * as float32 (the GPU canvas precision) and rounded to float32 on output. */
int orc_canvas_deform(orc_canvas *c, int x, int y, int w, int h, const float *disp);
void orc_render(const orc_canvas *c, int crop, uint8_t *out, int *out_w, int *out_h,
                double *crop_origin2);

/* invert_frame_boundary (mosaic.hpp:58-96). Returns the polygon size; writes
 * up to cap points into poly. */
int orc_invert_frame_boundary(int fw, int fh, const double *anchors, const double *warps,
                              int n, double alpha, double step, double *poly, int cap);

/* detail::blend_local (fieldest.hpp:75-97) over candidates `active` (indices
 * into apts/locals/probs). out5 = blended warp. Returns 0, -1 on empty. */
int orc_blend_local(const double *locals, const double *apts, const double *probs,
                    const int32_t *active, int nactive, double qx, double qy, double alpha,
                    int support, double *out5);

/* node_uncertainty (fieldest.hpp:44-52) over pts[m]. Returns NaN on bad input. */
double orc_node_uncertainty(double qx, double qy, const double *pts, int m, double beta);
/* Engine::blended_variance_at (slam.hpp:703-714) at every grid pixel. */
void orc_variance_field(double x0, double y0, int w, int h, const double *pos, const double *var, int n,
                        double alpha, double *out);

/* Dense grids (the north_star's per-pixel evaluation; SURVEY §8c route).
 * Query pixel (i, j) is the reference coordinate (x0 + i, y0 + j).
 *   node field : disp[j][i][2] = pixel_warp(p)(p) - p, support[j][i] in {0,1}
 *   emdq field : disp = blend_local(p)(p) - p, unc = node_uncertainty(p, apts[active])
 */
void orc_node_field_grid(double x0, double y0, int w, int h, const double *anchors,
                         const double *warps, int n, double alpha, double *disp,
                         uint8_t *support);
int orc_emdq_field_grid(double x0, double y0, int w, int h, const double *apts,
                        const double *locals, const double *probs, const int32_t *active,
                        int nactive, double alpha, int support, double beta, double *disp,
                        double *unc, int row_begin, int row_end);
/* orc_emdq_field_grid with a grid kNN search and OpenMP rows: bit-identical. */
int orc_emdq_field_grid_fast(double x0, double y0, int w, int h, const double *apts,
                             const double *locals, const double *probs, const int32_t *active,
                             int nactive, double alpha, int support, double beta, double *disp,
                             double *unc, int row_begin, int row_end);

/* ---- sparse front end (features.hpp), FP32 as the
 * reference computes it (no contraction) ---------------------------------- */
/* to_gray (image.hpp:63-75) */
void orc_to_gray(const uint8_t *im, int w, int h, int ch, float *out);
/* detect_features (features.hpp:140-205): kp = double[n][3] (x, y, response),
 * desc = float[n][64]; returns n (<= max_features). */
int orc_detect_features(const float *gray, int w, int h, int max_features, double quality,
                        int nms_radius, double *kp, float *desc);
/* match_features (features.hpp:208-254): out = double[n][5]; returns n. */
int orc_match_features(const double *kp_a, const float *desc_a, int na, const double *kp_b,
                       const float *desc_b, int nb, double ratio, double *out);

#ifdef __cplusplus
}
#endif
#endif
