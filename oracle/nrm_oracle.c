/*
 * nrm_oracle.c -- TEST INFRASTRUCTURE: plain-C restatement of the reference's
 * dense per-pixel stage (arxiv 2103.07414 reference, /root/reference/proj).
 * Used only as the parity checker (tests/, smoke(), bench.py cpu_baseline).
 *
 * Build: gcc -O2 -std=c99 -ffp-contract=off -fPIC -shared (see oracle/Makefile).
 * -ffp-contract=off keeps every a*b+c as two rounded FP64 operations, the way
 * g++ compiles the reference on x86-64, so results are bit-identical.
 */
#include "nrm_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define K_PIXEL_WEIGHT_CUTOFF 1e-6 /* mosaic.hpp:16 */
#define K_WEIGHT_CAP 30            /* mosaic.hpp:102 */
#define K_TILE 256                 /* mosaic.hpp:103 */

typedef struct { double w, z, dx, dy; } dq2;

/* DualQuat2::normalized (dualquat.hpp:47-52); returns 0 on degenerate. */
static int dq_normalized(dq2 in, dq2 *out) {
    const double n = hypot(in.w, in.z);
    if (n < 1e-300) return 0;
    out->w = in.w / n;
    out->z = in.z / n;
    out->dx = in.dx / n;
    out->dy = in.dy / n;
    return 1;
}

/* DualQuat2::apply (dualquat.hpp:75-80) then WarpFunction::apply scale (:107). */
void orc_warp_apply(const double *wp, double px, double py, double *out2) {
    const double scale = wp[0], w = wp[1], z = wp[2], dx = wp[3], dy = wp[4];
    const double c = w * w - z * z;
    const double s = 2.0 * w * z;
    const double ax = c * px - s * py + 2.0 * (dx * w - dy * z);
    const double ay = s * px + c * py + 2.0 * (dx * z + dy * w);
    out2[0] = ax * scale;
    out2[1] = ay * scale;
}

/* WarpFunction::unapply (dualquat.hpp:109-114). */
static int warp_unapply(const double *wp, double qx, double qy, double *out2) {
    const double scale = wp[0], w = wp[1], z = wp[2], dx = wp[3], dy = wp[4];
    if (!(scale > 0.0)) return 0;
    const double c = w * w - z * z;
    const double s = 2.0 * w * z;
    const double tx = 2.0 * (dx * w - dy * z);
    const double ty = 2.0 * (dx * z + dy * w);
    const double vx = qx / scale - tx;
    const double vy = qy / scale - ty;
    out2[0] = c * vx + s * vy;
    out2[1] = (-s) * vx + c * vy;
    return 1;
}

/* ------------------------------------------------------------------------ */
/* pixel_warp (mosaic.hpp:22-51)                                             */
/* ------------------------------------------------------------------------ */
int orc_pixel_warp(double x, double y, const double *anchors, const double *warps, int n,
                   double alpha, double *out5) {
    double wsum = 0.0;
    double acc_w = 0.0, acc_z = 0.0, acc_dx = 0.0, acc_dy = 0.0, acc_s = 0.0;
    double ref_w = 0.0, ref_z = 0.0;
    int have_ref = 0;
    for (int i = 0; i < n; ++i) {
        const double ddx = anchors[2 * i] - x, ddy = anchors[2 * i + 1] - y;
        const double d2 = ddx * ddx + ddy * ddy;
        const double w = exp(-alpha * d2);
        if (w <= K_PIXEL_WEIGHT_CUTOFF) continue;
        const double *q = &warps[5 * i];
        double qw = q[1], qz = q[2], qdx = q[3], qdy = q[4];
        if (!have_ref) {
            ref_w = qw;
            ref_z = qz;
            have_ref = 1;
        } else if (qw * ref_w + qz * ref_z < 0.0) {
            qw = -qw; qz = -qz; qdx = -qdx; qdy = -qdy;
        }
        acc_w += w * qw;
        acc_z += w * qz;
        acc_dx += w * qdx;
        acc_dy += w * qdy;
        acc_s += w * q[0];
        wsum += w;
    }
    if (!have_ref) return 0;
    dq2 mean = {acc_w / wsum, acc_z / wsum, acc_dx / wsum, acc_dy / wsum}, nq;
    if (!dq_normalized(mean, &nq)) return 0;
    out5[0] = acc_s / wsum;
    out5[1] = nq.w; out5[2] = nq.z; out5[3] = nq.dx; out5[4] = nq.dy;
    return 1;
}

/* ------------------------------------------------------------------------ */
/* Canvas (mosaic.hpp:100-182)                                               */
/* ------------------------------------------------------------------------ */
orc_canvas *orc_canvas_new(void) { return (orc_canvas *)calloc(1, sizeof(orc_canvas)); }

void orc_canvas_free(orc_canvas *c) {
    if (!c) return;
    free(c->color);
    free(c->weight);
    free(c);
}

void orc_canvas_info(const orc_canvas *c, int64_t *ox, int64_t *oy, int *w, int *h) {
    *ox = c->origin_x; *oy = c->origin_y; *w = c->width; *h = c->height;
}
double *orc_canvas_color(orc_canvas *c) { return c->color; }
uint8_t *orc_canvas_weight(orc_canvas *c) { return c->weight; }

static int64_t align_down(int64_t v) {
    return v >= 0 ? (v / K_TILE) * K_TILE : ((v - K_TILE + 1) / K_TILE) * K_TILE;
}

int orc_canvas_ensure_contains(orc_canvas *c, double x0, double y0, double x1, double y1) {
    const int64_t nx0_need = (int64_t)floor(x0), ny0_need = (int64_t)floor(y0);
    const int64_t nx1_need = (int64_t)ceil(x1) + 1, ny1_need = (int64_t)ceil(y1) + 1;
    const int empty = c->width == 0;
    if (!empty && nx0_need >= c->origin_x && ny0_need >= c->origin_y &&
        nx1_need <= c->origin_x + c->width && ny1_need <= c->origin_y + c->height)
        return 0;
    int64_t nx0 = align_down(nx0_need), ny0 = align_down(ny0_need);
    int64_t nx1 = nx1_need, ny1 = ny1_need;
    if (!empty) {
        if (c->origin_x < nx0) nx0 = c->origin_x;
        if (c->origin_y < ny0) ny0 = c->origin_y;
        if (c->origin_x + c->width > nx1) nx1 = c->origin_x + c->width;
        if (c->origin_y + c->height > ny1) ny1 = c->origin_y + c->height;
    }
    const int nw = (int)(((nx1 - nx0 + K_TILE - 1) / K_TILE) * K_TILE);
    const int nh = (int)(((ny1 - ny0 + K_TILE - 1) / K_TILE) * K_TILE);
    double *ncolor = (double *)calloc((size_t)nw * nh * 3, sizeof(double));
    uint8_t *nweight = (uint8_t *)calloc((size_t)nw * nh, 1);
    if (!ncolor || !nweight) { free(ncolor); free(nweight); return -1; }
    if (!empty) {
        const int ox = (int)(c->origin_x - nx0), oy = (int)(c->origin_y - ny0);
        for (int y = 0; y < c->height; ++y) {
            memcpy(&ncolor[((size_t)(y + oy) * nw + ox) * 3], &c->color[(size_t)y * c->width * 3],
                   sizeof(double) * (size_t)c->width * 3);
            memcpy(&nweight[(size_t)(y + oy) * nw + ox], &c->weight[(size_t)y * c->width],
                   (size_t)c->width);
        }
    }
    free(c->color);
    free(c->weight);
    c->color = ncolor;
    c->weight = nweight;
    c->origin_x = nx0;
    c->origin_y = ny0;
    c->width = nw;
    c->height = nh;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* sample_bilinear_rgb (image.hpp:78-92)                                     */
/* ------------------------------------------------------------------------ */
static void sample_bilinear_rgb(const uint8_t *im, int iw, int ih, int ch, double x, double y,
                                double *out3) {
    int x0 = (int)x, y0 = (int)y;
    const int xc = iw - 2 >= 0 ? iw - 2 : 0, yc = ih - 2 >= 0 ? ih - 2 : 0;
    if (x0 > xc) x0 = xc;
    if (y0 > yc) y0 = yc;
    const double fx = x - x0, fy = y - y0;
    const int x1 = x0 + 1 < iw - 1 ? x0 + 1 : iw - 1;
    const int y1 = y0 + 1 < ih - 1 ? y0 + 1 : ih - 1;
    for (int c = 0; c < 3; ++c) {
        const int k = ch == 1 ? 0 : c;
        const double v00 = im[((size_t)y0 * iw + x0) * ch + k], v10 = im[((size_t)y0 * iw + x1) * ch + k];
        const double v01 = im[((size_t)y1 * iw + x0) * ch + k], v11 = im[((size_t)y1 * iw + x1) * ch + k];
        out3[c] = ((1 - fx) * v00 + fx * v10) * (1 - fy) + ((1 - fx) * v01 + fx * v11) * fy;
    }
}

/* Rect::distance (geometry.hpp:73-77): hypot(max{x0-p,0,p-x1}, ...). */
static double rect_distance(double rx0, double ry0, double rx1, double ry1, double px, double py) {
    double dx = rx0 - px;
    if (dx < 0.0) dx = 0.0;
    if (dx < px - rx1) dx = px - rx1;
    double dy = ry0 - py;
    if (dy < 0.0) dy = 0.0;
    if (dy < py - ry1) dy = py - ry1;
    return hypot(dx, dy);
}

/* ------------------------------------------------------------------------ */
/* blend_frame (mosaic.hpp:196-296)                                          */
/* ------------------------------------------------------------------------ */
/* Bilinear sample of a float map with sample_bilinear_rgb's taps. */
static double sample_bilinear_f32(const float *m, int w, int h, double x, double y) {
    int x0 = (int)x, y0 = (int)y;
    const int xc = w - 2 >= 0 ? w - 2 : 0, yc = h - 2 >= 0 ? h - 2 : 0;
    if (x0 > xc) x0 = xc;
    if (y0 > yc) y0 = yc;
    const double fx = x - x0, fy = y - y0;
    const int x1 = x0 + 1 < w - 1 ? x0 + 1 : w - 1;
    const int y1 = y0 + 1 < h - 1 ? y0 + 1 : h - 1;
    const double a = m[(size_t)y0 * w + x0], b = m[(size_t)y0 * w + x1];
    const double c = m[(size_t)y1 * w + x0], d = m[(size_t)y1 * w + x1];
    return ((1.0 - fx) * a + fx * b) * (1.0 - fy) + ((1.0 - fx) * c + fx * d) * fy;
}

static int blend_frame_impl(orc_canvas *cv, const uint8_t *frame, int fw, int fh, int ch,
                            const double *anchors, const double *warps, int n, double alpha,
                            const double *poly, int npoly, const float *unc, int band_rank,
                            int band_count, int64_t *stats);

int orc_blend_frame(orc_canvas *cv, const uint8_t *frame, int fw, int fh, int ch,
                    const double *anchors, const double *warps, int n, double alpha,
                    const double *poly, int npoly, int64_t *stats) {
    return blend_frame_impl(cv, frame, fw, fh, ch, anchors, warps, n, alpha, poly, npoly, NULL, 0, 1, stats);
}

/* Multi-GPU restatement (nrm_canvas_set_band): blend_frame
 * restricted to the canvas rows of block-cyclic 64-row stripes
 * floor(y / 64) mod band_count == band_rank (absolute reference rows).
 * footprint_pixels is the whole window (the same on every rank); the other
 * counts cover the owned rows only, so they sum to the reference's over the
 * ranks. band_count = 1 is orc_blend_frame. */
int orc_blend_frame_band(orc_canvas *cv, const uint8_t *frame, int fw, int fh, int ch,
                         const double *anchors, const double *warps, int n, double alpha,
                         const double *poly, int npoly, int band_rank, int band_count, int64_t *stats) {
    return blend_frame_impl(cv, frame, fw, fh, ch, anchors, warps, n, alpha, poly, npoly, NULL, band_rank,
                            band_count, stats);
}

/* Extension (not in the reference): the uncertainty-weighted update of
 * nrm_blend_frame_weighted; unc == 1 everywhere gives orc_blend_frame. */
int orc_blend_frame_weighted(orc_canvas *cv, const uint8_t *frame, int fw, int fh, int ch,
                             const double *anchors, const double *warps, int n, double alpha,
                             const double *poly, int npoly, const float *unc, int64_t *stats) {
    return blend_frame_impl(cv, frame, fw, fh, ch, anchors, warps, n, alpha, poly, npoly, unc, 0, 1, stats);
}

static int band_owns(int64_t abs_row, int band_rank, int band_count) {
    if (band_count <= 1) return 1;
    int64_t s = abs_row >= 0 ? abs_row / 64 : -((-abs_row + 63) / 64);
    int64_t m = s % band_count;
    if (m < 0) m += band_count;
    return m == band_rank;
}

static int blend_frame_impl(orc_canvas *cv, const uint8_t *frame, int fw, int fh, int ch,
                            const double *anchors, const double *warps, int n, double alpha,
                            const double *poly, int npoly, const float *unc, int band_rank,
                            int band_count, int64_t *stats) {
    stats[0] = stats[1] = stats[2] = stats[3] = 0;
    if (fw == 0 || fh == 0 || npoly < 3) return 0;

    /* polygon_bbox (geometry.hpp:180-190) then Rect::expanded(4) */
    double bx0 = DBL_MAX, by0 = DBL_MAX, bx1 = -DBL_MAX, by1 = -DBL_MAX;
    for (int i = 0; i < npoly; ++i) {
        const double px = poly[2 * i], py = poly[2 * i + 1];
        bx0 = px < bx0 ? px : bx0;   /* std::min(a, b) == (b < a) ? b : a */
        by0 = py < by0 ? py : by0;
        bx1 = bx1 < px ? px : bx1;   /* std::max(a, b) == (a < b) ? b : a */
        by1 = by1 < py ? py : by1;
    }
    bx0 -= 4.0; by0 -= 4.0; bx1 += 4.0; by1 += 4.0;
    if (orc_canvas_ensure_contains(cv, bx0, by0, bx1, by1)) return -1;

    const double orgx = (double)cv->origin_x, orgy = (double)cv->origin_y;
    const int px0 = (int)floor(bx0 - orgx), py0 = (int)floor(by0 - orgy);
    const int px1 = (int)ceil(bx1 - orgx), py1 = (int)ceil(by1 - orgy);
    const int bw = px1 - px0 + 1, bh = py1 - py0 + 1;
    if (bw <= 0 || bh <= 0) return 0;
    stats[0] = (int64_t)bw * bh;

    const double max_d2 = -log(K_PIXEL_WEIGHT_CUTOFF) / alpha;
    const double max_d = sqrt(max_d2);
    const int ntx = (bw + K_TILE - 1) / K_TILE;
    int *tile_nodes = (int *)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1) * ntx);
    int *tile_count = (int *)calloc((size_t)ntx, sizeof(int));
    if (!tile_nodes || !tile_count) { free(tile_nodes); free(tile_count); return -1; }
    for (int tx = 0; tx < ntx; ++tx) {
        const int xe = bw < (tx + 1) * K_TILE ? bw : (tx + 1) * K_TILE;
        const double rx0 = orgx + px0 + tx * K_TILE, ry0 = orgy + py0;
        const double rx1 = orgx + px0 + xe, ry1 = orgy + py1 + 1.0;
        for (int i = 0; i < n; ++i)
            if (rect_distance(rx0, ry0, rx1, ry1, anchors[2 * i], anchors[2 * i + 1]) <= max_d)
                tile_nodes[(size_t)tx * n + tile_count[tx]++] = i;
    }

    const double fx_max = fw - 1.0, fy_max = fh - 1.0;
    int64_t blended = 0, no_support = 0, out_of_frame = 0;
    /* rows are independent (each pixel is written once; the counts are
     * order-free integer sums), so OpenMP rows give the serial result */
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : blended, no_support, out_of_frame)
    for (int ry = 0; ry < bh; ++ry) {
        const int cy = py0 + ry;
        const double ref_y = orgy + cy;
        if (!band_owns(cv->origin_y + cy, band_rank, band_count)) continue;
        for (int tx = 0; tx < ntx; ++tx) {
            const int *nodes = &tile_nodes[(size_t)tx * n];
            const int nn = tile_count[tx];
            const int cx_end = px0 + (bw < (tx + 1) * K_TILE ? bw : (tx + 1) * K_TILE);
            for (int cx = px0 + tx * K_TILE; cx < cx_end; ++cx) {
                const double xr = orgx + cx, yr = ref_y;
                double wsum = 0, aw = 0, az = 0, adx = 0, ady = 0, as = 0;
                double ref_w = 0, ref_z = 0;
                int have_ref = 0;
                for (int k = 0; k < nn; ++k) {
                    const int ni = nodes[k];
                    const double ddx = anchors[2 * ni] - xr, ddy = anchors[2 * ni + 1] - yr;
                    const double d2 = ddx * ddx + ddy * ddy;
                    const double w = exp(-alpha * d2);
                    if (w <= K_PIXEL_WEIGHT_CUTOFF) continue;
                    const double *q = &warps[5 * ni];
                    double qw = q[1], qz = q[2], qdx = q[3], qdy = q[4];
                    if (!have_ref) {
                        ref_w = qw; ref_z = qz; have_ref = 1;
                    } else if (qw * ref_w + qz * ref_z < 0.0) {
                        qw = -qw; qz = -qz; qdx = -qdx; qdy = -qdy;
                    }
                    aw += w * qw; az += w * qz;
                    adx += w * qdx; ady += w * qdy;
                    as += w * q[0];
                    wsum += w;
                }
                if (!have_ref) { ++no_support; continue; }
                dq2 mean = {aw / wsum, az / wsum, adx / wsum, ady / wsum}, nq;
                if (!dq_normalized(mean, &nq)) { ++no_support; continue; } /* reference throws */
                const double wp[5] = {as / wsum, nq.w, nq.z, nq.dx, nq.dy};
                double yv[2];
                orc_warp_apply(wp, xr, yr, yv);
                if (!(yv[0] >= 0.0 && yv[0] <= fx_max && yv[1] >= 0.0 && yv[1] <= fy_max)) {
                    ++out_of_frame;
                    continue;
                }
                double rgb[3];
                sample_bilinear_rgb(frame, fw, fh, ch, yv[0], yv[1], rgb);
                double *c = &cv->color[((size_t)cy * cv->width + cx) * 3];
                uint8_t *wgt = &cv->weight[(size_t)cy * cv->width + cx];
                const double wd = *wgt;
                if (unc) {
                    double u = sample_bilinear_f32(unc, fw, fh, yv[0], yv[1]);
                    const double cf = 1.0 / (u > 1.0 ? u : 1.0);
                    const double a = wd + 1.0 - cf;
                    for (int k = 0; k < 3; ++k) c[k] = (a * c[k] + cf * (rgb[k] / 255.0)) / (wd + 1.0);
                } else {
                    c[0] = (wd * c[0] + rgb[0] / 255.0) / (wd + 1.0);
                    c[1] = (wd * c[1] + rgb[1] / 255.0) / (wd + 1.0);
                    c[2] = (wd * c[2] + rgb[2] / 255.0) / (wd + 1.0);
                }
                if (*wgt < K_WEIGHT_CAP) ++*wgt;
                ++blended;
            }
        }
    }
    free(tile_nodes);
    free(tile_count);
    stats[1] = blended;
    stats[2] = no_support;
    stats[3] = out_of_frame;
    return 0;
}

/* Extension (no reference counterpart): canvas deformation
 * new(p) = old(p + d(p)) over a rectangle; see nrm_canvas_deform. */
int orc_canvas_deform(orc_canvas *cv, int x0, int y0, int w, int h, const float *disp) {
    const int W = cv->width, H = cv->height;
    double *nc = (double *)malloc(sizeof(double) * 3 * (size_t)(w > 0 ? w : 1) * (h > 0 ? h : 1));
    uint8_t *nw = (uint8_t *)malloc((size_t)(w > 0 ? w : 1) * (h > 0 ? h : 1));
    if (!nc || !nw) { free(nc); free(nw); return -1; }
    for (int j = 0; j < h; ++j) {
        for (int i = 0; i < w; ++i) {
            const size_t o = (size_t)j * w + i;
            const double sx = (double)(x0 + i) + (double)disp[2 * o];
            const double sy = (double)(y0 + j) + (double)disp[2 * o + 1];
            double c3[3] = {0.0, 0.0, 0.0};
            uint8_t cw = 0;
            if (sx >= 0.0 && sx <= W - 1.0 && sy >= 0.0 && sy <= H - 1.0) {
                /* FP64 source position, FP32 weights and blend (nrm_canvas_deform):
                 * this file is built with -ffp-contract=off, like the kernel's
                 * explicit round-to-nearest float operations */
                int tx0 = (int)sx, ty0 = (int)sy;
                if (tx0 > W - 2) tx0 = W - 2 >= 0 ? W - 2 : 0;
                if (ty0 > H - 2) ty0 = H - 2 >= 0 ? H - 2 : 0;
                const float fx = (float)(sx - tx0), fy = (float)(sy - ty0);
                const int tx1 = tx0 + 1 < W - 1 ? tx0 + 1 : W - 1, ty1 = ty0 + 1 < H - 1 ? ty0 + 1 : H - 1;
                const float gx = 1.0f - fx, gy = 1.0f - fy;
                const int txs[4] = {tx0, tx1, tx0, tx1}, tys[4] = {ty0, ty0, ty1, ty1};
                const float bw[4] = {gx * gy, fx * gy, gx * fy, fx * fy};
                float n3[3] = {0.0f, 0.0f, 0.0f}, den = 0.0f, best = -1.0f;
                for (int t = 0; t < 4; ++t) {
                    const size_t idx = (size_t)tys[t] * W + txs[t];
                    const uint8_t wt = cv->weight[idx];
                    if (wt == 0) continue;
                    for (int k = 0; k < 3; ++k) n3[k] = n3[k] + bw[t] * (float)cv->color[3 * idx + k];
                    den = den + bw[t];
                    if (bw[t] > best) { best = bw[t]; cw = wt; }
                }
                if (den > 0.0f) {
                    const float inv = 1.0f / den; /* correctly rounded, then three products */
                    for (int k = 0; k < 3; ++k) c3[k] = (double)(n3[k] * inv);
                } else {
                    cw = 0;
                }
            }
            for (int k = 0; k < 3; ++k) nc[3 * o + k] = c3[k];
            nw[o] = cw;
        }
    }
    for (int j = 0; j < h; ++j)
        for (int i = 0; i < w; ++i) {
            const size_t o = (size_t)j * w + i, idx = (size_t)(y0 + j) * W + (x0 + i);
            for (int k = 0; k < 3; ++k) cv->color[3 * idx + k] = nc[3 * o + k];
            cv->weight[idx] = nw[o];
        }
    free(nc);
    free(nw);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* render (mosaic.hpp:301-331)                                               */
/* ------------------------------------------------------------------------ */
void orc_render(const orc_canvas *cv, int crop, uint8_t *out, int *out_w, int *out_h,
                double *crop_origin2) {
    if (crop_origin2) { crop_origin2[0] = (double)cv->origin_x; crop_origin2[1] = (double)cv->origin_y; }
    *out_w = 0; *out_h = 0;
    if (cv->width == 0) return;
    int x0 = 0, y0 = 0, x1 = cv->width - 1, y1 = cv->height - 1;
    if (crop) {
        x0 = cv->width; y0 = cv->height; x1 = -1; y1 = -1;
        for (int y = 0; y < cv->height; ++y)
            for (int x = 0; x < cv->width; ++x)
                if (cv->weight[(size_t)y * cv->width + x] > 0) {
                    if (x < x0) x0 = x;
                    if (y < y0) y0 = y;
                    if (x > x1) x1 = x;
                    if (y > y1) y1 = y;
                }
        if (x1 < x0) return;
        if (crop_origin2) {
            crop_origin2[0] = (double)cv->origin_x + (double)x0;
            crop_origin2[1] = (double)cv->origin_y + (double)y0;
        }
    }
    *out_w = x1 - x0 + 1;
    *out_h = y1 - y0 + 1;
    if (!out) return;
    memset(out, 0, (size_t)(*out_w) * (*out_h) * 4);
    for (int y = y0; y <= y1; ++y)
        for (int x = x0; x <= x1; ++x) {
            uint8_t *px = &out[((size_t)(y - y0) * (*out_w) + (x - x0)) * 4];
            if (cv->weight[(size_t)y * cv->width + x] > 0) {
                const double *c = &cv->color[((size_t)y * cv->width + x) * 3];
                for (int k = 0; k < 3; ++k) {
                    double v = c[k];
                    v = v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v); /* std::clamp */
                    px[k] = (uint8_t)lround(v * 255.0);
                }
                px[3] = 255;
            }
        }
}

/* ------------------------------------------------------------------------ */
/* invert_frame_boundary (mosaic.hpp:58-96)                                  */
/* ------------------------------------------------------------------------ */
int orc_invert_frame_boundary(int fw, int fh, const double *anchors, const double *warps,
                              int n, double alpha, double step, double *poly, int cap) {
    const double w1 = fw - 1.0, h1 = fh - 1.0;
    int ns = 0;
    double *pos = (double *)malloc(sizeof(double) * 2 * (size_t)(n > 0 ? n : 1));
    if (!pos) return -1;
    for (int i = 0; i < n; ++i) orc_warp_apply(&warps[5 * i], anchors[2 * i], anchors[2 * i + 1], &pos[2 * i]);

#define NRM_SAMPLE(SX, SY)                                                         \
    do {                                                                           \
        const double yx = (SX), yy = (SY);                                         \
        int nearest = 0;                                                           \
        double best = DBL_MAX;                                                     \
        for (int i = 0; i < n; ++i) {                                              \
            const double ex = pos[2 * i] - yx, ey = pos[2 * i + 1] - yy;           \
            const double d2 = ex * ex + ey * ey;                                   \
            if (d2 < best) { best = d2; nearest = i; }                             \
        }                                                                          \
        double x0x = yx, x0y = yy;                                                 \
        if (n > 0) {                                                               \
            x0x = anchors[2 * nearest] + (yx - pos[2 * nearest]);                  \
            x0y = anchors[2 * nearest + 1] + (yy - pos[2 * nearest + 1]);          \
        }                                                                          \
        for (int it = 0; it < 15; ++it) {                                          \
            double wp[5], nx[2];                                                   \
            if (!orc_pixel_warp(x0x, x0y, anchors, warps, n, alpha, wp)) break;    \
            if (!warp_unapply(wp, yx, yy, nx)) break;                              \
            const double mx = nx[0] - x0x, my = nx[1] - x0y;                       \
            const double move = sqrt(mx * mx + my * my);                           \
            x0x = nx[0]; x0y = nx[1];                                              \
            if (move < 1e-7) break;                                                \
        }                                                                          \
        if (ns < cap) { poly[2 * ns] = x0x; poly[2 * ns + 1] = x0y; }              \
        ++ns;                                                                      \
    } while (0)

    for (double x = 0; x < w1; x += step) NRM_SAMPLE(x, 0.0);
    for (double y = 0; y < h1; y += step) NRM_SAMPLE(w1, y);
    for (double x = w1; x > 0; x -= step) NRM_SAMPLE(x, h1);
    for (double y = h1; y > 0; y -= step) NRM_SAMPLE(0.0, y);
#undef NRM_SAMPLE
    free(pos);
    return ns;
}

/* ------------------------------------------------------------------------ */
/* detail::blend_local (fieldest.hpp:75-97) + dq_blend (dualquat.hpp:133-162) */
/* ------------------------------------------------------------------------ */
#define ORC_MAX_SUPPORT 64

/* (d2, j) lexicographic order, as std::pair<double,int> operator< */
static int key_less(double da, int ja, double db, int jb) {
    return da < db || (!(db < da) && ja < jb);
}

/* Inserts key (d2, j) into the sorted kk-prefix kd/kj holding cnt keys:
 * partial_sort of the first kk (d2, j) keys, as a bounded insertion (keys
 * are distinct in j, so the prefix is unique). */
static void knn_insert(double d2, int j, double *kd, int *kj, int *cnt, int kk) {
    if (*cnt == kk && !key_less(d2, j, kd[kk - 1], kj[kk - 1])) return;
    int pos = *cnt < kk ? (*cnt)++ : kk - 1;
    while (pos > 0 && key_less(d2, j, kd[pos - 1], kj[pos - 1])) {
        kd[pos] = kd[pos - 1];
        kj[pos] = kj[pos - 1];
        --pos;
    }
    kd[pos] = d2;
    kj[pos] = j;
}

/* The blend of fieldest.hpp:86-96 over the kk selected keys (ascending). */
static int blend_keys(const double *locals, const double *probs, const double *kd, const int *kj, int kk,
                      double alpha, double *out5) {
    const double d2min = kd[0];
    double w[ORC_MAX_SUPPORT];
    for (int i = 0; i < kk; ++i) {
        const double p = probs[kj[i]];
        w[i] = exp(-alpha * (kd[i] - d2min)) * (p < 1e-6 ? 1e-6 : p); /* std::max(p, 1e-6) */
    }
    /* dq_blend */
    int ref = kk;
    double wsum = 0.0;
    for (int i = 0; i < kk; ++i) {
        if (w[i] > 0.0 && ref == kk) ref = i;
        wsum += w[i];
    }
    if (ref == kk) return -1;
    const double *qr = &locals[5 * kj[ref]];
    double sw = 0.0, sz = 0.0, sdx = 0.0, sdy = 0.0, ss = 0.0;
    for (int i = 0; i < kk; ++i) {
        const double wi = w[i];
        if (wi <= 0.0) continue;
        const double *q = &locals[5 * kj[i]];
        double qw = q[1], qz = q[2], qdx = q[3], qdy = q[4];
        if (qw * qr[1] + qz * qr[2] < 0.0) { qw = -qw; qz = -qz; qdx = -qdx; qdy = -qdy; }
        sw += wi * qw;
        sz += wi * qz;
        sdx += wi * qdx;
        sdy += wi * qdy;
        ss += wi * q[0];
    }
    dq2 mean = {sw / wsum, sz / wsum, sdx / wsum, sdy / wsum}, nq;
    if (!dq_normalized(mean, &nq)) return -1;
    out5[0] = ss / wsum;
    out5[1] = nq.w; out5[2] = nq.z; out5[3] = nq.dx; out5[4] = nq.dy;
    return 0;
}

int orc_blend_local(const double *locals, const double *apts, const double *probs,
                    const int32_t *active, int nactive, double qx, double qy, double alpha,
                    int support, double *out5) {
    if (nactive <= 0 || support <= 0) return -1;
    if (support > ORC_MAX_SUPPORT) support = ORC_MAX_SUPPORT;
    const int kk = support < nactive ? support : nactive;
    double kd[ORC_MAX_SUPPORT];
    int kj[ORC_MAX_SUPPORT];
    int cnt = 0;
    for (int a = 0; a < nactive; ++a) {
        const int j = active[a];
        const double ex = qx - apts[2 * j], ey = qy - apts[2 * j + 1];
        knn_insert(ex * ex + ey * ey, j, kd, kj, &cnt, kk);
    }
    return blend_keys(locals, probs, kd, kj, kk, alpha, out5);
}

/* node_uncertainty (fieldest.hpp:44-52) with bounded_exp (geometry.hpp:85-88). */
double orc_node_uncertainty(double qx, double qy, const double *pts, int m, double beta) {
    if (!(beta > 0.0) || m <= 0) return NAN;
    double best = DBL_MAX;
    for (int i = 0; i < m; ++i) {
        const double ex = qx - pts[2 * i], ey = qy - pts[2 * i + 1];
        const double d2 = ex * ex + ey * ey;
        best = d2 < best ? d2 : best; /* std::min(best, d2) == (d2 < best) ? d2 : best */
    }
    double arg = beta * best;
    if (55.0 < arg) arg = 55.0; /* std::min(arg, 55.0) */
    return exp(arg);
}

/* ------------------------------------------------------------------------ */
/* Dense grids                                                               */
/* ------------------------------------------------------------------------ */
void orc_node_field_grid(double x0, double y0, int w, int h, const double *anchors,
                         const double *warps, int n, double alpha, double *disp,
                         uint8_t *support) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int j = 0; j < h; ++j)
        for (int i = 0; i < w; ++i) {
            const double px = x0 + i, py = y0 + j;
            double wp[5], yv[2];
            const size_t o = (size_t)j * w + i;
            if (orc_pixel_warp(px, py, anchors, warps, n, alpha, wp)) {
                orc_warp_apply(wp, px, py, yv);
                disp[2 * o] = yv[0] - px;
                disp[2 * o + 1] = yv[1] - py;
                support[o] = 1;
            } else {
                disp[2 * o] = 0.0;
                disp[2 * o + 1] = 0.0;
                support[o] = 0;
            }
        }
}

int orc_emdq_field_grid(double x0, double y0, int w, int h, const double *apts,
                        const double *locals, const double *probs, const int32_t *active,
                        int nactive, double alpha, int support, double beta, double *disp,
                        double *unc, int row_begin, int row_end) {
    if (nactive <= 0) return -1;
    double *pts = (double *)malloc(sizeof(double) * 2 * (size_t)nactive);
    if (!pts) return -1;
    for (int a = 0; a < nactive; ++a) {
        pts[2 * a] = apts[2 * active[a]];
        pts[2 * a + 1] = apts[2 * active[a] + 1];
    }
    if (row_begin < 0) row_begin = 0;
    if (row_end > h || row_end < 0) row_end = h;
    int rc = 0;
    for (int j = row_begin; j < row_end; ++j)
        for (int i = 0; i < w; ++i) {
            const double px = x0 + i, py = y0 + j;
            const size_t o = (size_t)j * w + i;
            double wp[5], yv[2];
            if (orc_blend_local(locals, apts, probs, active, nactive, px, py, alpha, support, wp)) {
                rc = -1;
                continue;
            }
            orc_warp_apply(wp, px, py, yv);
            disp[2 * o] = yv[0] - px;
            disp[2 * o + 1] = yv[1] - py;
            unc[o] = orc_node_uncertainty(px, py, pts, nactive, beta);
        }
    free(pts);
    return rc;
}

/* The same dense EMDQ field with a uniform-grid kNN search (cells of about
 * four candidates, rings searched outward until the next ring cannot hold a
 * key below the current k-th) and OpenMP over rows. The kk selected keys,
 * their order and all arithmetic are those of orc_blend_local /
 * orc_node_uncertainty, so every output is bit-identical to the full scan
 * (tests/test_oracle_golden.py checks it); it only makes the canvas-scale
 * configurations (C2 / C4 / C5 full frames) checkable in seconds. The
 * uncertainty is bounded_exp(beta * d2) of the nearest key: the minimum over
 * all candidates of the same d2 expression node_uncertainty evaluates. */
int orc_emdq_field_grid_fast(double x0, double y0, int w, int h, const double *apts,
                             const double *locals, const double *probs, const int32_t *active,
                             int nactive, double alpha, int support, double beta, double *disp,
                             double *unc, int row_begin, int row_end) {
    if (nactive <= 0 || support <= 0) return -1;
    if (support > ORC_MAX_SUPPORT) support = ORC_MAX_SUPPORT;
    const int kk = support < nactive ? support : nactive;
    double bx0 = DBL_MAX, by0 = DBL_MAX, bx1 = -DBL_MAX, by1 = -DBL_MAX;
    for (int a = 0; a < nactive; ++a) {
        const double px = apts[2 * active[a]], py = apts[2 * active[a] + 1];
        bx0 = px < bx0 ? px : bx0;
        by0 = py < by0 ? py : by0;
        bx1 = px > bx1 ? px : bx1;
        by1 = py > by1 ? py : by1;
    }
    const double area = (bx1 - bx0 + 1.0) * (by1 - by0 + 1.0);
    double cs = sqrt(4.0 * area / nactive);
    if (!(cs >= 1.0)) cs = 1.0;
    int gw = (int)((bx1 - bx0) / cs) + 1, gh = (int)((by1 - by0) / cs) + 1;
    if (gw > 4096) gw = 4096;
    if (gh > 4096) gh = 4096;
    const double csx = (bx1 - bx0) / gw + 1e-9, csy = (by1 - by0) / gh + 1e-9;
    int *start = (int *)calloc((size_t)gw * gh + 1, sizeof(int));
    int *items = (int *)malloc(sizeof(int) * (size_t)nactive);
    int *fill = (int *)calloc((size_t)gw * gh, sizeof(int));
    if (!start || !items || !fill) { free(start); free(items); free(fill); return -1; }
#define ORC_CELL(px, py, cx, cy)                                        \
    do {                                                                \
        cx = (int)(((px) - bx0) / csx); cy = (int)(((py) - by0) / csy); \
        cx = cx < 0 ? 0 : (cx >= gw ? gw - 1 : cx);                     \
        cy = cy < 0 ? 0 : (cy >= gh ? gh - 1 : cy);                     \
    } while (0)
    for (int a = 0; a < nactive; ++a) {
        int cx, cy;
        ORC_CELL(apts[2 * active[a]], apts[2 * active[a] + 1], cx, cy);
        ++start[(size_t)cy * gw + cx + 1];
    }
    for (size_t c = 0; c < (size_t)gw * gh; ++c) start[c + 1] += start[c];
    for (int a = 0; a < nactive; ++a) {
        int cx, cy;
        ORC_CELL(apts[2 * active[a]], apts[2 * active[a] + 1], cx, cy);
        const size_t c = (size_t)cy * gw + cx;
        items[start[c] + fill[c]++] = active[a];
    }
    free(fill);
    if (row_begin < 0) row_begin = 0;
    if (row_end > h || row_end < 0) row_end = h;
    const double cmin = csx < csy ? csx : csy;
    int rc = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : rc)
    for (int j = row_begin; j < row_end; ++j) {
        for (int i = 0; i < w; ++i) {
            const double qx = x0 + i, qy = y0 + j;
            const size_t o = (size_t)j * w + i;
            double kd[ORC_MAX_SUPPORT];
            int kj[ORC_MAX_SUPPORT];
            int cnt = 0, cx, cy;
            ORC_CELL(qx, qy, cx, cy);
            /* distance from q to the boundary of its (clamped) cell block */
            const double ox = qx < bx0 ? bx0 - qx : (qx > bx1 ? qx - bx1 : 0.0);
            const double oy = qy < by0 ? by0 - qy : (qy > by1 ? qy - by1 : 0.0);
            const double outside2 = ox * ox + oy * oy; /* every candidate is at least this far (squared) */
            for (int r = 0;; ++r) {
                const int xa = cx - r, xb = cx + r, ya = cy - r, yb = cy + r;
                for (int yy = ya; yy <= yb; ++yy) {
                    if (yy < 0 || yy >= gh) continue;
                    const int step = (yy == ya || yy == yb) ? 1 : (xb - xa > 0 ? xb - xa : 1);
                    for (int xx = xa; xx <= xb; xx += step) {
                        if (xx < 0 || xx >= gw) continue;
                        const size_t c = (size_t)yy * gw + xx;
                        for (int t = start[c]; t < start[c + 1]; ++t) {
                            const int jj = items[t];
                            const double ex = qx - apts[2 * jj], ey = qy - apts[2 * jj + 1];
                            knn_insert(ex * ex + ey * ey, jj, kd, kj, &cnt, kk);
                        }
                    }
                }
                if (xa <= 0 && ya <= 0 && xb >= gw - 1 && yb >= gh - 1) break; /* every cell seen */
                if (cnt == kk) {
                    /* a candidate outside rings 0..r lies r full cells away
                     * along one axis, and never closer than the bbox on either:
                     * d2 >= ox^2 + oy^2 + (r cmin)^2 */
                    const double lim2 = outside2 + (r * cmin) * (r * cmin);
                    if (lim2 * (1.0 - 1e-9) > kd[kk - 1]) break;
                }
            }
            double wp[5], yv[2];
            if (blend_keys(locals, probs, kd, kj, kk, alpha, wp)) {
                rc = 1;
                continue;
            }
            orc_warp_apply(wp, qx, qy, yv);
            disp[2 * o] = yv[0] - qx;
            disp[2 * o + 1] = yv[1] - qy;
            double arg = beta * kd[0];
            if (55.0 < arg) arg = 55.0;
            unc[o] = exp(arg);
        }
    }
#undef ORC_CELL
    free(start);
    free(items);
    return rc ? -1 : 0;
}

/* Engine::blended_variance_at (slam.hpp:703-714) at every pixel (x0 + i,
 * y0 + j) of a grid: d2min over the node positions, then the
 * exp(-alpha (d2 - d2min))-weighted mean of the node variances (0 without
 * nodes). The reference's operation order. */
void orc_variance_field(double x0, double y0, int w, int h, const double *pos, const double *var, int n,
                        double alpha, double *out) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int j = 0; j < h; ++j)
        for (int i = 0; i < w; ++i) {
            const double px = x0 + i, py = y0 + j;
            double d2min = DBL_MAX;
            for (int k = 0; k < n; ++k) {
                const double dx = pos[2 * k] - px, dy = pos[2 * k + 1] - py;
                const double d2 = dx * dx + dy * dy;
                d2min = d2 < d2min ? d2 : d2min; /* std::min(d2min, d2) */
            }
            double wsum = 0.0, acc = 0.0;
            for (int k = 0; k < n; ++k) {
                const double dx = pos[2 * k] - px, dy = pos[2 * k + 1] - py;
                const double wk = exp(-alpha * ((dx * dx + dy * dy) - d2min));
                wsum += wk;
                acc += wk * var[k];
            }
            out[(size_t)j * w + i] = wsum > 0.0 ? acc / wsum : 0.0;
        }
}

/* ==========================================================================
 * Sparse front end (features.hpp). FP32 arithmetic in the
 * reference's order; this file is built with -ffp-contract=off, so every
 * float operation rounds separately, like the reference's SSE code.
 * ========================================================================== */

/* to_gray (image.hpp:63-75) */
void orc_to_gray(const uint8_t *im, int w, int h, int ch, float *out) {
    const size_t n = (size_t)w * (size_t)h;
    for (size_t i = 0; i < n; ++i) {
        if (ch == 1) {
            out[i] = im[i] * (1.f / 255.f);
        } else {
            const uint8_t *p = im + i * (size_t)ch;
            out[i] = (0.299f * p[0] + 0.587f * p[1] + 0.114f * p[2]) * (1.f / 255.f);
        }
    }
}

typedef struct orc_kp {
    double x, y, resp;
    int idx; /* raster order of detection (stable-sort tie-break) */
} orc_kp;

static int orc_kp_cmp(const void *pa, const void *pb) {
    const orc_kp *a = (const orc_kp *)pa, *b = (const orc_kp *)pb;
    /* features.hpp:186-191: response desc, y asc, x asc; stable */
    if (a->resp != b->resp) return a->resp > b->resp ? -1 : 1;
    if (a->y != b->y) return a->y < b->y ? -1 : 1;
    if (a->x != b->x) return a->x < b->x ? -1 : 1;
    return (a->idx > b->idx) - (a->idx < b->idx);
}

/* subpixel_offset (features.hpp:103-108) */
static double orc_subpixel_offset(float rm, float r0, float rp) {
    const double denom = (double)rm - 2.0 * r0 + rp;
    if (fabs(denom) < 1e-20) return 0.0;
    const double off = 0.5 * ((double)rm - rp) / denom;
    return off < -0.5 ? -0.5 : (off > 0.5 ? 0.5 : off);
}

/* corner_response (features.hpp:58-101) + detect_features (140-205) */
int orc_detect_features(const float *gray, int w, int h, int max_features, double quality,
                        int r, double *kp, float *desc) {
    const int margin = 8 + 2; /* kPatchRadius + 2 (features.hpp:54-55) */
    if (w < 2 * margin + 1 || h < 2 * margin + 1) return 0;
    const size_t n = (size_t)w * (size_t)h;
    float *ix = (float *)calloc(n, sizeof(float)), *iy = (float *)calloc(n, sizeof(float));
    float *resp = (float *)calloc(n, sizeof(float));
    if (!ix || !iy || !resp) {
        free(ix), free(iy), free(resp);
        return -1;
    }
#define G(x, y) gray[(size_t)(y) * w + (x)]
    for (int y = 1; y + 1 < h; ++y)
        for (int x = 1; x + 1 < w; ++x) {
            ix[(size_t)y * w + x] = (G(x + 1, y - 1) - G(x - 1, y - 1)) + 2.f * (G(x + 1, y) - G(x - 1, y)) +
                                    (G(x + 1, y + 1) - G(x - 1, y + 1));
            iy[(size_t)y * w + x] = (G(x - 1, y + 1) - G(x - 1, y - 1)) + 2.f * (G(x, y + 1) - G(x, y - 1)) +
                                    (G(x + 1, y + 1) - G(x + 1, y - 1));
        }
#undef G
    for (int y = 3; y < h - 3; ++y)
        for (int x = 3; x < w - 3; ++x) {
            float sxx = 0.f, syy = 0.f, sxy = 0.f;
            for (int dy = -2; dy <= 2; ++dy)
                for (int dx = -2; dx <= 2; ++dx) {
                    const float gx = ix[(size_t)(y + dy) * w + x + dx], gy = iy[(size_t)(y + dy) * w + x + dx];
                    sxx += gx * gx;
                    syy += gy * gy;
                    sxy += gx * gy;
                }
            const float tr = 0.5f * (sxx + syy);
            const float q = 0.25f * (sxx - syy) * (sxx - syy) + sxy * sxy;
            const float det = sqrtf(q > 0.f ? q : 0.f);
            resp[(size_t)y * w + x] = tr - det;
        }
    float max_resp = 0.f;
    for (size_t i = 0; i < n; ++i)
        if (resp[i] > max_resp) max_resp = resp[i];
    const float threshold = (float)quality * max_resp;
    int count = 0, cap = 1024;
    orc_kp *list = (orc_kp *)malloc((size_t)cap * sizeof(orc_kp));
    if (max_resp > 0.f && list) {
        for (int y = margin; y < h - margin; ++y)
            for (int x = margin; x < w - margin; ++x) {
                const float v = resp[(size_t)y * w + x];
                if (v <= threshold) continue;
                int is_max = 1;
                for (int dy = -r; dy <= r && is_max; ++dy)
                    for (int dx = -r; dx <= r; ++dx) {
                        if (dx == 0 && dy == 0) continue;
                        const float nb = resp[(size_t)(y + dy) * w + x + dx];
                        const int earlier = dy < 0 || (dy == 0 && dx < 0);
                        if (nb > v || (nb == v && earlier)) {
                            is_max = 0;
                            break;
                        }
                    }
                if (!is_max) continue;
                if (count == cap) {
                    cap *= 2;
                    orc_kp *nl = (orc_kp *)realloc(list, (size_t)cap * sizeof(orc_kp));
                    if (!nl) break;
                    list = nl;
                }
                orc_kp *k = &list[count];
                k->x = x + orc_subpixel_offset(resp[(size_t)y * w + x - 1], v, resp[(size_t)y * w + x + 1]);
                k->y = y + orc_subpixel_offset(resp[(size_t)(y - 1) * w + x], v, resp[(size_t)(y + 1) * w + x]);
                k->resp = v;
                k->idx = count++;
            }
    }
    free(ix), free(iy), free(resp);
    if (!list) return -1;
    qsort(list, (size_t)count, sizeof(orc_kp), orc_kp_cmp);
    if (count > max_features) count = max_features;
    /* fill_descriptor (features.hpp:110-134) */
    for (int i = 0; i < count; ++i) {
        kp[3 * i] = list[i].x;
        kp[3 * i + 1] = list[i].y;
        kp[3 * i + 2] = list[i].resp;
        const int cx = (int)lround(list[i].x), cy = (int)lround(list[i].y);
        float patch[64], mean = 0.f, norm2 = 0.f;
        for (int by = 0; by < 8; ++by)
            for (int bx = 0; bx < 8; ++bx) {
                const int px = cx - 8 + 2 * bx, py = cy - 8 + 2 * by;
                const float v = 0.25f * (gray[(size_t)py * w + px] + gray[(size_t)py * w + px + 1] +
                                         gray[(size_t)(py + 1) * w + px] + gray[(size_t)(py + 1) * w + px + 1]);
                patch[by * 8 + bx] = v;
                mean += v;
            }
        mean /= 64;
        for (int k = 0; k < 64; ++k) {
            patch[k] -= mean;
            norm2 += patch[k] * patch[k];
        }
        const float norm = sqrtf(norm2);
        for (int k = 0; k < 64; ++k) desc[64 * (size_t)i + k] = norm > 1e-12f ? patch[k] / norm : 0.f;
    }
    free(list);
    return count;
}

/* match_features (features.hpp:208-254) */
int orc_match_features(const double *kp_a, const float *desc_a, int na, const double *kp_b,
                       const float *desc_b, int nb, double ratio, double *out) {
    if (na == 0 || nb < 2) return 0;
    const double ratio_sq = ratio * ratio;
    int n = 0;
    for (int i = 0; i < na; ++i) {
        const float *da = desc_a + 64 * (size_t)i;
        float d1 = FLT_MAX, d2 = FLT_MAX;
        int j1 = -1;
        for (int j = 0; j < nb; ++j) {
            const float *db = desc_b + 64 * (size_t)j;
            float ssd = 0.f;
            for (int k = 0; k < 64; k += 8) {
                for (int u = 0; u < 8; ++u) {
                    const float d = da[k + u] - db[k + u];
                    ssd += d * d;
                }
                if (ssd > d2) break;
            }
            if (ssd < d1) {
                d2 = d1;
                d1 = ssd;
                j1 = j;
            } else if (ssd < d2) {
                d2 = ssd;
            }
        }
        if (j1 >= 0 && (double)d1 < ratio_sq * (double)d2) {
            double *o = out + 5 * (size_t)n++;
            o[0] = kp_a[3 * i];
            o[1] = kp_a[3 * i + 1];
            o[2] = kp_b[3 * j1];
            o[3] = kp_b[3 * j1 + 1];
            o[4] = 1.0 - sqrt((double)d1 / ((double)d2 > 1e-30 ? (double)d2 : 1e-30));
        }
    }
    return n;
}
