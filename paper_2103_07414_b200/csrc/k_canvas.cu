// k_canvas.cu -- canvas-wide passes: render (mosaic.hpp:301-331), occupancy (mosaic.hpp:121-127) and the
// host-mirror transfers behind Canvas::color()/weight() (mosaic.hpp:111-120).
// All are HBM-bound streaming kernels: one pixel per thread, coalesced rows.
#include <cmath>

#include "nrm_common.cuh"
#include "nrm_internal.h"

namespace nrm {
namespace {

struct CanvasView {
    const float* r;
    const float* g;
    const float* b;
    const uint8_t* w;
    long long pitch;
    long long ox, oy;  // logical origin relative to physical (0,0)
    long long abs_y0;  // absolute reference row of logical row 0
    int band_rank, band_count;
};

__device__ __forceinline__ bool owns_row(const CanvasView& v, int y) {
    if (v.band_count <= 1) return true;
    const long long ay = v.abs_y0 + y;
    long long s = ay / kStripeRows;
    if (ay % kStripeRows != 0 && ay < 0) --s;
    long long m = s % v.band_count;
    if (m < 0) m += v.band_count;
    return m == v.band_rank;
}

CanvasView view_of(const nrm_canvas* cv) {
    CanvasView v;
    v.r = cv->r;
    v.g = cv->g;
    v.b = cv->b;
    v.w = cv->w;
    v.pitch = cv->cap_w;
    v.ox = cv->origin_x - cv->phys_x0;
    v.oy = cv->origin_y - cv->phys_y0;
    v.abs_y0 = cv->origin_y;
    v.band_rank = cv->band_rank;
    v.band_count = cv->band_count;
    return v;
}

__global__ void k_render(CanvasView v, int x0, int y0, int w, int h, uchar4* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= w) return;
    const int x = x0 + i, y = y0 + j;
    uchar4 px = make_uchar4(0, 0, 0, 0);
    if (owns_row(v, y)) {
        const long long idx = (v.oy + y) * v.pitch + (v.ox + x);
        if (v.w[idx] > 0) {
            auto q = [](float c) -> unsigned char {
                double d = (double)c;
                d = d < 0.0 ? 0.0 : (1.0 < d ? 1.0 : d);  // std::clamp(c, 0, 1)
                return (unsigned char)lround(d * 255.0);
            };
            px = make_uchar4(q(v.r[idx]), q(v.g[idx]), q(v.b[idx]), 255);
        }
    }
    out[(size_t)j * w + i] = px;
}

// count[0] = occupied pixels; bbox4 = {minx, miny, maxx, maxy} (atomics; init by caller).
// Grid-stride over rows, block-level reduction, five atomics per block.
__global__ void __launch_bounds__(256) k_occupied(CanvasView v, int w, int h, unsigned long long* count, int* bbox4) {
    __shared__ int red[5][8];
    long long cnt = 0;
    int mnx = 0x7fffffff, mny = 0x7fffffff, mxx = -1, mxy = -1;
    for (int j = blockIdx.x; j < h; j += gridDim.x) {
        if (!owns_row(v, j)) continue;
        const uint8_t* row = v.w + (v.oy + j) * v.pitch + v.ox;
        for (int i = threadIdx.x; i < w; i += blockDim.x) {
            if (row[i] > 0) {
                ++cnt;
                mnx = min(mnx, i);
                mxx = max(mxx, i);
                mny = min(mny, j);
                mxy = max(mxy, j);
            }
        }
    }
    int c32 = (int)cnt;
    for (int o = 16; o > 0; o >>= 1) {
        c32 += __shfl_xor_sync(0xffffffffu, c32, o);
        mnx = min(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
        mny = min(mny, __shfl_xor_sync(0xffffffffu, mny, o));
        mxx = max(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
        mxy = max(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
    }
    const int wid = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][wid] = c32; red[1][wid] = mnx; red[2][wid] = mny; red[3][wid] = mxx; red[4][wid] = mxy;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long tc = 0;
        for (int k = 0; k < 8; ++k) {
            tc += red[0][k];
            mnx = min(mnx, red[1][k]); mny = min(mny, red[2][k]);
            mxx = max(mxx, red[3][k]); mxy = max(mxy, red[4][k]);
        }
        if (tc) {
            atomicAdd(count, (unsigned long long)tc);
            atomicMin(&bbox4[0], mnx);
            atomicMin(&bbox4[1], mny);
            atomicMax(&bbox4[2], mxx);
            atomicMax(&bbox4[3], mxy);
        }
    }
}

__global__ void k_canvas_read(CanvasView v, int x0, int y0, int w, int h, double* __restrict__ rgb,
                              uint8_t* __restrict__ wout) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= w) return;
    const long long idx = (v.oy + y0 + j) * v.pitch + (v.ox + x0 + i);
    const size_t o = (size_t)j * w + i;
    if (rgb) {
        rgb[3 * o] = v.r[idx];
        rgb[3 * o + 1] = v.g[idx];
        rgb[3 * o + 2] = v.b[idx];
    }
    if (wout) wout[o] = v.w[idx];
}

__global__ void k_canvas_write(float* r, float* g, float* b, uint8_t* wp, long long pitch, long long ox,
                               long long oy, int x0, int y0, int w, int h,
                               const double* __restrict__ rgb, const uint8_t* __restrict__ win) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= w) return;
    const long long idx = (oy + y0 + j) * pitch + (ox + x0 + i);
    const size_t o = (size_t)j * w + i;
    if (rgb) {
        r[idx] = (float)rgb[3 * o];
        g[idx] = (float)rgb[3 * o + 1];
        b[idx] = (float)rgb[3 * o + 2];
    }
    if (win) wp[idx] = win[o];
}

// Canvas deformation (extension, north_star; no
// reference counterpart): new(p) = old(p + d(p)) over a region, bilinear in
// FP64 with the taps of sample_bilinear_rgb (image.hpp:78-92) restricted to
// occupied pixels (weights renormalised), weight from the nearest occupied
// tap; a source outside the canvas or with no occupied tap leaves the pixel
// unoccupied. d == 0 reproduces the canvas bit for bit. Output goes to
// scratch planes (sources may lie anywhere in the canvas).
__global__ void k_canvas_deform(CanvasView v, int W, int H, int x0, int y0, int w, int h,
                                const float2* __restrict__ disp, float* __restrict__ outr, float* __restrict__ outg,
                                float* __restrict__ outb, uint8_t* __restrict__ outw) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= w) return;
    const size_t o = (size_t)j * w + i;
    const float2 d = disp[o];
    const double sx = xadd((double)(x0 + i), (double)d.x), sy = xadd((double)(y0 + j), (double)d.y);
    float cr = 0.f, cg = 0.f, cb = 0.f;
    uint8_t cw = 0;
    if (sx >= 0.0 && sx <= W - 1.0 && sy >= 0.0 && sy <= H - 1.0) {
        int tx0 = (int)sx, ty0 = (int)sy;
        if (tx0 > W - 2) tx0 = W - 2 >= 0 ? W - 2 : 0;
        if (ty0 > H - 2) ty0 = H - 2 >= 0 ? H - 2 : 0;
        const double fx = xsub(sx, (double)tx0), fy = xsub(sy, (double)ty0);
        const int tx1 = tx0 + 1 < W - 1 ? tx0 + 1 : W - 1, ty1 = ty0 + 1 < H - 1 ? ty0 + 1 : H - 1;
        const double gx = xsub(1.0, fx), gy = xsub(1.0, fy);
        const int txs[4] = {tx0, tx1, tx0, tx1}, tys[4] = {ty0, ty0, ty1, ty1};
        const double bw[4] = {xmul(gx, gy), xmul(fx, gy), xmul(gx, fy), xmul(fx, fy)};
        double nr = 0.0, ng = 0.0, nb = 0.0, den = 0.0, best = -1.0;
        for (int t = 0; t < 4; ++t) {
            const long long idx = (v.oy + tys[t]) * v.pitch + (v.ox + txs[t]);
            const uint8_t wt = v.w[idx];
            if (wt == 0) continue;
            nr = xadd(nr, xmul(bw[t], (double)v.r[idx]));
            ng = xadd(ng, xmul(bw[t], (double)v.g[idx]));
            nb = xadd(nb, xmul(bw[t], (double)v.b[idx]));
            den = xadd(den, bw[t]);
            if (bw[t] > best) {
                best = bw[t];
                cw = wt;
            }
        }
        if (den > 0.0) {
            cr = (float)(nr / den);
            cg = (float)(ng / den);
            cb = (float)(nb / den);
        } else {
            cw = 0;
        }
    }
    outr[o] = cr;
    outg[o] = cg;
    outb[o] = cb;
    outw[o] = cw;
}

}  // namespace

cudaError_t launch_canvas_deform(const nrm_canvas* cv, int x, int y, int w, int h, const float2* disp, float* scratch,
                                 cudaStream_t st, int64_t* launches) {
    if (w <= 0 || h <= 0) return cudaSuccess;
    const size_t npx = (size_t)w * h;
    float* r = scratch;
    float* g = r + npx;
    float* b = g + npx;
    uint8_t* wt = reinterpret_cast<uint8_t*>(b + npx);
    prof_mark("k_canvas_deform", st);
    k_canvas_deform<<<dim3((w + 255) / 256, h), 256, 0, st>>>(view_of(cv), cv->width, cv->height, x, y, w, h, disp,
                                                              r, g, b, wt);
    ++*launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // scratch -> canvas planes
    const long long ox = cv->origin_x - cv->phys_x0, oy = cv->origin_y - cv->phys_y0;
    const size_t off = (size_t)(oy + y) * cv->cap_w + (size_t)(ox + x);
    float* planes[3] = {cv->r, cv->g, cv->b};
    const float* src[3] = {r, g, b};
    for (int k = 0; k < 3; ++k) {
        e = cudaMemcpy2DAsync(planes[k] + off, (size_t)cv->cap_w * sizeof(float), src[k], (size_t)w * sizeof(float),
                              (size_t)w * sizeof(float), (size_t)h, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return e;
    }
    return cudaMemcpy2DAsync(cv->w + off, (size_t)cv->cap_w, wt, (size_t)w, (size_t)w, (size_t)h,
                             cudaMemcpyDeviceToDevice, st);
}

cudaError_t launch_render(const nrm_canvas* cv, int x, int y, int w, int h, uint8_t* out,
                          cudaStream_t st, int64_t* launches) {
    if (w <= 0 || h <= 0) return cudaSuccess;
    prof_mark("k_render", st);
    k_render<<<dim3((w + 255) / 256, h), 256, 0, st>>>(view_of(cv), x, y, w, h, reinterpret_cast<uchar4*>(out));
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_occupied(const nrm_canvas* cv, unsigned long long* count, int* bbox4,
                            cudaStream_t st, int64_t* launches) {
    if (cv->width <= 0 || cv->height <= 0) return cudaSuccess;
    const int blocks = cv->height < 148 * 8 ? cv->height : 148 * 8;
    prof_mark("k_occupied", st);
    k_occupied<<<blocks, 256, 0, st>>>(view_of(cv), cv->width, cv->height, count, bbox4);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_canvas_read(const nrm_canvas* cv, int x, int y, int w, int h, double* rgb,
                               uint8_t* weight, cudaStream_t st, int64_t* launches) {
    if (w <= 0 || h <= 0) return cudaSuccess;
    prof_mark("k_canvas_read", st);
    k_canvas_read<<<dim3((w + 255) / 256, h), 256, 0, st>>>(view_of(cv), x, y, w, h, rgb, weight);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_canvas_write(nrm_canvas* cv, int x, int y, int w, int h, const double* rgb,
                                const uint8_t* weight, cudaStream_t st, int64_t* launches) {
    if (w <= 0 || h <= 0) return cudaSuccess;
    prof_mark("k_canvas_write", st);
    k_canvas_write<<<dim3((w + 255) / 256, h), 256, 0, st>>>(cv->r, cv->g, cv->b, cv->w, cv->cap_w,
                                                            cv->origin_x - cv->phys_x0,
                                                            cv->origin_y - cv->phys_y0, x, y, w, h, rgb,
                                                            weight);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace nrm
