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

}  // namespace

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
