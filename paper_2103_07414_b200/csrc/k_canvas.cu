// k_canvas.cu -- canvas-wide passes: render (mosaic.hpp:301-331), occupancy (mosaic.hpp:121-127) and the
// host-mirror transfers behind Canvas::color()/weight() (mosaic.hpp:111-120).
// All are HBM-bound streaming kernels: one pixel per thread, coalesced rows.
#include <cmath>
#include <utility>

#include "nrm_common.cuh"
#include "nrm_internal.h"
#include "frame_rgba.cuh"

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

// Rows are walked grid-stride over gridDim.y (<= 65535), so canvases of any
// height (up to the 2^30 rows ensure_contains allows) launch.
constexpr int kMaxGridY = 65535;
inline int grid_y(int h) { return h < kMaxGridY ? h : kMaxGridY; }

__global__ void k_render(CanvasView v, int x0, int y0, int w, int h, uchar4* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= w) return;
    for (int j = blockIdx.y; j < h; j += gridDim.y) {
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
    if (i >= w) return;
    for (int j = blockIdx.y; j < h; j += gridDim.y) {
        const long long idx = (v.oy + y0 + j) * v.pitch + (v.ox + x0 + i);
        const size_t o = (size_t)j * w + i;
        if (rgb) {
            rgb[3 * o] = v.r[idx];
            rgb[3 * o + 1] = v.g[idx];
            rgb[3 * o + 2] = v.b[idx];
        }
        if (wout) wout[o] = v.w[idx];
    }
}

__global__ void k_canvas_write(float* r, float* g, float* b, uint8_t* wp, long long pitch, long long ox,
                               long long oy, int x0, int y0, int w, int h,
                               const double* __restrict__ rgb, const uint8_t* __restrict__ win) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= w) return;
    for (int j = blockIdx.y; j < h; j += gridDim.y) {
        const long long idx = (oy + y0 + j) * pitch + (ox + x0 + i);
        const size_t o = (size_t)j * w + i;
        if (rgb) {
            r[idx] = (float)rgb[3 * o];
            g[idx] = (float)rgb[3 * o + 1];
            b[idx] = (float)rgb[3 * o + 2];
        }
        if (win) wp[idx] = win[o];
    }
}

// Halo rows for banded canvases: canvas rows rows[k] (logical
// canvas coordinates), all logical columns, packed as per-row SoA
// {R[w], G[w], B[w]} float32 followed by W[w] uint8 -> 13 w bytes per row.
// Rows start on 16-byte boundaries of the physical planes (origins and the
// pitch are multiples of 256 px), so one thread moves 4 pixels with float4 /
// uchar4 accesses.
__global__ void __launch_bounds__(256) k_rows_pack(CanvasView v, const int* __restrict__ rows, int nrows, int w,
                                                   unsigned char* __restrict__ buf) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;  // quad index in the row
    if (4 * q >= w) return;
    const size_t row_bytes = (size_t)13 * w;
    for (int k = blockIdx.y; k < nrows; k += gridDim.y) {
        const long long base = (v.oy + rows[k]) * v.pitch + v.ox + 4 * q;
        float* fr = reinterpret_cast<float*>(buf + (size_t)k * row_bytes);
        reinterpret_cast<float4*>(fr)[q] = *reinterpret_cast<const float4*>(v.r + base);
        reinterpret_cast<float4*>(fr + w)[q] = *reinterpret_cast<const float4*>(v.g + base);
        reinterpret_cast<float4*>(fr + 2 * w)[q] = *reinterpret_cast<const float4*>(v.b + base);
        reinterpret_cast<uchar4*>(fr + 3 * w)[q] = *reinterpret_cast<const uchar4*>(v.w + base);
    }
}

__global__ void __launch_bounds__(256) k_rows_unpack(float* r, float* g, float* b, uint8_t* wp, long long pitch,
                                                     long long ox, long long oy, const int* __restrict__ rows,
                                                     int nrows, int w, const unsigned char* __restrict__ buf) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (4 * q >= w) return;
    const size_t row_bytes = (size_t)13 * w;
    for (int k = blockIdx.y; k < nrows; k += gridDim.y) {
        const long long base = (oy + rows[k]) * pitch + ox + 4 * q;
        const float* fr = reinterpret_cast<const float*>(buf + (size_t)k * row_bytes);
        *reinterpret_cast<float4*>(r + base) = reinterpret_cast<const float4*>(fr)[q];
        *reinterpret_cast<float4*>(g + base) = reinterpret_cast<const float4*>(fr + w)[q];
        *reinterpret_cast<float4*>(b + base) = reinterpret_cast<const float4*>(fr + 2 * w)[q];
        *reinterpret_cast<uchar4*>(wp + base) = reinterpret_cast<const uchar4*>(fr + 3 * w)[q];
    }
}

// Canvas deformation (extension, north_star; no
// reference counterpart): new(p) = old(p + d(p)) over a region, bilinear in
// FP64 with the taps of sample_bilinear_rgb (image.hpp:78-92) restricted to
// occupied pixels (weights renormalised), weight from the nearest occupied
// tap; a source outside the canvas or with no occupied tap leaves the pixel
// unoccupied. d == 0 reproduces the canvas bit for bit.
struct Px {
    float r, g, b;
    uint8_t w;
};
// FP64 source position (the displacement is added exactly at any canvas
// coordinate), FP32 bilinear weights and blend with explicit round-to-nearest
// operations (no contraction), restated bit for bit by orc_canvas_deform.
__device__ __forceinline__ Px deform_sample(const CanvasView& v, int W, int H, int x, int y, float2 d) {
    const double sx = xadd((double)x, (double)d.x), sy = xadd((double)y, (double)d.y);
    Px o{0.f, 0.f, 0.f, 0};
    if (!(sx >= 0.0 && sx <= W - 1.0 && sy >= 0.0 && sy <= H - 1.0)) return o;
    int tx0 = (int)sx, ty0 = (int)sy;
    if (tx0 > W - 2) tx0 = W - 2 >= 0 ? W - 2 : 0;
    if (ty0 > H - 2) ty0 = H - 2 >= 0 ? H - 2 : 0;
    const float fx = (float)xsub(sx, (double)tx0), fy = (float)xsub(sy, (double)ty0);
    const int dx1 = tx0 + 1 < W - 1 ? 1 : W - 1 - tx0;  // tx1 - tx0 (0 on a one-pixel-wide canvas)
    const int dy1 = ty0 + 1 < H - 1 ? 1 : H - 1 - ty0;
    const float gx = __fsub_rn(1.f, fx), gy = __fsub_rn(1.f, fy);
    const float bw[4] = {__fmul_rn(gx, gy), __fmul_rn(fx, gy), __fmul_rn(gx, fy), __fmul_rn(fx, fy)};
    const int txs[4] = {tx0, tx0 + dx1, tx0, tx0 + dx1}, tys[4] = {ty0, ty0, ty0 + dy1, ty0 + dy1};
    uint8_t wt[4];
    float tr[4], tg[4], tb[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {  // all 16 tap loads at once (one latency round)
        const long long idx = (v.oy + tys[t]) * v.pitch + (v.ox + txs[t]);
        wt[t] = __ldg(v.w + idx);
        tr[t] = __ldg(v.r + idx);
        tg[t] = __ldg(v.g + idx);
        tb[t] = __ldg(v.b + idx);
    }
    float nr = 0.f, ng = 0.f, nb = 0.f, den = 0.f, best = -1.f;
    uint8_t cw = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        if (wt[t] == 0) continue;
        nr = __fadd_rn(nr, __fmul_rn(bw[t], tr[t]));
        ng = __fadd_rn(ng, __fmul_rn(bw[t], tg[t]));
        nb = __fadd_rn(nb, __fmul_rn(bw[t], tb[t]));
        den = __fadd_rn(den, bw[t]);
        if (bw[t] > best) {
            best = bw[t];
            cw = wt[t];
        }
    }
    if (den > 0.f) {
        const float inv = __frcp_rn(den);  // correctly rounded 1 / den, then three products
        o.r = __fmul_rn(nr, inv);
        o.g = __fmul_rn(ng, inv);
        o.b = __fmul_rn(nb, inv);
        o.w = cw;
    }
    return o;
}

// Ping-pong pass over the whole logical canvas: 4 pixels per thread (the
// logical origin and the pitch are multiples of 256 px, so every quad is a
// 16-byte aligned float4 / uchar4 of each plane). Pixels of the region are
// resampled, the others copied, into the alternate planes (whose role is
// swapped with the canvas planes afterwards). Rows this rank does not own
// are skipped. Quads entirely inside the region never read their own pixels:
// per pixel the pass moves the algorithmic 13 B read (taps, shared between
// neighbours through L1/L2) + 8 B displacement + 13 B written (ncu:
// dram__bytes = 34.0 B/px, profiles/r02_deform_ncu.txt).
#ifndef NRM_DEF_MINB
#define NRM_DEF_MINB 4  // 64 registers, 4 CTAs per SM: 2.26 ms vs 3.30 ms unconstrained (16384^2, tools/deform_probe.py)
#endif
__global__ void __launch_bounds__(256, NRM_DEF_MINB) k_canvas_deform_pp(
    CanvasView v, int W, int H, int rx0, int ry0, int rw, int rh, const float2* __restrict__ disp,
    float* __restrict__ outr, float* __restrict__ outg, float* __restrict__ outb, uint8_t* __restrict__ outw) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    const int x = 4 * q;
    if (x >= W) return;
    const bool cols_all = x >= rx0 && x + 3 < rx0 + rw, cols_any = x + 3 >= rx0 && x < rx0 + rw;
    for (int y = blockIdx.y; y < H; y += gridDim.y) {
        if (!owns_row(v, y)) continue;
        const long long base = (v.oy + y) * v.pitch + v.ox + x;
        const bool row_in = y >= ry0 && y < ry0 + rh;
        float4 cr, cg, cb;
        uchar4 cw;
        if (!(row_in && cols_all)) {  // some pixels of the quad are copied through
            cr = *reinterpret_cast<const float4*>(v.r + base);
            cg = *reinterpret_cast<const float4*>(v.g + base);
            cb = *reinterpret_cast<const float4*>(v.b + base);
            cw = *reinterpret_cast<const uchar4*>(v.w + base);
        }
        if (row_in && cols_any) {
            const size_t o = (size_t)(y - ry0) * rw + (x - rx0);
            float2 dq[4];
            if (cols_all && (o & 1) == 0) {  // two 16-byte loads for the quad's displacements
                const float4 a = __ldg(reinterpret_cast<const float4*>(disp + o));
                const float4 b = __ldg(reinterpret_cast<const float4*>(disp + o) + 1);
                dq[0] = make_float2(a.x, a.y);
                dq[1] = make_float2(a.z, a.w);
                dq[2] = make_float2(b.x, b.y);
                dq[3] = make_float2(b.z, b.w);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int xi = x + k;
                    dq[k] = (xi >= rx0 && xi < rx0 + rw) ? __ldg(disp + o + k) : make_float2(0.f, 0.f);
                }
            }
            float* pr = &cr.x;
            float* pg = &cg.x;
            float* pb = &cb.x;
            unsigned char* pw = &cw.x;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int xi = x + k;
                if (xi < rx0 || xi >= rx0 + rw) continue;
                const Px px = deform_sample(v, W, H, xi, y, dq[k]);
                pr[k] = px.r;
                pg[k] = px.g;
                pb[k] = px.b;
                pw[k] = px.w;
            }
        }
        *reinterpret_cast<float4*>(outr + base) = cr;
        *reinterpret_cast<float4*>(outg + base) = cg;
        *reinterpret_cast<float4*>(outb + base) = cb;
        *reinterpret_cast<uchar4*>(outw + base) = cw;
    }
}

// Small regions: resample into region-sized scratch planes, then copy the
// owned rows back (k_deform_commit) -- no pass over the rest of the canvas.
__global__ void k_canvas_deform_region(CanvasView v, int W, int H, int x0, int y0, int w, int h,
                                       const float2* __restrict__ disp, float* __restrict__ outr,
                                       float* __restrict__ outg, float* __restrict__ outb,
                                       uint8_t* __restrict__ outw) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= w) return;
    for (int j = blockIdx.y; j < h; j += gridDim.y) {
        if (!owns_row(v, y0 + j)) continue;
        const size_t o = (size_t)j * w + i;
        const Px p = deform_sample(v, W, H, x0 + i, y0 + j, disp[o]);
        outr[o] = p.r;
        outg[o] = p.g;
        outb[o] = p.b;
        outw[o] = p.w;
    }
}

__global__ void k_deform_commit(CanvasView v, float* r, float* g, float* b, uint8_t* wp, int x0, int y0, int w,
                                int h, const float* __restrict__ sr, const float* __restrict__ sg,
                                const float* __restrict__ sb, const uint8_t* __restrict__ sw) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= w) return;
    for (int j = blockIdx.y; j < h; j += gridDim.y) {
        if (!owns_row(v, y0 + j)) continue;
        const long long idx = (v.oy + y0 + j) * v.pitch + (v.ox + x0 + i);
        const size_t o = (size_t)j * w + i;
        r[idx] = sr[o];
        g[idx] = sg[o];
        b[idx] = sb[o];
        wp[idx] = sw[o];
    }
}

}  // namespace

__global__ void __launch_bounds__(RGBA_THREADS) k_frame_rgba(FrameSet fs, int fw, int fh, int fch,
                                                             uint8_t* __restrict__ out, size_t pitch,
                                                             size_t slot_bytes) {
    const int fr = blockIdx.y;
    const uint8_t* base = fs.f[0];  // a select, not a dynamic index (that would copy the parameters to local memory)
#pragma unroll
    for (int k = 1; k < kFrameSlots; ++k)
        if (fr == k) base = fs.f[k];
    rgba_convert(base, out + slot_bytes * fr, fw, fh, fch, pitch, blockIdx.x, gridDim.x);
}

cudaError_t launch_frame_rgba(const FrameSet& fs, int nf, int fw, int fh, int fch, uint8_t* out, size_t pitch,
                              size_t slot_bytes, cudaStream_t st, int64_t* launches) {
    if (nf <= 0 || nf > kFrameSlots) return cudaErrorInvalidValue;
    prof_mark("k_frame_rgba", st);
    const long long total = (long long)((fw + 3) / 4) * fh;
    const int blocks = (int)std::max(1LL, std::min((total + RGBA_THREADS * RGBA_GROUPS - 1) / (RGBA_THREADS * RGBA_GROUPS),
                                                   (long long)148 * 8));
    k_frame_rgba<<<dim3(blocks, nf), RGBA_THREADS, 0, st>>>(fs, fw, fh, fch, out, pitch, slot_bytes);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t canvas_alt_planes(nrm_canvas* cv, cudaStream_t st) {
    if (cv->ar) return cudaSuccess;
    const size_t npx = (size_t)cv->cap_w * (size_t)cv->cap_h;
    cudaError_t e = cudaMalloc(&cv->ar, npx * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&cv->ag, npx * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&cv->ab, npx * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&cv->aw, npx);
    // pixels outside the logical window must read as empty after a swap
    // (ensure_contains inside the reservation relies on it)
    if (e == cudaSuccess) e = cudaMemsetAsync(cv->ar, 0, npx * sizeof(float), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(cv->ag, 0, npx * sizeof(float), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(cv->ab, 0, npx * sizeof(float), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(cv->aw, 0, npx, st);
    if (e != cudaSuccess) {
        cudaFree(cv->ar);
        cudaFree(cv->ag);
        cudaFree(cv->ab);
        cudaFree(cv->aw);
        cv->ar = cv->ag = cv->ab = nullptr;
        cv->aw = nullptr;
    }
    return e;
}

bool deform_uses_ping_pong(const nrm_canvas* cv, int w, int h) {
    // a region of a quarter of the canvas or more: one pass over the canvas
    // (13 B read + 13 B written per pixel) beats scratch + copy-back (which
    // moves the region twice)
    return 4 * (double)w * (double)h >= (double)cv->width * (double)cv->height;
}

cudaError_t launch_canvas_deform(nrm_canvas* cv, int x, int y, int w, int h, const float2* disp, float* scratch,
                                 cudaStream_t st, int64_t* launches) {
    if (w <= 0 || h <= 0) return cudaSuccess;
    const CanvasView v = view_of(cv);
    if (deform_uses_ping_pong(cv, w, h)) {
        cudaError_t e = canvas_alt_planes(cv, st);
        if (e != cudaSuccess) return e;
        const int quads = cv->width / 4;
        prof_mark("k_canvas_deform", st);
        k_canvas_deform_pp<<<dim3((quads + 255) / 256, grid_y(cv->height)), 256, 0, st>>>(
            v, cv->width, cv->height, x, y, w, h, disp, cv->ar, cv->ag, cv->ab, cv->aw);
        ++*launches;
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        std::swap(cv->r, cv->ar);
        std::swap(cv->g, cv->ag);
        std::swap(cv->b, cv->ab);
        std::swap(cv->w, cv->aw);
        return cudaSuccess;
    }
    const size_t npx = (size_t)w * h;
    float* r = scratch;
    float* g = r + npx;
    float* b = g + npx;
    uint8_t* wt = reinterpret_cast<uint8_t*>(b + npx);
    prof_mark("k_canvas_deform", st);
    k_canvas_deform_region<<<dim3((w + 255) / 256, grid_y(h)), 256, 0, st>>>(v, cv->width, cv->height, x, y, w, h,
                                                                           disp, r, g, b, wt);
    ++*launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    prof_mark("k_deform_commit", st);
    k_deform_commit<<<dim3((w + 255) / 256, grid_y(h)), 256, 0, st>>>(v, cv->r, cv->g, cv->b, cv->w, x, y, w, h, r, g,
                                                                    b, wt);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_rows_pack(const nrm_canvas* cv, const int* d_rows, int nrows, void* d_buf, cudaStream_t st,
                             int64_t* launches) {
    if (nrows <= 0 || cv->width <= 0) return cudaSuccess;
    const int quads = cv->width / 4;
    prof_mark("k_rows_pack", st);
    k_rows_pack<<<dim3((quads + 255) / 256, grid_y(nrows)), 256, 0, st>>>(view_of(cv), d_rows, nrows, cv->width,
                                                                          static_cast<unsigned char*>(d_buf));
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_rows_unpack(nrm_canvas* cv, const int* d_rows, int nrows, const void* d_buf, cudaStream_t st,
                               int64_t* launches) {
    if (nrows <= 0 || cv->width <= 0) return cudaSuccess;
    const int quads = cv->width / 4;
    prof_mark("k_rows_unpack", st);
    k_rows_unpack<<<dim3((quads + 255) / 256, grid_y(nrows)), 256, 0, st>>>(
        cv->r, cv->g, cv->b, cv->w, cv->cap_w, cv->origin_x - cv->phys_x0, cv->origin_y - cv->phys_y0, d_rows, nrows,
        cv->width, static_cast<const unsigned char*>(d_buf));
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_render(const nrm_canvas* cv, int x, int y, int w, int h, uint8_t* out,
                          cudaStream_t st, int64_t* launches) {
    if (w <= 0 || h <= 0) return cudaSuccess;
    prof_mark("k_render", st);
    k_render<<<dim3((w + 255) / 256, grid_y(h)), 256, 0, st>>>(view_of(cv), x, y, w, h, reinterpret_cast<uchar4*>(out));
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
    k_canvas_read<<<dim3((w + 255) / 256, grid_y(h)), 256, 0, st>>>(view_of(cv), x, y, w, h, rgb, weight);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_canvas_write(nrm_canvas* cv, int x, int y, int w, int h, const double* rgb,
                                const uint8_t* weight, cudaStream_t st, int64_t* launches) {
    if (w <= 0 || h <= 0) return cudaSuccess;
    prof_mark("k_canvas_write", st);
    k_canvas_write<<<dim3((w + 255) / 256, grid_y(h)), 256, 0, st>>>(cv->r, cv->g, cv->b, cv->w, cv->cap_w,
                                                                    cv->origin_x - cv->phys_x0,
                                                                    cv->origin_y - cv->phys_y0, x, y, w, h, rgb,
                                                                    weight);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace nrm
