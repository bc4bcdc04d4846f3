// k_variance.cu -- dense node-variance field: Engine::blended_variance_at
// (slam.hpp:703-714) at every pixel of a grid. The reference evaluates it
// per feature to seed new feature tracks; as a per-pixel map it is the
// "node variance" source of uncertainty for the uncertainty-weighted blend
// (nrm_blend_frame_weighted takes any map).
//
//   v(p) = sum_i w_i var_i / sum_i w_i,  w_i = exp(-alpha (|x_i - p|^2 - d2min(p)))
//
// One thread per pixel, the node positions / variances staged through shared
// memory in chunks; two passes (d2min, then the weighted sums). Distances are
// FP64 (at canvas-scale coordinates FP32 d^2 would lose the exponent);
// exp(-alpha (d2 - d2min)) = 2^n 2^f with n = rint, |f| <= 1/2 in FP64 and
// 2^f on MUFU.EX2 (relative error < 3e-7); sums in FP32. Every node
// contributes, as in the reference (no cutoff), so the cost is O(n) per
// pixel: meant for frame lattices (tens to hundreds of nodes).
#include <cfloat>

#include "nrm_common.cuh"
#include "nrm_internal.h"

namespace nrm {
namespace {

constexpr int VT = 256;       // threads (16 x 16 pixels)
constexpr int VCHUNK = 256;   // nodes staged per chunk

__global__ void __launch_bounds__(VT) k_variance_field(double x0, double y0, int w, int h,
                                                       const double* __restrict__ pos,
                                                       const double* __restrict__ var, int n, double alpha,
                                                       float* __restrict__ out) {
    __shared__ double2 sp[VCHUNK];
    __shared__ float sv[VCHUNK];
    const int i = blockIdx.x * 16 + (threadIdx.x & 15), j = blockIdx.y * 16 + (threadIdx.x >> 4);
    const bool valid = i < w && j < h;
    const double px = x0 + i, py = y0 + j;
    double d2min = DBL_MAX;
    for (int c0 = 0; c0 < n; c0 += VCHUNK) {  // pass 1: nearest node
        const int cn = min(VCHUNK, n - c0);
        __syncthreads();
        for (int k = threadIdx.x; k < cn; k += VT) sp[k] = make_double2(pos[2 * (c0 + k)], pos[2 * (c0 + k) + 1]);
        __syncthreads();
        for (int k = 0; k < cn; ++k) {
            const double dx = sp[k].x - px, dy = sp[k].y - py;
            d2min = fmin(d2min, fma(dx, dx, dy * dy));
        }
    }
    const double nal = -alpha * kLog2e;
    float wsum = 0.f, acc = 0.f;
    for (int c0 = 0; c0 < n; c0 += VCHUNK) {  // pass 2: weighted mean
        const int cn = min(VCHUNK, n - c0);
        __syncthreads();
        for (int k = threadIdx.x; k < cn; k += VT) {
            sp[k] = make_double2(pos[2 * (c0 + k)], pos[2 * (c0 + k) + 1]);
            sv[k] = (float)var[c0 + k];
        }
        __syncthreads();
        for (int k = 0; k < cn; ++k) {
            const double dx = sp[k].x - px, dy = sp[k].y - py;
            const double t = fmax(nal * (fma(dx, dx, dy * dy) - d2min), -200.0);
            const double nn = rint(t);
            const float wk = ex2_approx((float)(t - nn)) * exp2f((float)nn);
            wsum += wk;
            acc = fmaf(wk, sv[k], acc);
        }
    }
    if (valid) out[(size_t)j * w + i] = wsum > 0.f ? acc / wsum : 0.f;
}

}  // namespace

cudaError_t launch_variance_field(double x0, double y0, int w, int h, const double* pos, const double* var, int n,
                                  double alpha, float* out, cudaStream_t st, int64_t* launches) {
    if (w <= 0 || h <= 0) return cudaSuccess;
    prof_mark("k_variance_field", st);
    k_variance_field<<<dim3((w + 15) / 16, (h + 15) / 16), VT, 0, st>>>(x0, y0, w, h, pos, var, n, alpha, out);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace nrm
