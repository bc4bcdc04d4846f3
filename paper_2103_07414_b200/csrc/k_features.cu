// k_features.cu -- the sparse front end before the EM:
// to_gray (image.hpp:63-75), detect_features (features.hpp:140-205) and
// match_features (features.hpp:208-254) on the GPU, bit-identical to the
// reference.
//
// The reference computes in FP32 (and FP64 for the subpixel offsets and the
// match scores) with a fixed operation order and no FMA contraction. Every
// kernel here spells its arithmetic with round-to-nearest intrinsics in that
// order, so the corner responses, the non-maximum-suppression decisions, the
// keypoint order, the descriptors and the ratio-test decisions are the
// reference's bit for bit.
//
//   k_gray        u8 -> FP32 gray
//   k_response    Sobel + 5 x 5 box-summed structure tensor -> min eigenvalue,
//                 fused through a shared-memory tile; per-CTA maximum
//   k_nms         threshold = quality * max, (2r+1)^2 suppression with the
//                 earliest-raster tie rule, FP64 subpixel offsets; appends
//                 candidates
//   k_select      one CTA: radix-select of the max_features-th response,
//                 then a shared-memory bitonic sort of the survivors by
//                 (response desc, y asc, x asc, raster index); the same CTA
//                 sorts all candidates in global memory in the pathological
//                 case of more than 2048 survivors tied at the cut
//   k_descriptors one thread per keypoint (the reference's sequential sums)
//   k_match       8 query descriptors x a 128-candidate chunk per CTA (staged
//                 in shared memory), 4 candidates per lane, full FP32 SSDs in
//                 the reference's order, (d1, j1, d2) merged exactly as the
//                 sequential scan would; k_match_compact merges the chunks,
//                 applies the FP64 ratio test and compacts in query order
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "nrm_common.cuh"
#include "nrm_internal.h"

namespace nrm {
namespace {

constexpr int kDim = 64;          // FrameFeatures::kDescriptorDim (features.hpp:42)
constexpr int kPatchRadius = 8;   // features.hpp:54
constexpr int kMargin = kPatchRadius + 2;
constexpr int kSum = 2;           // 5 x 5 box (features.hpp:79)
constexpr int RT_W = 32, RT_H = 16;  // response tile
constexpr int SEL_T = 1024, SEL_CAP = 2048;

__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }

// to_gray (image.hpp:63-75)
__global__ void k_gray(const uint8_t* __restrict__ im, int n, int ch, float* __restrict__ g) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    constexpr float k = 1.f / 255.f;
    if (ch == 1) {
        g[i] = fmul((float)im[i], k);
    } else {
        const uint8_t* p = im + (size_t)i * ch;
        const float s = fadd(fadd(fmul(0.299f, (float)p[0]), fmul(0.587f, (float)p[1])), fmul(0.114f, (float)p[2]));
        g[i] = fmul(s, k);
    }
}

// corner_response (features.hpp:58-101) for one RT_W x RT_H tile. The Sobel
// gradients are zero on the image border (the reference never writes them);
// the response is zero outside [3, w-3) x [3, h-3).
__global__ void __launch_bounds__(RT_W * RT_H) k_response(const float* __restrict__ g, int w, int h,
                                                          float* __restrict__ resp, unsigned* __restrict__ maxbits) {
    constexpr int GW = RT_W + 2 * (kSum + 1), GH = RT_H + 2 * (kSum + 1);  // gray with a 3-px halo
    constexpr int DW = RT_W + 2 * kSum, DH = RT_H + 2 * kSum;              // gradients with a 2-px halo
    __shared__ float sg[GH][GW];
    __shared__ float sx[DH][DW], sy[DH][DW];
    __shared__ unsigned smax;
    const int x0 = blockIdx.x * RT_W, y0 = blockIdx.y * RT_H;
    const int t = threadIdx.x;
    if (t == 0) smax = 0u;
    for (int e = t; e < GW * GH; e += RT_W * RT_H) {
        const int gx = x0 - (kSum + 1) + e % GW, gy = y0 - (kSum + 1) + e / GW;
        sg[e / GW][e % GW] = (gx >= 0 && gx < w && gy >= 0 && gy < h) ? g[(size_t)gy * w + gx] : 0.f;
    }
    __syncthreads();
    for (int e = t; e < DW * DH; e += RT_W * RT_H) {
        const int dx = e % DW, dy = e / DW;
        const int x = x0 - kSum + dx, y = y0 - kSum + dy;
        float ix = 0.f, iy = 0.f;
        if (x >= 1 && x + 1 < w && y >= 1 && y + 1 < h) {
            const int cx = dx + 1, cy = dy + 1;  // position in sg
            // ix = (g(x+1,y-1) - g(x-1,y-1)) + 2 (g(x+1,y) - g(x-1,y)) + (g(x+1,y+1) - g(x-1,y+1))
            ix = fadd(fadd(fsub(sg[cy - 1][cx + 1], sg[cy - 1][cx - 1]), fmul(2.f, fsub(sg[cy][cx + 1], sg[cy][cx - 1]))),
                      fsub(sg[cy + 1][cx + 1], sg[cy + 1][cx - 1]));
            // iy = (g(x-1,y+1) - g(x-1,y-1)) + 2 (g(x,y+1) - g(x,y-1)) + (g(x+1,y+1) - g(x+1,y-1))
            iy = fadd(fadd(fsub(sg[cy + 1][cx - 1], sg[cy - 1][cx - 1]), fmul(2.f, fsub(sg[cy + 1][cx], sg[cy - 1][cx]))),
                      fsub(sg[cy + 1][cx + 1], sg[cy - 1][cx + 1]));
        }
        sx[dy][dx] = ix;
        sy[dy][dx] = iy;
    }
    __syncthreads();
    const int lx = t % RT_W, ly = t / RT_W;
    const int x = x0 + lx, y = y0 + ly;
    float r = 0.f;
    if (y >= kSum + 1 && y < h - kSum - 1 && x >= kSum + 1 && x < w - kSum - 1) {
        float sxx = 0.f, syy = 0.f, sxy = 0.f;
        for (int dy = 0; dy <= 2 * kSum; ++dy)
#pragma unroll
            for (int dx = 0; dx <= 2 * kSum; ++dx) {
                const float gx = sx[ly + dy][lx + dx], gy = sy[ly + dy][lx + dx];
                sxx = fadd(sxx, fmul(gx, gx));
                syy = fadd(syy, fmul(gy, gy));
                sxy = fadd(sxy, fmul(gx, gy));
            }
        const float tr = fmul(0.5f, fadd(sxx, syy));
        const float dd = fsub(sxx, syy);
        const float det = __fsqrt_rn(fmaxf(0.f, fadd(fmul(fmul(0.25f, dd), dd), fmul(sxy, sxy))));
        r = fsub(tr, det);
    }
    if (x < w && y < h) resp[(size_t)y * w + x] = r;
    // maximum over the image (max_resp starts at 0: only positive values matter)
    if (r > 0.f) atomicMax(&smax, __float_as_uint(r));
    __syncthreads();
    if (t == 0 && smax) atomicMax(maxbits, smax);
}

// Candidate keypoint before sorting.
struct Cand {
    double x, y;   // subpixel position
    float resp;
    int idx;       // raster index (stable-sort tie-break)
};

// subpixel_offset (features.hpp:103-108), FP64 from FP32 samples
__device__ __forceinline__ double subpixel_offset(float rm, float r0, float rp) {
    const double denom = __dadd_rn(__dsub_rn((double)rm, __dmul_rn(2.0, (double)r0)), (double)rp);
    if (fabs(denom) < 1e-20) return 0.0;
    const double off = __ddiv_rn(__dmul_rn(0.5, __dsub_rn((double)rm, (double)rp)), denom);
    return fmin(fmax(off, -0.5), 0.5);
}

// Non-maximum suppression (features.hpp:153-182) on a 32 x 8 tile of
// responses staged in shared memory with an r-pixel halo (r <= kMargin).
constexpr int NMS_W = 32, NMS_H = 8, NMS_HALO = kMargin;
__global__ void __launch_bounds__(NMS_W * NMS_H) k_nms(const float* __restrict__ resp, int w, int h, int r,
                                                       float quality, const unsigned* __restrict__ maxbits,
                                                       Cand* __restrict__ out, unsigned* __restrict__ count,
                                                       unsigned cap) {
    constexpr int SW = NMS_W + 2 * NMS_HALO, SH = NMS_H + 2 * NMS_HALO;
    __shared__ float sr[SH][SW + 1];
    const int x0 = kMargin + blockIdx.x * NMS_W, y0 = kMargin + blockIdx.y * NMS_H;
    const int t = threadIdx.x;
    const int tw = NMS_W + 2 * r, th = NMS_H + 2 * r;  // staged window for this radius
    for (int e = t; e < tw * th; e += NMS_W * NMS_H) {
        const int sx = e % tw, sy = e / tw;
        const int gx = x0 - r + sx, gy = y0 - r + sy;
        sr[sy][sx] = (gx < w && gy < h) ? resp[(size_t)gy * w + gx] : 0.f;  // gx, gy >= 0 since r <= kMargin
    }
    __syncthreads();
    const int lx = t % NMS_W, ly = t / NMS_W;
    const int x = x0 + lx, y = y0 + ly;
    if (x >= w - kMargin || y >= h - kMargin) return;
    const float thr = fmul(quality, __uint_as_float(*maxbits));
    const float v = sr[ly + r][lx + r];
    if (!(v > thr)) return;
    for (int dy = -r; dy <= r; ++dy) {
        const float* row = &sr[ly + r + dy][lx + r];
        for (int dx = -r; dx <= r; ++dx) {
            if (dx == 0 && dy == 0) continue;
            const float n = row[dx];
            const bool earlier = dy < 0 || (dy == 0 && dx < 0);
            if (n > v || (n == v && earlier)) return;
        }
    }
    Cand c;
    c.x = __dadd_rn((double)x, subpixel_offset(resp[(size_t)y * w + x - 1], v, resp[(size_t)y * w + x + 1]));
    c.y = __dadd_rn((double)y, subpixel_offset(resp[(size_t)(y - 1) * w + x], v, resp[(size_t)(y + 1) * w + x]));
    c.resp = v;
    c.idx = y * w + x;
    const unsigned slot = atomicAdd(count, 1u);
    if (slot < cap) out[slot] = c;
}

// The reference's keypoint order (stable_sort by response desc, y asc, x asc
// over the raster-ordered list, features.hpp:186-191).
__device__ __forceinline__ bool cand_before(const Cand& a, const Cand& b) {
    if (a.resp != b.resp) return a.resp > b.resp;
    if (a.y != b.y) return a.y < b.y;
    if (a.x != b.x) return a.x < b.x;
    return a.idx < b.idx;
}

// In-place bitonic sort of n <= SEL_CAP candidates in shared memory (padded
// with sentinels that sort last).
__device__ void block_bitonic(Cand* s, int n) {
    int np = 1;
    while (np < n) np <<= 1;
    for (int i = n + threadIdx.x; i < np; i += blockDim.x) s[i] = Cand{0.0, 0.0, -1.f, 0x7fffffff};
    __syncthreads();
    for (int k = 2; k <= np; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < np; i += blockDim.x) {
                const int l = i ^ j;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    const Cand a = s[i], b = s[l];
                    if (up ? cand_before(b, a) : cand_before(a, b)) {
                        s[i] = b;
                        s[l] = a;
                    }
                }
            }
            __syncthreads();
        }
}

// Top-k selection + sort. status[0] = kept count; status[1] = 1 when more
// than SEL_CAP candidates tied at the cut and the CTA sorted all of them in
// global memory instead.
__global__ void __launch_bounds__(SEL_T) k_select(Cand* __restrict__ cand, const unsigned* __restrict__ count,
                                                  unsigned cap, int kmax, Cand* __restrict__ kept,
                                                  int* __restrict__ status) {
    extern __shared__ __align__(16) unsigned char sel_raw[];
    Cand* s = reinterpret_cast<Cand*>(sel_raw);  // SEL_CAP entries (dynamic shared memory)
    __shared__ unsigned hist[256];
    __shared__ unsigned sh_prefix, sh_need, sh_n;
    const int t = threadIdx.x;
    const int n = (int)min(*count, cap);
    if (n <= SEL_CAP) {
        for (int i = t; i < n; i += SEL_T) s[i] = cand[i];
        __syncthreads();
        block_bitonic(s, n);
        const int m = min(n, kmax);
        for (int i = t; i < m; i += SEL_T) kept[i] = s[i];
        if (t == 0) status[0] = m, status[1] = 0;
        return;
    }
    // radix select of the kmax-th largest response (positive floats order as
    // unsigned integers), 8 bits per pass from the top
    unsigned prefix = 0u, need = (unsigned)kmax;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = t; i < 256; i += SEL_T) hist[i] = 0u;
        __syncthreads();
        const unsigned hi_mask = shift == 24 ? 0u : (0xffffffffu << (shift + 8));
        for (int i = t; i < n; i += SEL_T) {
            const unsigned key = __float_as_uint(cand[i].resp);
            if ((key & hi_mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (t == 0) {
            unsigned acc = 0u;
            int b = 255;
            for (; b > 0; --b) {
                if (acc + hist[b] >= need) break;
                acc += hist[b];
            }
            sh_prefix = prefix | ((unsigned)b << shift);
            sh_need = need - acc;
        }
        __syncthreads();
        prefix = sh_prefix;
        need = sh_need;
        __syncthreads();
    }
    // survivors: response >= pivot (prefix is the pivot's bit pattern)
    if (t == 0) sh_n = 0u;
    __syncthreads();
    for (int i = t; i < n; i += SEL_T) {
        const Cand c = cand[i];
        if (__float_as_uint(c.resp) >= prefix) {
            const unsigned slot = atomicAdd(&sh_n, 1u);
            if (slot < SEL_CAP) s[slot] = c;
        }
    }
    __syncthreads();
    const int m = (int)sh_n;
    if (m > SEL_CAP) {
        // more than SEL_CAP tied at the cut (periodic textures): this CTA
        // sorts every candidate in global memory (padded to a power of two
        // with sentinels; cand has room for it)
        int np = 1;
        while (np < n) np <<= 1;
        for (int i = n + t; i < np; i += SEL_T) cand[i] = Cand{0.0, 0.0, -1.f, 0x7fffffff};
        __syncthreads();
        for (int k = 2; k <= np; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = t; i < np; i += SEL_T) {
                    const int l = i ^ j;
                    if (l > i) {
                        const bool up = (i & k) == 0;
                        const Cand a = cand[i], b = cand[l];
                        if (up ? cand_before(b, a) : cand_before(a, b)) {
                            cand[i] = b;
                            cand[l] = a;
                        }
                    }
                }
                __syncthreads();
            }
        const int kk = min(n, kmax);
        for (int i = t; i < kk; i += SEL_T) kept[i] = cand[i];
        if (t == 0) status[0] = kk, status[1] = 1;
        return;
    }
    block_bitonic(s, m);
    const int k = min(m, kmax);
    for (int i = t; i < k; i += SEL_T) kept[i] = s[i];
    if (t == 0) status[0] = k, status[1] = 0;
}

// Keypoints (x, y, response) and descriptors (fill_descriptor,
// features.hpp:110-134) of the kept candidates.
__global__ void k_descriptors(const float* __restrict__ g, int w, const Cand* __restrict__ kept,
                              const int* __restrict__ status, double* __restrict__ kp, float* __restrict__ desc) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= status[0]) return;
    const Cand c = kept[i];
    kp[3 * i] = c.x;
    kp[3 * i + 1] = c.y;
    kp[3 * i + 2] = (double)c.resp;
    const int cx = (int)llround(c.x), cy = (int)llround(c.y);
    float patch[kDim];
    float mean = 0.f;
#pragma unroll
    for (int by = 0; by < 8; ++by)
#pragma unroll
        for (int bx = 0; bx < 8; ++bx) {
            const int px = cx - kPatchRadius + 2 * bx, py = cy - kPatchRadius + 2 * by;
            const float* r0 = g + (size_t)py * w + px;
            const float* r1 = r0 + w;
            const float v = fmul(0.25f, fadd(fadd(fadd(r0[0], r0[1]), r1[0]), r1[1]));
            patch[by * 8 + bx] = v;
            mean = fadd(mean, v);
        }
    mean = __fdiv_rn(mean, (float)kDim);
    float norm2 = 0.f;
#pragma unroll
    for (int k = 0; k < kDim; ++k) {
        patch[k] = fsub(patch[k], mean);
        norm2 = fadd(norm2, fmul(patch[k], patch[k]));
    }
    const float norm = __fsqrt_rn(norm2);
    float* o = desc + (size_t)i * kDim;
    if (norm > 1e-12f) {
#pragma unroll
        for (int k = 0; k < kDim; ++k) o[k] = __fdiv_rn(patch[k], norm);
    } else {
#pragma unroll
        for (int k = 0; k < kDim; ++k) o[k] = 0.f;
    }
}

// Candidate descriptors transposed to [dim][nb] so a warp's lanes read
// consecutive candidates.
__global__ void k_transpose_desc(const float* __restrict__ d, int n, float* __restrict__ dt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * kDim) return;
    const int j = i / kDim, k = i % kDim;
    dt[(size_t)k * n + j] = d[i];
}

// match_features (features.hpp:208-254). CTA = 8 query descriptors a_i (one
// warp each) x one chunk of MCHUNK candidates staged in shared memory; each
// lane scans 4 candidates j ascending (4 independent FP32 SSD chains in the
// reference's order) with the reference's (d1, j1, d2) update. Summaries merge
// exactly -- the smallest index wins a tie for d1 and d2 is the second
// smallest of the multiset -- across lanes here and across chunks in
// k_match_compact, which is what the sequential scan computes. The reference's
// early exit (ssd > d2) never changes d1, j1 or d2, so full sums are used.
constexpr int MCHUNK = 128;
struct MatchPart {
    float d1, d2;
    int j1, pad;
};
__device__ __forceinline__ void merge_part(float& d1, int& j1, float& d2, float e1, int k1, float e2) {
    const float lo = fminf(d1, e1), hi = fmaxf(d1, e1);
    const int jn = (d1 < e1 || (d1 == e1 && (unsigned)j1 < (unsigned)k1)) ? j1 : k1;  // j = -1 only with FLT_MAX
    d2 = fminf(hi, fminf(d2, e2));
    d1 = lo;
    j1 = jn;
}
__global__ void __launch_bounds__(256) k_match(const float* __restrict__ da, int na, const float* __restrict__ dbt,
                                               int nb, MatchPart* __restrict__ part) {
    __shared__ float sb[kDim][MCHUNK];
    __shared__ float sa[8][kDim];
    const int t = threadIdx.x, lane = t & 31, wv = t >> 5;
    const int j0 = blockIdx.y * MCHUNK, nj = min(MCHUNK, nb - j0);
    for (int e = t; e < kDim * MCHUNK; e += 256) {
        const int k = e / MCHUNK, j = e % MCHUNK;
        sb[k][j] = j < nj ? dbt[(size_t)k * nb + j0 + j] : 0.f;
    }
    const int i = blockIdx.x * 8 + wv;
    for (int k = lane; k < kDim; k += 32) sa[wv][k] = i < na ? da[(size_t)i * kDim + k] : 0.f;
    __syncthreads();
    if (i >= na) return;
    float ssd[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
    for (int k = 0; k < kDim; ++k) {
        const float a = sa[wv][k];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float d = fsub(a, sb[k][lane + 32 * u]);
            ssd[u] = fadd(ssd[u], fmul(d, d));
        }
    }
    float d1 = FLT_MAX, d2 = FLT_MAX;
    int j1 = -1;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        if (lane + 32 * u >= nj) continue;
        if (ssd[u] < d1) {
            d2 = d1;
            d1 = ssd[u];
            j1 = j0 + lane + 32 * u;
        } else if (ssd[u] < d2) {
            d2 = ssd[u];
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float e1 = __shfl_xor_sync(0xffffffffu, d1, o), e2 = __shfl_xor_sync(0xffffffffu, d2, o);
        const int k1 = __shfl_xor_sync(0xffffffffu, j1, o);
        merge_part(d1, j1, d2, e1, k1, e2);
    }
    if (lane == 0) part[(size_t)i * gridDim.y + blockIdx.y] = MatchPart{d1, d2, j1, 0};
}

// Compaction of the matches in query order (one CTA, na <= 8192).
// Each query's chunk summaries are merged first, then the ratio test (FP64,
// features.hpp:241-245) decides.
__global__ void __launch_bounds__(1024) k_match_compact(const MatchPart* __restrict__ part, int nchunks, int na,
                                                        double ratio_sq, const double* __restrict__ kpa,
                                                        const double* __restrict__ kpb, double* __restrict__ out,
                                                        int* __restrict__ nout) {
    __shared__ int warp_tot[32];
    __shared__ int carry;
    const int t = threadIdx.x, lane = t & 31, wv = t >> 5;
    if (t == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < na; base += 1024) {
        const int i = base + t;
        int bj = -1;
        double sc = 0.0;
        if (i < na) {
            MatchPart p = part[(size_t)i * nchunks];
            for (int c = 1; c < nchunks; ++c) {
                const MatchPart q = part[(size_t)i * nchunks + c];
                merge_part(p.d1, p.j1, p.d2, q.d1, q.j1, q.d2);
            }
            if (p.j1 >= 0 && (double)p.d1 < __dmul_rn(ratio_sq, (double)p.d2)) {
                bj = p.j1;
                sc = __dsub_rn(1.0, __dsqrt_rn(__ddiv_rn((double)p.d1, fmax((double)p.d2, 1e-30))));
            }
        }
        const bool hit = bj >= 0;
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) warp_tot[wv] = __popc(m);
        __syncthreads();
        int before = carry;
        for (int w = 0; w < wv; ++w) before += warp_tot[w];
        if (hit) {
            const int o = before + __popc(m & ((1u << lane) - 1u));
            double* r = out + 5 * (size_t)o;
            r[0] = kpa[3 * i];
            r[1] = kpa[3 * i + 1];
            r[2] = kpb[3 * bj];
            r[3] = kpb[3 * bj + 1];
            r[4] = sc;
        }
        __syncthreads();
        if (t == 0) {
            int s = 0;
            for (int w = 0; w < 32; ++w) s += warp_tot[w];
            carry += s;
        }
        __syncthreads();
    }
    if (t == 0) *nout = carry;
}

}  // namespace

size_t features_scratch_bytes(int w, int h, int r, int kmax) {
    const size_t px = (size_t)w * h;
    const size_t cap = features_cand_cap(w, h, r);
    size_t np = 1;
    while (np < cap) np <<= 1;
    return px * 4 * 2 + np * sizeof(Cand) + (size_t)kmax * sizeof(Cand) + 256;
}

size_t features_cand_cap(int w, int h, int r) {
    // maxima are more than r apart (the tie rule keeps one per window)
    const size_t a = (size_t)(w + r) / (size_t)(r + 1) + 1, b = (size_t)(h + r) / (size_t)(r + 1) + 1;
    return std::min((size_t)w * h, a * b);
}

cudaError_t launch_detect_features(const FeatLaunch& F, cudaStream_t st, int64_t* launches) {
    const int w = F.w, h = F.h;
    const size_t px = (size_t)w * h;
    char* base = static_cast<char*>(F.scratch);
    float* gray = F.gray_in ? const_cast<float*>(F.gray_in) : reinterpret_cast<float*>(base);
    float* resp = reinterpret_cast<float*>(base + px * 4);
    const unsigned cap = (unsigned)features_cand_cap(w, h, F.nms_radius);
    unsigned npow = 1;
    while (npow < cap) npow <<= 1;
    Cand* cand = reinterpret_cast<Cand*>(base + px * 8);
    Cand* kept = cand + npow;
    unsigned* counters = reinterpret_cast<unsigned*>(kept + F.max_features);  // [0] max bits, [1] count
    int* status = F.status;
    cudaError_t e = cudaMemsetAsync(counters, 0, 2 * sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    if (!F.gray_in) {
        prof_mark("k_gray", st);
        k_gray<<<(unsigned)((px + 255) / 256), 256, 0, st>>>(F.image, (int)px, F.ch, gray);
        ++*launches;
    }
    prof_mark("k_response", st);
    k_response<<<dim3((w + RT_W - 1) / RT_W, (h + RT_H - 1) / RT_H), RT_W * RT_H, 0, st>>>(gray, w, h, resp,
                                                                                          counters);
    ++*launches;
    const int iw = w - 2 * kMargin, ih = h - 2 * kMargin;
    prof_mark("k_nms", st);
    k_nms<<<dim3((iw + NMS_W - 1) / NMS_W, (ih + NMS_H - 1) / NMS_H), NMS_W * NMS_H, 0, st>>>(
        resp, w, h, F.nms_radius, F.quality, counters, cand, counters + 1, cap);
    ++*launches;
    prof_mark("k_select", st);
    constexpr int sel_smem = SEL_CAP * (int)sizeof(Cand);
    e = cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, sel_smem);
    if (e != cudaSuccess) return e;
    k_select<<<1, SEL_T, sel_smem, st>>>(cand, counters + 1, cap, F.max_features, kept, status);
    ++*launches;
    prof_mark("k_descriptors", st);
    k_descriptors<<<(F.max_features + 127) / 128, 128, 0, st>>>(gray, w, kept, status, F.kp, F.desc);
    ++*launches;
    return cudaGetLastError();
}

size_t match_scratch_bytes(int na, int nb) {
    const size_t nchunks = (size_t)(nb + MCHUNK - 1) / MCHUNK;
    return (size_t)nb * kDim * 4 + 16 + (size_t)na * nchunks * sizeof(MatchPart) + 64;
}

cudaError_t launch_match_features(const MatchLaunch& M, cudaStream_t st, int64_t* launches) {
    char* base = static_cast<char*>(M.scratch);
    float* dbt = reinterpret_cast<float*>(base);
    MatchPart* part = reinterpret_cast<MatchPart*>(base + (((size_t)M.nb * kDim * 4 + 15) & ~size_t(15)));
    const int nchunks = (M.nb + MCHUNK - 1) / MCHUNK;
    prof_mark("k_transpose_desc", st);
    k_transpose_desc<<<(M.nb * kDim + 255) / 256, 256, 0, st>>>(M.desc_b, M.nb, dbt);
    ++*launches;
    prof_mark("k_match", st);
    k_match<<<dim3((M.na + 7) / 8, nchunks), 256, 0, st>>>(M.desc_a, M.na, dbt, M.nb, part);
    ++*launches;
    prof_mark("k_match_compact", st);
    k_match_compact<<<1, 1024, 0, st>>>(part, nchunks, M.na, M.ratio * M.ratio, M.kp_a, M.kp_b, M.out, M.nout);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace nrm
