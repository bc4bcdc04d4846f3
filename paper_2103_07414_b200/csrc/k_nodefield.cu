// k_nodefield.cu -- K1 (fused node field + mosaic update, blend_frame
// mosaic.hpp:196-296) and K2 (dense node field, pixel_warp mosaic.hpp:22-51
// at every grid pixel), plus the exact-tier exception pass, the batched
// pixel_warp and invert_frame_boundary (mosaic.hpp:58-96).
//
// K1/K2 design:
//   CTA = one 64 x 32 pixel tile (256 threads, 8 rows per thread).
//   Prologue: (K1) cp.async the tile's canvas R/G/B/W rows into shared memory
//   so the read-modify-write latency overlaps the compute; (FP64) cull nodes
//   against the tile into an ordered list, classifying each as "inner"
//   (weight > 1e-6 at every tile pixel), "ring" (the 1e-6 cutoff crosses the
//   tile) or out; pick a per-tile output origin; conjugate every listed warp
//   into tile-local coordinates (T(-P) q T(o)); build separable Gaussian
//   tables ex[k][col], ey[k][row] (exp(-a(dx^2+dy^2)) = exp(-a dx^2)
//   exp(-a dy^2), MUFU.EX2).
//   Main loop (FP32): per (pixel, node) one FMUL for the weight and six FFMA
//   accumulations; ring nodes add the cutoff test.
//   Epilogue: normalise, apply, FP64 recombination with the tile origin,
//   frame-bounds test, FP32 bilinear sample of the raw frame, capped running
//   average from the staged canvas values.
//   Pixels whose discrete decisions are within rounding of a threshold (ring
//   weight ~1e-6, frame edge within 4e-3 px) or tiles whose warps are not in
//   one hemisphere go to an exception queue that the exact FP64 pass
//   (xpixel_warp, the reference's operation order and libm) resolves. That
//   pass also finalises BlendStats and resets the per-context counters.
#include <cmath>
#include <vector>

#include "nrm_common.cuh"
#include "nrm_internal.h"
#include "frame_rgba.cuh"

namespace nrm {
namespace {

#ifndef NRM_K1_CHUNK
#define NRM_K1_CHUNK 64   // nodes per table chunk (multiple of 8)
#endif
#ifndef NRM_K1_MINB
#define NRM_K1_MINB 4     // K1: resident CTAs per SM (64 registers)
#endif
#ifndef NRM_K2_MINB
#define NRM_K2_MINB 2     // K2: resident CTAs per SM (128 registers: 6.08 ms vs 6.38 at 3 CTAs, 16384^2 C4 field)
#endif
// Planning tiles are 64 x 32 px. A K1 CTA takes one 32 x 32 half (one m16
// tile per warp, 64 registers, 4 CTAs/SM); a K2 CTA takes the whole tile (two
// m16 tiles per warp, 128 registers, 2 CTAs/SM), which pays off there because
// its canvas-wide lattices list ~80 nodes per tile.
constexpr int TW = 64, TH = 32, HW = 32, NT = 256, CHUNK = NRM_K1_CHUNK;
template <int MODE> struct K1Shape {
    static constexpr int MT = MODE == 1 ? 2 : 1;  // m16 tiles per warp
    static constexpr int CW = 32 * MT;            // CTA columns
    static constexpr int NH = TW / CW;            // CTAs per planning tile
    static constexpr int MINB = MODE == 1 ? NRM_K2_MINB : NRM_K1_MINB;
};
static_assert(CHUNK % 8 == 0 && CHUNK <= 64, "k-steps of 8 nodes; one table thread per node");
constexpr int KP = CHUNK + 4;  // [col][node] table pitch: conflict-free ldmatrix rows
constexpr int EYP = 40;        // [node][row] table pitch: conflict-free B-fragment reads
constexpr int NF_CAP = 512;           // listed nodes per tile plan (more: the tile goes to the exact pass)
// 8,192 tile plans (200 MB) per launch chunk: a 4K frame in one chunk (C4
// 680 -> 659 us against 2,048) and a 16384^2 canvas field in 16 (7.0 -> 6.2 ms)
#ifndef NRM_NF_CHUNK_TILES
#define NRM_NF_CHUNK_TILES 8192
#endif
constexpr int NF_CHUNK_TILES = NRM_NF_CHUNK_TILES;  // tile plans resident per launch chunk
constexpr int NF_PLAN_WARPS = 8;      // planning warps (tiles) per CTA
constexpr int NF_GROUP_TILES = 64;    // prefilter node lists per 64 tile columns (4096 px)
constexpr int EXC_THREADS = 128;
#ifndef NRM_EXC_BLOCKS
#define NRM_EXC_BLOCKS 148
#endif
#ifndef NRM_EXC_KC
#define NRM_EXC_KC 4
#endif
constexpr int EXC_BLOCKS = NRM_EXC_BLOCKS;  // exception-pass CTAs (one warp per queued pixel, grid-stride)
constexpr float kCutHi = (float)(1e-6 * (1.0 + 4e-6));
constexpr float kCutLo = (float)(1e-6 * (1.0 - 4e-6));
// Fast-tier accuracy. Its position error follows
//   err <= 5e-5 px + kLeverErr * S * |P|,
// S = max |s_i - s0| over the tile's listed warps, |P| = the tile's output
// coordinate magnitude: the blend's scale and translation channels carry
// first-order terms of size S |P| that cancel in exact arithmetic, and the
// FP32 weights / TF32 products resolve them to ~1e-6 relative
// (tools/precision_probe.py: 7.5e-7 typical, 9.3e-7 worst over i.i.d. random
// scales). Tiles with S |P| > kScaleLever go to the exact tier, so the fast
// tier stays within 5e-5 + 1.5e-6 * 640 ~= 1e-3 px, and the frame-bounds
// margin is twice that.
constexpr double kScaleLever = 640.0;  // px
constexpr double kBoundMargin = 2e-3;  // px
constexpr unsigned kRingBit = 0x80000000u;

// Per-tile plan written by k_nf_plan (one warp per tile), read by k_node_field.
enum NfStatus : int { NF_OK = 0, NF_EXACT = 1, NF_EMPTY = 2, NF_OUTSIDE = 3 };
struct __align__(16) NfHdr {
    double P[2], Y0[2], e0[2], s0;  // output origin / reference scale (FP64)
    int count, status, ninner, pad1;  // listed nodes; inner ones come first
};
struct __align__(16) NfEntry {
    float4 q;      // warp conjugated to the tile origin (T(-P) q T(o))
    double2 a;     // anchor (absolute, FP64) for the separable tables
    float d;       // scale - s0
    unsigned idx;  // node index | kRingBit
    unsigned pad[2];
};
struct __align__(16) NfPlan {
    NfHdr h;
    NfEntry e[NF_CAP];
};

// Per-chunk tables. The Gaussian factorises, w = ex[col] * ey[row]; the
// column factor is the MMA's A operand, split into TF32 hi + lo.
template <int CW>
struct Smem {
    float exh[CW][KP], exl[CW][KP];  // column factor [col][node], hi / lo
    float ey[CHUNK][EYP];            // row factor [node][row]
    float4 qt[CHUNK][2];             // B columns per inner node: qw, qz, qdx, qdy, ds, 1, 0, 0
    NfEntry e[CHUNK];
};

// K1 only: the tile's canvas values, staged with cp.async at kernel entry.
struct CanvasTile {
    float r[TH][HW], g[TH][HW], b[TH][HW];  // one 32 x 32 TMA box each (128-byte aligned)
    uint8_t w[TH][HW];
    unsigned long long bar;  // TMA completion
};
// CanvasTile's offset in the dynamic shared memory (TMA destinations: 128 B)
template <int CW>
__host__ __device__ constexpr size_t canvas_tile_offset() {
    return (sizeof(Smem<CW>) + 127) & ~size_t(127);
}


// One frame of a batched blend (frames with pairwise disjoint footprints).
struct NfBatchFrame {
    NodeFieldLaunch L;  // the frame's launch, with its own queue / counters / stats
    int ti0, tj0, tj1, s1, ntx, rows;
    int plan_off, cta_off;  // first plan / first K1 CTA of this frame
};

__host__ __device__ __forceinline__ int tile_row_of(int by, int tile_j0, int s1, int band_count) {
    if (band_count <= 1) return tile_j0 + by;
    const int s = s1 + (by >> 1) * band_count;
    return 2 * s + (by & 1);
}

// Marks a deferred pixel whose queue slot overflowed: the blend's weight
// byte gets bit 7 (weights never exceed kWeightCap = 30), the node field's
// displacement becomes NaN (or its support byte 0xFF without a displacement
// output). K1 has not written the pixel; the exact pass finds the marks by a
// scan of the launch window and resolves them like queued pixels.
constexpr uint8_t kSpillBit = 0x80;
template <int MODE>
__device__ __forceinline__ void spill_mark(const NodeFieldLaunch& L, int i, int j) {
    if (MODE == 1) {
        const size_t o = (size_t)(j - L.grid.j0) * (L.grid.i1 - L.grid.i0 + 1) + (i - L.grid.i0);
        if (L.disp)
            L.disp[o] = make_float2(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
        else if (L.support)
            L.support[o] = 0xFF;
    } else {
        const long long idx = (long long)(j - L.phys_y0) * L.pitch + (i - L.phys_x0);
        L.W[idx] = (uint8_t)(L.W[idx] | kSpillBit);
    }
}

template <int MODE>
__device__ __forceinline__ void defer_pixel(const NodeFieldLaunch& L, bool pred, int i, int j) {
    if (queue_push(pred, i, j, L.exc, L.exc_count, L.exc_cap)) spill_mark<MODE>(L, i, j);
}

// Pushes every valid pixel of the tile to the exception queue.
template <int MODE>
__device__ void tile_to_exceptions(const NodeFieldLaunch& L, int ci0, int ci1, int cj0, int cj1) {
    const int w = ci1 - ci0 + 1, h = cj1 - cj0 + 1;
    const int total = w * h;
    for (int base = 0; base < total; base += NT) {
        const int e = base + threadIdx.x;
        const bool v = e < total;
        defer_pixel<MODE>(L, v, ci0 + (v ? e % w : 0), cj0 + (v ? e / w : 0));
    }
}

// ---------------------------------------------------------------------------
// k_nf_plan: one warp per tile. Ordered FP64 cull of the nodes against the
// tile (inner: weight > 1e-6 at every tile pixel; ring: the cutoff crosses
// the tile), hemisphere arc of the listed warps and the reference node
// nearest the tile centre, the tile's output origin, and the listed warps
// conjugated into tile-local coordinates.
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// k_nf_prefilter: one CTA; the index-ordered list of nodes that can reach
// (weight > 1e-6, same conservative test as k_nf_plan) any pixel of the
// launch chunk's rectangle [xlo, xhi] x [ylo, yhi]. Planning and the exact
// pass then scan this list instead of all n nodes (canvas-wide lattices:
// thousands of nodes, ~100 per tile).
// ---------------------------------------------------------------------------
constexpr int PF_THREADS = 512;
__global__ void __launch_bounds__(PF_THREADS) k_nf_prefilter(NodeFieldLaunch L, int ti0, int ti1, int tj1, int nty) {
    __shared__ int wsum[PF_THREADS / 32];
    __shared__ int base;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int ci = blockIdx.y, gi = blockIdx.x;
    const int by0 = ci * L.chunk_rows, by1 = min(by0 + L.chunk_rows, nty) - 1;
    const int gx0 = ti0 + gi * NF_GROUP_TILES, gx1 = min(gx0 + NF_GROUP_TILES - 1, ti1);
    // the chunk's tile rows (block-cyclic with bands: their bounding range)
    const int r0 = tile_row_of(by0, L.tile_j0, L.band_s1, L.band_count);
    const int r1 = min(tile_row_of(by1, L.tile_j0, L.band_s1, L.band_count), tj1);
    const double xlo = L.grid.gx + max(gx0 * TW, L.grid.i0), xhi = L.grid.gx + min((gx1 + 1) * TW - 1, L.grid.i1);
    const double ylo = L.grid.gy + max(r0 * TH, L.grid.j0), yhi = L.grid.gy + min((r1 + 1) * TH - 1, L.grid.j1);
    const int li = ci * L.col_groups + gi;
    int* list = L.lists + (size_t)li * L.lstride;
    if (t == 0) base = 0;
    __syncthreads();
    for (int b0 = 0; b0 < L.n; b0 += PF_THREADS) {
        const int i = b0 + t;
        bool keep = false;
        if (i < L.n) {
            const double ax = __ldg(&L.anchors[2 * i]), ay = __ldg(&L.anchors[2 * i + 1]);
            const double dxn = fmax(fmax(xlo - ax, 0.0), ax - xhi);
            const double dyn = fmax(fmax(ylo - ay, 0.0), ay - yhi);
            keep = L.alpha * (dxn * dxn + dyn * dyn) <= kLnCutoff + 1e-6;
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) wsum[wid] = __popc(m);
        __syncthreads();
        int off = base;
        for (int w = 0; w < wid; ++w) off += wsum[w];
        if (keep) list[off + __popc(m & ((1u << lane) - 1u))] = i;
        __syncthreads();
        if (t == 0) {
            int tot = 0;
            for (int w = 0; w < PF_THREADS / 32; ++w) tot += wsum[w];
            base += tot;
        }
        __syncthreads();
    }
    if (t == 0) L.lcounts[li] = base;
}

// The node list of (launch chunk ci, tile column group gi): (list, count);
// all n nodes without lists.
__device__ __forceinline__ const int* chunk_nodes(const NodeFieldLaunch& L, int ci, int gi, int* n) {
    if (!L.lists) {
        *n = L.n;
        return nullptr;
    }
    const int li = ci * L.col_groups + gi;
    *n = L.lcounts[li];
    return L.lists + (size_t)li * L.lstride;
}

__device__ __forceinline__ void nf_plan_tile(const NodeFieldLaunch& L, NfPlan* __restrict__ plans, int g, int tile_i0,
                                             int tile_j0, int tile_j_last, int s1, int by0, int rows, int ntx,
                                             unsigned (*list_s)[NF_CAP]);

// The planner reads only the nodes, so it may run while the previous blend's
// exact pass finishes (programmatic dependent launch); it waits for that
// predecessor before exiting, which keeps the canvas order for the next
// kernel (k_node_field waits for the planner). The last `conv` CTAs convert
// the frame for the texture: the previous blend's k_node_field, the only
// reader of those rows, has finished before this launch can start (its exact
// pass, the PDL primary here, triggers only after waiting for that grid).
constexpr int NF_CONV_BLOCKS = 2 * 148;
// 3 CTAs per SM (80 registers, a few spills): alone it is slower (15.9
// against 13.7 us on C2), but beside K3 the C2 step gains 1.3 us
#ifndef NRM_NF_PLAN_MINB
#define NRM_NF_PLAN_MINB 3
#endif
__global__ void __launch_bounds__(NF_PLAN_WARPS * 32, NRM_NF_PLAN_MINB)
k_nf_plan(NodeFieldLaunch L, NfPlan* __restrict__ plans, int tile_i0, int tile_j0, int tile_j_last, int s1, int by0,
          int rows, int ntx, int conv) {
    static_assert(NF_PLAN_WARPS * 32 == RGBA_THREADS, "conversion CTA shape");
    __shared__ unsigned list_s[NF_PLAN_WARPS][NF_CAP];
    const int nplan = gridDim.x - conv;
    if ((int)blockIdx.x >= nplan) {
        rgba_convert(L.frame, L.frgba, L.fw, L.fh, L.fch, L.frgba_pitch, blockIdx.x - nplan, conv);
        pdl_wait();
        return;
    }
    nf_plan_tile(L, plans, blockIdx.x * NF_PLAN_WARPS + (threadIdx.x >> 5), tile_i0, tile_j0, tile_j_last, s1, by0,
                 rows, ntx, list_s);
    pdl_wait();
}

// Planner of a batched blend: one warp per tile over all frames' tiles.
__global__ void __launch_bounds__(NF_PLAN_WARPS * 32)
k_nf_plan_batch(const NfBatchFrame* __restrict__ F, int nf, NfPlan* __restrict__ plans, int total) {
    __shared__ unsigned list_s[NF_PLAN_WARPS][NF_CAP];
    const int gt = blockIdx.x * NF_PLAN_WARPS + (threadIdx.x >> 5);
    if (gt < total) {
        int f = 0;
        while (f + 1 < nf && gt >= F[f + 1].plan_off) ++f;
        const NfBatchFrame& fr = F[f];
        nf_plan_tile(fr.L, plans + fr.plan_off, gt - fr.plan_off, fr.ti0, fr.tj0, fr.tj1, fr.s1, 0, fr.rows, fr.ntx,
                     list_s);
    }
    pdl_wait();
}

__device__ __forceinline__ void nf_plan_tile(const NodeFieldLaunch& L, NfPlan* __restrict__ plans, int g, int tile_i0,
                                             int tile_j0, int tile_j_last, int s1, int by0, int rows, int ntx,
                                             unsigned (*list_s)[NF_CAP]) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (g >= rows * ntx) return;
    unsigned* list = list_s[wid];
    NfPlan& pl = plans[g];
    const int tix = tile_i0 + g % ntx;
    const int tjy = tile_row_of(by0 + g / ntx, tile_j0, s1, L.band_count);
    const int ti0 = tix * TW, tj0 = tjy * TH;
    const int ci0 = max(ti0, L.grid.i0), ci1 = min(ti0 + TW - 1, L.grid.i1);
    const int cj0 = max(tj0, L.grid.j0), cj1 = min(tj0 + TH - 1, L.grid.j1);
    if (tjy < tile_j0 || tjy > tile_j_last || ci0 > ci1 || cj0 > cj1) {
        if (lane == 0) pl.h.status = NF_OUTSIDE;
        return;
    }
    const double ox = L.grid.gx + ti0, oy = L.grid.gy + tj0;  // unclipped tile origin
    const double xlo = L.grid.gx + ci0, xhi = L.grid.gx + ci1;
    const double ylo = L.grid.gy + cj0, yhi = L.grid.gy + cj1;
    const double alpha = L.alpha;

    // cull + classify: inner nodes (index order), then ring nodes (index order)
    auto classify = [&](int i) {
        int status = 0;  // 0 out, 1 inner, 2 ring
        if (i < L.n) {
            const double2 a = make_double2(__ldg(&L.anchors[2 * i]), __ldg(&L.anchors[2 * i + 1]));
            const double dxn = fmax(fmax(xlo - a.x, 0.0), a.x - xhi);
            const double dyn = fmax(fmax(ylo - a.y, 0.0), a.y - yhi);
            const double dxf = fmax(a.x - xlo, xhi - a.x), dyf = fmax(a.y - ylo, yhi - a.y);
            const double amin = alpha * (dxn * dxn + dyn * dyn);
            const double amax = alpha * (dxf * dxf + dyf * dyf);
            if (amin <= kLnCutoff + 1e-6) status = amax < kLnCutoff - 1e-5 ? 1 : 2;
        }
        return status;
    };
    int count = 0, ninner = 0;
    int nsrc;
    const int* src = chunk_nodes(L, by0 / L.chunk_rows, (g % ntx) / NF_GROUP_TILES, &nsrc);
    for (int pass = 1; pass <= 2; ++pass) {
        for (int base = 0; base < nsrc; base += 32) {
            const int e = base + lane;
            const int i = e < nsrc ? (src ? src[e] : e) : L.n;  // L.n: out of range -> not listed
            const bool take = classify(i) == pass;
            const unsigned m = __ballot_sync(0xffffffffu, take);
            const int pos = count + __popc(m & ((1u << lane) - 1u));
            if (take && pos < NF_CAP) list[pos] = (unsigned)i | (pass == 2 ? kRingBit : 0u);
            count += __popc(m);
        }
        if (pass == 1) ninner = count;
    }
    if (count > NF_CAP || count == 0) {
        if (lane == 0) {
            pl.h.count = count;
            pl.h.status = count == 0 ? NF_EMPTY : NF_EXACT;
        }
        return;
    }
    __syncwarp();
    // hemisphere arc + reference node (nearest the tile centre, lowest index
    // on ties); the listed warps are loaded once and kept in registers
    constexpr int KPL = 4;  // entries per lane held in registers (count <= 128)
    W5 qk[KPL];
    double2 ak[KPL];
    const unsigned i0 = list[0] & ~kRingBit;
    const double phi0 = atan2(__ldg(&L.warps[5 * i0 + 2]), __ldg(&L.warps[5 * i0 + 1]));
    double lo = 0.0, hi = 0.0, best = 1e300;
    int besti = 0x7fffffff;
    const double cxm = ox + 0.5 * TW, cym = oy + 0.5 * TH;
    auto arc = [&](unsigned i, const W5& q, const double2& a) {
        double rel = atan2(q.z, q.w) - phi0;
        if (rel > M_PI) rel -= 2.0 * M_PI;
        if (rel < -M_PI) rel += 2.0 * M_PI;
        lo = fmin(lo, rel);
        hi = fmax(hi, rel);
        const double ddx = a.x - cxm, ddy = a.y - cym;
        const double d2 = ddx * ddx + ddy * ddy;
        if (d2 < best || (d2 == best && (int)i < besti)) {
            best = d2;
            besti = (int)i;
        }
    };
#pragma unroll
    for (int r = 0; r < KPL; ++r) {
        const int k = lane + 32 * r;
        if (k < count) {
            const unsigned i = list[k] & ~kRingBit;
            qk[r] = load_w5(&L.warps[5 * i]);
            ak[r] = make_double2(__ldg(&L.anchors[2 * i]), __ldg(&L.anchors[2 * i + 1]));
        }
    }
#pragma unroll
    for (int r = 0; r < KPL; ++r)
        if (lane + 32 * r < count) arc(list[lane + 32 * r] & ~kRingBit, qk[r], ak[r]);
    for (int k = lane + 32 * KPL; k < count; k += 32) {
        const unsigned i = list[k] & ~kRingBit;
        arc(i, load_w5(&L.warps[5 * i]), make_double2(__ldg(&L.anchors[2 * i]), __ldg(&L.anchors[2 * i + 1])));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        const double bd = __shfl_xor_sync(0xffffffffu, best, o);
        const int bi = __shfl_xor_sync(0xffffffffu, besti, o);
        if (bd < best || (bd == best && bi < besti)) {
            best = bd;
            besti = bi;
        }
    }
    const W5 qr = load_w5(&L.warps[5 * besti]);
    double yx, yy;
    xapply(qr, ox, oy, &yx, &yy);
    const double s0 = qr.s;
    const double Y00 = rint(yx), Y01 = rint(yy);
    const double P0 = Y00 / s0, P1 = Y01 / s0;
    // scale lever S |P| of the fast tier's error model (see kScaleLever)
    double sdev = 0.0;
#pragma unroll
    for (int r = 0; r < KPL; ++r)
        if (lane + 32 * r < count) sdev = fmax(sdev, fabs(qk[r].s - s0));
    for (int k = lane + 32 * KPL; k < count; k += 32) sdev = fmax(sdev, fabs(__ldg(&L.warps[5 * (list[k] & ~kRingBit)]) - s0));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sdev = fmax(sdev, __shfl_xor_sync(0xffffffffu, sdev, o));
    const double lever = sdev * (fmax(fabs(P0), fabs(P1)) + (double)(TW + TH));
    const bool uniform = (hi - lo) < (0.5 * M_PI - 1e-6) && s0 > 0.0 && isfinite(P0) && isfinite(P1) &&
                         lever <= kScaleLever;
    if (lane == 0) {
        pl.h.P[0] = P0;
        pl.h.P[1] = P1;
        pl.h.Y0[0] = Y00;
        pl.h.Y0[1] = Y01;
        pl.h.e0[0] = fma(s0, P0, -Y00);
        pl.h.e0[1] = fma(s0, P1, -Y01);
        pl.h.s0 = s0;
        pl.h.count = count;
        pl.h.ninner = ninner;
        pl.h.status = uniform ? NF_OK : NF_EXACT;
    }
    if (!uniform) return;
    // listed warps in tile-local coordinates
    auto conj = [&](int k, const W5& q, const double2& a) {
        // qa = q * T(o): applies the tile-origin translation first
        const double hx = 0.5 * ox, hy = 0.5 * oy;
        const double qa_dx = (q.w * hx - q.z * hy) + q.dx;
        const double qa_dy = (q.w * hy + q.z * hx) + q.dy;
        // q' = T(-P) * qa
        const double px = 0.5 * P0, py = 0.5 * P1;
        const double qdx = qa_dx + (-px * q.w - py * q.z);
        const double qdy = qa_dy + (px * q.z - py * q.w);
        NfEntry en;
        en.q = make_float4((float)q.w, (float)q.z, (float)qdx, (float)qdy);
        en.a = a;
        en.d = (float)(q.s - s0);
        en.idx = list[k];
        en.pad[0] = en.pad[1] = 0u;
        pl.e[k] = en;
    };
#pragma unroll
    for (int r = 0; r < KPL; ++r)
        if (lane + 32 * r < count) conj(lane + 32 * r, qk[r], ak[r]);
    for (int k = lane + 32 * KPL; k < count; k += 32) {
        const unsigned i = list[k] & ~kRingBit;
        conj(k, load_w5(&L.warps[5 * i]), make_double2(__ldg(&L.anchors[2 * i]), __ldg(&L.anchors[2 * i + 1])));
    }
}

__device__ __forceinline__ void stage_entries(NfEntry* dst, const NfEntry* src, int n) {
    constexpr int kC = (int)(sizeof(NfEntry) / 16);
    for (int c = threadIdx.x; c < n * kC; c += NT)
        cp_async16(reinterpret_cast<char*>(dst) + 16 * c, reinterpret_cast<const char*>(src) + 16 * c);
}

// One K1/K2 CTA: slice bx of launch-grid column, launch row by (see the
// kernels below for the grid layouts).
template <int MODE>
__device__ __forceinline__ void nf_field_cta(const NodeFieldLaunch& L, const NfPlan* __restrict__ plans, int tile_i0,
                                             int tile_j0, int s1, int by0, int ntx, int bx, int by,
                                             unsigned char* smem_raw) {
    constexpr int MT = K1Shape<MODE>::MT, CW = K1Shape<MODE>::CW, NH = K1Shape<MODE>::NH;
    Smem<CW>& s = *reinterpret_cast<Smem<CW>*>(smem_raw);
    CanvasTile& ct = *reinterpret_cast<CanvasTile*>(smem_raw + canvas_tile_offset<CW>());
    const int t = threadIdx.x;
    const int half = bx % NH;  // this CTA's column slice of the planning tile
    const NfPlan& pl = plans[by * ntx + bx / NH];
    const int tix = tile_i0 + bx / NH;
    const int tjy = tile_row_of(by0 + by, tile_j0, s1, L.band_count);
    const int ti0 = tix * TW, tj0 = tjy * TH;  // planning tile origin
    const int hi0 = ti0 + CW * half;           // first column of this slice

    // ---- 0. stage the canvas slice (the whole 64 x 32 tile lies in the
    //         canvas: tiles and canvas bounds are both 32/64-aligned,
    //         mosaic.hpp:141-151) before the plan header arrives, then the
    //         first chunk of the tile's plan
    const bool tma = MODE != 1 && L.ctm_ok;  // launch-uniform
    if (tma) {  // four 32 x 32 boxes by TMA, one thread; everyone waits before the epilogue
        if (t == 0) {
            mbar_init(&ct.bar, 1);
            mbar_expect_tx(&ct.bar, (unsigned)(3 * sizeof(ct.r) + sizeof(ct.w)));
            const int x = hi0 - (int)L.phys_x0, y = tj0 - (int)L.phys_y0;
            tma_load_2d(ct.r, &L.ctm[0], x, y, &ct.bar);
            tma_load_2d(ct.g, &L.ctm[1], x, y, &ct.bar);
            tma_load_2d(ct.b, &L.ctm[2], x, y, &ct.bar);
            tma_load_2d(ct.w, &L.ctm[3], x, y, &ct.bar);
        }
    } else if (MODE != 1) {
        const long long base = (long long)(tj0 - L.phys_y0) * L.pitch + (hi0 - L.phys_x0);
        {  // float planes: thread = (row r, 16-byte chunk k) for rows r and r + 16
            const int k = t & 7, r = t >> 3;  // r < 32
            const long long o = base + (long long)r * L.pitch + 4 * k;
            cp_async16(&ct.r[r][4 * k], L.R + o);
            cp_async16(&ct.g[r][4 * k], L.G + o);
            cp_async16(&ct.b[r][4 * k], L.B + o);
        }
        if (t < 2 * TH) {  // weight plane: 2 chunks per row
            const int k = t & 1, r = t >> 1;
            cp_async16(&ct.w[r][16 * k], L.W + base + (long long)r * L.pitch + 16 * k);
        }
    }
    const int status = pl.h.status;
    const int ci0 = max(hi0, L.grid.i0), ci1 = min(hi0 + CW - 1, L.grid.i1);
    const int cj0 = max(tj0, L.grid.j0), cj1 = min(tj0 + TH - 1, L.grid.j1);
    // an early exit must not leave a copy into this CTA's shared memory in flight
    auto drain = [&]() {
        cp_async_wait_all();
        if (tma && t == 0) mbar_wait(&ct.bar, 0);
    };
    if (status == NF_OUTSIDE || ci0 > ci1) {  // outside the footprint rows / right of the grid
        drain();
        return;
    }
    const int count = pl.h.count;
    if (status == NF_OK) stage_entries(s.e, pl.e, min(CHUNK, count));
    cp_async_commit();

    if (status == NF_EXACT) {
        tile_to_exceptions<MODE>(L, ci0, ci1, cj0, cj1);
        drain();
        return;
    }

    // ---- B. no node reaches the tile: every pixel lacks support ----------
    if (status == NF_EMPTY) {
        int ns = 0;
        for (int e = t; e < (ci1 - ci0 + 1) * (cj1 - cj0 + 1); e += NT) {
            const int w = ci1 - ci0 + 1;
            const int i = ci0 + e % w, j = cj0 + e / w;
            if (MODE == 1) {
                const size_t o = (size_t)(j - L.grid.j0) * (L.grid.i1 - L.grid.i0 + 1) + (i - L.grid.i0);
                if (L.disp) L.disp[o] = make_float2(0.f, 0.f);
                if (L.support) L.support[o] = 0;
            }
            ++ns;
        }
        drain();
        if (MODE != 1) block_add3<NT>(L.acc, 0, ns, 0);
        return;
    }
    const double ox = L.grid.gx + ti0, oy = L.grid.gy + tj0;  // unclipped tile origin
    const double alpha = L.alpha;
    const double P0 = pl.h.P[0], P1 = pl.h.P[1], s0 = pl.h.s0;
    const int ninner = pl.h.ninner;

    // ---- D. main loop over node chunks -----------------------------------
    // Inner nodes run on the tensor cores. The sums are a product of two
    // factored matrices: for component j (qw, qz, qdx, qdy, s - s0, 1),
    //   D_j[col][row] = sum_k ex[k][col] * (ey[k][row] * q_k[j]),
    // i.e. A = ex (32 cols x K nodes), B_j = ey * q_j (K x 32 rows). Warp w
    // owns 16 columns x 8 rows: one m16 tile x 6 n8 tiles (one per
    // component, the 8 rows on n), so every thread ends with all six sums of
    // its 4 pixels. 3xTF32 split products keep ~2^-21 relative accuracy. Ring
    // nodes (the 1e-6 cutoff crosses the tile) follow on the CUDA cores with
    // the per-pixel cutoff test.
    const int lane = t & 31, wid = t >> 5, g = lane >> 2, tig = lane & 3;
    const int cw = 16 * MT * (wid & 1), rw = 8 * (wid >> 1);  // within the slice
    float acc[MT][6][4];  // [m tile][component][fragment f]: pixel (cw + 16 mt + 8 (f >> 1) + g, rw + 2 tig + (f & 1))
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int j = 0; j < 6; ++j)
#pragma unroll
            for (int f = 0; f < 4; ++f) acc[mt][j][f] = 0.f;
    unsigned amb = 0;

    const double nal = -alpha * kLog2e;
    const double hx0 = ox + CW * half;  // x of the slice's first column
    for (int c0 = 0; c0 < count; c0 += CHUNK) {
        const int cn = min(CHUNK, count - c0);
        const int kin = min(max(ninner - c0, 0), cn);  // inner nodes of this chunk come first
        const int cn8 = (cn + 7) & ~7;
        if (c0 > 0) {  // later chunks (tiles with more than CHUNK listed nodes)
            __syncthreads();
            stage_entries(s.e, pl.e + c0, cn);
            cp_async_commit();
        }
        cp_async_wait_all();
        __syncthreads();
        // Tables; padding up to a multiple of 8 nodes is zero. Column factor:
        // thread = (node, 8-column block), node fastest (conflict-free
        // stores); along a row the FP64 exponent -a (ax - x)^2 advances by
        // its exact second differences.
        {
            constexpr int CB = CW / 4;  // columns per thread
            const int k = t & 63, cb = (t >> 6) * CB;
            float* ph = &s.exh[cb][k];
            float* pq = &s.exl[cb][k];
            if (k < cn) {
                const double d0 = s.e[k].a.x - (hx0 + cb);
                double E = nal * d0 * d0, D = nal * (1.0 - 2.0 * d0);
                const double D2 = 2.0 * nal;
#pragma unroll 8
                for (int c = 0; c < CB; ++c) {
                    const float v = ex2_approx((float)E);
                    const float hi = tf32_hi(v);
                    ph[c * KP] = hi;
                    pq[c * KP] = v - hi;
                    E += D;
                    D += D2;
                }
            } else if (k < cn8) {
#pragma unroll 8
                for (int c = 0; c < CB; ++c) ph[c * KP] = pq[c * KP] = 0.f;
            }
        }
        {  // row factor: thread = (row, every 8th node)
            const int r = t & 31;
            const double y = oy + r;
            for (int k = t >> 5; k < cn8; k += 8) {
                float v = 0.f;
                if (k < cn) {
                    const double dy = s.e[k].a.y - y;
                    v = ex2_approx((float)(nal * dy * dy));
                }
                s.ey[k][r] = v;
            }
        }
        for (int k = t; k < cn8; k += NT) {
            const bool in = k < kin;  // ring nodes and padding: zero B columns
            s.qt[k][0] = in ? s.e[k].q : make_float4(0.f, 0.f, 0.f, 0.f);
            s.qt[k][1] = make_float4(in ? s.e[k].d : 0.f, in ? 1.f : 0.f, 0.f, 0.f);
        }
        __syncthreads();

        for (int kb = 0; kb < kin; kb += 8) {
            unsigned ah[MT][4], al[MT][4];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                ldsm_x4(&s.exh[cw + 16 * mt + (lane & 15)][kb + 4 * (lane >> 4)], ah[mt]);
                ldsm_x4(&s.exl[cw + 16 * mt + (lane & 15)][kb + 4 * (lane >> 4)], al[mt]);
            }
            const float ey0 = s.ey[kb + tig][rw + g], ey1 = s.ey[kb + tig + 4][rw + g];
            const float* qa = &s.qt[kb + tig][0].x;
            const float* qb = &s.qt[kb + tig + 4][0].x;
#pragma unroll
            for (int j = 0; j < 6; ++j) {
                const float b0 = ey0 * qa[j], b1 = ey1 * qb[j];
                const float b0h = tf32_hi(b0), b1h = tf32_hi(b1);
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    mma_tf32(acc[mt][j], al[mt], b0h, b1h);
                    mma_tf32(acc[mt][j], ah[mt], b0 - b0h, b1 - b1h);
                    mma_tf32(acc[mt][j], ah[mt], b0h, b1h);
                }
            }
        }
        for (int k = kin; k < cn; ++k) {  // ring nodes: the 1e-6 cutoff per pixel
            const float4 q = s.e[k].q;
            const float dd = s.e[k].d;
            const float2 eyv = *reinterpret_cast<const float2*>(&s.ey[k][rw + 2 * tig]);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
                for (int hc = 0; hc < 2; ++hc) {
                    const int c = cw + 16 * mt + 8 * hc + g;
                    const float exv = s.exh[c][k] + s.exl[c][k];
#pragma unroll
                    for (int hr = 0; hr < 2; ++hr) {
                        const int f = 2 * hc + hr;
                        float w = exv * (hr ? eyv.y : eyv.x);
                        const bool in = w > kCutHi;
                        amb |= (unsigned)((w >= kCutLo) && !in) << (4 * mt + f);
                        w = in ? w : 0.f;
                        acc[mt][0][f] = fmaf(w, q.x, acc[mt][0][f]);
                        acc[mt][1][f] = fmaf(w, q.y, acc[mt][1][f]);
                        acc[mt][2][f] = fmaf(w, q.z, acc[mt][2][f]);
                        acc[mt][3][f] = fmaf(w, q.w, acc[mt][3][f]);
                        acc[mt][4][f] = fmaf(w, dd, acc[mt][4][f]);
                        acc[mt][5][f] += w;
                    }
                }
            }
        }
    }

    if (tma) mbar_wait(&ct.bar, 0);  // the canvas tile has landed
    // ---- E. epilogue --------------------------------------------------------
    // Output position y = Y0 + r with the integer tile image origin Y0 and a
    // tile-relative remainder r = e0 + dl P + (s0 + dl) Q(u) that stays small
    // (|r| ~ 1e2 px): FP32 keeps it to ~1e-5 px at any canvas coordinate.
    const double Y00 = pl.h.Y0[0], Y01 = pl.h.Y0[1];
    const int Y0x = (int)Y00, Y0y = (int)Y01;  // rint() results: exact integers
    const float P0f = (float)P0, P1f = (float)P1, s0f = (float)s0;
    const float e00f = (float)pl.h.e0[0], e01f = (float)pl.h.e0[1];
    const float fxm = (float)(L.fw - 1), fym = (float)(L.fh - 1);
    // K2: displacement base (Y0 - tile origin), exact small integer - grid offset
    const float bdx = (float)(Y00 - ox), bdy = (float)(Y01 - oy);
    int nb = 0, nns = 0, noof = 0;
#pragma unroll
    for (int p = 0; p < 4 * MT; ++p) {
        const int mt = p >> 2, f = p & 3;
        const int hcol = cw + 16 * mt + 8 * (f >> 1) + g, r = rw + 2 * tig + (f & 1);  // within the slice
        const int col = CW * half + hcol;                                                // within the planning tile
        const int i = ti0 + col, jj = tj0 + r;
        const float s0v = acc[mt][0][f], s1v = acc[mt][1][f], s2v = acc[mt][2][f];
        const float s3v = acc[mt][3][f], s4v = acc[mt][4][f], s5v = acc[mt][5][f];
        const bool valid = i >= ci0 && i <= ci1 && jj >= cj0 && jj <= cj1;
        bool exc = false;
        if (valid) {
            if ((amb >> p) & 1u) {
                exc = true;
            } else if (s5v == 0.f) {
                ++nns;
                if (MODE == 1) {
                    const size_t o = (size_t)(jj - L.grid.j0) * (L.grid.i1 - L.grid.i0 + 1) + (i - L.grid.i0);
                    if (L.disp) L.disp[o] = make_float2(0.f, 0.f);
                    if (L.support) L.support[o] = 0;
                }
            } else {
                const float rn = rsqrtf(fmaf(s0v, s0v, s1v * s1v));
                const float qw = s0v * rn, qz = s1v * rn, qdx = s2v * rn, qdy = s3v * rn;
                const float cc = qw * qw - qz * qz, ss = 2.f * qw * qz;
                const float ux = (float)col, uy = (float)r;
                const float Qx = cc * ux - ss * uy + 2.f * (qdx * qw - qdy * qz);
                const float Qy = ss * ux + cc * uy + 2.f * (qdx * qz + qdy * qw);
                const float dl = __fdividef(s4v, s5v);  // s5 > 0, far from 2^126
                const float sbf = s0f + dl;
                const float rx = fmaf(sbf, Qx, fmaf(dl, P0f, e00f));
                const float ry = fmaf(sbf, Qy, fmaf(dl, P1f, e01f));
                if (MODE == 1) {
                    const size_t o = (size_t)(jj - L.grid.j0) * (L.grid.i1 - L.grid.i0 + 1) + (i - L.grid.i0);
                    if (L.disp) L.disp[o] = make_float2((bdx - ux) + rx, (bdy - uy) + ry);
                    if (L.support) L.support[o] = 1;
                } else {
                    const float yx = (float)Y0x + rx, yy = (float)Y0y + ry;  // margin test only
                    const float margin = fminf(fminf(yx, fxm - yx), fminf(yy, fym - yy));
                    if (margin < (float)-kBoundMargin) {
                        ++noof;
                    } else if (margin < (float)kBoundMargin) {
                        exc = true;
                    } else {
                        const int xc = L.fw - 2 >= 0 ? L.fw - 2 : 0, yc = L.fh - 2 >= 0 ? L.fh - 2 : 0;
                        const int x0 = min(Y0x + (int)floorf(rx), xc), y0 = min(Y0y + (int)floorf(ry), yc);
                        const float fx = rx - (float)(x0 - Y0x), fy = ry - (float)(y0 - Y0y);
                        const int x1 = min(x0 + 1, L.fw - 1), y1 = min(y0 + 1, L.fh - 1);
                        const unsigned row0 = (unsigned)y0 * (unsigned)L.fw, row1 = (unsigned)y1 * (unsigned)L.fw;
                        const float gx = 1.f - fx, gy = 1.f - fy;
                        float vr, vg, vbl;  // bilinear sample / 255
                        if (L.ftex) {
                            // three 2 x 2 gathers of the RGBA8 texture, already / 255:
                            // .w (x0, y0), .z (x1, y0), .x (x0, y1), .y (x1, y1); the
                            // clamped address mode gives x1 = min(x0 + 1, fw - 1) likewise
                            const float tx = (float)x0 + 1.f, ty = (float)y0 + 1.f;
                            const float4 cr = tex2Dgather<float4>((cudaTextureObject_t)L.ftex, tx, ty, 0);
                            const float4 cg = tex2Dgather<float4>((cudaTextureObject_t)L.ftex, tx, ty, 1);
                            const float4 cb = tex2Dgather<float4>((cudaTextureObject_t)L.ftex, tx, ty, 2);
                            vr = (gx * cr.w + fx * cr.z) * gy + (gx * cr.x + fx * cr.y) * fy;
                            vg = (gx * cg.w + fx * cg.z) * gy + (gx * cg.x + fx * cg.y) * fy;
                            vbl = (gx * cb.w + fx * cb.z) * gy + (gx * cb.x + fx * cb.y) * fy;
                        } else {
                            float va[3], vb[3], vc[3], vd[3];
                            texel_u32(L.frame, row0 + x0, L.fch, va);
                            texel_u32(L.frame, row0 + x1, L.fch, vb);
                            texel_u32(L.frame, row1 + x0, L.fch, vc);
                            texel_u32(L.frame, row1 + x1, L.fch, vd);
                            constexpr float k255 = 1.f / 255.f;
                            vr = ((gx * va[0] + fx * vb[0]) * gy + (gx * vc[0] + fx * vd[0]) * fy) * k255;
                            vg = ((gx * va[1] + fx * vb[1]) * gy + (gx * vc[1] + fx * vd[1]) * fy) * k255;
                            vbl = ((gx * va[2] + fx * vb[2]) * gy + (gx * vc[2] + fx * vd[2]) * fy) * k255;
                        }
                        const uint8_t wg = ct.w[r][hcol];
                        const float wd = (float)wg, inv = __fdividef(1.f, wd + 1.f);
                        const long long idx = (long long)(jj - L.phys_y0) * L.pitch + (i - L.phys_x0);
                        // reference rule: (w c + v) / (w + 1); weighted mode:
                        // ((w + 1 - cf) c + cf v) / (w + 1), identical for cf == 1
                        float a = wd, cf = 1.f;
                        if (MODE == 2) {
                            const float* U = L.unc;
                            const float u = (gx * U[row0 + x0] + fx * U[row0 + x1]) * gy +
                                            (gx * U[row1 + x0] + fx * U[row1 + x1]) * fy;
                            cf = __frcp_rn(fmaxf(u, 1.f));
                            a = wd + 1.f - cf;
                        }
                        // explicit FMAs: the same instructions in both modes, so
                        // cf == 1 reproduces the reference rule bit for bit
                        L.R[idx] = fmaf(a, ct.r[r][hcol], cf * vr) * inv;
                        L.G[idx] = fmaf(a, ct.g[r][hcol], cf * vg) * inv;
                        L.B[idx] = fmaf(a, ct.b[r][hcol], cf * vbl) * inv;
                        L.W[idx] = wg < kWeightCap ? (uint8_t)(wg + 1) : wg;
                        ++nb;
                    }
                }
            }
        }
        defer_pixel<MODE>(L, exc, i, jj);
    }
    if (MODE != 1) block_add3<NT>(L.acc, nb, nns, noof);
}

#ifndef NRM_K2_MMASYNC
// ---------------------------------------------------------------------------
// K2 on the 5th-generation tensor cores (tcgen05). CTA = one 64 x 32 planning
// tile, 256 threads. The inner-node sums are one product per chunk of 32
// listed nodes, D[col][n] += A[col][k] B[n][k] with
//   A = ex (M = 64 tile columns), B[32 j + row][k] = ey[k][row] q_k[j]
//   (N = 6 components x 32 rows = 192),
// 3xTF32 split products (Al Bh + Ah Bl + Ah Bh) accumulated in FP32 in tensor
// memory (64 lanes x 192 columns); one thread issues the MMAs and commits
// them to an mbarrier. Ring nodes (the 1e-6 cutoff crosses the tile) stay on
// the CUDA cores in registers; the epilogue adds the accumulator read back
// from tensor memory with tcgen05.ld (16x256b: the mma.sync fragment layout,
// so each thread owns 8 pixels as before). Operand layout and descriptors:
// nrm_common.cuh, validated by tools/probes/tcgen05_probe.cu.
// ---------------------------------------------------------------------------
constexpr int TC_K = 32;                                       // listed nodes per chunk (4 MMA k-steps)
constexpr int TC_M = TW, TC_N = 6 * TH;                        // 64 x 192
constexpr unsigned TC_IDESC = umma_idesc_tf32(TC_M, TC_N);
constexpr int TC_TMEM_COLS = 256;                              // >= TC_N, power of two
struct __align__(128) SmemTC {
    float ah[TC_K * TC_M], al[TC_K * TC_M];  // A = ex, K-major canonical (umma_kmajor_off), TF32 hi / lo
    float bh[TC_K * TC_N], bl[TC_K * TC_N];  // B = ey * q_j
    float ey[TC_K][EYP];                     // row factor [node][row] (ring nodes)
    float eyt[TH][TC_K + 4];                 // row factor [row][node] (B build: 16-byte reads)
    float qt[8][TC_K];                       // [component][node]: qw, qz, qdx, qdy, ds, 1 (zero for ring nodes)
    NfEntry e[TC_K];
    unsigned long long bar;                  // MMA completion
    unsigned tmem;                           // tensor-memory base address
};

__device__ __forceinline__ void nf_field_tc(const NodeFieldLaunch& L, const NfPlan* __restrict__ plans, int tile_i0,
                                            int tile_j0, int s1, int by0, int ntx, int bx, int by,
                                            unsigned char* smem_raw) {
    SmemTC& s = *reinterpret_cast<SmemTC*>(smem_raw);
    const int t = threadIdx.x;
    const NfPlan& pl = plans[by * ntx + bx];
    const int tix = tile_i0 + bx;
    const int tjy = tile_row_of(by0 + by, tile_j0, s1, L.band_count);
    const int ti0 = tix * TW, tj0 = tjy * TH;
    const int status = pl.h.status;
    const int ci0 = max(ti0, L.grid.i0), ci1 = min(ti0 + TW - 1, L.grid.i1);
    const int cj0 = max(tj0, L.grid.j0), cj1 = min(tj0 + TH - 1, L.grid.j1);
    if (status == NF_OUTSIDE || ci0 > ci1) return;
    if (status == NF_EXACT) {
        tile_to_exceptions<1>(L, ci0, ci1, cj0, cj1);
        return;
    }
    if (status == NF_EMPTY) {  // no node reaches the tile: no support anywhere
        const int w = ci1 - ci0 + 1;
        for (int e = t; e < w * (cj1 - cj0 + 1); e += NT) {
            const int i = ci0 + e % w, j = cj0 + e / w;
            const size_t o = (size_t)(j - L.grid.j0) * (L.grid.i1 - L.grid.i0 + 1) + (i - L.grid.i0);
            if (L.disp) L.disp[o] = make_float2(0.f, 0.f);
            if (L.support) L.support[o] = 0;
        }
        return;
    }
    const int count = pl.h.count, ninner = pl.h.ninner;
    stage_entries(s.e, pl.e, min(TC_K, count));
    cp_async_commit();
    if (t < 32) tmem_alloc<TC_TMEM_COLS>(&s.tmem);
    if (t == 0) mbar_init(&s.bar, 1);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const unsigned tmem = s.tmem;

    const double ox = L.grid.gx + ti0, oy = L.grid.gy + tj0;  // unclipped tile origin
    const double nal = -L.alpha * kLog2e;
    const int lane = t & 31, wid = t >> 5, g = lane >> 2, tig = lane & 3;
    // warp w reads tensor-memory lanes 32 (w % 4) .. + 15 = tile columns
    // cb = 16 (w % 4) .., and rows rb = 16 (w / 4) ..; thread pixels:
    // (cb + 8 (f >> 1) + g, rb + 8 mt + 2 tig + (f & 1))
    const int cb = 16 * (wid & 3), rb = 16 * (wid >> 2);
    float acc[2][6][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int j = 0; j < 6; ++j)
#pragma unroll
            for (int f = 0; f < 4; ++f) acc[mt][j][f] = 0.f;
    unsigned amb = 0, phase = 0;
    bool pending = false, any_mma = false;  // block-uniform
    for (int c0 = 0; c0 < count; c0 += TC_K) {
        const int cn = min(TC_K, count - c0);
        const int kin = min(max(ninner - c0, 0), cn);  // inner nodes of this chunk come first
        const int cn8 = (cn + 7) & ~7;
        if (c0 > 0) {
            if (pending) {  // the previous chunk's MMAs have read A and B
                mbar_wait(&s.bar, phase);
                phase ^= 1u;
                pending = false;
            }
            __syncthreads();  // and every thread is done with its ring nodes
            stage_entries(s.e, pl.e + c0, cn);
            cp_async_commit();
        }
        cp_async_wait_all();
        __syncthreads();
        // A (column factor, hi / lo): thread = (column, 4 consecutive nodes),
        // one 16-byte store of each half per group; (c, 4 kq) sits at byte
        // umma_kmajor_off = 16 TC_M kq + 128 (c / 8) + 16 (c % 8)
        for (int u = t; u < TC_M * (cn8 / 4); u += NT) {
            const int c = u & (TC_M - 1), kq = u / TC_M, k0 = 4 * kq;
            float h4[4], l4[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int k = k0 + i;
                float v = 0.f;
                if (k < cn) {
                    const double d = s.e[k].a.x - (ox + c);
                    v = ex2_approx((float)(nal * d * d));
                }
                h4[i] = tf32_hi(v);
                l4[i] = v - h4[i];
            }
            const int o = 4 * TC_M * kq + 32 * (c >> 3) + 4 * (c & 7);
            *reinterpret_cast<float4*>(&s.ah[o]) = make_float4(h4[0], h4[1], h4[2], h4[3]);
            *reinterpret_cast<float4*>(&s.al[o]) = make_float4(l4[0], l4[1], l4[2], l4[3]);
        }
        {  // row factor: thread = (row, every 8th node)
            const int r = t & 31;
            const double y = oy + r;
            for (int k = t >> 5; k < cn8; k += 8) {
                float v = 0.f;
                if (k < cn) {
                    const double dy = s.e[k].a.y - y;
                    v = ex2_approx((float)(nal * dy * dy));
                }
                s.ey[k][r] = v;
                s.eyt[r][k] = v;
            }
        }
        for (int k = t; k < cn8; k += NT) {
            const bool in = k < kin;  // ring nodes and padding: zero B rows
            const float4 q = s.e[k].q;
            s.qt[0][k] = in ? q.x : 0.f;
            s.qt[1][k] = in ? q.y : 0.f;
            s.qt[2][k] = in ? q.z : 0.f;
            s.qt[3][k] = in ? q.w : 0.f;
            s.qt[4][k] = in ? s.e[k].d : 0.f;
            s.qt[5][k] = in ? 1.f : 0.f;
        }
        __syncthreads();
        if (kin > 0) {
            // B (hi / lo): thread = (n = 32 j + row, 4 consecutive nodes); items
            // u = t + 256 i walk n by 64 (mod 192) and kq by 1 (+1 on wrap)
            const int kin8 = (kin + 7) & ~7, nq = kin8 / 4;
            int n = t < TC_N ? t : t - TC_N, kq = t < TC_N ? 0 : 1;
            while (kq < nq) {
                const int j = n >> 5, r = n & 31;
                const float4 e4 = *reinterpret_cast<const float4*>(&s.eyt[r][4 * kq]);
                const float4 q4 = *reinterpret_cast<const float4*>(&s.qt[j][4 * kq]);
                const float v0 = e4.x * q4.x, v1 = e4.y * q4.y, v2 = e4.z * q4.z, v3 = e4.w * q4.w;
                const float h0 = tf32_hi(v0), h1 = tf32_hi(v1), h2 = tf32_hi(v2), h3 = tf32_hi(v3);
                const int o = 4 * TC_N * kq + 32 * (n >> 3) + 4 * (n & 7);
                *reinterpret_cast<float4*>(&s.bh[o]) = make_float4(h0, h1, h2, h3);
                *reinterpret_cast<float4*>(&s.bl[o]) = make_float4(v0 - h0, v1 - h1, v2 - h2, v3 - h3);
                n += NT - TC_N;
                ++kq;
                if (n >= TC_N) {
                    n -= TC_N;
                    ++kq;
                }
            }
            fence_async_smem();
            tc_fence_before();
            __syncthreads();
            tc_fence_after();
            if (t == 0) {
                const unsigned a_h = smem_addr(s.ah), a_l = smem_addr(s.al), b_h = smem_addr(s.bh),
                               b_l = smem_addr(s.bl);
                for (int ks = 0; ks < nq / 2; ++ks) {
                    const unsigned oa = ks * 32 * TC_M, ob = ks * 32 * TC_N;
                    const unsigned long long dah = umma_desc(a_h + oa, 16 * TC_M, 128),
                                             dal = umma_desc(a_l + oa, 16 * TC_M, 128),
                                             dbh = umma_desc(b_h + ob, 16 * TC_N, 128),
                                             dbl = umma_desc(b_l + ob, 16 * TC_N, 128);
                    umma_tf32(tmem, dal, dbh, TC_IDESC, (any_mma || ks > 0) ? 1u : 0u);
                    umma_tf32(tmem, dah, dbl, TC_IDESC, 1u);
                    umma_tf32(tmem, dah, dbh, TC_IDESC, 1u);
                }
                umma_commit(&s.bar);
            }
            pending = true;
            any_mma = true;
        }
        // ring nodes on the CUDA cores, per-pixel 1e-6 cutoff (overlaps the MMAs)
        for (int k = kin; k < cn; ++k) {
            const float4 q = s.e[k].q;
            const float dd = s.e[k].d;
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const float2 eyv = *reinterpret_cast<const float2*>(&s.ey[k][rb + 8 * mt + 2 * tig]);
#pragma unroll
                for (int hc = 0; hc < 2; ++hc) {
                    const int c = cb + 8 * hc + g, o = umma_kmajor_off(c, k, TC_M) >> 2;
                    const float exv = s.ah[o] + s.al[o];
#pragma unroll
                    for (int hr = 0; hr < 2; ++hr) {
                        const int f = 2 * hc + hr;
                        float w = exv * (hr ? eyv.y : eyv.x);
                        const bool in = w > kCutHi;
                        amb |= (unsigned)((w >= kCutLo) && !in) << (4 * mt + f);
                        w = in ? w : 0.f;
                        acc[mt][0][f] = fmaf(w, q.x, acc[mt][0][f]);
                        acc[mt][1][f] = fmaf(w, q.y, acc[mt][1][f]);
                        acc[mt][2][f] = fmaf(w, q.z, acc[mt][2][f]);
                        acc[mt][3][f] = fmaf(w, q.w, acc[mt][3][f]);
                        acc[mt][4][f] = fmaf(w, dd, acc[mt][4][f]);
                        acc[mt][5][f] += w;
                    }
                }
            }
        }
    }
    if (pending) mbar_wait(&s.bar, phase);
    tc_fence_after();
    if (any_mma) {
        const unsigned tl = tmem + ((unsigned)(32 * (wid & 3)) << 16);
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            float v[8];
            tmem_ld_16x256b_x2(tl + (unsigned)(32 * j + rb), v);
#pragma unroll
            for (int f = 0; f < 4; ++f) {
                acc[0][j][f] += v[f];
                acc[1][j][f] += v[4 + f];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (wid == 0) tmem_dealloc<TC_TMEM_COLS>(tmem);

    // epilogue (K2 of nf_field_cta with this thread's pixel map)
    const double Y00 = pl.h.Y0[0], Y01 = pl.h.Y0[1];
    const float P0f = (float)pl.h.P[0], P1f = (float)pl.h.P[1], s0f = (float)pl.h.s0;
    const float e00f = (float)pl.h.e0[0], e01f = (float)pl.h.e0[1];
    const float bdx = (float)(Y00 - ox), bdy = (float)(Y01 - oy);
#pragma unroll
    for (int p = 0; p < 8; ++p) {
        const int mt = p >> 2, f = p & 3;
        const int col = cb + 8 * (f >> 1) + g, r = rb + 8 * mt + 2 * tig + (f & 1);
        const int i = ti0 + col, jj = tj0 + r;
        const float s0v = acc[mt][0][f], s1v = acc[mt][1][f], s2v = acc[mt][2][f];
        const float s3v = acc[mt][3][f], s4v = acc[mt][4][f], s5v = acc[mt][5][f];
        const bool valid = i >= ci0 && i <= ci1 && jj >= cj0 && jj <= cj1;
        bool exc = false;
        if (valid) {
            const size_t o = (size_t)(jj - L.grid.j0) * (L.grid.i1 - L.grid.i0 + 1) + (i - L.grid.i0);
            if ((amb >> p) & 1u) {
                exc = true;
            } else if (s5v == 0.f) {
                if (L.disp) L.disp[o] = make_float2(0.f, 0.f);
                if (L.support) L.support[o] = 0;
            } else {
                const float rn = rsqrtf(fmaf(s0v, s0v, s1v * s1v));
                const float qw = s0v * rn, qz = s1v * rn, qdx = s2v * rn, qdy = s3v * rn;
                const float cc = qw * qw - qz * qz, ss = 2.f * qw * qz;
                const float ux = (float)col, uy = (float)r;
                const float Qx = cc * ux - ss * uy + 2.f * (qdx * qw - qdy * qz);
                const float Qy = ss * ux + cc * uy + 2.f * (qdx * qz + qdy * qw);
                const float dl = __fdividef(s4v, s5v);  // s5 > 0, far from 2^126
                const float sbf = s0f + dl;
                const float rx = fmaf(sbf, Qx, fmaf(dl, P0f, e00f));
                const float ry = fmaf(sbf, Qy, fmaf(dl, P1f, e01f));
                if (L.disp) L.disp[o] = make_float2((bdx - ux) + rx, (bdy - uy) + ry);
                if (L.support) L.support[o] = 1;
            }
        }
        defer_pixel<1>(L, exc, i, jj);
    }
}
#endif

template <int MODE>
__global__ void __launch_bounds__(NT, K1Shape<MODE>::MINB)
k_node_field(const __grid_constant__ NodeFieldLaunch L, const NfPlan* __restrict__ plans, int tile_i0, int tile_j0,
             int s1, int by0, int ntx, int trig) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // last launch chunk: the exception pass may become resident during the
    // last wave (it waits for this grid before reading the queue); earlier
    // chunks are followed by the next chunk's planner, which rewrites the plans
    if (trig) pdl_trigger();
    pdl_wait();
#ifndef NRM_K2_MMASYNC
    if constexpr (MODE == 1) {
        nf_field_tc(L, plans, tile_i0, tile_j0, s1, by0, ntx, blockIdx.x, blockIdx.y, smem_raw);
        return;
    }
#endif
    nf_field_cta<MODE>(L, plans, tile_i0, tile_j0, s1, by0, ntx, blockIdx.x, blockIdx.y, smem_raw);
}

// Batched blends of frames with pairwise disjoint footprints (the order of
// their updates is then irrelevant): one launch over all frames' CTAs.
template <int MODE>
__global__ void __launch_bounds__(NT, K1Shape<MODE>::MINB)
k_node_field_batch(const NfBatchFrame* __restrict__ F, int nf, const NfPlan* __restrict__ plans) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int NH = K1Shape<MODE>::NH;
    pdl_wait();
    int f = 0;
    while (f + 1 < nf && (int)blockIdx.x >= F[f + 1].cta_off) ++f;
    const NfBatchFrame& fr = F[f];
    if (fr.L.ctm_ok && threadIdx.x == 0) {
        // the frame table's tensor maps were copied in by the host: acquire
        // them for the TMA unit (its descriptor cache may hold this address's
        // maps from an earlier call)
#pragma unroll
        for (int k = 0; k < 4; ++k)
            asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;\n" ::"l"(&fr.L.ctm[k]) : "memory");
    }
    const int lc = (int)blockIdx.x - fr.cta_off, per_row = fr.ntx * NH;
    nf_field_cta<MODE>(fr.L, plans + fr.plan_off, fr.ti0, fr.tj0, fr.s1, 0, fr.ntx, lc % per_row, lc / per_row,
                       smem_raw);
}

// Exact-tier resolution of queued pixels (mosaic.hpp:243-283 semantics), one
// CTA. It then writes BlendStats (footprint + partial sums) and restores the
// per-context state (acc = 0, exc_count = 0) for the next call.
// Warp-cooperative pixel_warp (mosaic.hpp:22-51) for one pixel: lanes
// evaluate the node weights in parallel (exact tier), then every lane sums the
// contributors' products in ascending node order -- the reference's order, so
// the result is bit-identical -- with shuffles. All lanes end with the result.
// stage: optional per-warp shared scratch (32 x 6 doubles) for the ordered sum.
__device__ int xpixel_warp_warp(double x, double y, const double* __restrict__ anchors,
                                const double* __restrict__ warps, const int* __restrict__ src, int n, double alpha,
                                W5* out, double* stage = nullptr) {
    constexpr int KC = NRM_EXC_KC;  // node chunks whose weights are evaluated together
    const int lane = threadIdx.x & 31;
    const double na = -alpha;
    double wsum = 0.0, aw = 0.0, az = 0.0, adx = 0.0, ady = 0.0, as = 0.0;
    double accj = 0.0;  // staged path: lane j < 6 keeps sum j (aw, az, adx, ady, as, wsum)
    double ref_w = 0.0, ref_z = 0.0;
    bool have_ref = false;
    for (int g0 = 0; g0 < n; g0 += 32 * KC) {
        double w[KC], q[KC][5];
        bool contrib[KC];
#pragma unroll
        for (int c = 0; c < KC; ++c) {  // independent: loads and exps overlap
            const int e = g0 + 32 * c + lane;
            w[c] = 0.0;
            contrib[c] = false;
#pragma unroll
            for (int k = 0; k < 5; ++k) q[c][k] = 0.0;
            if (e < n) {
                const int i = src ? src[e] : e;  // src: index-ordered subset
                const double d2 = xdist2(__ldg(&anchors[2 * i]), __ldg(&anchors[2 * i + 1]), x, y);
                w[c] = xexp(xmul(na, d2));
                contrib[c] = !(w[c] <= kPixelWeightCutoff);
#pragma unroll
                for (int k = 0; k < 5; ++k) q[c][k] = __ldg(&warps[5 * i + k]);
            }
        }
#pragma unroll
        for (int c = 0; c < KC; ++c) {  // ordered accumulation, chunk by chunk
            const unsigned m = __ballot_sync(0xffffffffu, contrib[c]);
            if (!m) continue;
            double* qc = q[c];
            if (!have_ref) {  // first contributing node in index order
                const int sl = __ffs(m) - 1;
                ref_w = __shfl_sync(0xffffffffu, qc[1], sl);
                ref_z = __shfl_sync(0xffffffffu, qc[2], sl);
                have_ref = true;
                if (lane != sl && xadd(xmul(qc[1], ref_w), xmul(qc[2], ref_z)) < 0.0) {
                    qc[1] = -qc[1]; qc[2] = -qc[2]; qc[3] = -qc[3]; qc[4] = -qc[4];
                }
            } else if (xadd(xmul(qc[1], ref_w), xmul(qc[2], ref_z)) < 0.0) {
                qc[1] = -qc[1]; qc[2] = -qc[2]; qc[3] = -qc[3]; qc[4] = -qc[4];
            }
            if (stage) {
                // contributors' terms in index order through shared memory; lane j
                // < 6 adds term j of each in turn (the same sequence of rounded
                // adds per sum, the six sums' latency chains side by side)
                if (contrib[c]) {
                    double* d = stage + 6 * __popc(m & ((1u << lane) - 1u));
                    d[0] = xmul(w[c], qc[1]);
                    d[1] = xmul(w[c], qc[2]);
                    d[2] = xmul(w[c], qc[3]);
                    d[3] = xmul(w[c], qc[4]);
                    d[4] = xmul(w[c], qc[0]);
                    d[5] = w[c];
                }
                __syncwarp();
                if (lane < 6) {
                    const int cnt = __popc(m);
#pragma unroll 8
                    for (int e = 0; e < cnt; ++e) accj = xadd(accj, stage[6 * e + lane]);
                }
                __syncwarp();
                continue;
            }
            const double p0 = xmul(w[c], qc[1]), p1 = xmul(w[c], qc[2]), p2 = xmul(w[c], qc[3]);
            const double p3 = xmul(w[c], qc[4]), p4 = xmul(w[c], qc[0]);
            for (unsigned mm = m; mm; mm &= mm - 1) {
                const int jl = __ffs(mm) - 1;
                aw = xadd(aw, __shfl_sync(0xffffffffu, p0, jl));
                az = xadd(az, __shfl_sync(0xffffffffu, p1, jl));
                adx = xadd(adx, __shfl_sync(0xffffffffu, p2, jl));
                ady = xadd(ady, __shfl_sync(0xffffffffu, p3, jl));
                as = xadd(as, __shfl_sync(0xffffffffu, p4, jl));
                wsum = xadd(wsum, __shfl_sync(0xffffffffu, w[c], jl));
            }
        }
    }
    if (stage) {  // lanes 0..5 hold the sums
        aw = __shfl_sync(0xffffffffu, accj, 0);
        az = __shfl_sync(0xffffffffu, accj, 1);
        adx = __shfl_sync(0xffffffffu, accj, 2);
        ady = __shfl_sync(0xffffffffu, accj, 3);
        as = __shfl_sync(0xffffffffu, accj, 4);
        wsum = __shfl_sync(0xffffffffu, accj, 5);
    }
    XPW s{wsum, aw, az, adx, ady, as, ref_w, ref_z, have_ref};
    return xpw_finish(s, out);
}

// Queued pixel q of launch L, resolved by one warp in the exact tier. Returns
// (valid in lane 0) 0 blended, 1 no support, 2 out of frame, -1 (field mode).
template <int MODE>
__device__ __forceinline__ int exc_pixel(const NodeFieldLaunch& L, int2 p, double* stage) {
    const int lane = threadIdx.x & 31;
    const double fxm = L.fw - 1.0, fym = L.fh - 1.0;
    const double x = L.grid.gx + p.x, y = L.grid.gy + p.y;
    W5 wp;
    // the pixel's launch chunk: tile row -> launch row (inverse of tile_row_of)
    const int tjy = floordiv(p.y, TH);
    const int by = L.band_count <= 1 ? tjy - L.tile_j0
                                     : 2 * (((tjy >> 1) - L.band_s1) / L.band_count) + (tjy & 1);
    int nsrc;
    const int tix = floordiv(p.x, TW) - floordiv(L.grid.i0, TW);
    const int* src = chunk_nodes(L, by / L.chunk_rows, tix / NF_GROUP_TILES, &nsrc);
    // blend modes: the pixel's canvas values do not depend on the exact
    // evaluation, so lane 0 issues their loads first and their latency hides
    // behind it (the pass is a latency chain at the end of the K1 stream)
    const long long idx = (long long)(p.y - L.phys_y0) * L.pitch + (p.x - L.phys_x0);
    uint8_t wg = 0;
    float cr = 0.f, cg = 0.f, cb = 0.f;
    if (MODE != 1 && lane == 0) {
        wg = L.W[idx];
        cr = L.R[idx];
        cg = L.G[idx];
        cb = L.B[idx];
    }
    const int rc = xpixel_warp_warp(x, y, L.anchors, L.warps, src, nsrc, L.alpha, &wp, stage);
    if (lane != 0) return -1;
    if (MODE == 1) {
        const size_t o = (size_t)(p.y - L.grid.j0) * (L.grid.i1 - L.grid.i0 + 1) + (p.x - L.grid.i0);
        if (rc == 0) {
            double yx, yy;
            xapply(wp, x, y, &yx, &yy);
            if (L.disp) L.disp[o] = make_float2((float)(yx - x), (float)(yy - y));
            if (L.support) L.support[o] = 1;
        } else {
            if (L.disp) L.disp[o] = make_float2(0.f, 0.f);
            if (L.support) L.support[o] = 0;
        }
        return -1;
    }
    if (rc != 0) return 1;
    double yx, yy;
    xapply(wp, x, y, &yx, &yy);
    if (!(yx >= 0.0 && yx <= fxm && yy >= 0.0 && yy <= fym)) return 2;
    double rgb[3];
    xsample_bilinear(L.frame, L.fw, L.fh, L.fch, yx, yy, rgb);
    const double wd = wg;
    // reference operation order, no contraction (mosaic.hpp:278-282); the
    // weighted mode runs the same operations with a = w + 1 - cf, cf <= 1
    double a = wd, cf = 1.0;
    if (MODE == 2) {  // weighted mode (see NodeFieldLaunch::unc)
        cf = 1.0 / fmax(xsample_bilinear_f32(L.unc, L.fw, L.fh, yx, yy), 1.0);
        a = xsub(xadd(wd, 1.0), cf);
    }
    L.R[idx] = (float)(xadd(xmul(a, (double)cr), xmul(cf, rgb[0] / 255.0)) / xadd(wd, 1.0));
    L.G[idx] = (float)(xadd(xmul(a, (double)cg), xmul(cf, rgb[1] / 255.0)) / xadd(wd, 1.0));
    L.B[idx] = (float)(xadd(xmul(a, (double)cb), xmul(cf, rgb[2] / 255.0)) / xadd(wd, 1.0));
    L.W[idx] = wg < kWeightCap ? (uint8_t)(wg + 1) : wg;
    return 0;
}

__device__ __forceinline__ bool band_owns_abs_row(const NodeFieldLaunch& L, int j) {
    return L.band_count <= 1 || posmod(floordiv(j, kStripeRows), L.band_count) == L.band_rank;
}

// Spilled pixels of a launch (queue overflow, see spill_mark): a scan of the
// launch window, one warp per 32 consecutive pixels; each marked pixel is
// unmarked and resolved by the whole warp. `fn(p, r)` receives each result.
template <int MODE, class Fn>
__device__ __forceinline__ void exc_scan(const NodeFieldLaunch& L, double* stage, unsigned gw, unsigned nwarps,
                                         Fn fn) {
    const int lane = threadIdx.x & 31;
    const long long wdt = L.grid.i1 - L.grid.i0 + 1, hgt = L.grid.j1 - L.grid.j0 + 1;
    const long long total = wdt * hgt;
    for (long long base = (long long)gw * 32; base < total; base += (long long)nwarps * 32) {
        const long long e = base + lane;
        int i = 0, j = 0;
        bool mk = false;
        if (e < total) {
            j = L.grid.j0 + (int)(e / wdt);
            i = L.grid.i0 + (int)(e % wdt);
            if (band_owns_abs_row(L, j)) {
                if (MODE == 1) {
                    const size_t o = (size_t)e;
                    if (L.disp) {
                        mk = isnan(L.disp[o].x);
                    } else if (L.support && L.support[o] == 0xFF) {
                        mk = true;
                        L.support[o] = 0;
                    }
                } else {
                    const long long idx = (long long)(j - L.phys_y0) * L.pitch + (i - L.phys_x0);
                    const uint8_t wv = L.W[idx];
                    if (wv & kSpillBit) {
                        mk = true;
                        L.W[idx] = (uint8_t)(wv & (uint8_t)~kSpillBit);
                    }
                }
            }
        }
        unsigned m = __ballot_sync(0xffffffffu, mk);
        __syncwarp();
        while (m) {
            const int l = __ffs(m) - 1;
            m &= m - 1;
            const int2 p = make_int2(__shfl_sync(0xffffffffu, i, l), __shfl_sync(0xffffffffu, j, l));
            fn(exc_pixel<MODE>(L, p, stage));
        }
    }
}

// The deferred pixels of one launch -- the queued ones, then (after a queue
// overflow) the spilled ones -- one warp per pixel spread over the grid;
// returns this thread's partial BlendStats counts (lane 0 of each warp).
template <int MODE>
__device__ __forceinline__ void exc_run(const NodeFieldLaunch& L, double* stage, int& nb, int& nns, int& noof) {
    const unsigned total = *L.exc_count;
    const unsigned cnt = min(total, L.exc_cap);
    const unsigned gw = blockIdx.x * (EXC_THREADS / 32) + (threadIdx.x >> 5), nwarps = gridDim.x * (EXC_THREADS / 32);
    auto tally = [&](int r) {
        nb += r == 0;
        nns += r == 1;
        noof += r == 2;
    };
    for (unsigned q = gw; q < cnt; q += nwarps) tally(exc_pixel<MODE>(L, L.exc[q], stage));
    if (total > L.exc_cap) exc_scan<MODE>(L, stage, gw, nwarps, tally);
}

// Block-sums the partial counts into L.acc (blend modes).
template <int MODE>
__device__ __forceinline__ void exc_accumulate(const NodeFieldLaunch& L, int nb, int nns, int noof,
                                               int (*red)[EXC_THREADS / 32]) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        nb += __shfl_xor_sync(0xffffffffu, nb, o);
        nns += __shfl_xor_sync(0xffffffffu, nns, o);
        noof += __shfl_xor_sync(0xffffffffu, noof, o);
    }
    if (lane == 0) {
        red[0][wid] = nb;
        red[1][wid] = nns;
        red[2][wid] = noof;
    }
    __syncthreads();
    if (threadIdx.x == 0 && MODE != 1) {
        unsigned long long tot[3] = {0, 0, 0};
        for (int k = 0; k < 3; ++k)
            for (int w = 0; w < EXC_THREADS / 32; ++w) tot[k] += (unsigned long long)red[k][w];
        for (int k = 0; k < 3; ++k)
            if (tot[k]) atomicAdd(&L.acc[k], tot[k]);
    }
    __syncthreads();
}

// BlendStats and the per-launch state reset (one thread of the last CTA).
template <int MODE>
__device__ __forceinline__ void exc_finalize(const NodeFieldLaunch& L) {
    if (MODE != 1) {
        volatile unsigned long long* acc = L.acc;
        if (L.stats_out) {
            L.stats_out[0] = L.footprint;
            L.stats_out[1] = acc[0];
            L.stats_out[2] = acc[1];
            L.stats_out[3] = acc[2];
        }
        acc[0] = acc[1] = acc[2] = 0;
    }
    if (L.exc_last) *L.exc_last = *L.exc_count;  // queued + spilled
    if (L.exc_overflow && *L.exc_count > L.exc_cap) atomicAdd(L.exc_overflow, 1u);  // diagnostics: spilled launches
    *L.exc_count = 0;
}

template <int MODE>
__global__ void __launch_bounds__(EXC_THREADS) k_node_exceptions(NodeFieldLaunch L) {
    __shared__ int red[3][EXC_THREADS / 32];
    __shared__ bool last;
    __shared__ double stage[EXC_THREADS / 32][32 * 6];
    // the exact evaluation's dependent reads of inputs no kernel writes (the
    // exp table, small node arrays) start before the wait for the field grid,
    // so a queued pixel finds them in this SM's L1
    prefetch_l1(reinterpret_cast<const char*>(kExpTab) + 128 * (threadIdx.x & 15));
    if (L.n <= 256) {
        for (int o = 128 * threadIdx.x; o < 16 * L.n; o += 128 * EXC_THREADS)
            prefetch_l1(reinterpret_cast<const char*>(L.anchors) + o);
        for (int o = 128 * threadIdx.x; o < 40 * L.n; o += 128 * EXC_THREADS)
            prefetch_l1(reinterpret_cast<const char*>(L.warps) + o);
    }
    pdl_wait();
    // the field grid triggered this pass early: the next blend's planner
    // (which rewrites the frame texture) may start only once it has finished;
    // it may still overlap this pass (it only reads nodes)
    pdl_trigger();
    int nb = 0, nns = 0, noof = 0;
    exc_run<MODE>(L, stage[threadIdx.x >> 5], nb, nns, noof);
    exc_accumulate<MODE>(L, nb, nns, noof, red);
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(L.exc_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    // the last CTA finalises BlendStats and restores the per-context state
    if (last && threadIdx.x == 0) {
        __threadfence();
        exc_finalize<MODE>(L);
        *L.exc_done = 0;
    }
}

// Exact pass of a batched blend: the queued pixels of all frames spread over
// all warps (one warp per pixel; counts go straight to each frame's counters),
// then the last CTA finalises every frame's BlendStats.
template <int MODE>
__global__ void __launch_bounds__(EXC_THREADS) k_node_exceptions_batch(const NfBatchFrame* __restrict__ F, int nf) {
    __shared__ unsigned pre[17];  // prefix sums of the queue lengths (nf <= 16)
    __shared__ bool last;
    __shared__ double stage[EXC_THREADS / 32][32 * 6];
    pdl_trigger();
    pdl_wait();
    if (threadIdx.x == 0) {
        pre[0] = 0u;
        for (int f = 0; f < nf; ++f) pre[f + 1] = pre[f] + min(*F[f].L.exc_count, F[f].L.exc_cap);
    }
    __syncthreads();
    const unsigned total = pre[nf];
    const unsigned gw = blockIdx.x * (EXC_THREADS / 32) + (threadIdx.x >> 5), nwarps = gridDim.x * (EXC_THREADS / 32);
    for (unsigned i = gw; i < total; i += nwarps) {
        int f = 0;
        while (i >= pre[f + 1]) ++f;
        const NodeFieldLaunch& L = F[f].L;
        const int r = exc_pixel<MODE>(L, L.exc[i - pre[f]], stage[threadIdx.x >> 5]);
        if (MODE != 1 && r >= 0) atomicAdd(&L.acc[r], 1ull);
    }
    for (int f = 0; f < nf; ++f) {  // spilled pixels of frames whose queue overflowed
        const NodeFieldLaunch& L = F[f].L;
        if (*L.exc_count <= L.exc_cap) continue;
        exc_scan<MODE>(L, stage[threadIdx.x >> 5], gw, nwarps, [&](int r) {
            if (MODE != 1 && r >= 0) atomicAdd(&L.acc[r], 1ull);
        });
    }
    __syncthreads();
    unsigned* done = F[0].L.exc_done;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        for (int f = 0; f < nf; ++f) exc_finalize<MODE>(F[f].L);
        *done = 0;
    }
}

__global__ void k_pixel_warp_points(const double* __restrict__ pts, int npts,
                                    const double* __restrict__ anchors,
                                    const double* __restrict__ warps, int n, double alpha,
                                    double* __restrict__ out, uint8_t* __restrict__ valid) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= npts) return;
    W5 wp;
    const int rc = xpixel_warp(pts[2 * k], pts[2 * k + 1], anchors, warps, n, alpha, &wp);
    valid[k] = rc == 0 ? 1 : (rc == 2 ? 2 : 0);
    double* o = &out[5 * k];
    if (rc == 0) {
        o[0] = wp.s; o[1] = wp.w; o[2] = wp.z; o[3] = wp.dx; o[4] = wp.dy;
    } else {
        o[0] = o[1] = o[2] = o[3] = o[4] = 0.0;
    }
}

// invert_frame_boundary (mosaic.hpp:58-96): poly holds the frame-boundary
// samples on entry (generated on the host by the reference's own loops) and
// their preimages on exit.
__global__ void k_invert_boundary(const double* __restrict__ anchors,
                                  const double* __restrict__ warps, int n, double alpha,
                                  double* __restrict__ poly, int ns) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ns) return;
    const double yx = poly[2 * k], yy = poly[2 * k + 1];
    int nearest = 0;
    double best = 1.7976931348623157e308, px_n = 0.0, py_n = 0.0;
    for (int i = 0; i < n; ++i) {
        const W5 q = load_w5(&warps[5 * i]);
        double px, py;
        xapply(q, anchors[2 * i], anchors[2 * i + 1], &px, &py);
        const double d2 = xdist2(px, py, yx, yy);
        if (d2 < best) {
            best = d2;
            nearest = i;
            px_n = px;
            py_n = py;
        }
    }
    double x0 = yx, y0 = yy;
    if (n > 0) {
        x0 = xadd(anchors[2 * nearest], xsub(yx, px_n));
        y0 = xadd(anchors[2 * nearest + 1], xsub(yy, py_n));
    }
    for (int it = 0; it < 15; ++it) {
        W5 wp;
        if (xpixel_warp(x0, y0, anchors, warps, n, alpha, &wp) != 0) break;
        double nx, ny;
        if (!xunapply(wp, yx, yy, &nx, &ny)) break;
        const double move = sqrt(xdist2(nx, ny, x0, y0));
        x0 = nx;
        y0 = ny;
        if (move < 1e-7) break;
    }
    poly[2 * k] = x0;
    poly[2 * k + 1] = y0;
}

__global__ void k_selftest_libm(const double* __restrict__ x, const double* __restrict__ y, int n,
                                double* __restrict__ ex, double* __restrict__ hy) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    ex[k] = xexp(x[k]);
    hy[k] = xhypot(x[k], y[k]);
}

}  // namespace

cudaError_t launch_selftest_libm(const double* x, const double* y, int n, double* ex, double* hy,
                                 cudaStream_t st, int64_t* launches) {
    if (n <= 0) return cudaSuccess;
    prof_mark("k_selftest_libm", st);
    k_selftest_libm<<<(n + 255) / 256, 256, 0, st>>>(x, y, n, ex, hy);
    ++*launches;
    return cudaGetLastError();
}

// Launch geometry shared by the scratch sizing and the launcher.
struct NfGeom {
    int ti0, ti1, tj0, tj1, ntx, nty, s1, chunk_rows, nchunks;
};
NfGeom nf_geom(const NodeFieldLaunch& L) {
    NfGeom g;
    g.ti0 = floordiv(L.grid.i0, TW);
    g.ti1 = floordiv(L.grid.i1, TW);
    g.tj0 = floordiv(L.grid.j0, TH);
    g.tj1 = floordiv(L.grid.j1, TH);
    g.ntx = g.ti1 - g.ti0 + 1;
    g.nty = g.tj1 - g.tj0 + 1;
    g.s1 = 0;
    if (L.band_count > 1) {
        const int stripe_lo = floordiv(g.tj0 * TH, kStripeRows);
        g.s1 = stripe_lo + posmod(L.band_rank - stripe_lo, L.band_count);
        int cnt = 0;
        for (int by = 0;; ++by) {
            const int s = g.s1 + (by >> 1) * L.band_count;
            const int row = 2 * s + (by & 1);
            if (row > g.tj1) break;
            cnt = by + 1;
        }
        g.nty = cnt;
    }
    g.chunk_rows = g.ntx > 0 ? max(1, NF_CHUNK_TILES / g.ntx) : 1;
    g.nchunks = (g.ntx > 0 && g.nty > 0) ? (g.nty + g.chunk_rows - 1) / g.chunk_rows : 0;
    return g;
}
constexpr int kPrefilterMinNodes = 257;  // small lattices: every node reaches every tile anyway

size_t node_field_scratch_bytes(const NodeFieldLaunch& L) {
    const NfGeom g = nf_geom(L);
    size_t b = (size_t)NF_CHUNK_TILES * sizeof(NfPlan);
    const size_t nl = (size_t)g.nchunks * (size_t)((g.ntx + NF_GROUP_TILES - 1) / NF_GROUP_TILES);
    if (L.n >= kPrefilterMinNodes) b += (nl * (size_t)L.n + nl + 64) * sizeof(int);
    return b;
}

cudaError_t launch_node_field(const NodeFieldLaunch& L0, int mode, cudaStream_t st, int64_t* launches) {
    const NfGeom g = nf_geom(L0);
    NodeFieldLaunch L = L0;
    L.chunk_rows = g.chunk_rows;
    L.tile_j0 = g.tj0;
    L.band_s1 = g.s1;
    NfPlan* plans = static_cast<NfPlan*>(L.plans);
    if (L.n >= kPrefilterMinNodes && g.nchunks > 0) {
        L.lstride = L.n;
        L.col_groups = (g.ntx + NF_GROUP_TILES - 1) / NF_GROUP_TILES;
        L.lists = reinterpret_cast<int*>(reinterpret_cast<char*>(L.plans) + (size_t)NF_CHUNK_TILES * sizeof(NfPlan));
        L.lcounts = L.lists + (size_t)g.nchunks * L.col_groups * L.lstride;
    }
    const size_t base = canvas_tile_offset<K1Shape<0>::CW>();
#ifndef NRM_K2_MMASYNC
    const size_t smem_k2 = sizeof(SmemTC);
#else
    const size_t smem_k2 = sizeof(Smem<K1Shape<1>::CW>);
#endif
    const size_t smem = mode != 1 ? base + sizeof(CanvasTile) : smem_k2;
    const int nh = mode == 1 ? K1Shape<1>::NH : K1Shape<0>::NH;
    const int kmode = mode == 1 ? 1 : (L.unc ? 2 : 0);  // 2: uncertainty-weighted blend
    auto k_field = kmode == 0 ? k_node_field<0> : (kmode == 1 ? k_node_field<1> : k_node_field<2>);
    auto k_exc = kmode == 0 ? k_node_exceptions<0> : (kmode == 1 ? k_node_exceptions<1> : k_node_exceptions<2>);
    if (L.lists) {  // all chunks' node lists in one launch
        prof_mark("k_nf_prefilter", st);
        k_nf_prefilter<<<dim3(L.col_groups, g.nchunks), PF_THREADS, 0, st>>>(L, g.ti0, g.ti1, g.tj1, g.nty);
        ++*launches;
    }
    cudaFuncSetAttribute(k_field, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int ci = 0; ci < g.nchunks; ++ci) {
        const int by0 = ci * g.chunk_rows;
        const int rows = min(g.chunk_rows, g.nty - by0);
        if ((size_t)rows * g.ntx > (size_t)NF_CHUNK_TILES) return cudaErrorInvalidValue;  // ntx > chunk
        prof_mark("k_nf_plan", st);
        const int conv = (ci == 0 && L.frgba) ? NF_CONV_BLOCKS : 0;
        cudaError_t e = launch_pdl(k_nf_plan, dim3((rows * g.ntx + NF_PLAN_WARPS - 1) / NF_PLAN_WARPS + conv),
                                   dim3(NF_PLAN_WARPS * 32), 0, st, L, plans, g.ti0, g.tj0, g.tj1, g.s1, by0, rows,
                                   g.ntx, conv);
        ++*launches;
        if (e != cudaSuccess) return e;
        prof_mark("k_node_field", st);
        e = launch_pdl(k_field, dim3(nh * g.ntx, rows), dim3(NT), smem, st, L,
                                         static_cast<const NfPlan*>(plans), g.ti0, g.tj0, g.s1, by0, g.ntx,
                                         ci == g.nchunks - 1 ? 1 : 0);
        ++*launches;
        if (e != cudaSuccess) return e;
    }
    prof_mark("k_node_exceptions", st);
    const cudaError_t e = launch_pdl(k_exc, dim3(EXC_BLOCKS), dim3(EXC_THREADS), 0, st, L);
    ++*launches;
    return e;
}

size_t node_field_batch_scratch_bytes(int nf) {
    return (((size_t)nf * sizeof(NfBatchFrame) + 255) & ~size_t(255)) + (size_t)NF_CHUNK_TILES * sizeof(NfPlan);
}

cudaError_t launch_node_field_batch(const NodeFieldLaunch* Ls, int nf, void* scratch, cudaStream_t st,
                                    int64_t* launches) {
    std::vector<NfBatchFrame> F((size_t)nf);
    int tiles = 0, ctas = 0;
    for (int f = 0; f < nf; ++f) {
        const NfGeom g = nf_geom(Ls[f]);
        if (g.nchunks > 1 || Ls[f].n >= kPrefilterMinNodes) return cudaErrorNotSupported;
        NfBatchFrame& fr = F[f];
        fr.L = Ls[f];
        fr.L.chunk_rows = g.chunk_rows;
        fr.L.tile_j0 = g.tj0;
        fr.L.band_s1 = g.s1;
        fr.L.lists = nullptr;
        fr.ti0 = g.ti0;
        fr.tj0 = g.tj0;
        fr.tj1 = g.tj1;
        fr.s1 = g.s1;
        fr.ntx = g.nchunks ? g.ntx : 0;
        fr.rows = g.nchunks ? g.nty : 0;
        fr.plan_off = tiles;
        fr.cta_off = ctas;
        tiles += fr.rows * fr.ntx;
        ctas += fr.rows * fr.ntx * K1Shape<0>::NH;
    }
    if (tiles > NF_CHUNK_TILES) return cudaErrorNotSupported;
    NfBatchFrame* dF = static_cast<NfBatchFrame*>(scratch);
    NfPlan* plans = reinterpret_cast<NfPlan*>(static_cast<char*>(scratch) +
                                              (((size_t)nf * sizeof(NfBatchFrame) + 255) & ~size_t(255)));
    cudaError_t e = cudaMemcpyAsync(dF, F.data(), (size_t)nf * sizeof(NfBatchFrame), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    if (tiles > 0) {
        prof_mark("k_nf_plan", st);
        e = launch_pdl(k_nf_plan_batch, dim3((tiles + NF_PLAN_WARPS - 1) / NF_PLAN_WARPS), dim3(NF_PLAN_WARPS * 32),
                       0, st, static_cast<const NfBatchFrame*>(dF), nf, plans, tiles);
        ++*launches;
        if (e != cudaSuccess) return e;
        const size_t smem = canvas_tile_offset<K1Shape<0>::CW>() + sizeof(CanvasTile);
        cudaFuncSetAttribute(k_node_field_batch<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        prof_mark("k_node_field", st);
        e = launch_pdl(k_node_field_batch<0>, dim3(ctas), dim3(NT), smem, st, static_cast<const NfBatchFrame*>(dF),
                       nf, static_cast<const NfPlan*>(plans));
        ++*launches;
        if (e != cudaSuccess) return e;
    }
    prof_mark("k_node_exceptions", st);
    e = launch_pdl(k_node_exceptions_batch<0>, dim3(EXC_BLOCKS), dim3(EXC_THREADS), 0, st,
                   static_cast<const NfBatchFrame*>(dF), nf);
    ++*launches;
    return e;
}

cudaError_t launch_pixel_warp_points(const double* pts, int npts, const double* anchors,
                                     const double* warps, int n, double alpha, double* out,
                                     uint8_t* valid, cudaStream_t st, int64_t* launches) {
    if (npts <= 0) return cudaSuccess;
    prof_mark("k_pixel_warp_points", st);
    k_pixel_warp_points<<<(npts + 127) / 128, 128, 0, st>>>(pts, npts, anchors, warps, n, alpha, out, valid);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_invert_boundary(int, int, const double* anchors, const double* warps, int n,
                                   double alpha, double, double* poly, int nsamples,
                                   cudaStream_t st, int64_t* launches) {
    if (nsamples <= 0) return cudaSuccess;
    prof_mark("k_invert_boundary", st);
    k_invert_boundary<<<(nsamples + 63) / 64, 64, 0, st>>>(anchors, warps, n, alpha, poly, nsamples);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace nrm
