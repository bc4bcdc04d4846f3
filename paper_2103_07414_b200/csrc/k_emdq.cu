// k_emdq.cu -- K3: dense EMDQ field + per-pixel uncertainty.
//
// Per grid pixel p (SURVEY §8c route):
//   field(p) = detail::blend_local(locals, apts, probs, active, p, alpha, S)(p)
//              (fieldest.hpp:75-97: the S nearest candidates by (d^2, j),
//               w = exp(-alpha (d^2 - d2min)) * max(prob, 1e-6), dq_blend
//               with the nearest as hemisphere reference, dualquat.hpp:133-162)
//   unc(p)   = node_uncertainty(p, apts[active], beta) = bounded_exp(beta d2min)
//              (fieldest.hpp:44-52; the nearest inlier is the kNN's first).
//
// The kNN membership decides which warps are blended, so it must equal the
// reference's exactly. Design:
//   k_super (64 x 64 supertiles): a 256-bin histogram of squared centre
//     distances bounds the S-th neighbour distance R; every point that can be
//     among the S nearest of a supertile pixel lies within R + 2 hd of its
//     centre. Those points form the supertile list (plus a rotation-arc flag).
//   k_plan (one warp per 16 x 16 tile, no block barriers): the same bound
//     over the supertile list, then an FP64 classification of the tile's
//     candidates against the tile rectangle: "in" (fewer than S others can
//     ever be closer), "out" (at least S are always closer) or ambiguous. In
//     and ambiguous ones become packed records in tile-local coordinates with
//     their warps conjugated to the tile origin (T(-P) q T(o)); the ambiguous
//     are then re-classified per 8 x 4 sub-tile (FP32, conservative margins),
//     leaving ~2 free slots per pixel. Plans go to HBM (L2-resident).
//   k_pixels (one CTA per tile, plan staged by one TMA bulk copy, warp =
//     sub-tile, one pixel per thread): one pass over the sure members
//     accumulating weighted warps (weights on MUFU.EX2 relative to a
//     tile-wide d^2 floor: the common factor cancels in dq_blend's
//     normalisation), an early-reject sorted insertion of the ambiguous
//     (closest first) into the m = S - |in| free slots, their accumulation and
//     the epilogue. When the selected and rejected boundary keys are within
//     the FP32 error bound, the pixel is queued for the exact tier.
//   k_emdq_exceptions (after each chunk's k_pixels): the queued pixels, a
//     warp per pixel, in the exact tier (FP64, reference operation order and
//     libm: the kNN set and blend are bit-identical to the reference's).
//   Tiles whose candidates span more than a quarter turn of rotation
//   (hemisphere flips possible) or overflow a capacity run the exact tier in
//   k_pixels, a thread per pixel.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>

#include "nrm_common.cuh"
#include "nrm_internal.h"

namespace nrm {
namespace {

constexpr int ET = 16;            // tile edge
constexpr int ENT = ET * ET;      // threads
constexpr int NW = ENT / 32;      // warps
constexpr int CAND_CAP = 512;     // tile candidates
constexpr int SCAP = 192;         // staged (in + ambiguous) per tile
constexpr int MAX_SUPPORT = 32;
constexpr int ST = 64;            // supertile edge (4 x 4 tiles)
constexpr int WCAP_S = 256;       // per-warp gather capacity in the supertile pass
constexpr int SLIST_CAP = 1024;   // supertile list capacity
constexpr int SFLAG_OVERFLOW = 1, SFLAG_NONUNIFORM = 2;
// tile plans per launch chunk (4 KB each): a 4K frame (32,400 tiles) in one
// chunk, so one k_plan / k_pixels / exception-pass tail instead of two
// (C4 694 -> 687 us, C5 1105 -> 1090 us against 16,384)
#ifndef NRM_EMDQ_CHUNK_TILES
#define NRM_EMDQ_CHUNK_TILES 32768
#endif
constexpr int EMDQ_CHUNK_TILES = NRM_EMDQ_CHUNK_TILES;
#ifndef NRM_PIX_MINB
#define NRM_PIX_MINB 4  // k_pixels resident CTAs per SM (register budget: 64)
#endif  // tile plans resident per launch chunk

// Gathered candidate arrays (one entry per active index, in active order).
struct Cand {
    const double* x;
    const double* y;
    const float2* c32;   // coarse absolute coordinates for culling
    const double* l;     // 5 per entry
    const double* p;     // max(prob, 1e-6)
    const double* phi;   // atan2(z, w)
    const int* j;        // original index (reference tie-break)
};

struct SuperLists {
    int* list;   // [nsuper][SLIST_CAP]
    int* count;  // [nsuper]
    int* flag;   // [nsuper]
    int nsx;     // supertiles per row
};

constexpr int TREC = 64;          // staged records per tile (in + ambiguous)
constexpr int TCAND = 128;        // tile candidates before classification
#ifndef NRM_PLAN_WARPS
#define NRM_PLAN_WARPS 4  // 4-tile CTAs: finer than 8 for the last of ~2.3 waves (51.2 -> 48.9 us on C2)
#endif
constexpr int PLAN_WARPS = NRM_PLAN_WARPS;  // planning warps (tiles) per CTA
constexpr int TFLAG_EXACT_SUPER = 1, TFLAG_EXACT_STAGED = 2;
constexpr double kLocalMax = 256.0;    // px: staged tile-local coordinates (|u| < 2^8, ulp 2^-15)
constexpr double kScaleLever = 640.0;  // px: max S |P| for the fast tier (k_nodefield.cu)
constexpr int NEAR_CAP = 8;       // per sub-tile: candidates that can be the nearest

// Per-tile plan written by k_plan, read by k_pixels (one 16 x 16 tile).
struct __align__(16) TileHdr {
    double P[2], Y0[2], e0[2], s0;  // output origin / reference scale (FP64)
    float d2ref, d2top;             // tile-wide d^2 floor / ceiling of the staged points
    int nin, ne, flags, pad;
    unsigned char nx[NW], na[NW];   // per sub-tile: extra sure members, ambiguous
    unsigned char nn[NW];           // per sub-tile: possible-nearest list size (255: scan all)
};

// One tile's plan, contiguous so k_pixels stages it with 16-byte loads.
struct __align__(16) TilePlan {
    TileHdr hdr;
    float4 rec0[TREC];                  // ux, uy (tile-local), prob, s - s0
    float4 rec1[TREC];                  // conjugated dual quaternion
    double2 axy[TREC];                  // absolute coordinates (exact d^2 for the uncertainty)
    int sidx[TREC];                     // candidate indices (exact-tier fallback)
    unsigned char sub[NW][TREC];        // per sub-tile: extra sure, then ambiguous
    unsigned char near[NW][NEAR_CAP];   // per sub-tile: points that can be the nearest
};

struct TilePlans {
    TilePlan* plan;        // [chunk tiles]
    int tx0, ty0, ntx;     // chunk: first tile column/row, tiles per row
};

// Per-warp planning scratch.
struct PlanWarp {
    int hist[256];
    int cand[TCAND];
    double dmin2[TCAND], dmax2[TCAND], dc2[TCAND];  // dmin2: float2 bounds; dmax2: ambiguous keys
    unsigned char cls[TCAND];
    int sidx[TREC];
    float2 wd[TREC];
    float ux[TREC], uy[TREC];
    unsigned char wcls[TREC];
    float R;
    double ref[7];
};

// Pixel-kernel shared memory (one tile).
struct PixSmem {
    TilePlan p;                        // staged by one TMA bulk copy
    float ex[TREC][ET], ey[TREC][ET];  // separable weights: w = ex[k][col] * ey[k][row]
    unsigned long long bar;            // TMA completion
};
static_assert(sizeof(TilePlan) % 16 == 0, "TMA bulk copies move 16-byte multiples");
struct SSmem {
    int hist[256];
    int wcnt[NW];
    int wcand[NW][WCAP_S];
    double red_lo[NW], red_hi[NW];
    double mincos;
    float R;
};
constexpr int SUPER_CC_CAP = 8192;  // candidates whose coarse coordinates k_super caches in shared memory
#ifndef NRM_SUPER_FUSED_GATHER_MAX
#define NRM_SUPER_FUSED_GATHER_MAX 2048
#endif
constexpr int SUPER_FUSED_GATHER_MAX = NRM_SUPER_FUSED_GATHER_MAX;  // above: a separate k_gather first

// Candidate bins for large candidate sets: 64 px cells on the supertile grid
// plus a margin ring that takes every candidate outside it. EmdqLaunch::
// cell_cnt holds a CTA ticket and count[nc] (persistent-zero), EmdqLaunch::cells start[nc + 1]
// | cursor[nc] | candidate index[N], nc = (nsx + 2) (nsy + 2).
constexpr int BIN_MAX_N = 1 << 17;  // k_super keeps an N-bit membership bitmap in shared memory
struct CellGrid {
    float x0, y0;  // absolute coordinates of supertile (0, 0)'s first pixel
    int nsx, nsy;
};
__host__ __device__ __forceinline__ int cell_count_of(const CellGrid& cg) { return (cg.nsx + 2) * (cg.nsy + 2); }
__device__ __forceinline__ int cell_of(const CellGrid& cg, float2 c) {
    int cx = (int)floorf((c.x - cg.x0) * (1.f / ST)), cy = (int)floorf((c.y - cg.y0) * (1.f / ST));
    cx = min(max(cx, -1), cg.nsx);
    cy = min(max(cy, -1), cg.nsy);
    return (cy + 1) * (cg.nsx + 2) + (cx + 1);
}

// One CTA (the last k_gather CTA to finish): exclusive scan of the cell
// counts into start / cursor; the counts are zeroed for the next call.
__device__ void bin_scan_block(int* __restrict__ cnt, int* __restrict__ cells, int nc, int n) {
    __shared__ int wsum[32];
    __shared__ int carry;
    int* start = cells;
    int* cur = cells + nc + 1;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = blockDim.x >> 5;
    if (t == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nc; base += blockDim.x) {
        const int c = base + t;
        const int v = c < nc ? __ldcg(&cnt[c]) : 0;  // other CTAs' atomics: read at L2
        int x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) wsum[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int w = lane < nw ? wsum[lane] : 0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, w, d);
                if (lane >= d) w += y;
            }
            if (lane < nw) wsum[lane] = w;
        }
        __syncthreads();
        const int excl = carry + (wid > 0 ? wsum[wid - 1] : 0) + x - v;
        if (c < nc) {
            start[c] = excl;
            cur[c] = excl;
            cnt[c] = 0;
        }
        __syncthreads();
        if (t == blockDim.x - 1) carry = excl + v;
        __syncthreads();
    }
    if (t == 0) start[nc] = n;
}

// Candidate indices grouped by cell (the order inside a cell is arbitrary:
// k_super's lists come out in index order through its bitmap).
__global__ void k_bin_scatter(const float2* __restrict__ c32, int n, CellGrid cg, int* __restrict__ cells) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    const int nc = cell_count_of(cg);
    const int pos = atomicAdd(&cells[nc + 1 + cell_of(cg, c32[a])], 1);
    cells[2 * nc + 1 + pos] = a;
}

__device__ __forceinline__ void gather_one(const double* __restrict__ apts, const double* __restrict__ locals,
                                           const double* __restrict__ probs, const int32_t* __restrict__ active,
                                           int a, double* cx, double* cy, float2* c32, double* cl, double* cp,
                                           double* cphi, int* cj, int* cnt, const CellGrid& cg) {
    const int j = active[a];
    const double x = apts[2 * j], y = apts[2 * j + 1];
    cx[a] = x;
    cy[a] = y;
    c32[a] = make_float2((float)x, (float)y);
    if (cnt) atomicAdd(&cnt[1 + cell_of(cg, c32[a])], 1);  // bin counts (zero on entry)
#pragma unroll
    for (int k = 0; k < 5; ++k) cl[5 * a + k] = locals[5 * j + k];
    const double p = probs[j];
    cp[a] = p < 1e-6 ? 1e-6 : p;  // std::max(probs[j], 1e-6)
    cphi[a] = atan2(locals[5 * j + 2], locals[5 * j + 1]);
    cj[a] = j;
}

// cnt (binned calls): [0] a CTA ticket, [1 + cell] the bin counts, both
// persistent-zero; the last CTA scans the counts into `bins`.
__global__ void k_gather(const double* __restrict__ apts, const double* __restrict__ locals,
                         const double* __restrict__ probs, const int32_t* __restrict__ active,
                         int nactive, double* cx, double* cy, float2* c32, double* cl, double* cp,
                         double* cphi, int* cj, int* cnt, int* bins, CellGrid cg) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a < nactive) gather_one(apts, locals, probs, active, a, cx, cy, c32, cl, cp, cphi, cj, cnt, cg);
    if (cnt) {
        __shared__ bool last;
        __syncthreads();  // this CTA's counts are issued
        if (threadIdx.x == 0) {
            __threadfence();
            last = atomicAdd(&cnt[0], 1) == (int)gridDim.x - 1;
        }
        __syncthreads();
        if (last) {
            __threadfence();
            bin_scan_block(cnt + 1, bins, cell_count_of(cg), nactive);
            if (threadIdx.x == 0) cnt[0] = 0;
        }
    }
}

__device__ __forceinline__ bool key_less(double da, int ja, double db, int jb) {
    return da < db || (!(db < da) && ja < jb);
}

__device__ __forceinline__ int hist_bin(float d2) {
    // 8 sub-bins per octave from d2 = 1; bin 0 also takes d2 < 1, 255 the rest.
    const int b = (int)(__float_as_uint(d2) >> 20) - (127 << 3);
    return b < 0 ? 0 : (b > 254 ? 255 : b);
}
__device__ __forceinline__ float bin_upper(int b) { return __uint_as_float((unsigned)(b + 1 + (127 << 3)) << 20); }

// Warp 0: from a 256-bin histogram, an upper bound on the S-th smallest
// squared distance -> R (with slack for the FP32 coarse coordinates).
__device__ __forceinline__ void radius_from_hist(const int* hist, int S, int lane, float* R) {
    int v[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        v[k] = hist[lane * 8 + k];
        sum += v[k];
    }
    int incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += n;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, incl >= S);
    if (hit == 0) {
        if (lane == 0) *R = INFINITY;
        return;
    }
    if (lane == __ffs(hit) - 1) {
        int acc = incl - sum, b = lane * 8 + 7;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            acc += v[k];
            if (acc >= S) {
                b = lane * 8 + k;
                break;
            }
        }
        *R = (b >= 255) ? INFINITY : sqrtf(bin_upper(b)) * 1.0001f + 0.05f;
    }
}

// ---------------------------------------------------------------------------
// Supertile pass: candidate superset + rotation arc for each 64 x 64 block.
// ---------------------------------------------------------------------------
// Gathered candidate arrays written by k_super (the gather is fused into it).
struct GatherOut {
    double *x, *y, *l, *p, *phi;
    float2* c32;
    int* j;
};

// Also gathers the active candidates (grid-stride; k_gather's former job) for
// the later kernels. Its own reads go through `active` directly, since other
// CTAs are writing the gathered arrays concurrently; the values are the same.
// gathered: the candidates were gathered by k_gather before this grid (large
// candidate sets): every CTA then reads the contiguous coarse coordinates
// G.c32 instead of the active -> apts chain of dependent loads.
__global__ void __launch_bounds__(ENT) k_super(EmdqLaunch L, GatherOut G, SuperLists SL, int S, float pad,
                                              int gathered, CellGrid cg) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_wait();
    SSmem& s = *reinterpret_cast<SSmem*>(smem_raw);
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    // this call's count of exact-tier pixels (k_pixels adds to it)
    if (L.exact_count && t == 0 && blockIdx.x == 0 && blockIdx.y == 0) *L.exact_count = 0u;
    if (!gathered) {
        const int nb = gridDim.x * gridDim.y;
        for (int a = (blockIdx.y * gridDim.x + blockIdx.x) * ENT + t; a < L.nactive; a += nb * ENT) {
            const int j = L.active[a];
            const double x = L.apts[2 * j], y = L.apts[2 * j + 1];
            G.x[a] = x;
            G.y[a] = y;
            G.c32[a] = make_float2((float)x, (float)y);
#pragma unroll
            for (int k = 0; k < 5; ++k) G.l[5 * a + k] = L.locals[5 * j + k];
            const double p = L.probs[j];
            G.p[a] = p < 1e-6 ? 1e-6 : p;  // std::max(probs[j], 1e-6)
            G.phi[a] = atan2(L.locals[5 * j + 2], L.locals[5 * j + 1]);
            G.j[a] = j;
        }
    }
    const int N = L.nactive;
    // coarse coordinates of every candidate, cached in shared memory (one
    // pass of dependent global loads instead of two)
    float2* cc = !L.cells && N <= SUPER_CC_CAP
                     ? reinterpret_cast<float2*>(smem_raw + ((sizeof(SSmem) + 15) & ~size_t(15)))
                     : nullptr;
    auto coarse_g = [&](int a) {
        if (gathered) return G.c32[a];
        const int j = L.active[a];
        return make_float2((float)L.apts[2 * j], (float)L.apts[2 * j + 1]);
    };
    if (cc)
        for (int a = t; a < N; a += ENT) cc[a] = coarse_g(a);
    auto coarse = [&](int a) { return cc ? cc[a] : coarse_g(a); };
    auto phi_of = [&](int a) {
        const int j = L.active[a];
        return atan2(L.locals[5 * j + 2], L.locals[5 * j + 1]);
    };
    const int sid = blockIdx.y * SL.nsx + blockIdx.x;
    const int i0 = L.grid.i0 + blockIdx.x * ST, j0 = L.grid.j0 + blockIdx.y * ST;
    const int i1 = min(i0 + ST - 1, L.grid.i1), j1 = min(j0 + ST - 1, L.grid.j1);
    const double xlo = L.grid.gx + i0, xhi = L.grid.gx + i1, ylo = L.grid.gy + j0, yhi = L.grid.gy + j1;
    const float cx = (float)(0.5 * (xlo + xhi)), cy = (float)(0.5 * (ylo + yhi));
    const float hd = (float)(0.5 * sqrt((xhi - xlo) * (xhi - xlo) + (yhi - ylo) * (yhi - ylo)));

    s.hist[t] = 0;
    // per-warp contiguous chunks keep the list order deterministic
    const int per = (N + NW - 1) / NW;
    const int a0 = wid * per, a1 = min(N, a0 + per);
    int cnt = 0;
    if (L.cells) {
        // Binned: the same histogram bin of the S-th nearest and the same list
        // as the full scans below, from the cells near the supertile only.
        const int ncx = cg.nsx + 2, ncy = cg.nsy + 2, nc = ncx * ncy;
        const int* cstart = L.cells;
        const int* cidx = L.cells + 2 * nc + 1;
        unsigned* bits = reinterpret_cast<unsigned*>(smem_raw + ((sizeof(SSmem) + 15) & ~size_t(15)));
        for (int w = t; w < (N + 31) / 32; w += ENT) bits[w] = 0u;
        const int scx = blockIdx.x + 1, scy = blockIdx.y + 1;
        // (a) ring search: the smallest square of (2r + 1)^2 cells around the
        //     supertile holding >= S candidates bounds the S-th nearest by the
        //     square's far corner (rho); a non-empty margin cell in the square
        //     (candidates outside the grid, unbounded) or too few: rho = inf
        if (wid == 0) {
            int cum = 0, r = 0;
            bool unbounded = false;
            for (;; ++r) {
                int c = 0;
                for (int dy = -r + lane; dy <= r; dy += 32) {
                    const int y = scy + dy;
                    if (y < 0 || y >= ncy) continue;
                    const int xl = max(scx - r, 0), xh = min(scx + r, ncx - 1);
                    auto cell_n = [&](int x) { return cstart[y * ncx + x + 1] - cstart[y * ncx + x]; };
                    auto margin = [&](int x) { return x == 0 || x == ncx - 1 || y == 0 || y == ncy - 1; };
                    if (dy == -r || dy == r) {
                        const int n = cstart[y * ncx + xh + 1] - cstart[y * ncx + xl];
                        c += n;
                        if (n > 0)
                            for (int x = xl; x <= xh; ++x) unbounded |= margin(x) && cell_n(x) > 0;
                    } else {
                        if (scx - r >= 0) {
                            c += cell_n(scx - r);
                            unbounded |= margin(scx - r) && cell_n(scx - r) > 0;
                        }
                        if (scx + r < ncx) {
                            c += cell_n(scx + r);
                            unbounded |= margin(scx + r) && cell_n(scx + r) > 0;
                        }
                    }
                }
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
                cum += c;
                if (cum >= S || (scx - r <= 0 && scy - r <= 0 && scx + r >= ncx - 1 && scy + r >= ncy - 1)) break;
            }
            unbounded = __any_sync(0xffffffffu, unbounded) || cum < S;
            if (lane == 0) {
                float rho = INFINITY;
                if (!unbounded) {
                    const float sx0 = cg.x0 + ST * (float)(blockIdx.x - r), sx1 = cg.x0 + ST * (float)(blockIdx.x + r + 1);
                    const float sy0 = cg.y0 + ST * (float)(blockIdx.y - r), sy1 = cg.y0 + ST * (float)(blockIdx.y + r + 1);
                    const float dxm = fmaxf(cx - sx0, sx1 - cx), dym = fmaxf(cy - sy0, sy1 - cy);
                    rho = sqrtf(dxm * dxm + dym * dym) + 2.f;
                }
                s.R = rho;  // (reused: the scan radius, then the list radius)
            }
        }
        __syncthreads();
        // the cell rows and columns a disc of radius rad around the centre touches
        auto window = [&](float rad, int& x_lo, int& x_hi, int& y_lo, int& y_hi) {
            if (!(rad < 1e30f)) {
                x_lo = 0, x_hi = ncx - 1, y_lo = 0, y_hi = ncy - 1;
                return;
            }
            x_lo = max(0, (int)floorf((cx - rad - cg.x0) * (1.f / ST)) + 1 - 1);
            x_hi = min(ncx - 1, (int)floorf((cx + rad - cg.x0) * (1.f / ST)) + 1 + 1);
            y_lo = max(0, (int)floorf((cy - rad - cg.y0) * (1.f / ST)) + 1 - 1);
            y_hi = min(ncy - 1, (int)floorf((cy + rad - cg.y0) * (1.f / ST)) + 1 + 1);
        };
        int x_lo, x_hi, y_lo, y_hi;
        window(s.R, x_lo, x_hi, y_lo, y_hi);
        // (b) histogram over the window: every candidate within rho is in it
        //     and at least S are, so the first bin whose cumulative count
        //     reaches S is the full histogram's
        for (int y = y_lo + wid; y <= y_hi; y += NW) {  // a warp per cell row: the rows' load chains overlap
            const int e0 = cstart[y * ncx + x_lo], e1 = cstart[y * ncx + x_hi + 1];
            for (int e = e0 + lane; e < e1; e += 32) {
                const float2 c = G.c32[cidx[e]];
                const float dx = c.x - cx, dy = c.y - cy;
                atomicAdd(&s.hist[hist_bin(fmaf(dx, dx, dy * dy))], 1);
            }
        }
        __syncthreads();
        if (wid == 0) radius_from_hist(s.hist, S, lane, &s.R);
        __syncthreads();
        const float lim = s.R + 2.f * hd + 1.f + pad, lim2 = lim * lim;
        // (c) membership over the list window (the full scan's test), as bits
        window(lim, x_lo, x_hi, y_lo, y_hi);
        for (int y = y_lo + wid; y <= y_hi; y += NW) {
            const int e0 = cstart[y * ncx + x_lo], e1 = cstart[y * ncx + x_hi + 1];
            for (int e = e0 + lane; e < e1; e += 32) {
                const int a = cidx[e];
                const float2 c = G.c32[a];
                const float dx = c.x - cx, dy = c.y - cy;
                if (!(fmaf(dx, dx, dy * dy) > lim2)) atomicOr(&bits[a >> 5], 1u << (a & 31));
            }
        }
        __syncthreads();
        // (d) each warp's index range, in index order (the full scan's chunks)
        if (a0 < a1) {
            const int wlast = (a1 - 1) >> 5;
            for (int wb = a0 >> 5; wb <= wlast; wb += 32) {
                const int word = wb + lane;
                unsigned b = 0u;
                if (word <= wlast) {
                    b = bits[word];
                    const int lo = word * 32;
                    if (lo < a0) b &= ~0u << (a0 - lo);
                    if (a1 - lo < 32) b &= (1u << (a1 - lo)) - 1u;
                }
                const int nb = __popc(b);
                int incl = nb;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, d);
                    if (lane >= d) incl += y;
                }
                int pos = cnt + incl - nb;
                while (b) {
                    const int k = __ffs(b) - 1;
                    b &= b - 1u;
                    if (pos < WCAP_S) s.wcand[wid][pos] = word * 32 + k;
                    ++pos;
                }
                cnt += __shfl_sync(0xffffffffu, incl, 31);
            }
        }
    } else {
        __syncthreads();
        for (int a = t; a < N; a += ENT) {
            const float2 c = coarse(a);
            const float dx = c.x - cx, dy = c.y - cy;
            atomicAdd(&s.hist[hist_bin(fmaf(dx, dx, dy * dy))], 1);
        }
        __syncthreads();
        if (wid == 0) radius_from_hist(s.hist, S, lane, &s.R);
        __syncthreads();
        const float lim = s.R + 2.f * hd + 1.f + pad, lim2 = lim * lim;
        for (int base = a0; base < a1; base += 32) {
            const int a = base + lane;
            bool keep = false;
            if (a < a1) {
                const float2 c = coarse(a);
                const float dx = c.x - cx, dy = c.y - cy;
                keep = !(fmaf(dx, dx, dy * dy) > lim2);
            }
            const unsigned msk = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const int pos = cnt + __popc(msk & ((1u << lane) - 1u));
                if (pos < WCAP_S) s.wcand[wid][pos] = a;
            }
            cnt += __popc(msk);
        }
    }
    if (lane == 0) s.wcnt[wid] = cnt;
    __syncthreads();
    int off = 0, total = 0;
    for (int w = 0; w < NW; ++w) {
        const int c = s.wcnt[w];
        if (w < wid) off += c;
        total += c;
    }
    bool overflow = total > SLIST_CAP;
    for (int w = 0; w < NW; ++w) overflow |= s.wcnt[w] > WCAP_S;
    if (!overflow) {
        for (int k = lane; k < cnt; k += 32) SL.list[(size_t)sid * SLIST_CAP + off + k] = s.wcand[wid][k];
    }
    // Rotation arc over the list, relative to the first listed point: are
    // all phi = atan2(z, w) within less than a quarter turn? First a
    // conservative test without atan2: every listed real part within
    // pi/4 - 5e-7 of the first one's (cosine of the angle between the (w, z)
    // vectors) bounds the spread below pi/2 - 1e-6. Only tiles that fail it
    // take the exact atan2 pass (the original criterion).
    constexpr double kCosQuarterArc = 0.7071072;  // > cos(pi/4 - 5e-7)
    int first = -1;
    for (int w = 0; w < NW && first < 0; ++w)
        if (s.wcnt[w] > 0) first = s.wcand[w][0];
    double mc = 1.0;
    if (total > 0 && !overflow) {
        const int jf = L.active[first];
        const double w0 = L.locals[5 * jf + 1], z0 = L.locals[5 * jf + 2];
        const double n0 = w0 * w0 + z0 * z0;
        for (int k = lane; k < cnt; k += 32) {
            const int j = L.active[s.wcand[wid][k]];
            const double w = L.locals[5 * j + 1], z = L.locals[5 * j + 2];
            mc = fmin(mc, (w0 * w + z0 * z) / sqrt(n0 * (w * w + z * z)));
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) mc = fmin(mc, __shfl_xor_sync(0xffffffffu, mc, d));
    if (lane == 0) s.red_lo[wid] = mc;
    __syncthreads();
    if (t == 0) {
        for (int w = 0; w < NW; ++w) mc = fmin(mc, s.red_lo[w]);
        s.mincos = mc;
    }
    __syncthreads();
    bool nonuniform = false;
    if (!(s.mincos > kCosQuarterArc) && total > 0 && !overflow) {  // block-uniform
        double lo = 0.0, hi = 0.0;
        const double phi0 = phi_of(first);
        for (int k = lane; k < cnt; k += 32) {
            double rel = phi_of(s.wcand[wid][k]) - phi0;
            if (rel > M_PI) rel -= 2.0 * M_PI;
            if (rel < -M_PI) rel += 2.0 * M_PI;
            lo = fmin(lo, rel);
            hi = fmax(hi, rel);
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, d));
            hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, d));
        }
        __syncthreads();  // red_lo reuse
        if (lane == 0) {
            s.red_lo[wid] = lo;
            s.red_hi[wid] = hi;
        }
        __syncthreads();
        for (int w = 0; w < NW; ++w) {
            lo = fmin(lo, s.red_lo[w]);
            hi = fmax(hi, s.red_hi[w]);
        }
        nonuniform = !((hi - lo) < (0.5 * M_PI - 1e-6));
    }
    if (t == 0) {
        int f = 0;
        if (overflow) f |= SFLAG_OVERFLOW;
        if (nonuniform) f |= SFLAG_NONUNIFORM;
        SL.flag[sid] = f;
        SL.count[sid] = overflow ? N : total;
    }
}

// ---------------------------------------------------------------------------
// Exact tier: detail::blend_local at (qx, qy) over candidate entries
// idx[0..n) (or 0..n when idx is null) in the reference's operation order,
// skipping the candidate whose original index is `excl` (leave-one-out, the
// EM E-step fieldest.hpp:195-209; -1: none). Returns 0 with the blended warp
// and the nearest squared distance, 1 when no candidate remains, 2 when
// dq_blend would throw (no positive weight or a degenerate real part).
// ---------------------------------------------------------------------------
template <int MS>
__device__ int emdq_blend_exact(double qx, double qy, const int* __restrict__ idx, int n, int S, const Cand& C,
                                double alpha, int excl, W5* out, double* d2min_out) {
    double sd[MS];
    int sj[MS], sa[MS];
#pragma unroll
    for (int s = 0; s < MS; ++s) {
        sd[s] = DBL_MAX;
        sj[s] = INT_MAX;
        sa[s] = -1;
    }
    int navail = 0;
    for (int e = 0; e < n; ++e) {
        const int a = idx ? idx[e] : e;
        const int j = C.j[a];
        if (j == excl) continue;
        ++navail;
        const double d2 = xdist2(qx, qy, C.x[a], C.y[a]);
        bool lt[MS];
#pragma unroll
        for (int s = 0; s < MS; ++s) lt[s] = key_less(d2, j, sd[s], sj[s]);
#pragma unroll
        for (int s = MS - 1; s >= 0; --s) {
            if (s < S) {
                if (s > 0 && lt[s - 1]) {
                    sd[s] = sd[s - 1];
                    sj[s] = sj[s - 1];
                    sa[s] = sa[s - 1];
                } else if (lt[s]) {
                    sd[s] = d2;
                    sj[s] = j;
                    sa[s] = a;
                }
            }
        }
    }
    const int kk = min(S, navail);  // std::min(support, cand.size())
    *d2min_out = sd[0];
    if (kk == 0) return 1;
    // dq_blend (dualquat.hpp:133-162) over the sorted kk nearest
    const double d2min = sd[0];
    const double na = -alpha;
    double w[MS];
    double wsum = 0.0;
    int ref = -1;
#pragma unroll
    for (int s = 0; s < MS; ++s) {
        w[s] = 0.0;
        if (s < kk) {
            w[s] = xmul(xexp(xmul(na, xsub(sd[s], d2min))), C.p[sa[s]]);
            if (w[s] > 0.0 && ref < 0) ref = s;
            wsum = xadd(wsum, w[s]);
        }
    }
    double sw = 0.0, sz = 0.0, sdx = 0.0, sdy = 0.0, ss = 0.0;
    double rw = 0.0, rz = 0.0;
#pragma unroll
    for (int s = 0; s < MS; ++s)
        if (s == ref) {
            rw = C.l[5 * sa[s] + 1];
            rz = C.l[5 * sa[s] + 2];
        }
#pragma unroll
    for (int s = 0; s < MS; ++s) {
        if (s < kk && w[s] > 0.0) {
            const double* q = &C.l[5 * sa[s]];
            double qw = q[1], qz = q[2], qdx = q[3], qdy = q[4];
            if (xadd(xmul(qw, rw), xmul(qz, rz)) < 0.0) {
                qw = -qw; qz = -qz; qdx = -qdx; qdy = -qdy;
            }
            sw = xadd(sw, xmul(w[s], qw));
            sz = xadd(sz, xmul(w[s], qz));
            sdx = xadd(sdx, xmul(w[s], qdx));
            sdy = xadd(sdy, xmul(w[s], qdy));
            ss = xadd(ss, xmul(w[s], q[0]));
        }
    }
    if (ref < 0) return 2;
    const double mw = sw / wsum, mz = sz / wsum, mdx = sdx / wsum, mdy = sdy / wsum;
    const double nr = xhypot(mw, mz);
    if (!(nr >= 1e-300)) return 2;
    *out = W5{ss / wsum, mw / nr, mz / nr, mdx / nr, mdy / nr};
    return 0;
}

// Dense-grid exact pixel: displacement (NaN where dq_blend would throw) and
// the uncertainty bounded_exp(beta d2min) (node_uncertainty, fieldest.hpp:44-52).
template <int MS>
__device__ void emdq_exact(double qx, double qy, const int* __restrict__ idx, int n, int S, const Cand& C,
                           double alpha, double beta, float2* out_d, float* out_u) {
    W5 f;
    double d2min;
    const int rc = emdq_blend_exact<MS>(qx, qy, idx, n, S, C, alpha, -1, &f, &d2min);
    float2 dout;
    if (rc == 0) {
        double yx, yy;
        xapply(f, qx, qy, &yx, &yy);
        dout = make_float2((float)(yx - qx), (float)(yy - qy));
    } else {
        dout = make_float2(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
    }
    if (out_d) *out_d = dout;
    if (out_u) {
        double arg = xmul(beta, d2min);
        if (55.0 < arg) arg = 55.0;
        *out_u = (float)xexp(arg);
    }
}

template <int MAXS>
__device__ __noinline__ void exact_dispatch(double qx, double qy, const int* idx, int n, int S, const Cand C,
                                            double alpha, double beta, float2* od, float* ou) {
    if (S <= 16 || MAXS <= 16)
        emdq_exact<16>(qx, qy, idx, n, S, C, alpha, beta, od, ou);
    else
        emdq_exact<MAXS>(qx, qy, idx, n, S, C, alpha, beta, od, ou);
}

// ---------------------------------------------------------------------------
// k_plan: one warp per 16 x 16 tile (no block barriers).
//   radius bound over the supertile list -> candidates -> FP64 in/out/
//   ambiguous classification against the tile -> staged records (in: index
//   order, ambiguous: by centre distance) in tile-local coordinates with
//   conjugated warps -> per 8 x 4 sub-tile refinement of the ambiguous.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(PLAN_WARPS * 32)
k_plan(EmdqLaunch L, Cand C, SuperLists SL, TilePlans TP, int ntiles, int S) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_wait();
    // this chunk's exact-tier queue starts empty (the previous chunk's
    // exception pass, or the previous call's, precedes this grid)
    if (L.exq_count && threadIdx.x == 0 && blockIdx.x == 0) *L.exq_count = 0u;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    PlanWarp& w = reinterpret_cast<PlanWarp*>(smem_raw)[wid];
    const int g = blockIdx.x * PLAN_WARPS + wid;  // tile index within the chunk
    if (g >= ntiles) return;
    const int tx = TP.tx0 + g % TP.ntx, ty = TP.ty0 + g / TP.ntx;
    const int ti0 = L.grid.i0 + tx * ET, tj0 = L.grid.j0 + ty * ET;
    const int ti1 = min(ti0 + ET - 1, L.grid.i1), tj1 = min(tj0 + ET - 1, L.grid.j1);
    const double ox = L.grid.gx + ti0, oy = L.grid.gy + tj0;
    const double xlo = ox, xhi = L.grid.gx + ti1, ylo = oy, yhi = L.grid.gy + tj1;
    const double cxm = 0.5 * (xlo + xhi), cym = 0.5 * (ylo + yhi);
    const double hd = 0.5 * sqrt((xhi - xlo) * (xhi - xlo) + (yhi - ylo) * (yhi - ylo));
    const float cxf = (float)cxm, cyf = (float)cym;
    const int sid = (ty / (ST / ET)) * SL.nsx + tx / (ST / ET);
    const int sflag = SL.flag[sid];
    const int nsrc = SL.count[sid];
    const int* src = (sflag & SFLAG_OVERFLOW) ? nullptr : SL.list + (size_t)sid * SLIST_CAP;
    TilePlan& tp = TP.plan[g];
    TileHdr* hdr = &tp.hdr;
    int flags = 0;

    // 1. radius bound
#pragma unroll
    for (int k = 0; k < 8; ++k) w.hist[lane + 32 * k] = 0;
    __syncwarp();
    for (int e = lane; e < nsrc; e += 32) {
        const float2 c = C.c32[src ? src[e] : e];
        const float dx = c.x - cxf, dy = c.y - cyf;
        atomicAdd(&w.hist[hist_bin(fmaf(dx, dx, dy * dy))], 1);
    }
    __syncwarp();
    radius_from_hist(w.hist, S, lane, &w.R);
    __syncwarp();
    const float lim = w.R + (float)(2.0 * hd) + 1.0f, lim2 = lim * lim;

    // 2. ordered gather
    int nc = 0;
    for (int base = 0; base < nsrc; base += 32) {
        const int e = base + lane;
        int a = -1;
        if (e < nsrc) {
            a = src ? src[e] : e;
            const float2 c = C.c32[a];
            const float dx = c.x - cxf, dy = c.y - cyf;
            if (fmaf(dx, dx, dy * dy) > lim2) a = -1;
        }
        const unsigned msk = __ballot_sync(0xffffffffu, a >= 0);
        if (a >= 0) {
            const int pos = nc + __popc(msk & ((1u << lane) - 1u));
            if (pos < TCAND) w.cand[pos] = a;
        }
        nc += __popc(msk);
    }
    if (nc > TCAND) flags |= TFLAG_EXACT_SUPER;
    nc = min(nc, TCAND);
    __syncwarp();

    // 3. classification against the tile rectangle. The bounds are FP64 and
    //    rounded outwards to FP32 (dmin down, dmax up), and the FP32 margins
    //    (1e-6 relative) dwarf the FP64 rounding of the pixels' exact d^2, so
    //    "in" and "out" stay conservative.
    float2* dmm = reinterpret_cast<float2*>(w.dmin2);  // {dmin^2, dmax^2} per candidate
    for (int k = lane; k < nc; k += 32) {
        const int a = w.cand[k];
        const double ax = C.x[a], ay = C.y[a];
        const double dxn = fmax(fmax(xlo - ax, 0.0), ax - xhi), dyn = fmax(fmax(ylo - ay, 0.0), ay - yhi);
        const double dxf = fmax(ax - xlo, xhi - ax), dyf = fmax(ay - ylo, yhi - ay);
        dmm[k] = make_float2(__double2float_rd(dxn * dxn + dyn * dyn), __double2float_ru(dxf * dxf + dyf * dyf));
        w.dc2[k] = (ax - cxm) * (ax - cxm) + (ay - cym) * (ay - cym);
    }
    __syncwarp();
    for (int k = lane; k < nc; k += 32) {
        const float2 dk = dmm[k];
        const float hi = fmaf(dk.y, 1.000001f, 1e-6f), lo = fmaf(dk.x, 0.999999f, -1e-6f);
        int cle = -1, clt = 0;  // l == k always counts in cle, never in clt
#pragma unroll 4
        for (int l = 0; l < nc; ++l) {
            const float2 dl = dmm[l];
            cle += dl.x <= hi;
            clt += dl.y < lo;
        }
        w.cls[k] = cle < S ? 1 : (clt >= S ? 0 : 2);
    }
    __syncwarp();

    // 4. staging order + tile reference. The ambiguous are staged closest to
    //    the tile centre first (a heuristic order for the pixels' early-reject
    //    insertion, not a correctness property): unique 32-bit keys = FP32
    //    centre distance with the candidate slot in the low 7 bits.
    unsigned* akey = reinterpret_cast<unsigned*>(w.dmax2);
    int* acand = reinterpret_cast<int*>(akey + TCAND);
    int ni = 0, na = 0;
    for (int base = 0; base < nc; base += 32) {
        const int k = base + lane;
        const int c = k < nc ? w.cls[k] : 0;
        const unsigned below = (1u << lane) - 1u;
        const unsigned mi = __ballot_sync(0xffffffffu, c == 1);
        if (c == 1 && ni + __popc(mi & below) < TREC) w.sidx[ni + __popc(mi & below)] = w.cand[k];
        const unsigned ma = __ballot_sync(0xffffffffu, c == 2);
        if (c == 2) {
            akey[na + __popc(ma & below)] = (__float_as_uint((float)w.dc2[k]) & ~127u) | (unsigned)k;
            acand[na + __popc(ma & below)] = w.cand[k];
        }
        ni += __popc(mi);
        na += __popc(ma);
    }
    __syncwarp();
    const int ne = ni + na;
    if (ni > S || ne < S || ne > TREC) flags |= TFLAG_EXACT_SUPER;
    double best = 1e300;
    int bestk = 0x7fffffff;
    if (!(flags & TFLAG_EXACT_SUPER)) {
        for (int e = lane; e < na; e += 32) {
            const unsigned key = akey[e];
            int r = 0;
            for (int l = 0; l < na; ++l) r += akey[l] < key;
            w.sidx[ni + r] = acand[e];
        }
        for (int k = lane; k < nc; k += 32) {
            const int c = w.cls[k];
            const double dk = w.dc2[k];
            if (c != 0 && (dk < best || (dk == best && k < bestk))) {
                best = dk;
                bestk = k;
            }
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const double bd = __shfl_xor_sync(0xffffffffu, best, d);
        const int bk = __shfl_xor_sync(0xffffffffu, bestk, d);
        if (bd < best || (bd == best && bk < bestk)) {
            best = bd;
            bestk = bk;
        }
    }
    if (flags & TFLAG_EXACT_SUPER) {
        if (lane == 0) {
            hdr->flags = flags;
            hdr->ne = 0;
            hdr->nin = 0;
        }
        return;
    }
    if (lane == 0) {
        const W5 qr = load_w5(&C.l[5 * w.cand[bestk]]);
        double yx, yy;
        xapply(qr, ox, oy, &yx, &yy);
        const double Y0 = rint(yx), Y1 = rint(yy);
        const double P0 = Y0 / qr.s, P1 = Y1 / qr.s;
        w.ref[0] = P0;
        w.ref[1] = P1;
        w.ref[2] = Y0;
        w.ref[3] = Y1;
        w.ref[4] = fma(qr.s, P0, -Y0);
        w.ref[5] = fma(qr.s, P1, -Y1);
        w.ref[6] = qr.s;
    }
    __syncwarp();
    const double P0 = w.ref[0], P1 = w.ref[1], s0 = w.ref[6];
    if (!(s0 > 0.0) || !isfinite(P0) || !isfinite(P1)) flags |= TFLAG_EXACT_STAGED;
    if (sflag & SFLAG_NONUNIFORM) flags |= TFLAG_EXACT_STAGED;

    // 5. records (tile-local coordinates, conjugated warps)
    float4* r0g = tp.rec0;
    float4* r1g = tp.rec1;
    int* sg = tp.sidx;
    float d2lo = FLT_MAX, d2hi = 0.f;
    double sdev = 0.0, umax = 0.0;
    for (int k = lane; k < ne; k += 32) {
        const int a = w.sidx[k];
        const W5 q = load_w5(&C.l[5 * a]);
        sdev = fmax(sdev, fabs(q.s - s0));
        const double hx = 0.5 * ox, hy = 0.5 * oy;
        const double qa_dx = (q.w * hx - q.z * hy) + q.dx;  // q * T(o)
        const double qa_dy = (q.w * hy + q.z * hx) + q.dy;
        const double px = 0.5 * P0, py = 0.5 * P1;         // T(-P) * (q * T(o))
        r1g[k] = make_float4((float)q.w, (float)q.z, (float)(qa_dx + (-px * q.w - py * q.z)),
                             (float)(qa_dy + (px * q.z - py * q.w)));
        const double ux = C.x[a] - ox, uy = C.y[a] - oy;
        umax = fmax(umax, fmax(fabs(ux), fabs(uy)));
        r0g[k] = make_float4((float)ux, (float)uy, (float)C.p[a], (float)(q.s - s0));
        sg[k] = a;
        tp.axy[k] = make_double2(C.x[a], C.y[a]);
        w.ux[k] = (float)ux;
        w.uy[k] = (float)uy;
        const double dxn = fmax(fmax(-ux, 0.0), ux - (xhi - xlo)), dyn = fmax(fmax(-uy, 0.0), uy - (yhi - ylo));
        const double dxf = fmax(ux, (xhi - xlo) - ux), dyf = fmax(uy, (yhi - ylo) - uy);
        d2lo = fminf(d2lo, (float)(dxn * dxn + dyn * dyn));
        d2hi = fmaxf(d2hi, (float)(dxf * dxf + dyf * dyf));
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        d2lo = fminf(d2lo, __shfl_xor_sync(0xffffffffu, d2lo, d));
        d2hi = fmaxf(d2hi, __shfl_xor_sync(0xffffffffu, d2hi, d));
        sdev = fmax(sdev, __shfl_xor_sync(0xffffffffu, sdev, d));
        umax = fmax(umax, __shfl_xor_sync(0xffffffffu, umax, d));
    }
    if ((float)L.alpha * (d2hi - d2lo) >= 60.f) flags |= TFLAG_EXACT_STAGED;
    // Margins of the FP32 tier: tile-local coordinates below
    // kLocalMax px carry <= 2^-9 ulp ~ 1.5e-5 px of rounding, which the d^2
    // tolerance d2_tol covers; and the field error model of the node field
    // (k_nodefield.cu kScaleLever) bounds the scale lever S |P|.
    if (umax >= kLocalMax || sdev * (fmax(fabs(P0), fabs(P1)) + 2.0 * ET) > kScaleLever)
        flags |= TFLAG_EXACT_STAGED;
    __syncwarp();

    // 6. per sub-tile refinement of the tile-ambiguous (FP32, conservative margins)
    unsigned char* subg = &tp.sub[0][0];
    unsigned char* nearg = &tp.near[0][0];
    int my_nx = 0, my_na = 0, my_nn = 0;  // lane st < NW keeps sub-tile st's counts
    if (!(flags & TFLAG_EXACT_STAGED) && ne <= 32) {
        // Lane l holds staged point l. Sorted copies of the {min, max} squared
        // distances to the sub-tile (a bitonic network over the lanes) turn
        // each point's "how many others can be closer" counts into two binary
        // searches: the same counts, hence the same classes, as the all-pairs
        // loop of the general path below. Two sub-tiles at a time for ILP.
        constexpr int NP = 2;
        const unsigned below = (1u << lane) - 1u;
        const float ax = lane < ne ? w.ux[lane] : 0.f, ay = lane < ne ? w.uy[lane] : 0.f;
        for (int st0 = 0; st0 < NW; st0 += NP) {
            float dmn[NP], dmx[NP], sa[NP], sb[NP];
            bool ok[NP];
#pragma unroll
            for (int u = 0; u < NP; ++u) {
                const int st = st0 + u;
                const float wx0 = (float)((st & 1) * 8), wy0 = (float)((st >> 1) * 4);
                const float wx1 = fminf(wx0 + 7.f, (float)(ti1 - ti0)), wy1 = fminf(wy0 + 3.f, (float)(tj1 - tj0));
                ok[u] = !(wx0 > wx1 || wy0 > wy1);
                dmn[u] = dmx[u] = INFINITY;
                if (lane < ne) {
                    const float dxn = fmaxf(fmaxf(wx0 - ax, 0.f), ax - wx1), dyn = fmaxf(fmaxf(wy0 - ay, 0.f), ay - wy1);
                    const float dxf = fmaxf(ax - wx0, wx1 - ax), dyf = fmaxf(ay - wy0, wy1 - ay);
                    dmn[u] = fmaf(dxn, dxn, dyn * dyn);
                    dmx[u] = fmaf(dxf, dxf, dyf * dyf);
                }
                sa[u] = dmn[u];
                sb[u] = dmx[u];
            }
#pragma unroll
            for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
                for (int j = k >> 1; j > 0; j >>= 1) {
                    const bool take_min = ((lane & k) == 0) == ((lane & j) == 0);
#pragma unroll
                    for (int u = 0; u < NP; ++u) {
                        const float pa = __shfl_xor_sync(0xffffffffu, sa[u], j);
                        const float pb = __shfl_xor_sync(0xffffffffu, sb[u], j);
                        sa[u] = take_min ? fminf(sa[u], pa) : fmaxf(sa[u], pa);
                        sb[u] = take_min ? fminf(sb[u], pb) : fmaxf(sb[u], pb);
                    }
                }
            // The classes only compare the counts with S: cle = #{l : dmin_l <= hi_k} - 1 < S
            // <=> hi_k < the (S+1)-th smallest dmin (lane S of the sorted copy; none when
            // S >= 32), and clt = #{l : dmax_l < lo_k} >= S <=> the S-th smallest dmax
            // (lane S - 1) < lo_k: the same classes as counting, from two broadcasts.
#pragma unroll
            for (int u = 0; u < NP; ++u) {
                const int st = st0 + u;
                const float hi = dmx[u] * (1.f + 1e-5f) + 1e-2f, lo = dmn[u] * (1.f - 1e-5f) - 1e-2f;
                const float tin = __shfl_sync(0xffffffffu, sa[u], S < 32 ? S : 31);
                const float tout = __shfl_sync(0xffffffffu, sb[u], S - 1);
                const bool in = S >= 32 || hi < tin;
                // points that can be the nearest somewhere in the sub-tile
                const float thr = __shfl_sync(0xffffffffu, sb[u], 0) * (1.f + 1e-5f) + 1e-2f;
                const unsigned mn = __ballot_sync(0xffffffffu, dmn[u] <= thr);
                int c = 0;
                if (lane >= ni && lane < ne) c = in ? 1 : (tout >= lo ? 2 : 0);
                const unsigned mi = __ballot_sync(0xffffffffu, c == 1), ma = __ballot_sync(0xffffffffu, c == 2);
                int nx = 255, nw = 0, nn = 0;
                if (ok[u]) {  // warp-uniform
                    nn = __popc(mn);
                    if (nn > NEAR_CAP)
                        nn = 255;
                    else if ((mn >> lane) & 1u)
                        nearg[st * NEAR_CAP + __popc(mn & below)] = (unsigned char)lane;
                    nx = __popc(mi);
                    nw = __popc(ma);
                    if (c == 1) subg[st * TREC + __popc(mi & below)] = (unsigned char)lane;
                    if (c == 2) subg[st * TREC + nx + __popc(ma & below)] = (unsigned char)lane;
                }
                if (lane == st) {
                    my_nx = nx;
                    my_na = nw;
                    my_nn = nn;
                }
            }
        }
    } else {  // general path (more than 32 staged points): all pairs
        for (int st = 0; st < NW; ++st) {
            const float wx0 = (float)((st & 1) * 8), wy0 = (float)((st >> 1) * 4);
            const float wx1 = fminf(wx0 + 7.f, (float)(ti1 - ti0)), wy1 = fminf(wy0 + 3.f, (float)(tj1 - tj0));
            int nx = 0, nw = 0, nn = 0;
            if (!(wx0 > wx1 || wy0 > wy1) && !(flags & TFLAG_EXACT_STAGED)) {
                for (int k = lane; k < ne; k += 32) {
                    const float ax = w.ux[k], ay = w.uy[k];
                    const float dxn = fmaxf(fmaxf(wx0 - ax, 0.f), ax - wx1), dyn = fmaxf(fmaxf(wy0 - ay, 0.f), ay - wy1);
                    const float dxf = fmaxf(ax - wx0, wx1 - ax), dyf = fmaxf(ay - wy0, wy1 - ay);
                    w.wd[k] = make_float2(fmaf(dxn, dxn, dyn * dyn), fmaf(dxf, dxf, dyf * dyf));
                }
                __syncwarp();
                // points that can be the nearest somewhere in the sub-tile
                float thr = FLT_MAX;
                for (int k = lane; k < ne; k += 32) thr = fminf(thr, w.wd[k].y);
    #pragma unroll
                for (int d = 16; d > 0; d >>= 1) thr = fminf(thr, __shfl_xor_sync(0xffffffffu, thr, d));
                thr = thr * (1.f + 1e-5f) + 1e-2f;
                for (int base = 0; base < ne; base += 32) {
                    const int k = base + lane;
                    const bool cand = k < ne && w.wd[k].x <= thr;
                    const unsigned mn = __ballot_sync(0xffffffffu, cand);
                    const int pos = nn + __popc(mn & ((1u << lane) - 1u));
                    if (cand && pos < NEAR_CAP) nearg[st * NEAR_CAP + pos] = (unsigned char)k;
                    nn += __popc(mn);
                }
                if (nn > NEAR_CAP) nn = 255;
                for (int base = ni; base < ne; base += 32) {
                    const int k = base + lane;
                    int c = 0;
                    if (k < ne) {
                        const float2 dk = w.wd[k];
                        const float hi = dk.y * (1.f + 1e-5f) + 1e-2f, lo = dk.x * (1.f - 1e-5f) - 1e-2f;
                        int cle = -1, clt = 0;  // l == k always counts in cle
    #pragma unroll 4
                        for (int l = 0; l < ne; ++l) {
                            const float2 dl = w.wd[l];
                            cle += dl.x <= hi;
                            clt += dl.y < lo;
                        }
                        c = cle < S ? 1 : (clt >= S ? 0 : 2);
                        w.wcls[k] = (unsigned char)c;
                    }
                    const unsigned mi = __ballot_sync(0xffffffffu, c == 1);
                    if (c == 1) subg[st * TREC + nx + __popc(mi & ((1u << lane) - 1u))] = (unsigned char)k;
                    nx += __popc(mi);
                }
                __syncwarp();
                for (int base = ni; base < ne; base += 32) {
                    const int k = base + lane;
                    const int c = k < ne ? w.wcls[k] : 0;
                    const unsigned ma = __ballot_sync(0xffffffffu, c == 2);
                    if (c == 2) subg[st * TREC + nx + nw + __popc(ma & ((1u << lane) - 1u))] = (unsigned char)k;
                    nw += __popc(ma);
                }
                __syncwarp();
            } else {
                nx = 255;  // sub-tile without valid pixels, or exact tile
            }
            if (lane == st) {
                my_nx = nx;
                my_na = nw;
                my_nn = nn;
            }
        }
    }
    if (lane < NW) {
        hdr->nx[lane] = (unsigned char)my_nx;
        hdr->na[lane] = (unsigned char)my_na;
        hdr->nn[lane] = (unsigned char)my_nn;
    }
    if (lane == 0) {
        hdr->P[0] = P0;
        hdr->P[1] = P1;
        hdr->Y0[0] = w.ref[2];
        hdr->Y0[1] = w.ref[3];
        hdr->e0[0] = w.ref[4];
        hdr->e0[1] = w.ref[5];
        hdr->s0 = s0;
        hdr->d2ref = d2lo;
        hdr->d2top = d2hi;
        hdr->nin = ni;
        hdr->ne = ne;
        hdr->flags = flags;
    }
}

// ---------------------------------------------------------------------------
// Fast tier for one pixel (col, row = tile-local pixel position).
//   sure members: records [0, nin) plus sub-list [0, nxin)
//   ambiguous:    sub-list [nxin, nxin + namb), closest-to-centre first
// Weights come from the tile's separable tables (w = ex[k][col] ey[k][row],
// prob and the tile-wide d^2 floor folded into ey); the ambiguous are ranked
// by their FP32 squared distance.
// ---------------------------------------------------------------------------
struct FastOut {
    float s0, s1, s2, s3, s4, s5;  // sums: w*qw, w*qz, w*qdx, w*qdy, w*(s-s0), w
    bool exact;                    // boundary near-tie: rerun in the exact tier
};

#ifndef NRM_PIX_UNROLL
#define NRM_PIX_UNROLL 4
#endif
constexpr int kPixUnroll = NRM_PIX_UNROLL;  // member-accumulation loops of k_pixels

// Bound on |FP32 d^2 - exact d^2| for tile-local coordinates.
__device__ __forceinline__ float d2_tol(float d2) { return 2e-6f * d2 + 2e-3f; }

template <int MS>
__device__ __forceinline__ void fast_pixel(int col, int row, int nin, const unsigned char* __restrict__ wl,
                                           int nxin, int namb, int m, const TilePlan& p, const float (*ex)[ET],
                                           const float (*ey)[ET], FastOut& o) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, a4 = 0.f, a5 = 0.f;
    auto take = [&](int k) {
        const float w = ex[k][col] * ey[k][row];
        const float4 q = p.rec1[k];
        a0 = fmaf(w, q.x, a0);
        a1 = fmaf(w, q.y, a1);
        a2 = fmaf(w, q.z, a2);
        a3 = fmaf(w, q.w, a3);
        a4 = fmaf(w, p.rec0[k].w, a4);
        a5 += w;
    };
#pragma unroll (kPixUnroll)
    for (int k = 0; k < nin; ++k) take(k);
#pragma unroll (kPixUnroll)
    for (int e = 0; e < nxin; ++e) take(wl[e]);
    bool exact = false;
    const float ux = (float)col, uy = (float)row;
    const unsigned char* amb = wl + nxin;
    if (MS > 0 && m > 0) {  // m == 0: the sure members fill S, nothing to select
        // sorted insertion of the ambiguous keys (closest-to-centre first, so
        // most later keys are rejected by one compare) into the m <= MS slots
        // at the top of sd[]; the slots below hold -1 (< any d^2) and never
        // move, so the network and the worst member (sd[MS - 1]) are static
        float sd[MS > 0 ? MS : 1];
        int sk[MS > 0 ? MS : 1];
#pragma unroll
        for (int q = 0; q < MS; ++q) {
            sd[q] = q < MS - m ? -1.f : FLT_MAX;
            sk[q] = 0;
        }
        float rej = FLT_MAX;
        for (int e = 0; e < namb; ++e) {
            const int k = amb[e];
            const float2 u = *reinterpret_cast<const float2*>(&p.rec0[k]);
            const float dx = u.x - ux, dy = u.y - uy;
            const float d2 = fmaf(dx, dx, dy * dy);
            if (!(d2 < sd[MS - 1])) {
                rej = fminf(rej, d2);
                continue;
            }
            rej = fminf(rej, sd[MS - 1]);  // the current last member is evicted (or a sentinel)
            bool lt[MS > 0 ? MS : 1];
#pragma unroll
            for (int q = 0; q < MS; ++q) lt[q] = d2 < sd[q];
#pragma unroll
            for (int q = MS - 1; q >= 0; --q) {
                if (q > 0 && lt[q - 1]) {
                    sd[q] = sd[q - 1];
                    sk[q] = sk[q - 1];
                } else if (lt[q]) {
                    sd[q] = d2;
                    sk[q] = k;
                }
            }
        }
        const float worst = sd[MS > 0 ? MS - 1 : 0];
        // near-tie between the last member and the first rejected key
        if (rej < FLT_MAX && !(rej - worst > d2_tol(rej))) exact = true;
        // the members sit in the top m slots; m is warp-uniform, so these
        // branches do not diverge and no register selection is needed
#pragma unroll
        for (int q = 0; q < MS; ++q)
            if (q >= MS - m) take(sk[q]);
    } else if (MS == 0 && m > 0) {
        // many free slots (rare): repeated minimum selection; pass m + 1
        // finds the first rejected key for the near-tie test
        unsigned taken = 0u;
        float last = 0.f;
        for (int r = 0; r <= m; ++r) {
            float best = FLT_MAX;
            int bi = -1;
            for (int e = 0; e < namb; ++e) {
                if ((taken >> e) & 1u) continue;
                const float2 u = *reinterpret_cast<const float2*>(&p.rec0[amb[e]]);
                const float dx = u.x - ux, dy = u.y - uy;
                const float d2 = fmaf(dx, dx, dy * dy);
                if (d2 < best) {
                    best = d2;
                    bi = e;
                }
            }
            if (r == m) {
                if (bi >= 0 && !(best - last > d2_tol(best))) exact = true;
                break;
            }
            taken |= 1u << bi;
            last = best;
            take(amb[bi]);
        }
    }
    o = FastOut{a0, a1, a2, a3, a4, a5, exact};
}

__device__ __forceinline__ void fast_dispatch(int col, int row, int nin, const unsigned char* wl, int nxin,
                                              int namb, int m, const TilePlan& p, const float (*ex)[ET],
                                              const float (*ey)[ET], FastOut& o) {
    if (m <= 4)
        fast_pixel<4>(col, row, nin, wl, nxin, namb, m, p, ex, ey, o);
    else if (m <= 8)
        fast_pixel<8>(col, row, nin, wl, nxin, namb, m, p, ex, ey, o);
    else
        fast_pixel<0>(col, row, nin, wl, nxin, namb, m, p, ex, ey, o);
}

// ---------------------------------------------------------------------------
// One 16 x 16 tile whose plan is staged in shared memory (warp w = 8 x 4
// sub-tile w). Contains one block barrier, taken by all threads or none
// (the tile flags are uniform).
// ---------------------------------------------------------------------------
template <int MAXS>
__device__ __forceinline__ void pixels_tile(const EmdqLaunch& L, const Cand& C, const SuperLists& SL, const TilePlan& sp,
                                            float (*ex)[ET], float (*ey)[ET], int tx, int ty, int S) {
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int ti0 = L.grid.i0 + tx * ET, tj0 = L.grid.j0 + ty * ET;
    const int ti1 = min(ti0 + ET - 1, L.grid.i1), tj1 = min(tj0 + ET - 1, L.grid.j1);
    const TileHdr& h = sp.hdr;
    const int flags = h.flags;

    const int lx = (wid & 1) * 8 + (lane & 7), ly = (wid >> 1) * 4 + (lane >> 3);
    const int pi = ti0 + lx, pj = tj0 + ly;
    const bool valid = pi <= ti1 && pj <= tj1;
    const size_t o = (size_t)(pj - L.grid.j0) * (L.grid.i1 - L.grid.i0 + 1) + (pi - L.grid.i0);
    float2* od = (valid && L.disp) ? &L.disp[o] : nullptr;
    float* ou = (valid && L.unc) ? &L.unc[o] : nullptr;

    // Exact-tier pixels. Whole tiles or sub-tiles flagged for the exact tier
    // run it here, a thread per pixel (all lanes busy). Single pixels on a
    // near-tie (~4e-5 of them on C2) are queued for k_emdq_exceptions (a warp
    // per pixel) instead: resolved here, each cost its thread ~10 us of
    // serial FP64 work and cold instruction fetches, which held the whole
    // CTA and, at 86 pixels, a third of this kernel's time. Every lane
    // reaches the push below (no early returns).
    bool inline_exact = true;  // tile / sub-tile flagged for the exact tier
    bool queue_exact = false;  // a single pixel on a near-tie
    const int* xsrc = nullptr;  // inline exact: candidate list (staged list or supertile list)
    int xn = 0;
    if (!(flags & TFLAG_EXACT_SUPER)) {  // tile-uniform
        const int ne = h.ne, nin = h.nin;
        const int nxin = h.nx[wid], namb = h.na[wid], nnear = h.nn[wid];
        // separable weight tables (prob and the tile-wide d^2 floor folded into
        // ey): thread = (record k, 4 columns / rows); the per-record terms once,
        // float4 stores (ex[k][4q .. 4q+3], ey[k][4q .. 4q+3])
        if (!(flags & TFLAG_EXACT_STAGED)) {
            const int k = t >> 2, c0 = 4 * (t & 3);
            if (k < ne) {
                const float nal = (float)(-L.alpha * kLog2e), d2ref = h.d2ref;
                const float4 r0 = sp.rec0[k];
                const float cx = fminf(fmaxf(r0.x, 0.f), (float)(ET - 1)), cy = fminf(fmaxf(r0.y, 0.f), (float)(ET - 1));
                const float dxr = (r0.x - cx) * (r0.x - cx), dyr = (r0.y - cy) * (r0.y - cy);
                const float base = nal * (dxr + dyr - d2ref);
                float vx[4], vy[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float dx = r0.x - (float)(c0 + i), dy = r0.y - (float)(c0 + i);
                    vx[i] = ex2_approx(nal * (dx * dx - dxr));
                    vy[i] = ex2_approx(fmaf(nal, dy * dy - dyr, base)) * r0.z;
                }
                *reinterpret_cast<float4*>(&ex[k][c0]) = make_float4(vx[0], vx[1], vx[2], vx[3]);
                *reinterpret_cast<float4*>(&ey[k][c0]) = make_float4(vy[0], vy[1], vy[2], vy[3]);
            }
        }
        __syncthreads();
        xsrc = sp.sidx;
        xn = ne;
        const int wi = nin + nxin, m = S - wi;
        if (!(flags & TFLAG_EXACT_STAGED) && !(nxin == 255 || m < 0 || wi + namb < S || namb > 32)) {
            inline_exact = false;
            FastOut fo;
            if (valid) {
                fast_dispatch(lx, ly, nin, sp.sub[wid], nxin, namb, m, sp, ex, ey, fo);
                queue_exact = fo.exact || !(fo.s5 > 0.f);
            }
            if (valid && !queue_exact) {
                const double qx = L.grid.gx + pi, qy = L.grid.gy + pj;
                const float rn = rsqrtf(fmaf(fo.s0, fo.s0, fo.s1 * fo.s1));
                const float qw = fo.s0 * rn, qz = fo.s1 * rn, qdx = fo.s2 * rn, qdy = fo.s3 * rn;
                const float cc = qw * qw - qz * qz, ss = 2.f * qw * qz;
                const float ux = (float)lx, uy = (float)ly;
                const float Qx = cc * ux - ss * uy + 2.f * (qdx * qw - qdy * qz);
                const float Qy = ss * ux + cc * uy + 2.f * (qdx * qz + qdy * qw);
                const float dlb = __fdividef(fo.s4, fo.s5);  // s5 > 0 (checked above)
                // displacement y - q = (Y0 - tile origin - u) + (e0 + dl P + (s0 + dl) Q(u)):
                // the first part is a small per-tile constant (bd, FP64 -> FP32), the
                // second stays ~1e2 px, so FP32 keeps it to ~1e-5 px at any coordinate
                // (the K1/K2 epilogue; error model: k_nodefield.cu kScaleLever)
                if (od) {
                    const float sbf = (float)h.s0 + dlb;
                    const float rx = fmaf(sbf, Qx, fmaf(dlb, (float)h.P[0], (float)h.e0[0]));
                    const float ry = fmaf(sbf, Qy, fmaf(dlb, (float)h.P[1], (float)h.e0[1]));
                    const float bdx = (float)(h.Y0[0] - (L.grid.gx + ti0)), bdy = (float)(h.Y0[1] - (L.grid.gy + tj0));
                    *od = make_float2((bdx - ux) + rx, (bdy - uy) + ry);
                }
                if (ou) {
                    // bounded_exp(beta d2min) (fieldest.hpp:44-52) to FP32 output
                    // precision: d2min in FP64 over the points that can be the nearest in
                    // this sub-tile; exp(x) = 2^n 2^f, n = rint(x log2 e), |f| <= 1/2 in
                    // FP64, 2^f on MUFU.EX2 (relative error < 3e-7, inside the 1e-6 bar)
                    double d2m = DBL_MAX;
                    const int nl = nnear == 255 ? ne : nnear;
                    for (int e = 0; e < nl; ++e) {
                        const int k = nnear == 255 ? e : sp.near[wid][e];
                        const double2 a = sp.axy[k];
                        const double dx = qx - a.x, dy = qy - a.y;
                        d2m = fmin(d2m, fma(dx, dx, dy * dy));
                    }
                    const double tx = fmin(L.beta * d2m, 55.0) * 1.4426950408889634;
                    const double n = rint(tx);
                    *ou = ex2_approx((float)(tx - n)) * __int_as_float(((int)n + 127) << 23);
                }
            }
        }
    }
    if (flags & TFLAG_EXACT_SUPER) {
        const int sid = (ty / (ST / ET)) * SL.nsx + tx / (ST / ET);
        xsrc = (SL.flag[sid] & SFLAG_OVERFLOW) ? nullptr : SL.list + (size_t)sid * SLIST_CAP;
        xn = xsrc ? SL.count[sid] : L.nactive;
    }
    if ((inline_exact || queue_exact) && valid && L.exact_count) atomicAdd(L.exact_count, 1u);
    // queued unless there is no queue or the slot was past its capacity
    if (inline_exact) {
        if (valid) exact_dispatch<MAXS>(L.grid.gx + pi, L.grid.gy + pj, xsrc, xn, S, C, L.alpha, L.beta, od, ou);
    } else if (L.exq ? queue_push(queue_exact, pi, pj, L.exq, L.exq_count, L.exq_cap) : queue_exact) {
        exact_dispatch<MAXS>(L.grid.gx + pi, L.grid.gy + pj, xsrc, xn, S, C, L.alpha, L.beta, od, ou);
    }
}

// k_pixels: one CTA per tile.
template <int MAXS>
__global__ void __launch_bounds__(ENT, NRM_PIX_MINB)
k_pixels(EmdqLaunch L, Cand C, SuperLists SL, TilePlans TP, int S) {
    __shared__ __align__(128) PixSmem s;
    const int g = blockIdx.y * TP.ntx + blockIdx.x;
    // the tile plan (4 KB) arrives by one TMA bulk copy (cp.async.bulk): one
    // thread arms the barrier and issues it, no register round trip
    if (threadIdx.x == 0) mbar_init(&s.bar, 1);
    __syncthreads();
    pdl_wait();
    if (threadIdx.x == 0) {
        mbar_expect_tx(&s.bar, (unsigned)sizeof(TilePlan));
        bulk_g2s(&s.p, &TP.plan[g], (unsigned)sizeof(TilePlan), &s.bar);
    }
    mbar_wait(&s.bar, 0);
    pixels_tile<MAXS>(L, C, SL, s.p, s.ex, s.ey, TP.tx0 + blockIdx.x, TP.ty0 + blockIdx.y, S);
}

// ---------------------------------------------------------------------------
// k_emdq_exceptions: the dense field's exact-tier pixels (queued by
// k_pixels), one warp per pixel, bit-identical to emdq_exact / the
// reference's blend_local + node_uncertainty (fieldest.hpp:44-52, 75-97):
//   * the S nearest by (d^2, j) over the tile's staged list (the tile plan
//     of this launch chunk, at most 64 candidates): each candidate's rank
//     among all of them in one pass over the warp's keys in shared memory
//     (FP64 d^2 as xdist2);
//   * lane s holds member s: its weight exp(-alpha (d^2 - d2min)) prob in
//     parallel (glibc-exact exp), then the reference's ordered sums (wsum,
//     then the hemisphere-aligned weighted warps) as a shuffle chain;
//   * lane 0 normalises, applies and writes the displacement and the
//     uncertainty bounded_exp(beta d2min).
// ---------------------------------------------------------------------------
#ifndef NRM_EXQ_BLOCKS
#define NRM_EXQ_BLOCKS 148
#endif
constexpr int EXQ_THREADS = 128, EXQ_BLOCKS = NRM_EXQ_BLOCKS;  // grid-stride; warps without a pixel exit
struct ExqWarp {
    uint4 key[TREC];      // d^2 bits (lo, hi), j
    int4 mem[MAX_SUPPORT];  // members in order: candidate, -, d^2 bits (lo, hi)
};
__shared__ ExqWarp exq_smem[EXQ_THREADS / 32];
__device__ __forceinline__ void warp_min_key(double& d, int& j, int& a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double od = __shfl_xor_sync(0xffffffffu, d, o);
        const int oj = __shfl_xor_sync(0xffffffffu, j, o), oa = __shfl_xor_sync(0xffffffffu, a, o);
        if (key_less(od, oj, d, j)) {
            d = od;
            j = oj;
            a = oa;
        }
    }
}

__device__ void exact_pixel_warp(const EmdqLaunch& L, const Cand& C, const TilePlans& TP, int S, int pi, int pj) {
    const int lane = threadIdx.x & 31;
    const double qx = L.grid.gx + pi, qy = L.grid.gy + pj;
    // the pixel's tile plan (this launch chunk): its staged list (in +
    // ambiguous, at most TREC) holds every candidate of the pixel's S nearest
    const int g = ((pj - L.grid.j0) / ET - TP.ty0) * TP.ntx + (pi - L.grid.i0) / ET - TP.tx0;
    const int* src = TP.plan[g].sidx;
    const int n = min(TP.plan[g].hdr.ne, TREC);  // queued pixels come from planned (non-exact) tiles: ne <= TREC
    // 1. the kk = min(S, n) nearest, in (d^2, j) order: every staged
    //    candidate (n <= TREC = 64, two per lane) gets its rank among all n by
    //    one pass over the warp's keys in shared memory (d^2 >= 0, so its bits
    //    compare as integers; ties by j); the one of rank s goes to lane s.
    ExqWarp& xw = exq_smem[threadIdx.x >> 5];
    double my_d2 = DBL_MAX;
    int my_a = -1;
    const int kk = min(S, n);
    {
        unsigned long long ku[2];
        int kj[2], ka[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int e = lane + 32 * r;
            ku[r] = ~0ull;
            kj[r] = INT_MAX;
            ka[r] = -1;
            if (e < n) {
                const int a = src[e];
                ka[r] = a;
                kj[r] = C.j[a];
                ku[r] = (unsigned long long)__double_as_longlong(xdist2(qx, qy, C.x[a], C.y[a]));
                xw.key[e] = make_uint4((unsigned)ku[r], (unsigned)(ku[r] >> 32), (unsigned)kj[r], 0u);
            }
        }
        __syncwarp();
        int rank[2] = {0, 0};
        for (int e = 0; e < n; ++e) {
            const uint4 o = xw.key[e];  // broadcast
            const unsigned long long ou = ((unsigned long long)o.y << 32) | o.x;
            const int oj = (int)o.z;
#pragma unroll
            for (int r = 0; r < 2; ++r) rank[r] += (ou < ku[r] || (ou == ku[r] && oj < kj[r])) ? 1 : 0;
        }
#pragma unroll
        for (int r = 0; r < 2; ++r)
            if (ka[r] >= 0 && rank[r] < kk) xw.mem[rank[r]] = make_int4(ka[r], 0, (int)(unsigned)ku[r], (int)(ku[r] >> 32));
        __syncwarp();
        if (lane < kk) {
            const int4 m = xw.mem[lane];
            my_a = m.x;
            my_d2 = __longlong_as_double((long long)(((unsigned long long)(unsigned)m.w << 32) | (unsigned)m.z));
        }
        __syncwarp();  // the warp's next pixel rewrites the keys
    }
    const double d2min = __shfl_sync(0xffffffffu, my_d2, 0);  // DBL_MAX when kk == 0
    // 2. weights, in parallel (emdq_blend_exact's expressions)
    const bool mem = lane < kk;
    double w = 0.0;
    if (mem) w = xmul(xexp(xmul(-L.alpha, xsub(my_d2, d2min))), C.p[my_a]);
    const unsigned pos = __ballot_sync(0xffffffffu, mem && w > 0.0);
    int rc = kk == 0 ? 1 : (pos ? 0 : 2);
    double wsum = 0.0;
    for (int s = 0; s < kk; ++s) wsum = xadd(wsum, __shfl_sync(0xffffffffu, w, s));
    // 3. hemisphere-aligned weighted warps, summed in member order
    const int ref = pos ? __ffs(pos) - 1 : 0;
    double q0 = 0.0, qw = 0.0, qz = 0.0, qdx = 0.0, qdy = 0.0;
    if (mem) {
        const double* q = &C.l[5 * my_a];
        q0 = q[0];
        qw = q[1];
        qz = q[2];
        qdx = q[3];
        qdy = q[4];
    }
    const double rw = __shfl_sync(0xffffffffu, qw, ref), rz = __shfl_sync(0xffffffffu, qz, ref);
    if (xadd(xmul(qw, rw), xmul(qz, rz)) < 0.0) {
        qw = -qw;
        qz = -qz;
        qdx = -qdx;
        qdy = -qdy;
    }
    const double p0 = xmul(w, qw), p1 = xmul(w, qz), p2 = xmul(w, qdx), p3 = xmul(w, qdy), p4 = xmul(w, q0);
    double sw = 0.0, sz = 0.0, sdx = 0.0, sdy = 0.0, ss = 0.0;
    for (unsigned m = pos; m; m &= m - 1u) {  // contributing members (w > 0) in order
        const int s = __ffs(m) - 1;
        sw = xadd(sw, __shfl_sync(0xffffffffu, p0, s));
        sz = xadd(sz, __shfl_sync(0xffffffffu, p1, s));
        sdx = xadd(sdx, __shfl_sync(0xffffffffu, p2, s));
        sdy = xadd(sdy, __shfl_sync(0xffffffffu, p3, s));
        ss = xadd(ss, __shfl_sync(0xffffffffu, p4, s));
    }
    if (lane != 0) return;
    W5 f;
    if (rc == 0) {
        const double mw = sw / wsum, mz = sz / wsum, mdx = sdx / wsum, mdy = sdy / wsum;
        const double nr = xhypot(mw, mz);
        if (!(nr >= 1e-300))
            rc = 2;
        else
            f = W5{ss / wsum, mw / nr, mz / nr, mdx / nr, mdy / nr};
    }
    const size_t o = (size_t)(pj - L.grid.j0) * (L.grid.i1 - L.grid.i0 + 1) + (pi - L.grid.i0);
    if (L.disp) {
        float2 dout = make_float2(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
        if (rc == 0) {
            double yx, yy;
            xapply(f, qx, qy, &yx, &yy);
            dout = make_float2((float)(yx - qx), (float)(yy - qy));
        }
        L.disp[o] = dout;
    }
    if (L.unc) {
        double arg = xmul(L.beta, d2min);
        if (55.0 < arg) arg = 55.0;
        L.unc[o] = (float)xexp(arg);
    }
}

// One launch per chunk of tiles, after that chunk's k_pixels (the next
// chunk's k_plan empties the queue and rewrites the plans).
__global__ void __launch_bounds__(EXQ_THREADS) k_emdq_exceptions(EmdqLaunch L, Cand C, TilePlans TP, int S) {
    pdl_wait();
    const unsigned cnt = min(*L.exq_count, L.exq_cap);
    const unsigned gw = blockIdx.x * (EXQ_THREADS / 32) + (threadIdx.x >> 5), nw = gridDim.x * (EXQ_THREADS / 32);
    for (unsigned i = gw; i < cnt; i += nw) {
        const int2 p = L.exq[i];
        exact_pixel_warp(L, C, TP, S, p.x, p.y);
    }
}

// ---------------------------------------------------------------------------
// k_points: one thread per scattered query, exact tier over the candidate
// list of the supertile holding the query (k_super with one extra neighbour
// when a candidate is left out, and a margin for queries between pixels).
// ---------------------------------------------------------------------------
template <int MAXS>
__global__ void __launch_bounds__(128) k_points(EmdqLaunch L, Cand C, SuperLists SL, PointsLaunch P, int S,
                                                int nsy) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= P.nq) return;
    const double qx = P.q[2 * k], qy = P.q[2 * k + 1];
    const int excl = P.excl ? P.excl[k] : -1;
    const int* src = nullptr;
    int n = L.nactive;
    if (!P.full_scan) {
        int sx = (int)floor((qx - L.grid.gx - L.grid.i0) / ST), sy = (int)floor((qy - L.grid.gy - L.grid.j0) / ST);
        sx = min(max(sx, 0), SL.nsx - 1);
        sy = min(max(sy, 0), nsy - 1);
        const int sid = sy * SL.nsx + sx;
        src = (SL.flag[sid] & SFLAG_OVERFLOW) ? nullptr : SL.list + (size_t)sid * SLIST_CAP;
        n = SL.count[sid];
    }
    W5 f;
    double d2min;
    const int rc = (S <= 16 || MAXS <= 16) ? emdq_blend_exact<16>(qx, qy, src, n, S, C, L.alpha, excl, &f, &d2min)
                                           : emdq_blend_exact<MAXS>(qx, qy, src, n, S, C, L.alpha, excl, &f, &d2min);
    if (P.status) P.status[k] = rc;
    if (P.warps) {
        double* o = &P.warps[5 * k];
        if (rc == 0) {
            o[0] = f.s; o[1] = f.w; o[2] = f.z; o[3] = f.dx; o[4] = f.dy;
        } else {
            o[0] = o[1] = o[2] = o[3] = o[4] = 0.0;
        }
    }
    if (P.pred) {
        double yx = 0.0, yy = 0.0;
        if (rc == 0) xapply(f, qx, qy, &yx, &yy);
        P.pred[2 * k] = yx;
        P.pred[2 * k + 1] = yy;
    }
    if (P.unc) {
        double arg = xmul(L.beta, d2min);
        if (55.0 < arg) arg = 55.0;  // bounded_exp (geometry.hpp:85-88)
        P.unc[k] = xexp(arg);
    }
}

__global__ void k_points_bbox(const double* __restrict__ q, int nq, double* out4) {
    __shared__ double red[4][32];
    double mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    for (int k = threadIdx.x; k < nq; k += blockDim.x) {
        const double x = q[2 * k], y = q[2 * k + 1];
        mnx = fmin(mnx, x);
        mny = fmin(mny, y);
        mxx = fmax(mxx, x);
        mxy = fmax(mxy, y);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        mnx = fmin(mnx, __shfl_xor_sync(0xffffffffu, mnx, d));
        mny = fmin(mny, __shfl_xor_sync(0xffffffffu, mny, d));
        mxx = fmax(mxx, __shfl_xor_sync(0xffffffffu, mxx, d));
        mxy = fmax(mxy, __shfl_xor_sync(0xffffffffu, mxy, d));
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        red[0][w] = mnx;
        red[1][w] = mny;
        red[2][w] = mxx;
        red[3][w] = mxy;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int v = 1; v < (int)(blockDim.x >> 5); ++v) {
            mnx = fmin(mnx, red[0][v]);
            mny = fmin(mny, red[1][v]);
            mxx = fmax(mxx, red[2][v]);
            mxy = fmax(mxy, red[3][v]);
        }
        out4[0] = mnx;
        out4[1] = mny;
        out4[2] = mxx;
        out4[3] = mxy;
    }
}

}  // namespace

// Exact-tier queue of a dense field: the fast tier defers ~4e-5 of the pixels
// on C2 (86 of 2.07 M), plus whole tiles flagged for the exact tier; 1/32 of
// the grid, at least 2^16 slots of 8 B. A push past the capacity resolves its
// pixel in place (k_pixels), so nothing depends on the size.
static unsigned emdq_queue_cap(const FieldGrid& g) {
    const size_t px = (size_t)(g.i1 - g.i0 + 1) * (size_t)(g.j1 - g.j0 + 1);
    return (unsigned)std::min<size_t>(std::max<size_t>((size_t)1 << 16, px / 32), (size_t)1 << 30);
}
static size_t emdq_queue_bytes(const FieldGrid& g) { return (size_t)emdq_queue_cap(g) * sizeof(int2) + 16; }

void emdq_cell_bytes(int nactive, const FieldGrid& g, size_t* count_bytes, size_t* bin_bytes) {
    *count_bytes = *bin_bytes = 0;
    if (nactive <= SUPER_FUSED_GATHER_MAX || nactive > BIN_MAX_N) return;
    const int nsx = (g.i1 - g.i0 + ST) / ST, nsy = (g.j1 - g.j0 + ST) / ST;
    const size_t nc = (size_t)(nsx + 2) * (nsy + 2);
    *count_bytes = (nc + 1) * sizeof(int);  // a CTA ticket, then the counts
    *bin_bytes = (2 * nc + 1 + (size_t)nactive) * sizeof(int);
}

size_t emdq_scratch_bytes(int nactive, const FieldGrid& g, bool tile_plans) {
    const size_t na = (size_t)nactive;
    const int nsx = (g.i1 - g.i0 + ST) / ST, nsy = (g.j1 - g.j0 + ST) / ST;
    const size_t nsuper = (size_t)nsx * nsy;
    const size_t plans = tile_plans ? (size_t)EMDQ_CHUNK_TILES * sizeof(TilePlan) + 256 + emdq_queue_bytes(g) : 0;
    return na * 9 * sizeof(double) + na * sizeof(float2) + na * sizeof(int) + nsuper * (SLIST_CAP + 2) * sizeof(int) +
           plans + 1024;
}

cudaError_t launch_emdq_field(const EmdqLaunch& L, cudaStream_t st, int64_t* launches) {
    if (L.nactive <= 0) return cudaErrorInvalidValue;
    const size_t na = (size_t)L.nactive;
    // scratch layout (emdq_scratch_bytes): x, y, l[5], p, phi (double) | c32 (float2) | j (int) |
    // supertile lists | tile plans (one chunk)
    Cand C;
    C.x = L.cx;
    C.y = L.cy;
    C.l = L.cl;
    C.p = L.cp;
    double* phi = L.cp + na;
    C.phi = phi;
    float2* c32 = reinterpret_cast<float2*>(phi + na);
    C.c32 = c32;
    int* cj = reinterpret_cast<int*>(c32 + na);
    C.j = cj;
    SuperLists SL;
    SL.nsx = (L.grid.i1 - L.grid.i0 + ST) / ST;
    const int nsy = (L.grid.j1 - L.grid.j0 + ST) / ST;
    const size_t nsuper = (size_t)SL.nsx * nsy;
    SL.list = cj + na;
    SL.count = SL.list + nsuper * SLIST_CAP;
    SL.flag = SL.count + nsuper;
    char* pbase = reinterpret_cast<char*>(SL.flag + nsuper);
    pbase = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(pbase) + 255) & ~uintptr_t(255));
    TilePlans TP;
    TP.plan = reinterpret_cast<TilePlan*>(pbase);
    EmdqLaunch LQ = L;  // with the exact-tier queue behind the tile plans
    {
        char* qb = pbase + (size_t)EMDQ_CHUNK_TILES * sizeof(TilePlan);
        qb = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(qb) + 255) & ~uintptr_t(255));
        LQ.exq_count = reinterpret_cast<unsigned*>(qb);
        LQ.exq = reinterpret_cast<int2*>(qb + 16);
        LQ.exq_cap = emdq_queue_cap(L.grid);
        if (L.exq_cap_override > 0 && (uint64_t)L.exq_cap_override < LQ.exq_cap) LQ.exq_cap = (unsigned)L.exq_cap_override;
    }

    const GatherOut G{L.cx, L.cy, L.cl, L.cp, phi, c32, cj};
    const int S = L.support < L.nactive ? L.support : L.nactive;
    const CellGrid cg{(float)(L.grid.gx + L.grid.i0), (float)(L.grid.gy + L.grid.j0), SL.nsx, nsy};
    if (L.nactive <= SUPER_FUSED_GATHER_MAX || L.nactive > BIN_MAX_N || !LQ.cell_cnt) LQ.cells = LQ.cell_cnt = nullptr;
    const bool binned = LQ.cells != nullptr;  // set by the caller when emdq_cell_bytes() > 0
    const size_t ssm = ((sizeof(SSmem) + 15) & ~size_t(15)) +
                       (binned ? (size_t)((L.nactive + 31) / 32) * sizeof(unsigned)
                               : (L.nactive <= SUPER_CC_CAP ? (size_t)L.nactive * sizeof(float2) : 0));
    cudaFuncSetAttribute(k_super, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
    // programmatic launch: its CTAs become resident while the stream's previous
    // kernel drains and wait in pdl_wait() before touching any scratch
    // small candidate sets: the gather is fused into k_super (one launch less
    // on the critical chain); large ones: k_gather first, so that every
    // supertile CTA reads the contiguous coarse coordinates
    const int gathered = L.nactive > SUPER_FUSED_GATHER_MAX ? 1 : 0;
    if (gathered) {
        prof_mark("k_gather", st);
        k_gather<<<(L.nactive + 255) / 256, 256, 0, st>>>(L.apts, L.locals, L.probs, L.active, L.nactive, L.cx, L.cy,
                                                           c32, L.cl, L.cp, phi, cj, LQ.cell_cnt, LQ.cells, cg);
        ++*launches;
        cudaError_t eg = cudaGetLastError();
        if (eg != cudaSuccess) return eg;
        if (binned) {  // (k_gather's last CTA scanned the counts)
            prof_mark("k_bin_scatter", st);
            k_bin_scatter<<<(L.nactive + 255) / 256, 256, 0, st>>>(c32, L.nactive, cg, LQ.cells);
            *launches += 1;
            eg = cudaGetLastError();
            if (eg != cudaSuccess) return eg;
        }
    }
    prof_mark("k_super", st);
    cudaError_t e = launch_pdl(k_super, dim3(SL.nsx, nsy), dim3(ENT), ssm, st, LQ, G, SL, S, 0.f, gathered, cg);
    ++*launches;
    if (e != cudaSuccess) return e;
    const int ntx = (L.grid.i1 - L.grid.i0 + ET) / ET;
    const int nty = (L.grid.j1 - L.grid.j0 + ET) / ET;
    const int rows_per_chunk = EMDQ_CHUNK_TILES / ntx > 0 ? EMDQ_CHUNK_TILES / ntx : 1;
    const size_t psm = sizeof(PlanWarp) * PLAN_WARPS;
    cudaFuncSetAttribute(k_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm);
    for (int ty0 = 0; ty0 < nty; ty0 += rows_per_chunk) {
        const int rows = min(rows_per_chunk, nty - ty0);
        if ((size_t)rows * ntx > (size_t)EMDQ_CHUNK_TILES) return cudaErrorInvalidValue;  // ntx > chunk
        TP.tx0 = 0;
        TP.ty0 = ty0;
        TP.ntx = ntx;
        const int ntiles = rows * ntx;
        prof_mark("k_plan", st);
        e = launch_pdl(k_plan, dim3((ntiles + PLAN_WARPS - 1) / PLAN_WARPS), dim3(PLAN_WARPS * 32), psm, st, LQ, C, SL,
                       TP, ntiles, S);
        if (e != cudaSuccess) return e;
        ++*launches;
        prof_mark("k_pixels", st);
        e = launch_pdl(S <= 16 ? k_pixels<16> : k_pixels<MAX_SUPPORT>, dim3(ntx, rows), dim3(ENT), 0, st, LQ, C, SL,
                       TP, S);
        ++*launches;
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        prof_mark("k_emdq_exceptions", st);
        e = launch_pdl(k_emdq_exceptions, dim3(EXQ_BLOCKS), dim3(EXQ_THREADS), 0, st, LQ, C, TP, S);
        ++*launches;
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace nrm

namespace nrm {

cudaError_t launch_points_bbox(const double* q, int nq, double* out4, cudaStream_t st, int64_t* launches) {
    prof_mark("k_points_bbox", st);
    k_points_bbox<<<1, 1024, 0, st>>>(q, nq, out4);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_emdq_points(const EmdqLaunch& L, const PointsLaunch& P, cudaStream_t st, int64_t* launches) {
    if (L.nactive <= 0 || P.nq <= 0) return cudaErrorInvalidValue;
    const size_t na = (size_t)L.nactive;
    Cand C;
    C.x = L.cx;
    C.y = L.cy;
    C.l = L.cl;
    C.p = L.cp;
    double* phi = L.cp + na;
    C.phi = phi;
    float2* c32 = reinterpret_cast<float2*>(phi + na);
    C.c32 = c32;
    int* cj = reinterpret_cast<int*>(c32 + na);
    C.j = cj;
    SuperLists SL;
    SL.nsx = (L.grid.i1 - L.grid.i0 + ST) / ST;
    const int nsy = (L.grid.j1 - L.grid.j0 + ST) / ST;
    const size_t nsuper = (size_t)SL.nsx * nsy;
    SL.list = cj + na;
    SL.count = SL.list + nsuper * SLIST_CAP;
    SL.flag = SL.count + nsuper;

    cudaError_t e = cudaSuccess;
    const int S = L.support < L.nactive ? L.support : L.nactive;
    // one more neighbour when a candidate may be left out; queries lie within
    // one pixel of their supertile's pixel rectangle
    const int Ssup = min(L.nactive, S + (P.excl ? 1 : 0));
    if (P.full_scan) {
        prof_mark("k_gather", st);
        k_gather<<<(L.nactive + 255) / 256, 256, 0, st>>>(L.apts, L.locals, L.probs, L.active, L.nactive, L.cx,
                                                           L.cy, c32, L.cl, L.cp, phi, cj, nullptr, nullptr, CellGrid{});
        ++*launches;
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    } else {
        const GatherOut G{L.cx, L.cy, L.cl, L.cp, phi, c32, cj};
        const size_t ssm = ((sizeof(SSmem) + 15) & ~size_t(15)) +
                           (L.nactive <= SUPER_CC_CAP ? (size_t)L.nactive * sizeof(float2) : 0);
        cudaFuncSetAttribute(k_super, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
        prof_mark("k_super", st);
        EmdqLaunch Lp = L;
        Lp.cells = Lp.cell_cnt = nullptr;  // the point queries' supertiles scan every candidate
        k_super<<<dim3(SL.nsx, nsy), ENT, ssm, st>>>(Lp, G, SL, Ssup, 3.f, 0, CellGrid{});
        ++*launches;
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    prof_mark("k_points", st);
    if (S <= 16)
        k_points<16><<<(P.nq + 127) / 128, 128, 0, st>>>(L, C, SL, P, S, nsy);
    else
        k_points<MAX_SUPPORT><<<(P.nq + 127) / 128, 128, 0, st>>>(L, C, SL, P, S, nsy);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace nrm
