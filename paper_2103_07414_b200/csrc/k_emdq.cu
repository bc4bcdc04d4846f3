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
// kNN membership decides which warps are blended, so it must match the
// reference exactly: d^2 is computed in the exact tier (same FP64 operation
// order as dist2) and ranked by the reference's (d^2, j) key.
//
// CTA = 16 x 16 pixel tile, one pixel per thread.
//   1. radius bound: 256-bin histogram of squared centre distances gives
//      R >= r_S(centre); every pixel's S nearest lie within R + 2*hd of the
//      centre (hd = tile half-diagonal).
//   2. candidates inside that disc are classified against the tile
//      rectangle: "sure-in" (fewer than S other candidates can ever be
//      closer), "sure-out" (at least S are always closer) or ambiguous.
//   3. per pixel: exact d^2 for sure-in + ambiguous, sorted insertion of the
//      ambiguous into the m = S - |sure-in| free slots, then the blend:
//      weights on MUFU.EX2 (FP32), accumulation and normalisation in FP64.
#include <cfloat>
#include <climits>
#include <cmath>

#include "nrm_common.cuh"
#include "nrm_internal.h"

namespace nrm {
namespace {

constexpr int ET = 16;            // tile edge
constexpr int ENT = ET * ET;      // threads
constexpr int CAND_CAP = 512;     // candidates per tile
constexpr int MAX_SUPPORT = 32;

struct ESmem {
    int hist[256];
    int cand[CAND_CAP];
    double dmin2[CAND_CAP], dmax2[CAND_CAP];
    unsigned char cls[CAND_CAP];  // 0 out, 1 in, 2 ambiguous
    // staged blend-eligible points: [0, n_in) sure-in, [n_in, n_in + n_amb) ambiguous
    double px[CAND_CAP], py[CAND_CAP], pp[CAND_CAP];
    double pl[CAND_CAP][5];
    int pj[CAND_CAP];
    int stage[CAND_CAP];
    int warp_cnt[ENT / 32];
    int ncand, n_in, n_amb, slow;
    float R;
};

__global__ void k_gather(const double* __restrict__ apts, const double* __restrict__ locals,
                         const double* __restrict__ probs, const int32_t* __restrict__ active,
                         int nactive, double* cx, double* cy, double* cl, double* cp, int* cj) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= nactive) return;
    const int j = active[a];
    cx[a] = apts[2 * j];
    cy[a] = apts[2 * j + 1];
#pragma unroll
    for (int k = 0; k < 5; ++k) cl[5 * a + k] = locals[5 * j + k];
    const double p = probs[j];
    cp[a] = p < 1e-6 ? 1e-6 : p;  // std::max(probs[j], 1e-6)
    cj[a] = j;
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

// One pixel: S-nearest selection + blend. E* point into smem (fast tiles) or
// the gathered global arrays (slow tiles: n_in = 0, every point ambiguous).
template <int MS>
__device__ void emdq_pixel(double qx, double qy, int n_in, int n_amb, int m,
                           const double* __restrict__ Ex, const double* __restrict__ Ey,
                           const double* __restrict__ Ep, const double* __restrict__ El,
                           const int* __restrict__ Ej, double alpha, double beta, float2* out_d,
                           float* out_u) {
    // sure-in: nearest key among them
    double best_d = DBL_MAX;
    int best_j = INT_MAX, best_k = -1;
    for (int k = 0; k < n_in; ++k) {
        const double d2 = xdist2(qx, qy, Ex[k], Ey[k]);
        if (key_less(d2, Ej[k], best_d, best_j)) {
            best_d = d2;
            best_j = Ej[k];
            best_k = k;
        }
    }
    // ambiguous: keep the m smallest (d2, j) keys, sorted ascending
    double sd[MS > 0 ? MS : 1];
    int sj[MS > 0 ? MS : 1], sk[MS > 0 ? MS : 1];
    if (MS > 0) {
#pragma unroll
        for (int s = 0; s < MS; ++s) {
            sd[s] = DBL_MAX;
            sj[s] = INT_MAX;
            sk[s] = -1;
        }
        double wd = DBL_MAX;
        int wj = INT_MAX;
        for (int a = 0; a < n_amb; ++a) {
            const int k = n_in + a;
            const double d2 = xdist2(qx, qy, Ex[k], Ey[k]);
            const int j = Ej[k];
            if (!key_less(d2, j, wd, wj)) continue;
            bool lt[MS > 0 ? MS : 1];
#pragma unroll
            for (int s = 0; s < MS; ++s) lt[s] = key_less(d2, j, sd[s], sj[s]);
#pragma unroll
            for (int s = MS - 1; s >= 0; --s) {
                if (s < m) {
                    if (s > 0 && lt[s - 1]) {
                        sd[s] = sd[s - 1];
                        sj[s] = sj[s - 1];
                        sk[s] = sk[s - 1];
                    } else if (lt[s]) {
                        sd[s] = d2;
                        sj[s] = j;
                        sk[s] = k;
                    }
                }
            }
#pragma unroll
            for (int s = 0; s < MS; ++s)
                if (s == m - 1) {
                    wd = sd[s];
                    wj = sj[s];
                }
        }
        if (m > 0 && key_less(sd[0], sj[0], best_d, best_j)) {
            best_d = sd[0];
            best_j = sj[0];
            best_k = sk[0];
        }
    }
    const double d2min = best_d;
    const double rw = El[5 * best_k + 1], rz = El[5 * best_k + 2];
    const float nal = (float)(-alpha * kLog2e);
    double wsum = 0.0, sw = 0.0, sz = 0.0, sdx = 0.0, sdy = 0.0, ss = 0.0;
    auto accum = [&](int k, double d2) {
        const float arg = (float)(d2 - d2min) * nal;
        const double w = (double)ex2_approx(arg) * Ep[k];
        wsum += w;
        if (w <= 0.0) return;
        const double* q = &El[5 * k];
        double qw = q[1], qz = q[2], qdx = q[3], qdy = q[4];
        if (xadd(xmul(qw, rw), xmul(qz, rz)) < 0.0) {
            qw = -qw; qz = -qz; qdx = -qdx; qdy = -qdy;
        }
        sw = fma(w, qw, sw);
        sz = fma(w, qz, sz);
        sdx = fma(w, qdx, sdx);
        sdy = fma(w, qdy, sdy);
        ss = fma(w, q[0], ss);
    };
    for (int k = 0; k < n_in; ++k) accum(k, xdist2(qx, qy, Ex[k], Ey[k]));
    if (MS > 0) {
#pragma unroll
        for (int s = 0; s < MS; ++s)
            if (s < m) accum(sk[s], sd[s]);
    }
    const double inv = 1.0 / wsum;
    const double mw = sw * inv, mz = sz * inv, mdx = sdx * inv, mdy = sdy * inv;
    const double nr = xhypot(mw, mz);
    float2 dout = make_float2(0.f, 0.f);
    if (nr >= 1e-300) {
        W5 f{ss * inv, mw / nr, mz / nr, mdx / nr, mdy / nr};
        double yx, yy;
        xapply(f, qx, qy, &yx, &yy);
        dout = make_float2((float)(yx - qx), (float)(yy - qy));
    } else {
        dout = make_float2(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
    }
    if (out_d) *out_d = dout;
    if (out_u) {
        double arg = beta * d2min;
        if (55.0 < arg) arg = 55.0;
        *out_u = (float)xexp(arg);
    }
}

template <int MS>
__device__ __forceinline__ void emdq_dispatch_leaf(double qx, double qy, int n_in, int n_amb, int m,
                                                   const double* Ex, const double* Ey,
                                                   const double* Ep, const double* El,
                                                   const int* Ej, double alpha, double beta,
                                                   float2* od, float* ou) {
    emdq_pixel<MS>(qx, qy, n_in, n_amb, m, Ex, Ey, Ep, El, Ej, alpha, beta, od, ou);
}

template <int MAXMS>
__device__ void emdq_dispatch(double qx, double qy, int n_in, int n_amb, int m, const double* Ex,
                              const double* Ey, const double* Ep, const double* El, const int* Ej,
                              double alpha, double beta, float2* od, float* ou) {
    if (m <= 0)
        emdq_dispatch_leaf<0>(qx, qy, n_in, n_amb, m, Ex, Ey, Ep, El, Ej, alpha, beta, od, ou);
    else if (m <= 2)
        emdq_dispatch_leaf<2>(qx, qy, n_in, n_amb, m, Ex, Ey, Ep, El, Ej, alpha, beta, od, ou);
    else if (m <= 4)
        emdq_dispatch_leaf<4>(qx, qy, n_in, n_amb, m, Ex, Ey, Ep, El, Ej, alpha, beta, od, ou);
    else if (m <= 8)
        emdq_dispatch_leaf<8>(qx, qy, n_in, n_amb, m, Ex, Ey, Ep, El, Ej, alpha, beta, od, ou);
    else if (m <= 16 || MAXMS <= 16)
        emdq_dispatch_leaf<16>(qx, qy, n_in, n_amb, m, Ex, Ey, Ep, El, Ej, alpha, beta, od, ou);
    else
        emdq_dispatch_leaf<MAXMS>(qx, qy, n_in, n_amb, m, Ex, Ey, Ep, El, Ej, alpha, beta, od, ou);
}

template <int MAXMS>
__global__ void __launch_bounds__(ENT)
k_emdq(EmdqLaunch L, const int* __restrict__ cj, int S) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ESmem& s = *reinterpret_cast<ESmem*>(smem_raw);
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int ti0 = L.grid.i0 + blockIdx.x * ET, tj0 = L.grid.j0 + blockIdx.y * ET;
    const int ti1 = min(ti0 + ET - 1, L.grid.i1), tj1 = min(tj0 + ET - 1, L.grid.j1);
    const double xlo = L.grid.gx + ti0, xhi = L.grid.gx + ti1;
    const double ylo = L.grid.gy + tj0, yhi = L.grid.gy + tj1;
    const double cxm = 0.5 * (xlo + xhi), cym = 0.5 * (ylo + yhi);
    const double hd = 0.5 * sqrt((xhi - xlo) * (xhi - xlo) + (yhi - ylo) * (yhi - ylo));
    const int N = L.nactive;

    // ---- 1. radius bound from a histogram of centre distances -----------
    s.hist[t] = 0;
    if (t == 0) {
        s.ncand = 0;
        s.slow = 0;
    }
    __syncthreads();
    for (int a = t; a < N; a += ENT) {
        const float dx = (float)(L.cx[a] - cxm), dy = (float)(L.cy[a] - cym);
        atomicAdd(&s.hist[hist_bin(dx * dx + dy * dy)], 1);
    }
    __syncthreads();
    if (t == 0) {
        int acc = 0, b = 0;
        for (; b < 256; ++b) {
            acc += s.hist[b];
            if (acc >= S) break;
        }
        // bin upper edges are exact floats; relative slack covers FP32 error
        s.R = (b >= 255) ? INFINITY : sqrtf(bin_upper(b)) * 1.0001f + 0.01f;
    }
    __syncthreads();
    const float lim = s.R + (float)(2.0 * hd) + 1.0f;
    const float lim2 = lim * lim;

    // ---- 2. ordered candidate gather --------------------------------------
    for (int base = 0; base < N; base += ENT) {
        const int a = base + t;
        bool keep = false;
        if (a < N) {
            const float dx = (float)(L.cx[a] - cxm), dy = (float)(L.cy[a] - cym);
            keep = !(dx * dx + dy * dy > lim2);
        }
        const unsigned msk = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s.warp_cnt[wid] = __popc(msk);
        __syncthreads();
        int off = s.ncand;
        for (int w = 0; w < wid; ++w) off += s.warp_cnt[w];
        if (keep) {
            const int pos = off + __popc(msk & ((1u << lane) - 1u));
            if (pos < CAND_CAP) s.cand[pos] = a;
            else s.slow = 1;
        }
        __syncthreads();
        if (t == 0) {
            int tot = 0;
            for (int w = 0; w < ENT / 32; ++w) tot += s.warp_cnt[w];
            s.ncand += tot;
        }
        __syncthreads();
    }
    const int nc = min(s.ncand, CAND_CAP);

    // ---- 3. classify against the tile rectangle (FP64) ----------------------
    if (!s.slow) {
        for (int k = t; k < nc; k += ENT) {
            const int a = s.cand[k];
            const double ax = L.cx[a], ay = L.cy[a];
            const double dxn = fmax(fmax(xlo - ax, 0.0), ax - xhi), dyn = fmax(fmax(ylo - ay, 0.0), ay - yhi);
            const double dxf = fmax(ax - xlo, xhi - ax), dyf = fmax(ay - ylo, yhi - ay);
            s.dmin2[k] = dxn * dxn + dyn * dyn;
            s.dmax2[k] = dxf * dxf + dyf * dyf;
        }
        __syncthreads();
        for (int k = t; k < nc; k += ENT) {
            const double hi = s.dmax2[k] * (1.0 + 1e-12) + 1e-9;
            const double lo = s.dmin2[k] * (1.0 - 1e-12) - 1e-9;
            int cle = 0, clt = 0;
            for (int l = 0; l < nc; ++l) {
                if (l == k) continue;
                cle += s.dmin2[l] <= hi;
                clt += s.dmax2[l] < lo;
            }
            s.cls[k] = cle < S ? 1 : (clt >= S ? 0 : 2);
        }
        __syncthreads();
        if (t == 0) {
            int ni = 0, na = 0;
            for (int k = 0; k < nc; ++k) {
                ni += s.cls[k] == 1;
                na += s.cls[k] == 2;
            }
            s.n_in = ni;
            s.n_amb = na;
            if (ni > S || ni + na < S || ni + na > CAND_CAP) s.slow = 1;
        }
        __syncthreads();
    }

    const int i = ti0 + (t % ET), j = tj0 + (t / ET);
    const bool valid = i <= ti1 && j <= tj1;
    const size_t o = (size_t)(j - L.grid.j0) * (L.grid.i1 - L.grid.i0 + 1) + (i - L.grid.i0);
    const double qx = L.grid.gx + i, qy = L.grid.gy + j;
    float2* od = (valid && L.disp) ? &L.disp[o] : nullptr;
    float* ou = (valid && L.unc) ? &L.unc[o] : nullptr;

    if (s.slow) {  // exact brute force over every candidate (pathological tiles)
        if (valid) emdq_dispatch<MAXMS>(qx, qy, 0, N, S, L.cx, L.cy, L.cp, L.cl, cj, L.alpha, L.beta, od, ou);
        return;
    }

    // ---- 4. stage sure-in then ambiguous (ordered) -----------------------
    if (t == 0) {
        int pi = 0, pa = s.n_in;
        for (int k = 0; k < nc; ++k) {
            const int c = s.cls[k];
            if (c == 0) continue;
            const int pos = c == 1 ? pi++ : pa++;
            s.stage[pos] = s.cand[k];
        }
    }
    __syncthreads();
    const int ne = s.n_in + s.n_amb;
    for (int pos = t; pos < ne; pos += ENT) {
        const int a = s.stage[pos];
        s.px[pos] = L.cx[a];
        s.py[pos] = L.cy[a];
        s.pp[pos] = L.cp[a];
        s.pj[pos] = cj[a];
#pragma unroll
        for (int q = 0; q < 5; ++q) s.pl[pos][q] = L.cl[5 * a + q];
    }
    __syncthreads();
    if (valid)
        emdq_dispatch<MAXMS>(qx, qy, s.n_in, s.n_amb, S - s.n_in, s.px, s.py, s.pp, &s.pl[0][0], s.pj,
                      L.alpha, L.beta, od, ou);
}

}  // namespace

cudaError_t launch_emdq_field(const EmdqLaunch& L, cudaStream_t st, int64_t* launches) {
    if (L.nactive <= 0) return cudaErrorInvalidValue;
    int* cj = reinterpret_cast<int*>(L.cp + L.nactive);  // scratch follows cp (see nrm_abi.cu)
    k_gather<<<(L.nactive + 255) / 256, 256, 0, st>>>(L.apts, L.locals, L.probs, L.active,
                                                       L.nactive, L.cx, L.cy, L.cl, L.cp, cj);
    ++*launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int S = L.support < L.nactive ? L.support : L.nactive;
    const int nx = (L.grid.i1 - L.grid.i0 + 1 + ET - 1) / ET;
    const int ny = (L.grid.j1 - L.grid.j0 + 1 + ET - 1) / ET;
    const size_t smem = sizeof(ESmem);
    if (S <= 16) {
        cudaFuncSetAttribute(k_emdq<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_emdq<16><<<dim3(nx, ny), ENT, smem, st>>>(L, cj, S);
    } else {
        cudaFuncSetAttribute(k_emdq<MAX_SUPPORT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_emdq<MAX_SUPPORT><<<dim3(nx, ny), ENT, smem, st>>>(L, cj, S);
    }
    ++*launches;
    return cudaGetLastError();
}

}  // namespace nrm
