// nrm_abi.cu -- host side of the C ABI (include/nrm_b200.h): contexts,
// HBM-resident canvases with the reference's growth bookkeeping, transfers
// and kernel orchestration. No compute happens on the host: every per-pixel
// result comes from the kernels in k_*.cu.
#include <cudaTypedefs.h>
#include <cstdlib>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <new>
#include <string>
#include <vector>

#include "nrm_common.cuh"
#include "nrm_internal.h"

namespace nrm {

namespace {
thread_local std::string g_last_error;

constexpr int64_t kTile64 = kTile;

int64_t align_down(int64_t v) { return v >= 0 ? (v / kTile64) * kTile64 : ((v - kTile64 + 1) / kTile64) * kTile64; }
int64_t align_up(int64_t v) { return -align_down(-v); }

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

#define NRM_CUDA(call)                                  \
    do {                                                \
        const cudaError_t e__ = (call);                 \
        if (e__ != cudaSuccess) return cuda_fail(e__, #call); \
    } while (0)

#define NRM_CHECK(rc_expr)             \
    do {                               \
        const int rc__ = (rc_expr);    \
        if (rc__ != NRM_OK) return rc__; \
    } while (0)

}  // namespace

namespace {
thread_local nrm_ctx* g_prof_ctx = nullptr;
}

void prof_mark(const char* name, cudaStream_t st) {
    nrm_ctx* c = g_prof_ctx;
    if (!c || !c->prof.on) return;
    Prof& p = c->prof;
    if (p.used == p.ev.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return;
        p.ev.push_back(e);
        p.name.push_back(nullptr);
    }
    p.name[p.used] = name;
    cudaEventRecord(p.ev[p.used], st);
    ++p.used;
}

bool prof_serialized() { return g_prof_ctx && g_prof_ctx->prof.on; }

ProfScope::ProfScope(nrm_ctx* c) : prev(g_prof_ctx) { g_prof_ctx = c; }
ProfScope::~ProfScope() {
    if (g_prof_ctx) prof_mark(nullptr, g_prof_ctx->stream);  // end of the call
    g_prof_ctx = prev;
}

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? NRM_ENOMEM : NRM_ECUDA;
}

cudaError_t DevBuf::ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(bytes, 256);
    const cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
}
void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
}

cudaError_t PinnedBuf::ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(bytes, 4096);
    const cudaError_t e = cudaHostAlloc(&p, want, cudaHostAllocDefault);
    if (e == cudaSuccess) cap = want;
    return e;
}
void PinnedBuf::release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
}

namespace {

int upload(nrm_ctx* c, DevBuf& dst, const void* src, size_t bytes) {
    NRM_CUDA(dst.ensure(bytes));
    if (bytes) NRM_CUDA(cudaMemcpyAsync(dst.p, src, bytes, cudaMemcpyHostToDevice, c->stream));
    return NRM_OK;
}

bool finite_all(const double* p, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(p[i])) return false;
    return true;
}

// ---- canvas storage ------------------------------------------------------
void free_planes(nrm_canvas* cv) {
    float* f[6] = {cv->r, cv->g, cv->b, cv->ar, cv->ag, cv->ab};
    for (float* p : f) cudaFree(p);
    cudaFree(cv->w);
    cudaFree(cv->aw);
    cv->r = cv->g = cv->b = cv->ar = cv->ag = cv->ab = nullptr;
    cv->w = cv->aw = nullptr;
}

// Reallocates physical storage to cover absolute [x0,x1) x [y0,y1) and
// copies the current logical window across; new pixels are zero.
int grow_physical(nrm_canvas* cv, int64_t x0, int64_t y0, int64_t x1, int64_t y1) {
    nrm_ctx* c = cv->ctx;
    const int64_t w64 = x1 - x0, h64 = y1 - y0;
    if (w64 <= 0 || h64 <= 0 || w64 > (1 << 30) || h64 > (1 << 30) || w64 * h64 > (int64_t)1 << 36)
        return fail(NRM_EINVAL, "canvas: requested extent too large");
    const size_t npx = (size_t)w64 * (size_t)h64;
    float *r = nullptr, *g = nullptr, *b = nullptr;
    uint8_t* w = nullptr;
    cudaError_t e = cudaMalloc(&r, npx * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&g, npx * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&b, npx * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&w, npx);
    if (e != cudaSuccess) {
        cudaFree(r);
        cudaFree(g);
        cudaFree(b);
        cudaFree(w);
        return cuda_fail(e, "canvas allocation");
    }
    // on any failure below the new planes are released (the canvas keeps its old storage)
    auto release_new = [&](cudaError_t err, const char* what) {
        cudaStreamSynchronize(c->stream);
        cudaFree(r);
        cudaFree(g);
        cudaFree(b);
        cudaFree(w);
        return cuda_fail(err, what);
    };
#define NRM_GROW(call)                                        \
    do {                                                      \
        const cudaError_t e__ = (call);                       \
        if (e__ != cudaSuccess) return release_new(e__, #call); \
    } while (0)
    NRM_GROW(cudaMemsetAsync(r, 0, npx * sizeof(float), c->stream));
    NRM_GROW(cudaMemsetAsync(g, 0, npx * sizeof(float), c->stream));
    NRM_GROW(cudaMemsetAsync(b, 0, npx * sizeof(float), c->stream));
    NRM_GROW(cudaMemsetAsync(w, 0, npx, c->stream));
    if (cv->width > 0 && cv->r) {
        const size_t spitch = (size_t)cv->cap_w, dpitch = (size_t)w64;
        const size_t soff = (size_t)(cv->origin_y - cv->phys_y0) * spitch + (size_t)(cv->origin_x - cv->phys_x0);
        const size_t doff = (size_t)(cv->origin_y - y0) * dpitch + (size_t)(cv->origin_x - x0);
        float* planes_old[3] = {cv->r, cv->g, cv->b};
        float* planes_new[3] = {r, g, b};
        for (int k = 0; k < 3; ++k)
            NRM_GROW(cudaMemcpy2DAsync(planes_new[k] + doff, dpitch * sizeof(float), planes_old[k] + soff,
                                       spitch * sizeof(float), (size_t)cv->width * sizeof(float),
                                       (size_t)cv->height, cudaMemcpyDeviceToDevice, c->stream));
        NRM_GROW(cudaMemcpy2DAsync(w + doff, dpitch, cv->w + soff, spitch, (size_t)cv->width,
                                   (size_t)cv->height, cudaMemcpyDeviceToDevice, c->stream));
        NRM_GROW(cudaStreamSynchronize(c->stream));
    }
#undef NRM_GROW
    free_planes(cv);
    cv->r = r;
    cv->g = g;
    cv->b = b;
    cv->w = w;
    cv->phys_x0 = x0;
    cv->phys_y0 = y0;
    cv->cap_w = (int)w64;
    cv->cap_h = (int)h64;
    return NRM_OK;
}

bool covers(const nrm_canvas* cv, int64_t x0, int64_t y0, int64_t x1, int64_t y1) {
    return cv->r && x0 >= cv->phys_x0 && y0 >= cv->phys_y0 && x1 <= cv->phys_x0 + cv->cap_w &&
           y1 <= cv->phys_y0 + cv->cap_h;
}

// Canvas::ensure_contains (mosaic.hpp:131-174) bookkeeping as a pure host
// function: the logical canvas (ox, oy, w, h) after growing to contain the
// rectangle. Returns NRM_OK; *grew = 0 when the canvas already contains it.
int plan_ensure_contains(int64_t ox, int64_t oy, int w, int h, double rx0, double ry0, double rx1, double ry1,
                         int64_t* nox, int64_t* noy, int64_t* nw, int64_t* nh, int* grew) {
    if (!(std::isfinite(rx0) && std::isfinite(ry0) && std::isfinite(rx1) && std::isfinite(ry1)))
        return fail(NRM_EINVAL, "ensure_contains: non-finite rectangle");
    if (std::fabs(rx0) > 1e9 || std::fabs(ry0) > 1e9 || std::fabs(rx1) > 1e9 || std::fabs(ry1) > 1e9)
        return fail(NRM_EINVAL, "ensure_contains: rectangle out of range");
    const int64_t nx0n = (int64_t)std::floor(rx0), ny0n = (int64_t)std::floor(ry0);
    const int64_t nx1n = (int64_t)std::ceil(rx1) + 1, ny1n = (int64_t)std::ceil(ry1) + 1;
    const bool empty = w == 0;
    *nox = ox;
    *noy = oy;
    *nw = w;
    *nh = h;
    *grew = 0;
    if (!empty && nx0n >= ox && ny0n >= oy && nx1n <= ox + w && ny1n <= oy + h) return NRM_OK;
    int64_t nx0 = align_down(nx0n), ny0 = align_down(ny0n);
    int64_t nx1 = nx1n, ny1 = ny1n;
    if (!empty) {
        nx0 = std::min(nx0, ox);
        ny0 = std::min(ny0, oy);
        nx1 = std::max(nx1, ox + (int64_t)w);
        ny1 = std::max(ny1, oy + (int64_t)h);
    }
    *nox = nx0;
    *noy = ny0;
    *nw = ((nx1 - nx0 + kTile64 - 1) / kTile64) * kTile64;
    *nh = ((ny1 - ny0 + kTile64 - 1) / kTile64) * kTile64;
    if (*nw > (1 << 30) || *nh > (1 << 30)) return fail(NRM_EINVAL, "ensure_contains: canvas too large");
    *grew = 1;
    return NRM_OK;
}

int ensure_contains(nrm_canvas* cv, double rx0, double ry0, double rx1, double ry1) {
    int64_t nx0, ny0, nw, nh;
    int grew = 0;
    NRM_CHECK(plan_ensure_contains(cv->origin_x, cv->origin_y, cv->width, cv->height, rx0, ry0, rx1, ry1, &nx0, &ny0,
                                   &nw, &nh, &grew));
    if (!grew) return NRM_OK;
    if (!covers(cv, nx0, ny0, nx0 + nw, ny0 + nh)) {
        int64_t px0 = nx0, py0 = ny0, px1 = nx0 + nw, py1 = ny0 + nh;
        if (cv->res_x1 > cv->res_x0) {
            px0 = std::min(px0, cv->res_x0);
            py0 = std::min(py0, cv->res_y0);
            px1 = std::max(px1, cv->res_x1);
            py1 = std::max(py1, cv->res_y1);
        }
        NRM_CHECK(grow_physical(cv, px0, py0, px1, py1));
    }
    cv->origin_x = nx0;
    cv->origin_y = ny0;
    cv->width = (int)nw;
    cv->height = (int)nh;
    return NRM_OK;
}

struct Bbox {
    double x0, y0, x1, y1;
};

// polygon_bbox (geometry.hpp:180-190) + Rect::expanded(4.0) (mosaic.hpp:203)
Bbox footprint_bbox(const double* poly, int npoly) {
    Bbox r{std::numeric_limits<double>::max(), std::numeric_limits<double>::max(),
           std::numeric_limits<double>::lowest(), std::numeric_limits<double>::lowest()};
    for (int i = 0; i < npoly; ++i) {
        r.x0 = std::min(r.x0, poly[2 * i]);
        r.y0 = std::min(r.y0, poly[2 * i + 1]);
        r.x1 = std::max(r.x1, poly[2 * i]);
        r.y1 = std::max(r.y1, poly[2 * i + 1]);
    }
    return {r.x0 - 4.0, r.y0 - 4.0, r.x1 + 4.0, r.y1 + 4.0};
}

// Per-context device state (c->misc, zeroed at context creation and restored
// by every exception pass): acc[3] (u64) | exc_count (u32) | overflow (u32).
// Diagnostics follow: last_exc (u32, pixels the last exception pass resolved),
// emdq_exact (u32, K3 pixels that took the exact tier, reset per call).
struct State {
    unsigned long long* acc;
    unsigned* exc_count;
    unsigned* overflow;
    unsigned* last_exc;
    unsigned* emdq_exact;
    unsigned* exc_done;
};
State state_of(nrm_ctx* c) {
    char* b = c->misc.as<char>();
    return {reinterpret_cast<unsigned long long*>(b), reinterpret_cast<unsigned*>(b + 24),
            reinterpret_cast<unsigned*>(b + 28), reinterpret_cast<unsigned*>(b + 32),
            reinterpret_cast<unsigned*>(b + 36), reinterpret_cast<unsigned*>(b + 40)};
}

// Exception-queue slots for a launch over `pixels` grid pixels. The fast
// tiers defer ~1e-5 of the pixels (34 of 2.6 M on C2), or whole tiles whose
// warps span more than a quarter turn; a deferral past the capacity is not
// lost but marked in the output and found by the exact pass's scan
// (k_nodefield.cu spill_mark), so the queue is sized for the common case:
// 1/64 of the pixels, at least 2^18 slots (8 B each).
size_t exception_capacity(const nrm_ctx* c, size_t pixels) {
    size_t cap = std::max<size_t>((size_t)1 << 18, pixels / 64);
    if (c->exc_cap_override > 0) cap = (size_t)c->exc_cap_override;
    return std::max<size_t>(1, std::min<size_t>({cap, pixels, (size_t)0x7fffffff}));
}

// K1's canvas tensor maps (TMA): the four planes as 2D tensors of cap_w x
// cap_h elements, box 32 x 32 (one K1 CTA's canvas tile). The encoder comes
// from the driver through the runtime (no libcuda link). Returns false (and
// K1 stages the tile with cp.async) when a plane does not meet TMA's
// alignment rules or the encoder is unavailable.
bool canvas_tensor_maps(const nrm_canvas* cv, NodeFieldLaunch& L) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    static const bool off = std::getenv("NRM_B200_NO_TMA") != nullptr;  // tests: the cp.async staging path
    if (off || !encode || cv->cap_w % 16 != 0) return false;
    const void* planes[4] = {cv->r, cv->g, cv->b, cv->w};
    for (int k = 0; k < 4; ++k) {
        if (reinterpret_cast<uintptr_t>(planes[k]) % 16 != 0) return false;
        const bool f32 = k < 3;
        const cuuint64_t dims[2] = {(cuuint64_t)cv->cap_w, (cuuint64_t)cv->cap_h};
        const cuuint64_t stride[1] = {(cuuint64_t)cv->cap_w * (f32 ? 4u : 1u)};
        const cuuint32_t box[2] = {32, 32}, estride[2] = {1, 1};
        if (encode(&L.ctm[k], f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 2,
                   const_cast<void*>(planes[k]), dims, stride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    return true;
}

// K1's frame textures: frames converted to RGBA8 rows (pitch a multiple of
// 128 B), frame k into slot k of the context's frame_rgba buffer, and a
// texture object per slot (point sampling, clamped addresses, normalised
// reads), rebuilt only when a slot's storage or the frame shape changes. A
// batch converts in one k_frame_rgba launch; a single frame (`fused`) hands
// the conversion to its planner launch (NodeFieldLaunch::frgba).
int frame_textures(nrm_ctx* c, int nf, const uint8_t* const* d_frames, int fw, int fh, int ch,
                   NodeFieldLaunch* const* Ls, bool fused) {
    if (nf <= 0 || nf > kFrameSlots) return fail(NRM_EINVAL, "frame texture count out of range");
    const size_t pitch = ((size_t)fw * 4 + 127) & ~size_t(127), bytes = pitch * (size_t)fh;
    if (c->frame_rgba.cap < bytes * (size_t)nf) {
        NRM_CUDA(cudaStreamSynchronize(c->stream));  // the old storage may still be sampled
        NRM_CUDA(c->frame_rgba.ensure(bytes * (size_t)nf));
    }
    if (fused) {
        if (nf != 1) return fail(NRM_EINVAL, "fused frame conversion takes one frame");
        Ls[0]->frgba = c->frame_rgba.as<uint8_t>();
        Ls[0]->frgba_pitch = pitch;
    } else {
        FrameSet fs = {};
        for (int k = 0; k < nf; ++k) fs.f[k] = d_frames[k];
        NRM_CUDA(launch_frame_rgba(fs, nf, fw, fh, ch, c->frame_rgba.as<uint8_t>(), pitch, bytes, c->stream,
                                   &c->launches));
    }
    for (int k = 0; k < nf; ++k) {
        uint8_t* dst = c->frame_rgba.as<uint8_t>() + bytes * (size_t)k;
        if (!c->ftex[k] || c->ftex_ptr[k] != dst || c->ftex_w[k] != fw || c->ftex_h[k] != fh ||
            c->ftex_pitch[k] != pitch) {
            if (c->ftex[k]) {
                NRM_CUDA(cudaStreamSynchronize(c->stream));  // no launch may still use the old object
                cudaDestroyTextureObject((cudaTextureObject_t)c->ftex[k]);
                c->ftex[k] = 0;
            }
            cudaResourceDesc rd = {};
            rd.resType = cudaResourceTypePitch2D;
            rd.res.pitch2D.devPtr = dst;
            rd.res.pitch2D.desc = cudaCreateChannelDesc<uchar4>();
            rd.res.pitch2D.width = (size_t)fw;
            rd.res.pitch2D.height = (size_t)fh;
            rd.res.pitch2D.pitchInBytes = pitch;
            cudaTextureDesc td = {};
            td.addressMode[0] = td.addressMode[1] = cudaAddressModeClamp;
            td.filterMode = cudaFilterModePoint;
            td.readMode = cudaReadModeNormalizedFloat;
            td.normalizedCoords = 0;
            cudaTextureObject_t t = 0;
            NRM_CUDA(cudaCreateTextureObject(&t, &rd, &td, nullptr));
            c->ftex[k] = (unsigned long long)t;
            c->ftex_ptr[k] = dst;
            c->ftex_w[k] = fw;
            c->ftex_h[k] = fh;
            c->ftex_pitch[k] = pitch;
        }
        Ls[k]->ftex = c->ftex[k];
    }
    return NRM_OK;
}

// Shared core of blend_frame: everything after the inputs are in HBM.
// d_stats: int64[4] on the device, written by the exception pass.
int blend_core(nrm_canvas* cv, const uint8_t* d_frame, int fw, int fh, int ch, const double* d_anchors,
               const double* d_warps, int n, double alpha, const double* poly, int npoly,
               unsigned long long* d_stats, const float* d_unc = nullptr) {
    nrm_ctx* c = cv->ctx;
    if (fw <= 0 || fh <= 0 || npoly < 3) {  // mosaic.hpp:201: empty stats, canvas untouched
        NRM_CUDA(cudaMemsetAsync(d_stats, 0, 4 * sizeof(unsigned long long), c->stream));
        return NRM_OK;
    }
    if (!finite_all(poly, (size_t)npoly * 2)) return fail(NRM_EINVAL, "blend_frame: non-finite polygon");
    const Bbox bb = footprint_bbox(poly, npoly);
    NRM_CHECK(ensure_contains(cv, bb.x0, bb.y0, bb.x1, bb.y1));
    const double orgx = (double)cv->origin_x, orgy = (double)cv->origin_y;
    const int px0 = (int)std::floor(bb.x0 - orgx), py0 = (int)std::floor(bb.y0 - orgy);
    const int px1 = (int)std::ceil(bb.x1 - orgx), py1 = (int)std::ceil(bb.y1 - orgy);
    const int bw = px1 - px0 + 1, bh = py1 - py0 + 1;
    if (bw <= 0 || bh <= 0) {  // mosaic.hpp:212
        NRM_CUDA(cudaMemsetAsync(d_stats, 0, 4 * sizeof(unsigned long long), c->stream));
        return NRM_OK;
    }
    const unsigned long long footprint = (unsigned long long)bw * (unsigned long long)bh;
    const size_t exc_cap = exception_capacity(c, footprint);
    NRM_CUDA(c->exc.ensure(exc_cap * sizeof(int2) + 64));
    const State st = state_of(c);

    NodeFieldLaunch L;
    L.frame = d_frame;
    L.fw = fw;
    L.fh = fh;
    L.fch = ch;
    L.unc = d_unc;
    L.anchors = d_anchors;
    L.warps = d_warps;
    L.n = n;
    L.alpha = alpha;
    // index space = absolute reference pixel coordinates
    L.grid.gx = 0.0;
    L.grid.gy = 0.0;
    L.grid.i0 = (int)(cv->origin_x + px0);
    L.grid.i1 = (int)(cv->origin_x + px1);
    L.grid.j0 = (int)(cv->origin_y + py0);
    L.grid.j1 = (int)(cv->origin_y + py1);
    L.R = cv->r;
    L.G = cv->g;
    L.B = cv->b;
    L.W = cv->w;
    L.pitch = cv->cap_w;
    L.phys_x0 = (int)cv->phys_x0;
    L.phys_y0 = (int)cv->phys_y0;
    L.band_rank = cv->band_rank;
    L.band_count = cv->band_count;
    L.acc = st.acc;
    L.stats_out = d_stats;
    L.footprint = footprint;
    L.exc = c->exc.as<int2>();
    L.exc_count = st.exc_count;
    L.exc_cap = (unsigned)exc_cap;
    L.exc_overflow = st.overflow;
    L.exc_last = st.last_exc;
    L.exc_done = st.exc_done;
    L.ctm_ok = canvas_tensor_maps(cv, L) ? 1 : 0;
    NRM_CUDA(c->tiles.ensure(node_field_scratch_bytes(L)));
    L.plans = c->tiles.p;
    if (ch == 3 || ch == 4) {
        NodeFieldLaunch* lp = &L;
        NRM_CHECK(frame_textures(c, 1, &d_frame, fw, fh, ch, &lp, true));
    }
    NRM_CUDA(launch_node_field(L, 0, c->stream, &c->launches));
    return NRM_OK;
}

int check_canvas(const nrm_canvas* cv) {
    if (!cv || !cv->ctx) return fail(NRM_ESTATE, "null canvas");
    return NRM_OK;
}

int check_region(const nrm_canvas* cv, int x, int y, int w, int h) {
    if (w < 0 || h < 0 || x < 0 || y < 0 || (int64_t)x + w > cv->width || (int64_t)y + h > cv->height)
        return fail(NRM_EINVAL, "canvas region out of bounds");
    return NRM_OK;
}

int validate_nodes(const double* anchors, const double* warps, int n, double alpha, bool host) {
    if (n < 0) return fail(NRM_EINVAL, "negative node count");
    if (n > 0 && (!anchors || !warps)) return fail(NRM_EINVAL, "null node arrays");
    if (!std::isfinite(alpha) || alpha < 0.0) return fail(NRM_EINVAL, "alpha must be finite and >= 0");
    if (host && n > 0 && (!finite_all(anchors, (size_t)n * 2) || !finite_all(warps, (size_t)n * 5)))
        return fail(NRM_EINVAL, "non-finite node arrays");
    return NRM_OK;
}

int grid_indices(const nrm_grid* g, FieldGrid* out) {
    if (!g || g->width < 0 || g->height < 0) return fail(NRM_EINVAL, "bad grid");
    if (!std::isfinite(g->x0) || !std::isfinite(g->y0)) return fail(NRM_EINVAL, "non-finite grid origin");
    out->gx = g->x0;
    out->gy = g->y0;
    out->i0 = 0;
    out->j0 = 0;
    out->i1 = g->width - 1;
    out->j1 = g->height - 1;
    return NRM_OK;
}

int node_field_core(nrm_ctx* c, const nrm_grid* grid, const double* d_anchors, const double* d_warps,
                    int n, double alpha, float* d_disp, uint8_t* d_support, int band_rank = 0, int band_count = 1,
                    bool absolute = false) {
    FieldGrid fg;
    NRM_CHECK(grid_indices(grid, &fg));
    if (absolute) {
        // stripes are anchored to absolute rows: index space = absolute pixels
        if (grid->x0 != std::floor(grid->x0) || grid->y0 != std::floor(grid->y0) || std::fabs(grid->x0) > 1e9 ||
            std::fabs(grid->y0) > 1e9)
            return fail(NRM_EINVAL, "node_field: a banded grid needs an integral origin");
        fg.gx = 0.0;
        fg.gy = 0.0;
        fg.i0 = (int)grid->x0;
        fg.j0 = (int)grid->y0;
        fg.i1 = fg.i0 + grid->width - 1;
        fg.j1 = fg.j0 + grid->height - 1;
    }
    const size_t npx = (size_t)grid->width * (size_t)grid->height;
    if (npx == 0) return NRM_OK;
    const size_t exc_cap = exception_capacity(c, npx);
    NRM_CUDA(c->exc.ensure(exc_cap * sizeof(int2) + 64));
    const State st = state_of(c);
    NodeFieldLaunch L;
    L.anchors = d_anchors;
    L.warps = d_warps;
    L.n = n;
    L.alpha = alpha;
    L.grid = fg;
    L.band_rank = band_rank;
    L.band_count = band_count;
    L.disp = reinterpret_cast<float2*>(d_disp);
    L.support = d_support;
    L.exc = c->exc.as<int2>();
    L.exc_count = st.exc_count;
    L.exc_cap = (unsigned)exc_cap;
    L.exc_overflow = st.overflow;
    L.exc_last = st.last_exc;
    L.exc_done = st.exc_done;
    NRM_CUDA(c->tiles.ensure(node_field_scratch_bytes(L)));
    L.plans = c->tiles.p;
    NRM_CUDA(launch_node_field(L, 1, c->stream, &c->launches));
    return NRM_OK;
}

int emdq_core(nrm_ctx* c, const nrm_grid* grid, const double* d_apts, const double* d_locals,
              const double* d_probs, int m_total, const int32_t* d_active, int nactive, double alpha,
              int support, double beta, float* d_disp, float* d_unc) {
    FieldGrid fg;
    NRM_CHECK(grid_indices(grid, &fg));
    if (nactive <= 0 || m_total <= 0) return fail(NRM_EINVAL, "emdq_field: no candidates");
    if (support < 1 || support > 32) return fail(NRM_EINVAL, "emdq_field: support must be in [1, 32]");
    if (!(beta > 0.0) || !std::isfinite(beta)) return fail(NRM_EINVAL, "node_uncertainty: beta must be positive");
    if (!std::isfinite(alpha) || alpha < 0.0) return fail(NRM_EINVAL, "alpha must be finite and >= 0");
    if ((size_t)grid->width * (size_t)grid->height == 0) return NRM_OK;
    const size_t na = (size_t)nactive;
    NRM_CUDA(c->pts.ensure(emdq_scratch_bytes(nactive, fg)));
    double* base = c->pts.as<double>();
    EmdqLaunch L;
    L.grid = fg;
    L.apts = d_apts;
    L.locals = d_locals;
    L.probs = d_probs;
    L.active = d_active;
    L.m_total = m_total;
    L.nactive = nactive;
    L.alpha = alpha;
    L.beta = beta;
    L.support = support;
    L.disp = reinterpret_cast<float2*>(d_disp);
    L.unc = d_unc;
    L.cx = base;
    L.cy = base + na;
    L.cl = base + 2 * na;
    L.cp = base + 7 * na;  // phi, c32, j, supertile lists and plans follow: see launch_emdq_field
    L.exact_count = state_of(c).emdq_exact;  // zeroed by k_super (no memset node in the PDL chain)
    L.exq_cap_override = c->exc_cap_override;
    size_t cnt_bytes = 0, bin_bytes = 0;
    emdq_cell_bytes(nactive, fg, &cnt_bytes, &bin_bytes);
    if (cnt_bytes) {  // large candidate sets: binned supertile scans
        const bool grow = c->emdq_cell_cnt.cap < cnt_bytes;
        NRM_CUDA(c->emdq_cell_cnt.ensure(cnt_bytes));
        // the bin counts start at zero; the last k_gather CTA re-zeroes every count it used
        if (grow) NRM_CUDA(cudaMemsetAsync(c->emdq_cell_cnt.p, 0, c->emdq_cell_cnt.cap, c->stream));
        NRM_CUDA(c->emdq_cells.ensure(bin_bytes));
        L.cell_cnt = c->emdq_cell_cnt.as<int>();
        L.cells = c->emdq_cells.as<int>();
    }
    NRM_CUDA(launch_emdq_field(L, c->stream, &c->launches));
    return NRM_OK;
}

// Scattered-query EMDQ (E-step / final field) on device arrays; bbox4 =
// {minx, miny, maxx, maxy} of the queries.
constexpr double kPointsSpanMax = 32768.0;  // wider query spreads scan every candidate
int points_core(nrm_ctx* c, const double* bbox4, const double* d_q, const int32_t* d_excl, int nq,
                const double* d_apts, const double* d_locals, const double* d_probs, int m_total,
                const int32_t* d_active, int nactive, double alpha, int support, double beta, double* d_warps,
                double* d_pred, double* d_unc, int32_t* d_status) {
    if (nq == 0) return NRM_OK;
    if (nactive <= 0 || m_total <= 0) return fail(NRM_EINVAL, "emdq_points: no candidates");
    if (support < 1 || support > 32) return fail(NRM_EINVAL, "emdq_points: support must be in [1, 32]");
    if (d_unc && (!(beta > 0.0) || !std::isfinite(beta)))
        return fail(NRM_EINVAL, "node_uncertainty: beta must be positive");
    if (!std::isfinite(alpha) || alpha < 0.0) return fail(NRM_EINVAL, "alpha must be finite and >= 0");
    for (int k = 0; k < 4; ++k)
        if (!std::isfinite(bbox4[k]) || std::fabs(bbox4[k]) > 1e9)
            return fail(NRM_EINVAL, "emdq_points: non-finite or out-of-range query");
    FieldGrid fg;
    fg.gx = 0.0;
    fg.gy = 0.0;
    fg.i0 = (int)std::floor(bbox4[0]);
    fg.j0 = (int)std::floor(bbox4[1]);
    fg.i1 = (int)std::floor(bbox4[2]);
    fg.j1 = (int)std::floor(bbox4[3]);
    PointsLaunch P;
    P.full_scan = (bbox4[2] - bbox4[0]) * (bbox4[3] - bbox4[1]) > kPointsSpanMax * kPointsSpanMax;
    if (P.full_scan) fg.i1 = fg.i0, fg.j1 = fg.j0;
    const size_t na = (size_t)nactive;
    NRM_CUDA(c->pts.ensure(emdq_scratch_bytes(nactive, fg, false)));
    double* base = c->pts.as<double>();
    EmdqLaunch L;
    L.grid = fg;
    L.apts = d_apts;
    L.locals = d_locals;
    L.probs = d_probs;
    L.active = d_active;
    L.m_total = m_total;
    L.nactive = nactive;
    L.alpha = alpha;
    L.beta = beta;
    L.support = support;
    L.cx = base;
    L.cy = base + na;
    L.cl = base + 2 * na;
    L.cp = base + 7 * na;
    P.q = d_q;
    P.excl = d_excl;
    P.nq = nq;
    P.warps = d_warps;
    P.pred = d_pred;
    P.unc = d_unc;
    P.status = d_status;
    NRM_CUDA(launch_emdq_points(L, P, c->stream, &c->launches));
    return NRM_OK;
}

}  // namespace
}  // namespace nrm

using namespace nrm;

extern "C" {

int nrm_abi_version(void) { return NRM_ABI_VERSION; }
const char* nrm_last_error(void) { return g_last_error.c_str(); }

int nrm_ctx_create(int device, nrm_ctx** out) {
    if (!out) return fail(NRM_EINVAL, "null out");
    *out = nullptr;
    int ndev = 0;
    NRM_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(NRM_EINVAL, "no such CUDA device");
    nrm_ctx* c = new (std::nothrow) nrm_ctx();
    if (!c) return fail(NRM_ENOMEM, "context allocation");
    c->device = device;
    DeviceGuard g(device);
    cudaError_t e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaStreamCreate");
    }
    c->stream = c->own_stream;
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    // per-context device state (see State): zero once, restored by every exception pass
    e = c->misc.ensure(256);
    if (e == cudaSuccess) e = cudaMemset(c->misc.p, 0, 256);
    if (e != cudaSuccess) {
        cudaStreamDestroy(c->own_stream);
        delete c;
        return cuda_fail(e, "context state allocation");
    }
    *out = c;
    return NRM_OK;
}

int nrm_ctx_destroy(nrm_ctx* c) {
    if (!c) return NRM_OK;
    DeviceGuard g(c->device);
    cudaStreamSynchronize(c->stream);
    for (unsigned long long t : c->ftex)
        if (t) cudaDestroyTextureObject((cudaTextureObject_t)t);
    DevBuf* bufs[] = {&c->frame_raw, &c->anchors, &c->warps, &c->exc,   &c->misc,  &c->stats, &c->pts,
                      &c->locals,    &c->probs,   &c->active, &c->out_a, &c->out_b, &c->tiles, &c->feat,
                      &c->feat_io,   &c->batch,  &c->halo,   &c->frame_rgba, &c->emdq_cells, &c->emdq_cell_cnt};
    for (DevBuf* b : bufs) b->release();
    c->staging.release();
    c->staging_out.release();
    for (cudaEvent_t e : c->prof.ev) cudaEventDestroy(e);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    delete c;
    return NRM_OK;
}

int nrm_ctx_set_stream(nrm_ctx* c, void* s) {
    if (!c) return fail(NRM_ESTATE, "null context");
    c->stream = s ? static_cast<cudaStream_t>(s) : c->own_stream;
    return NRM_OK;
}
void* nrm_ctx_stream(nrm_ctx* c) { return c ? (void*)c->stream : nullptr; }
int nrm_ctx_synchronize(nrm_ctx* c) {
    if (!c) return fail(NRM_ESTATE, "null context");
    DeviceGuard g(c->device);
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    NRM_CUDA(cudaGetLastError());
    return NRM_OK;
}
int nrm_ctx_launch_count(nrm_ctx* c, int64_t* out) {
    if (!c || !out) return fail(NRM_EINVAL, "null argument");
    *out = c->launches;
    return NRM_OK;
}

// ---- canvas ---------------------------------------------------------------
int nrm_canvas_create(nrm_ctx* c, nrm_canvas** out) {
    if (!c || !out) return fail(NRM_EINVAL, "null argument");
    nrm_canvas* cv = new (std::nothrow) nrm_canvas();
    if (!cv) return fail(NRM_ENOMEM, "canvas allocation");
    cv->ctx = c;
    *out = cv;
    return NRM_OK;
}

int nrm_canvas_destroy(nrm_canvas* cv) {
    if (!cv) return NRM_OK;
    if (cv->ctx) {
        DeviceGuard g(cv->ctx->device);
        cudaStreamSynchronize(cv->ctx->stream);
        free_planes(cv);
    }
    delete cv;
    return NRM_OK;
}

int nrm_canvas_reserve(nrm_canvas* cv, double x0, double y0, double x1, double y1) {
    NRM_CHECK(check_canvas(cv));
    if (!(std::isfinite(x0) && std::isfinite(y0) && std::isfinite(x1) && std::isfinite(y1)) || x1 < x0 || y1 < y0)
        return fail(NRM_EINVAL, "reserve: bad rectangle");
    DeviceGuard g(cv->ctx->device);
    cv->res_x0 = align_down((int64_t)std::floor(x0));
    cv->res_y0 = align_down((int64_t)std::floor(y0));
    cv->res_x1 = align_up((int64_t)std::ceil(x1) + 1);
    cv->res_y1 = align_up((int64_t)std::ceil(y1) + 1);
    int64_t px0 = cv->res_x0, py0 = cv->res_y0, px1 = cv->res_x1, py1 = cv->res_y1;
    if (cv->width > 0) {
        px0 = std::min(px0, cv->origin_x);
        py0 = std::min(py0, cv->origin_y);
        px1 = std::max(px1, cv->origin_x + cv->width);
        py1 = std::max(py1, cv->origin_y + cv->height);
    }
    if (!covers(cv, px0, py0, px1, py1)) NRM_CHECK(grow_physical(cv, px0, py0, px1, py1));
    NRM_CUDA(cudaStreamSynchronize(cv->ctx->stream));
    return NRM_OK;
}

int nrm_canvas_ensure_contains(nrm_canvas* cv, double x0, double y0, double x1, double y1) {
    NRM_CHECK(check_canvas(cv));
    DeviceGuard g(cv->ctx->device);
    NRM_CHECK(ensure_contains(cv, x0, y0, x1, y1));
    NRM_CUDA(cudaStreamSynchronize(cv->ctx->stream));
    return NRM_OK;
}

int nrm_canvas_info(const nrm_canvas* cv, int64_t* ox, int64_t* oy, int* w, int* h) {
    NRM_CHECK(check_canvas(cv));
    if (ox) *ox = cv->origin_x;
    if (oy) *oy = cv->origin_y;
    if (w) *w = cv->width;
    if (h) *h = cv->height;
    return NRM_OK;
}

int nrm_canvas_set_band(nrm_canvas* cv, int rank, int count) {
    NRM_CHECK(check_canvas(cv));
    if (count < 1 || rank < 0 || rank >= count) return fail(NRM_EINVAL, "set_band: need 0 <= rank < count");
    cv->band_rank = rank;
    cv->band_count = count;
    return NRM_OK;
}

int nrm_canvas_download(nrm_canvas* cv, int x, int y, int w, int h, double* rgb, uint8_t* weight) {
    NRM_CHECK(check_canvas(cv));
    NRM_CHECK(check_region(cv, x, y, w, h));
    if ((size_t)w * h == 0) return NRM_OK;
    nrm_ctx* c = cv->ctx;
    DeviceGuard g(c->device);
    const size_t npx = (size_t)w * h;
    NRM_CUDA(c->out_a.ensure(npx * 3 * sizeof(double)));
    NRM_CUDA(c->out_b.ensure(npx));
    NRM_CUDA(launch_canvas_read(cv, x, y, w, h, rgb ? c->out_a.as<double>() : nullptr,
                                weight ? c->out_b.as<uint8_t>() : nullptr, c->stream, &c->launches));
    if (rgb) NRM_CUDA(cudaMemcpyAsync(rgb, c->out_a.p, npx * 3 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (weight) NRM_CUDA(cudaMemcpyAsync(weight, c->out_b.p, npx, cudaMemcpyDeviceToHost, c->stream));
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    return NRM_OK;
}

int nrm_canvas_upload(nrm_canvas* cv, int x, int y, int w, int h, const double* rgb, const uint8_t* weight) {
    NRM_CHECK(check_canvas(cv));
    NRM_CHECK(check_region(cv, x, y, w, h));
    if ((size_t)w * h == 0) return NRM_OK;
    nrm_ctx* c = cv->ctx;
    DeviceGuard g(c->device);
    const size_t npx = (size_t)w * h;
    if (rgb) NRM_CHECK(upload(c, c->out_a, rgb, npx * 3 * sizeof(double)));
    if (weight) NRM_CHECK(upload(c, c->out_b, weight, npx));
    NRM_CUDA(launch_canvas_write(cv, x, y, w, h, rgb ? c->out_a.as<double>() : nullptr,
                                 weight ? c->out_b.as<uint8_t>() : nullptr, c->stream, &c->launches));
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    return NRM_OK;
}

// ---- extension: canvas deformation (north_star) ------------
static int deform_core(nrm_canvas* cv, int x, int y, int w, int h, const float* d_disp) {
    nrm_ctx* c = cv->ctx;
    const size_t npx = (size_t)w * h;
    if (!deform_uses_ping_pong(cv, w, h)) NRM_CUDA(c->out_b.ensure(npx * 13 + 64));
    NRM_CUDA(launch_canvas_deform(cv, x, y, w, h, reinterpret_cast<const float2*>(d_disp), c->out_b.as<float>(),
                                  c->stream, &c->launches));
    return NRM_OK;
}

int nrm_canvas_deform(nrm_canvas* cv, int x, int y, int w, int h, const float* disp) {
    NRM_CHECK(check_canvas(cv));
    NRM_CHECK(check_region(cv, x, y, w, h));
    if ((size_t)w * h == 0) return NRM_OK;
    if (!disp) return fail(NRM_EINVAL, "canvas_deform: null displacement field");
    nrm_ctx* c = cv->ctx;
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    NRM_CHECK(upload(c, c->out_a, disp, (size_t)w * h * 2 * sizeof(float)));
    NRM_CHECK(deform_core(cv, x, y, w, h, c->out_a.as<float>()));
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    return NRM_OK;
}

int nrm_canvas_deform_device(nrm_canvas* cv, int x, int y, int w, int h, const float* d_disp) {
    NRM_CHECK(check_canvas(cv));
    NRM_CHECK(check_region(cv, x, y, w, h));
    if ((size_t)w * h == 0) return NRM_OK;
    if (!d_disp) return fail(NRM_EINVAL, "canvas_deform: null displacement field");
    DeviceGuard g(cv->ctx->device);
    ProfScope prof_scope(cv->ctx);
    return deform_core(cv, x, y, w, h, d_disp);
}

// ---- halo rows of banded canvases -----------------------------
static int rows_common(nrm_canvas* cv, const int* rows, int nrows, const void* d_buf) {
    NRM_CHECK(check_canvas(cv));
    if (nrows < 0) return fail(NRM_EINVAL, "rows: negative count");
    if (nrows > 0 && (!rows || !d_buf)) return fail(NRM_EINVAL, "rows: null argument");
    for (int k = 0; k < nrows; ++k)
        if (rows[k] < 0 || rows[k] >= cv->height) return fail(NRM_EINVAL, "rows: row outside the canvas");
    if (nrows == 0) return NRM_OK;
    nrm_ctx* c = cv->ctx;
    NRM_CUDA(c->halo.ensure((size_t)nrows * sizeof(int)));
    NRM_CUDA(cudaMemcpyAsync(c->halo.p, rows, (size_t)nrows * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    return NRM_OK;
}

int nrm_canvas_pack_rows_device(nrm_canvas* cv, const int* rows, int nrows, void* d_buf) {
    if (cv && cv->ctx) {
        DeviceGuard g(cv->ctx->device);
        ProfScope prof_scope(cv->ctx);
        NRM_CHECK(rows_common(cv, rows, nrows, d_buf));
        NRM_CUDA(launch_rows_pack(cv, cv->ctx->halo.as<int>(), nrows, d_buf, cv->ctx->stream, &cv->ctx->launches));
        return NRM_OK;
    }
    return check_canvas(cv);
}

int nrm_canvas_unpack_rows_device(nrm_canvas* cv, const int* rows, int nrows, const void* d_buf) {
    if (cv && cv->ctx) {
        DeviceGuard g(cv->ctx->device);
        ProfScope prof_scope(cv->ctx);
        NRM_CHECK(rows_common(cv, rows, nrows, d_buf));
        NRM_CUDA(launch_rows_unpack(cv, cv->ctx->halo.as<int>(), nrows, d_buf, cv->ctx->stream,
                                    &cv->ctx->launches));
        return NRM_OK;
    }
    return check_canvas(cv);
}

static int occupied_scan(nrm_canvas* cv, unsigned long long* count, int bbox[4]) {
    nrm_ctx* c = cv->ctx;
    NRM_CUDA(c->stats.ensure(64));
    const int init[6] = {0, 0, 0x7fffffff, 0x7fffffff, -1, -1};
    NRM_CUDA(cudaMemcpyAsync(c->stats.p, init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    unsigned long long* d_count = c->stats.as<unsigned long long>();
    int* d_bbox = reinterpret_cast<int*>(d_count + 1);
    NRM_CUDA(launch_occupied(cv, d_count, d_bbox, c->stream, &c->launches));
    int out[6];
    NRM_CUDA(cudaMemcpyAsync(out, c->stats.p, sizeof(out), cudaMemcpyDeviceToHost, c->stream));
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    std::memcpy(count, out, sizeof(unsigned long long));
    std::memcpy(bbox, out + 2, 4 * sizeof(int));
    return NRM_OK;
}

int nrm_canvas_occupied_count(nrm_canvas* cv, int64_t* out) {
    NRM_CHECK(check_canvas(cv));
    if (!out) return fail(NRM_EINVAL, "null out");
    *out = 0;
    if (cv->width == 0) return NRM_OK;
    DeviceGuard g(cv->ctx->device);
    unsigned long long cnt = 0;
    int bb[4];
    NRM_CHECK(occupied_scan(cv, &cnt, bb));
    *out = (int64_t)cnt;
    return NRM_OK;
}

int nrm_canvas_occupied_bbox(nrm_canvas* cv, int* x0, int* y0, int* x1, int* y1) {
    NRM_CHECK(check_canvas(cv));
    int bb[4] = {0, 0, -1, -1};
    if (cv->width > 0) {
        DeviceGuard g(cv->ctx->device);
        unsigned long long cnt = 0;
        NRM_CHECK(occupied_scan(cv, &cnt, bb));
        if (cnt == 0) bb[0] = 0, bb[1] = 0, bb[2] = -1, bb[3] = -1;
    }
    if (x0) *x0 = bb[0];
    if (y0) *y0 = bb[1];
    if (x1) *x1 = bb[2];
    if (y1) *y1 = bb[3];
    return NRM_OK;
}

// ---- blend_frame ---------------------------------------------------------
namespace {
int blend_host(nrm_canvas* cv, const uint8_t* frame, int fw, int fh, int ch, const double* anchors,
               const double* warps, int n, double alpha, const double* poly, int npoly, const float* unc,
               nrm_blend_stats* out) {
    NRM_CHECK(check_canvas(cv));
    if (!out) return fail(NRM_EINVAL, "null stats");
    *out = nrm_blend_stats{0, 0, 0, 0};
    if (fw < 0 || fh < 0) return fail(NRM_EINVAL, "negative frame size");
    if (fw == 0 || fh == 0 || npoly < 3) return NRM_OK;  // mosaic.hpp:201
    if (ch != 1 && ch != 3 && ch != 4) return fail(NRM_EINVAL, "frame channels must be 1, 3 or 4");
    if (!frame || !poly) return fail(NRM_EINVAL, "null frame or polygon");
    NRM_CHECK(validate_nodes(anchors, warps, n, alpha, true));
    nrm_ctx* c = cv->ctx;
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    const size_t fbytes = (size_t)fw * fh * ch;
    const size_t ubytes = unc ? (size_t)fw * fh * sizeof(float) : 0;
    const size_t uoff = (fbytes + 255) & ~size_t(255);
    NRM_CUDA(c->frame_raw.ensure(uoff + ubytes));
    NRM_CUDA(cudaMemcpyAsync(c->frame_raw.p, frame, fbytes, cudaMemcpyHostToDevice, c->stream));
    const float* d_unc = nullptr;
    if (unc) {
        NRM_CUDA(cudaMemcpyAsync(c->frame_raw.as<char>() + uoff, unc, ubytes, cudaMemcpyHostToDevice, c->stream));
        d_unc = reinterpret_cast<const float*>(c->frame_raw.as<char>() + uoff);
    }
    NRM_CHECK(upload(c, c->anchors, anchors, (size_t)n * 2 * sizeof(double)));
    NRM_CHECK(upload(c, c->warps, warps, (size_t)n * 5 * sizeof(double)));
    NRM_CUDA(c->stats.ensure(64));
    NRM_CHECK(blend_core(cv, c->frame_raw.as<uint8_t>(), fw, fh, ch, c->anchors.as<double>(), c->warps.as<double>(), n,
                         alpha, poly, npoly, c->stats.as<unsigned long long>(), d_unc));
    NRM_CUDA(c->staging_out.ensure(64));
    NRM_CUDA(cudaMemcpyAsync(c->staging_out.p, c->stats.p, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    std::memcpy(out, c->staging_out.p, sizeof(nrm_blend_stats));
    return NRM_OK;
}

int blend_device(nrm_canvas* cv, const uint8_t* d_frame, int fw, int fh, int ch, const double* d_anchors,
                 const double* d_warps, int n, double alpha, const double* poly, int npoly, const float* d_unc,
                 int64_t* d_stats) {
    NRM_CHECK(check_canvas(cv));
    if (!d_stats) return fail(NRM_EINVAL, "null stats");
    if (fw < 0 || fh < 0) return fail(NRM_EINVAL, "negative frame size");
    NRM_CHECK(validate_nodes(d_anchors, d_warps, n, alpha, false));
    nrm_ctx* c = cv->ctx;
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    if (fw > 0 && fh > 0 && npoly >= 3) {
        if (ch != 1 && ch != 3 && ch != 4) return fail(NRM_EINVAL, "frame channels must be 1, 3 or 4");
        if (!d_frame || !poly) return fail(NRM_EINVAL, "null frame or polygon");
    }
    return blend_core(cv, d_frame, fw, fh, ch, d_anchors, d_warps, n, alpha, poly, npoly,
                      reinterpret_cast<unsigned long long*>(d_stats), d_unc);
}
}  // namespace

int nrm_blend_frame(nrm_canvas* cv, const uint8_t* frame, int fw, int fh, int ch, const double* anchors,
                    const double* warps, int n, double alpha, const double* poly, int npoly,
                    nrm_blend_stats* out) {
    return blend_host(cv, frame, fw, fh, ch, anchors, warps, n, alpha, poly, npoly, nullptr, out);
}

int nrm_blend_frame_device(nrm_canvas* cv, const uint8_t* d_frame, int fw, int fh, int ch, const double* d_anchors,
                           const double* d_warps, int n, double alpha, const double* poly, int npoly,
                           int64_t* d_stats) {
    return blend_device(cv, d_frame, fw, fh, ch, d_anchors, d_warps, n, alpha, poly, npoly, nullptr, d_stats);
}

int nrm_blend_frame_weighted(nrm_canvas* cv, const uint8_t* frame, int fw, int fh, int ch, const double* anchors,
                             const double* warps, int n, double alpha, const double* poly, int npoly,
                             const float* unc, nrm_blend_stats* out) {
    if (!unc && fw > 0 && fh > 0) return fail(NRM_EINVAL, "blend_frame_weighted: null uncertainty map");
    return blend_host(cv, frame, fw, fh, ch, anchors, warps, n, alpha, poly, npoly, unc, out);
}

int nrm_blend_frame_weighted_device(nrm_canvas* cv, const uint8_t* d_frame, int fw, int fh, int ch,
                                    const double* d_anchors, const double* d_warps, int n, double alpha,
                                    const double* poly, int npoly, const float* d_unc, int64_t* d_stats) {
    if (!d_unc && fw > 0 && fh > 0) return fail(NRM_EINVAL, "blend_frame_weighted: null uncertainty map");
    return blend_device(cv, d_frame, fw, fh, ch, d_anchors, d_warps, n, alpha, poly, npoly, d_unc, d_stats);
}

// ---- several frames per call ------------------------------------------------
int nrm_blend_frames_device(nrm_canvas* cv, int nf, const uint8_t* const* d_frames, int fw, int fh, int ch,
                            const double* const* d_anchors, const double* const* d_warps, const int* n, double alpha,
                            const double* const* polys, const int* npoly, int64_t* d_stats) {
    NRM_CHECK(check_canvas(cv));
    if (nf < 0) return fail(NRM_EINVAL, "blend_frames: negative frame count");
    if (nf == 0) return NRM_OK;
    if (!d_frames || !d_anchors || !d_warps || !n || !polys || !npoly || !d_stats)
        return fail(NRM_EINVAL, "blend_frames: null array");
    if (fw < 0 || fh < 0) return fail(NRM_EINVAL, "negative frame size");
    nrm_ctx* c = cv->ctx;
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    auto* stats = reinterpret_cast<unsigned long long*>(d_stats);
    // the reference's per-frame checks and canvas growth, in frame order
    struct Win {
        bool active;
        int i0, j0, i1, j1;
    };
    std::vector<Win> win((size_t)nf, Win{false, 0, 0, 0, 0});
    for (int f = 0; f < nf; ++f) {
        NRM_CHECK(validate_nodes(d_anchors[f], d_warps[f], n[f], alpha, false));
        if (fw <= 0 || fh <= 0 || npoly[f] < 3) continue;
        if (ch != 1 && ch != 3 && ch != 4) return fail(NRM_EINVAL, "frame channels must be 1, 3 or 4");
        if (!d_frames[f] || !polys[f]) return fail(NRM_EINVAL, "null frame or polygon");
        if (!finite_all(polys[f], (size_t)npoly[f] * 2)) return fail(NRM_EINVAL, "blend_frame: non-finite polygon");
        const Bbox bb = footprint_bbox(polys[f], npoly[f]);
        NRM_CHECK(ensure_contains(cv, bb.x0, bb.y0, bb.x1, bb.y1));
        // absolute pixel window (origins are integers, so this equals
        // blend_frame's window whatever the canvas grows to later)
        const double orgx = (double)cv->origin_x, orgy = (double)cv->origin_y;
        Win& w = win[f];
        w.i0 = (int)(cv->origin_x + (int64_t)std::floor(bb.x0 - orgx));
        w.j0 = (int)(cv->origin_y + (int64_t)std::floor(bb.y0 - orgy));
        w.i1 = (int)(cv->origin_x + (int64_t)std::ceil(bb.x1 - orgx));
        w.j1 = (int)(cv->origin_y + (int64_t)std::ceil(bb.y1 - orgy));
        w.active = w.i1 >= w.i0 && w.j1 >= w.j0;
    }
    // pairwise disjoint footprints: the order of the updates does not matter
    std::vector<int> act;
    bool disjoint = true;
    for (int f = 0; f < nf; ++f) {
        if (!win[f].active) continue;
        for (int e : act)
            if (!(win[f].i1 < win[e].i0 || win[e].i1 < win[f].i0 || win[f].j1 < win[e].j0 || win[e].j1 < win[f].j0))
                disjoint = false;
        act.push_back(f);
    }
    auto sequential = [&]() -> int {
        for (int f = 0; f < nf; ++f)
            NRM_CHECK(blend_core(cv, d_frames[f], fw, fh, ch, d_anchors[f], d_warps[f], n[f], alpha, polys[f],
                                 npoly[f], stats + 4 * f));
        return NRM_OK;
    };
    if (!disjoint || act.size() < 2 || act.size() > 16) return sequential();
    // per-frame counters (acc[3] u64 | exc_count u32 | pad), persistent-zero
    const size_t nact = act.size();
    const size_t need = nact * 32;
    if (c->batch.cap < need) {
        NRM_CUDA(c->batch.ensure(need));
        NRM_CUDA(cudaMemsetAsync(c->batch.p, 0, c->batch.cap, c->stream));
    }
    const State st = state_of(c);
    std::vector<size_t> cap(nact);
    size_t qtot = 0;
    for (size_t a = 0; a < nact; ++a) {
        const Win& w = win[act[a]];
        const unsigned long long fp = (unsigned long long)(w.i1 - w.i0 + 1) * (unsigned long long)(w.j1 - w.j0 + 1);
        cap[a] = exception_capacity(c, fp);
        qtot += cap[a];
    }
    NRM_CUDA(c->exc.ensure(qtot * sizeof(int2) + 64));
    std::vector<NodeFieldLaunch> Ls(nact);
    size_t qoff = 0;
    for (size_t a = 0; a < nact; ++a) {
        const int f = act[a];
        const Win& w = win[f];
        NodeFieldLaunch& L = Ls[a];
        L.frame = d_frames[f];
        L.fw = fw;
        L.fh = fh;
        L.fch = ch;
        L.anchors = d_anchors[f];
        L.warps = d_warps[f];
        L.n = n[f];
        L.alpha = alpha;
        L.grid.gx = 0.0;
        L.grid.gy = 0.0;
        L.grid.i0 = w.i0;
        L.grid.i1 = w.i1;
        L.grid.j0 = w.j0;
        L.grid.j1 = w.j1;
        L.R = cv->r;
        L.G = cv->g;
        L.B = cv->b;
        L.W = cv->w;
        L.pitch = cv->cap_w;
        L.phys_x0 = (int)cv->phys_x0;
        L.phys_y0 = (int)cv->phys_y0;
        L.band_rank = cv->band_rank;
        L.band_count = cv->band_count;
        char* fb = c->batch.as<char>() + 32 * a;
        L.acc = reinterpret_cast<unsigned long long*>(fb);
        L.exc_count = reinterpret_cast<unsigned*>(fb + 24);
        L.stats_out = stats + 4 * f;
        L.footprint = (unsigned long long)(w.i1 - w.i0 + 1) * (unsigned long long)(w.j1 - w.j0 + 1);
        L.exc = c->exc.as<int2>() + qoff;
        L.exc_cap = (unsigned)cap[a];
        L.exc_overflow = st.overflow;
        L.exc_last = st.last_exc;
        L.exc_done = st.exc_done;
        qoff += cap[a];
    }
    // one canvas, so one set of tensor maps, copied into every frame's launch
    // (the batch kernel reads them from its frame table in global memory)
    if (nact > 0 && canvas_tensor_maps(cv, Ls[0])) {
        Ls[0].ctm_ok = 1;
        for (size_t a = 1; a < nact; ++a) {
            for (int k = 0; k < 4; ++k) Ls[a].ctm[k] = Ls[0].ctm[k];
            Ls[a].ctm_ok = 1;
        }
    }
    if (ch == 3 || ch == 4) {  // one conversion launch for every active frame
        std::vector<const uint8_t*> fr(nact);
        std::vector<NodeFieldLaunch*> lp(nact);
        for (size_t a = 0; a < nact; ++a) {
            fr[a] = d_frames[act[a]];
            lp[a] = &Ls[a];
        }
        NRM_CHECK(frame_textures(c, (int)nact, fr.data(), fw, fh, ch, lp.data(), false));
    }
    NRM_CUDA(c->tiles.ensure(node_field_batch_scratch_bytes((int)nact)));
    const cudaError_t e = launch_node_field_batch(Ls.data(), (int)nact, c->tiles.p, c->stream, &c->launches);
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        return sequential();
    }
    NRM_CUDA(e);
    for (int f = 0; f < nf; ++f)
        if (!win[f].active) NRM_CUDA(cudaMemsetAsync(stats + 4 * f, 0, 4 * sizeof(unsigned long long), c->stream));
    return NRM_OK;
}

// ---- render ----------------------------------------------------------------
int nrm_render(nrm_canvas* cv, int crop, uint8_t* out, int* out_w, int* out_h, double* crop_origin2) {
    NRM_CHECK(check_canvas(cv));
    if (!out_w || !out_h) return fail(NRM_EINVAL, "null size outputs");
    if (crop_origin2) {
        crop_origin2[0] = (double)cv->origin_x;
        crop_origin2[1] = (double)cv->origin_y;
    }
    *out_w = 0;
    *out_h = 0;
    if (cv->width == 0) return NRM_OK;
    DeviceGuard g(cv->ctx->device);
    ProfScope prof_scope(cv->ctx);
    int x0 = 0, y0 = 0, x1 = cv->width - 1, y1 = cv->height - 1;
    if (crop) {
        unsigned long long cnt = 0;
        int bb[4];
        NRM_CHECK(occupied_scan(cv, &cnt, bb));
        if (cnt == 0) return NRM_OK;
        x0 = bb[0];
        y0 = bb[1];
        x1 = bb[2];
        y1 = bb[3];
        if (crop_origin2) {
            crop_origin2[0] = (double)cv->origin_x + (double)x0;
            crop_origin2[1] = (double)cv->origin_y + (double)y0;
        }
    }
    const int w = x1 - x0 + 1, h = y1 - y0 + 1;
    *out_w = w;
    *out_h = h;
    if (!out) return NRM_OK;
    nrm_ctx* c = cv->ctx;
    const size_t bytes = (size_t)w * h * 4;
    NRM_CUDA(c->out_b.ensure(bytes));
    NRM_CUDA(launch_render(cv, x0, y0, w, h, c->out_b.as<uint8_t>(), c->stream, &c->launches));
    NRM_CUDA(cudaMemcpyAsync(out, c->out_b.p, bytes, cudaMemcpyDeviceToHost, c->stream));
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    return NRM_OK;
}

int nrm_render_device(nrm_canvas* cv, int x, int y, int w, int h, uint8_t* d_out) {
    NRM_CHECK(check_canvas(cv));
    NRM_CHECK(check_region(cv, x, y, w, h));
    if (!d_out && (size_t)w * h) return fail(NRM_EINVAL, "null output");
    DeviceGuard g(cv->ctx->device);
    ProfScope prof_scope(cv->ctx);
    NRM_CUDA(launch_render(cv, x, y, w, h, d_out, cv->ctx->stream, &cv->ctx->launches));
    return NRM_OK;
}

// ---- node field ------------------------------------------------------------
int nrm_pixel_warp(nrm_ctx* c, const double* points, int npts, const double* anchors, const double* warps, int n,
                   double alpha, double* out_warps, uint8_t* valid) {
    if (!c) return fail(NRM_ESTATE, "null context");
    if (npts < 0 || (npts > 0 && (!points || !out_warps || !valid))) return fail(NRM_EINVAL, "bad point arrays");
    NRM_CHECK(validate_nodes(anchors, warps, n, alpha, true));
    if (npts == 0) return NRM_OK;
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    NRM_CHECK(upload(c, c->pts, points, (size_t)npts * 2 * sizeof(double)));
    NRM_CHECK(upload(c, c->anchors, anchors, (size_t)n * 2 * sizeof(double)));
    NRM_CHECK(upload(c, c->warps, warps, (size_t)n * 5 * sizeof(double)));
    NRM_CUDA(c->out_a.ensure((size_t)npts * 5 * sizeof(double)));
    NRM_CUDA(c->out_b.ensure((size_t)npts));
    NRM_CUDA(launch_pixel_warp_points(c->pts.as<double>(), npts, c->anchors.as<double>(), c->warps.as<double>(), n,
                                      alpha, c->out_a.as<double>(), c->out_b.as<uint8_t>(), c->stream, &c->launches));
    NRM_CUDA(cudaMemcpyAsync(out_warps, c->out_a.p, (size_t)npts * 5 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    NRM_CUDA(cudaMemcpyAsync(valid, c->out_b.p, (size_t)npts, cudaMemcpyDeviceToHost, c->stream));
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    for (int i = 0; i < npts; ++i)
        if (valid[i] == 2) return fail(NRM_EDEGENERATE, "DualQuat2: degenerate real part");
    return NRM_OK;
}

int nrm_node_field(nrm_ctx* c, const nrm_grid* grid, const double* anchors, const double* warps, int n, double alpha,
                   float* disp, uint8_t* support) {
    if (!c) return fail(NRM_ESTATE, "null context");
    NRM_CHECK(validate_nodes(anchors, warps, n, alpha, true));
    if (!grid || grid->width < 0 || grid->height < 0) return fail(NRM_EINVAL, "bad grid");
    const size_t npx = (size_t)grid->width * grid->height;
    if (npx == 0) return NRM_OK;
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    NRM_CHECK(upload(c, c->anchors, anchors, (size_t)n * 2 * sizeof(double)));
    NRM_CHECK(upload(c, c->warps, warps, (size_t)n * 5 * sizeof(double)));
    NRM_CUDA(c->out_a.ensure(npx * sizeof(float2)));
    NRM_CUDA(c->out_b.ensure(npx));
    NRM_CHECK(node_field_core(c, grid, c->anchors.as<double>(), c->warps.as<double>(), n, alpha,
                              disp ? c->out_a.as<float>() : nullptr, support ? c->out_b.as<uint8_t>() : nullptr));
    if (disp) NRM_CUDA(cudaMemcpyAsync(disp, c->out_a.p, npx * sizeof(float2), cudaMemcpyDeviceToHost, c->stream));
    if (support) NRM_CUDA(cudaMemcpyAsync(support, c->out_b.p, npx, cudaMemcpyDeviceToHost, c->stream));
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    return NRM_OK;
}

int nrm_node_field_device(nrm_ctx* c, const nrm_grid* grid, const double* d_anchors, const double* d_warps, int n,
                          double alpha, float* d_disp, uint8_t* d_support) {
    if (!c) return fail(NRM_ESTATE, "null context");
    NRM_CHECK(validate_nodes(d_anchors, d_warps, n, alpha, false));
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    return node_field_core(c, grid, d_anchors, d_warps, n, alpha, d_disp, d_support);
}

// ---- node variance field (Engine::blended_variance_at, slam.hpp:703-714) ----
int nrm_variance_field_device(nrm_ctx* c, const nrm_grid* grid, const double* d_pos, const double* d_var, int n,
                              double alpha, float* d_out) {
    if (!c) return fail(NRM_ESTATE, "null context");
    if (!grid || grid->width < 0 || grid->height < 0) return fail(NRM_EINVAL, "bad grid");
    if (!std::isfinite(grid->x0) || !std::isfinite(grid->y0)) return fail(NRM_EINVAL, "non-finite grid origin");
    if (n < 0 || (n > 0 && (!d_pos || !d_var))) return fail(NRM_EINVAL, "variance_field: bad node arrays");
    if (!std::isfinite(alpha) || alpha < 0.0) return fail(NRM_EINVAL, "alpha must be finite and >= 0");
    if ((size_t)grid->width * grid->height == 0) return NRM_OK;
    if (!d_out) return fail(NRM_EINVAL, "variance_field: null output");
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    NRM_CUDA(launch_variance_field(grid->x0, grid->y0, grid->width, grid->height, d_pos, d_var, n, alpha, d_out,
                                   c->stream, &c->launches));
    return NRM_OK;
}

int nrm_variance_field(nrm_ctx* c, const nrm_grid* grid, const double* pos, const double* var, int n, double alpha,
                       float* out) {
    if (!c) return fail(NRM_ESTATE, "null context");
    if (!grid || grid->width < 0 || grid->height < 0) return fail(NRM_EINVAL, "bad grid");
    if (n < 0 || (n > 0 && (!pos || !var))) return fail(NRM_EINVAL, "variance_field: bad node arrays");
    if (n > 0 && (!finite_all(pos, (size_t)n * 2) || !finite_all(var, (size_t)n)))
        return fail(NRM_EINVAL, "variance_field: non-finite node arrays");
    const size_t npx = (size_t)grid->width * grid->height;
    if (npx == 0) return NRM_OK;
    if (!out) return fail(NRM_EINVAL, "variance_field: null output");
    DeviceGuard g(c->device);
    NRM_CHECK(upload(c, c->anchors, pos, (size_t)n * 2 * sizeof(double)));
    NRM_CHECK(upload(c, c->warps, var, (size_t)n * sizeof(double)));
    NRM_CUDA(c->out_a.ensure(npx * sizeof(float)));
    NRM_CHECK(nrm_variance_field_device(c, grid, c->anchors.as<double>(), c->warps.as<double>(), n, alpha,
                                        c->out_a.as<float>()));
    NRM_CUDA(cudaMemcpyAsync(out, c->out_a.p, npx * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    return NRM_OK;
}

int nrm_node_field_band_device(nrm_ctx* c, const nrm_grid* grid, const double* d_anchors, const double* d_warps,
                               int n, double alpha, float* d_disp, uint8_t* d_support, int band_rank,
                               int band_count) {
    if (!c) return fail(NRM_ESTATE, "null context");
    if (band_count < 1 || band_rank < 0 || band_rank >= band_count)
        return fail(NRM_EINVAL, "node_field: need 0 <= band_rank < band_count");
    NRM_CHECK(validate_nodes(d_anchors, d_warps, n, alpha, false));
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    return node_field_core(c, grid, d_anchors, d_warps, n, alpha, d_disp, d_support, band_rank, band_count, true);
}

// ---- footprint -------------------------------------------------------------
int nrm_invert_frame_boundary(nrm_ctx* c, int fw, int fh, const double* anchors, const double* warps, int n,
                              double alpha, double step, double* poly, int cap, int* npoly) {
    if (!c) return fail(NRM_ESTATE, "null context");
    if (!npoly || (cap > 0 && !poly)) return fail(NRM_EINVAL, "null output");
    if (!(step > 0.0) || !std::isfinite(step)) return fail(NRM_EINVAL, "step must be positive");
    NRM_CHECK(validate_nodes(anchors, warps, n, alpha, true));
    // Boundary samples exactly as mosaic.hpp:62-67 generates them.
    std::vector<double> s;
    const double w1 = fw - 1.0, h1 = fh - 1.0;
    for (double x = 0; x < w1; x += step) s.insert(s.end(), {x, 0.0});
    for (double y = 0; y < h1; y += step) s.insert(s.end(), {w1, y});
    for (double x = w1; x > 0; x -= step) s.insert(s.end(), {x, h1});
    for (double y = h1; y > 0; y -= step) s.insert(s.end(), {0.0, y});
    const int ns = (int)(s.size() / 2);
    *npoly = ns;
    if (ns == 0) return NRM_OK;
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    NRM_CHECK(upload(c, c->pts, s.data(), s.size() * sizeof(double)));
    NRM_CHECK(upload(c, c->anchors, anchors, (size_t)n * 2 * sizeof(double)));
    NRM_CHECK(upload(c, c->warps, warps, (size_t)n * 5 * sizeof(double)));
    NRM_CUDA(launch_invert_boundary(fw, fh, c->anchors.as<double>(), c->warps.as<double>(), n, alpha, step,
                                    c->pts.as<double>(), ns, c->stream, &c->launches));
    const int m = std::min(ns, cap);
    if (m > 0)
        NRM_CUDA(cudaMemcpyAsync(poly, c->pts.p, (size_t)m * 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    return NRM_OK;
}

// ---- EMDQ field --------------------------------------------------------------
int nrm_emdq_field(nrm_ctx* c, const nrm_grid* grid, const double* apts, const double* locals, const double* probs,
                   int m_total, const int32_t* active, int nactive, double alpha, int support, double beta,
                   float* disp, float* unc) {
    if (!c) return fail(NRM_ESTATE, "null context");
    if (!grid || grid->width < 0 || grid->height < 0) return fail(NRM_EINVAL, "bad grid");
    if (m_total <= 0 || nactive <= 0 || !apts || !locals || !probs || !active)
        return fail(NRM_EINVAL, "emdq_field: empty or null candidate arrays");
    for (int a = 0; a < nactive; ++a)
        if (active[a] < 0 || active[a] >= m_total) return fail(NRM_EINVAL, "emdq_field: active index out of range");
    if (!finite_all(apts, (size_t)m_total * 2) || !finite_all(locals, (size_t)m_total * 5))
        return fail(NRM_EINVAL, "emdq_field: non-finite candidates");
    const size_t npx = (size_t)grid->width * grid->height;
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    NRM_CHECK(upload(c, c->anchors, apts, (size_t)m_total * 2 * sizeof(double)));
    NRM_CHECK(upload(c, c->locals, locals, (size_t)m_total * 5 * sizeof(double)));
    NRM_CHECK(upload(c, c->probs, probs, (size_t)m_total * sizeof(double)));
    NRM_CHECK(upload(c, c->active, active, (size_t)nactive * sizeof(int32_t)));
    NRM_CUDA(c->out_a.ensure(npx * sizeof(float2) + 16));
    NRM_CUDA(c->out_b.ensure(npx * sizeof(float) + 16));
    NRM_CHECK(emdq_core(c, grid, c->anchors.as<double>(), c->locals.as<double>(), c->probs.as<double>(), m_total,
                        c->active.as<int32_t>(), nactive, alpha, support, beta, disp ? c->out_a.as<float>() : nullptr,
                        unc ? c->out_b.as<float>() : nullptr));
    if (npx) {
        if (disp) NRM_CUDA(cudaMemcpyAsync(disp, c->out_a.p, npx * sizeof(float2), cudaMemcpyDeviceToHost, c->stream));
        if (unc) NRM_CUDA(cudaMemcpyAsync(unc, c->out_b.p, npx * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    }
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    return NRM_OK;
}

int nrm_emdq_field_device(nrm_ctx* c, const nrm_grid* grid, const double* d_apts, const double* d_locals,
                          const double* d_probs, int m_total, const int32_t* d_active, int nactive, double alpha,
                          int support, double beta, float* d_disp, float* d_unc) {
    if (!c) return fail(NRM_ESTATE, "null context");
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    return emdq_core(c, grid, d_apts, d_locals, d_probs, m_total, d_active, nactive, alpha, support, beta, d_disp,
                     d_unc);
}

// ---- EMDQ at scattered points (EM E-step, final field) -------------------------
int nrm_emdq_points(nrm_ctx* c, const double* q, const int32_t* exclude, int nq, const double* apts,
                    const double* locals, const double* probs, int m_total, const int32_t* active, int nactive,
                    double alpha, int support, double beta, double* warps, double* pred, double* unc,
                    int32_t* status) {
    if (!c) return fail(NRM_ESTATE, "null context");
    if (nq < 0 || (nq > 0 && !q)) return fail(NRM_EINVAL, "emdq_points: bad query array");
    if (m_total <= 0 || nactive <= 0 || !apts || !locals || !probs || !active)
        return fail(NRM_EINVAL, "emdq_points: empty or null candidate arrays");
    for (int a = 0; a < nactive; ++a)
        if (active[a] < 0 || active[a] >= m_total) return fail(NRM_EINVAL, "emdq_points: active index out of range");
    if (!finite_all(apts, (size_t)m_total * 2) || !finite_all(locals, (size_t)m_total * 5))
        return fail(NRM_EINVAL, "emdq_points: non-finite candidates");
    if (nq == 0) return NRM_OK;
    double bb[4] = {q[0], q[1], q[0], q[1]};
    for (int k = 0; k < nq; ++k) {
        const double x = q[2 * k], y = q[2 * k + 1];
        if (!std::isfinite(x) || !std::isfinite(y)) return fail(NRM_EINVAL, "emdq_points: non-finite query");
        bb[0] = std::min(bb[0], x);
        bb[1] = std::min(bb[1], y);
        bb[2] = std::max(bb[2], x);
        bb[3] = std::max(bb[3], y);
    }
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    const size_t nqs = (size_t)nq;
    // queries + exclusions share frame_raw; outputs share out_a
    NRM_CUDA(c->frame_raw.ensure(nqs * 2 * sizeof(double) + nqs * sizeof(int32_t) + 16));
    double* d_q = c->frame_raw.as<double>();
    int32_t* d_ex = exclude ? reinterpret_cast<int32_t*>(d_q + 2 * nqs) : nullptr;
    NRM_CUDA(cudaMemcpyAsync(d_q, q, nqs * 2 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    if (exclude) NRM_CUDA(cudaMemcpyAsync(d_ex, exclude, nqs * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
    NRM_CHECK(upload(c, c->anchors, apts, (size_t)m_total * 2 * sizeof(double)));
    NRM_CHECK(upload(c, c->locals, locals, (size_t)m_total * 5 * sizeof(double)));
    NRM_CHECK(upload(c, c->probs, probs, (size_t)m_total * sizeof(double)));
    NRM_CHECK(upload(c, c->active, active, (size_t)nactive * sizeof(int32_t)));
    NRM_CUDA(c->out_a.ensure(nqs * 8 * sizeof(double) + nqs * sizeof(int32_t) + 16));
    double* o = c->out_a.as<double>();
    double* d_w = warps ? o : nullptr;
    double* d_p = pred ? o + 5 * nqs : nullptr;
    double* d_u = unc ? o + 7 * nqs : nullptr;
    int32_t* d_s = status ? reinterpret_cast<int32_t*>(o + 8 * nqs) : nullptr;
    NRM_CHECK(points_core(c, bb, d_q, d_ex, nq, c->anchors.as<double>(), c->locals.as<double>(),
                          c->probs.as<double>(), m_total, c->active.as<int32_t>(), nactive, alpha, support, beta, d_w,
                          d_p, d_u, d_s));
    if (warps) NRM_CUDA(cudaMemcpyAsync(warps, d_w, nqs * 5 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (pred) NRM_CUDA(cudaMemcpyAsync(pred, d_p, nqs * 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (unc) NRM_CUDA(cudaMemcpyAsync(unc, d_u, nqs * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (status) NRM_CUDA(cudaMemcpyAsync(status, d_s, nqs * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    return NRM_OK;
}

int nrm_emdq_points_device(nrm_ctx* c, const double* d_q, const int32_t* d_exclude, int nq, const double* d_apts,
                           const double* d_locals, const double* d_probs, int m_total, const int32_t* d_active,
                           int nactive, double alpha, int support, double beta, double* d_warps, double* d_pred,
                           double* d_unc, int32_t* d_status) {
    if (!c) return fail(NRM_ESTATE, "null context");
    if (nq < 0 || (nq > 0 && !d_q)) return fail(NRM_EINVAL, "emdq_points: bad query array");
    if (nq == 0) return NRM_OK;
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    NRM_CUDA(c->misc.ensure(256));
    double* d_bb = reinterpret_cast<double*>(c->misc.as<char>() + 192);  // misc[192..224): scratch
    NRM_CUDA(launch_points_bbox(d_q, nq, d_bb, c->stream, &c->launches));
    double bb[4];
    NRM_CUDA(cudaMemcpyAsync(bb, d_bb, sizeof(bb), cudaMemcpyDeviceToHost, c->stream));
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    return points_core(c, bb, d_q, d_exclude, nq, d_apts, d_locals, d_probs, m_total, d_active, nactive, alpha,
                       support, beta, d_warps, d_pred, d_unc, d_status);
}

// ---- sparse front end (features.hpp) -------------------------------------------
namespace {
int detect_core(nrm_ctx* c, const uint8_t* d_image, const float* d_gray, int w, int h, int ch,
                const nrm_detector_config* cfg, double* d_kp, float* d_desc, int* d_n) {
    if (!cfg) return fail(NRM_EINVAL, "detect_features: null config");
    if (w < 0 || h < 0 || (w > 0 && h > 0 && !d_image && !d_gray)) return fail(NRM_EINVAL, "detect_features: bad image");
    if (!d_image && !d_gray) ch = 1;
    if (d_image && ch != 1 && ch != 3 && ch != 4) return fail(NRM_EINVAL, "detect_features: channels must be 1, 3 or 4");
    constexpr int kMargin = 10;  // kBorderMargin (features.hpp:55)
    if (cfg->max_features < 0 || cfg->nms_radius < 0 || !std::isfinite(cfg->quality_level))
        return fail(NRM_EINVAL, "detect_features: bad config");
    if (cfg->nms_radius > kMargin)  // the reference would read outside the response image
        return fail(NRM_EINVAL, "detect_features: nms_radius must be <= 10 (the border margin)");
    if (w < 2 * kMargin + 1 || h < 2 * kMargin + 1 || cfg->max_features == 0) {  // features.hpp:144
        NRM_CUDA(cudaMemsetAsync(d_n, 0, sizeof(int), c->stream));
        return NRM_OK;
    }
    NRM_CUDA(c->feat.ensure(features_scratch_bytes(w, h, cfg->nms_radius, cfg->max_features) + 64));
    FeatLaunch F;
    F.image = d_image;
    F.gray_in = d_gray;
    F.w = w;
    F.h = h;
    F.ch = ch;
    F.max_features = cfg->max_features;
    F.nms_radius = cfg->nms_radius;
    F.quality = static_cast<float>(cfg->quality_level);
    F.kp = d_kp;
    F.desc = d_desc;
    F.status = d_n;  // status[0] = count; status[1] lives in misc
    NRM_CUDA(c->misc.ensure(256));
    int* st2 = reinterpret_cast<int*>(c->misc.as<char>() + 224);  // misc[224..232): keypoint count, fallback flag
    F.status = st2;
    F.scratch = c->feat.p;
    NRM_CUDA(launch_detect_features(F, c->stream, &c->launches));
    NRM_CUDA(cudaMemcpyAsync(d_n, st2, sizeof(int), cudaMemcpyDeviceToDevice, c->stream));
    return NRM_OK;
}

int match_core(nrm_ctx* c, const double* d_kpa, const float* d_da, int na, const double* d_kpb, const float* d_db,
               int nb, double ratio, double* d_out, int* d_n) {
    if (na < 0 || nb < 0) return fail(NRM_EINVAL, "match_features: negative size");
    if (!std::isfinite(ratio)) return fail(NRM_EINVAL, "match_features: ratio must be finite");
    if (na == 0 || nb < 2) {  // features.hpp:211
        NRM_CUDA(cudaMemsetAsync(d_n, 0, sizeof(int), c->stream));
        return NRM_OK;
    }
    NRM_CUDA(c->feat.ensure(match_scratch_bytes(na, nb)));
    MatchLaunch M;
    M.kp_a = d_kpa;
    M.desc_a = d_da;
    M.na = na;
    M.kp_b = d_kpb;
    M.desc_b = d_db;
    M.nb = nb;
    M.ratio = ratio;
    M.out = d_out;
    M.nout = d_n;
    M.scratch = c->feat.p;
    NRM_CUDA(launch_match_features(M, c->stream, &c->launches));
    return NRM_OK;
}
}  // namespace

int nrm_detect_features(nrm_ctx* c, const uint8_t* image, int w, int h, int ch, const nrm_detector_config* cfg,
                        double* kp, float* desc, int* n) {
    if (!c) return fail(NRM_ESTATE, "null context");
    if (!n || !cfg || (cfg->max_features > 0 && (!kp || !desc))) return fail(NRM_EINVAL, "detect_features: null output");
    if (ch != 1 && ch != 3 && ch != 4) return fail(NRM_EINVAL, "detect_features: channels must be 1, 3 or 4");
    if (w < 0 || h < 0 || (w > 0 && h > 0 && !image)) return fail(NRM_EINVAL, "detect_features: bad image");
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    const size_t bytes = (size_t)w * h * ch;
    NRM_CHECK(upload(c, c->frame_raw, image, bytes));
    const int kmax = std::max(cfg->max_features, 0);
    NRM_CUDA(c->feat_io.ensure((size_t)kmax * (3 * sizeof(double) + 64 * sizeof(float)) + 16));
    double* d_kp = c->feat_io.as<double>();
    float* d_desc = reinterpret_cast<float*>(d_kp + 3 * (size_t)kmax);
    int* d_n = reinterpret_cast<int*>(d_desc + 64 * (size_t)kmax);
    NRM_CHECK(detect_core(c, c->frame_raw.as<uint8_t>(), nullptr, w, h, ch, cfg, d_kp, d_desc, d_n));
    NRM_CUDA(cudaMemcpyAsync(n, d_n, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    if (*n > 0) {
        NRM_CUDA(cudaMemcpyAsync(kp, d_kp, (size_t)*n * 3 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        NRM_CUDA(cudaMemcpyAsync(desc, d_desc, (size_t)*n * 64 * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
        NRM_CUDA(cudaStreamSynchronize(c->stream));
    }
    return NRM_OK;
}

int nrm_detect_features_gray(nrm_ctx* c, const float* gray, int w, int h, const nrm_detector_config* cfg, double* kp,
                             float* desc, int* n) {
    if (!c) return fail(NRM_ESTATE, "null context");
    if (!n || !cfg || (cfg->max_features > 0 && (!kp || !desc))) return fail(NRM_EINVAL, "detect_features: null output");
    if (w < 0 || h < 0 || (w > 0 && h > 0 && !gray)) return fail(NRM_EINVAL, "detect_features: bad image");
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    NRM_CHECK(upload(c, c->frame_raw, gray, (size_t)w * h * sizeof(float)));
    const int kmax = std::max(cfg->max_features, 0);
    NRM_CUDA(c->feat_io.ensure((size_t)kmax * (3 * sizeof(double) + 64 * sizeof(float)) + 16));
    double* d_kp = c->feat_io.as<double>();
    float* d_desc = reinterpret_cast<float*>(d_kp + 3 * (size_t)kmax);
    int* d_n = reinterpret_cast<int*>(d_desc + 64 * (size_t)kmax);
    NRM_CHECK(detect_core(c, nullptr, c->frame_raw.as<float>(), w, h, 1, cfg, d_kp, d_desc, d_n));
    NRM_CUDA(cudaMemcpyAsync(n, d_n, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    if (*n > 0) {
        NRM_CUDA(cudaMemcpyAsync(kp, d_kp, (size_t)*n * 3 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        NRM_CUDA(cudaMemcpyAsync(desc, d_desc, (size_t)*n * 64 * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
        NRM_CUDA(cudaStreamSynchronize(c->stream));
    }
    return NRM_OK;
}

int nrm_detect_features_device(nrm_ctx* c, const uint8_t* d_image, int w, int h, int ch,
                               const nrm_detector_config* cfg, double* d_kp, float* d_desc, int* d_n) {
    if (!c) return fail(NRM_ESTATE, "null context");
    if (!d_n || !cfg || (cfg->max_features > 0 && (!d_kp || !d_desc))) return fail(NRM_EINVAL, "detect_features: null output");
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    return detect_core(c, d_image, nullptr, w, h, ch, cfg, d_kp, d_desc, d_n);
}

int nrm_match_features(nrm_ctx* c, const double* kp_a, const float* desc_a, int na, const double* kp_b,
                       const float* desc_b, int nb, double ratio, double* out, int* n) {
    if (!c) return fail(NRM_ESTATE, "null context");
    if (!n || (na > 0 && (!kp_a || !desc_a || !out)) || (nb > 0 && (!kp_b || !desc_b)))
        return fail(NRM_EINVAL, "match_features: null array");
    if (na < 0 || nb < 0) return fail(NRM_EINVAL, "match_features: negative size");
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    const size_t sa = (size_t)na, sb = (size_t)nb;
    NRM_CUDA(c->feat_io.ensure((sa + sb) * (3 * sizeof(double) + 64 * sizeof(float)) + sa * 5 * sizeof(double) + 16));
    double* d_kpa = c->feat_io.as<double>();
    double* d_kpb = d_kpa + 3 * sa;
    double* d_out = d_kpb + 3 * sb;
    float* d_da = reinterpret_cast<float*>(d_out + 5 * sa);
    float* d_db = d_da + 64 * sa;
    int* d_n = reinterpret_cast<int*>(d_db + 64 * sb);
    if (na) {
        NRM_CUDA(cudaMemcpyAsync(d_kpa, kp_a, sa * 3 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        NRM_CUDA(cudaMemcpyAsync(d_da, desc_a, sa * 64 * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    }
    if (nb) {
        NRM_CUDA(cudaMemcpyAsync(d_kpb, kp_b, sb * 3 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        NRM_CUDA(cudaMemcpyAsync(d_db, desc_b, sb * 64 * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    }
    NRM_CHECK(match_core(c, d_kpa, d_da, na, d_kpb, d_db, nb, ratio, d_out, d_n));
    NRM_CUDA(cudaMemcpyAsync(n, d_n, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    if (*n > 0) {
        NRM_CUDA(cudaMemcpyAsync(out, d_out, (size_t)*n * 5 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        NRM_CUDA(cudaStreamSynchronize(c->stream));
    }
    return NRM_OK;
}

int nrm_match_features_device(nrm_ctx* c, const double* d_kp_a, const float* d_desc_a, int na, const double* d_kp_b,
                              const float* d_desc_b, int nb, double ratio, double* d_out, int* d_n) {
    if (!c) return fail(NRM_ESTATE, "null context");
    if (!d_n || (na > 0 && (!d_kp_a || !d_desc_a || !d_out)) || (nb > 0 && (!d_kp_b || !d_desc_b)))
        return fail(NRM_EINVAL, "match_features: null array");
    DeviceGuard g(c->device);
    ProfScope prof_scope(c);
    return match_core(c, d_kp_a, d_desc_a, na, d_kp_b, d_desc_b, nb, ratio, d_out, d_n);
}

// ---- diagnostics -------------------------------------------------------------
int nrm_selftest_libm(nrm_ctx* c, const double* x, const double* y, int n, double* exp_out, double* hypot_out) {
    if (!c) return fail(NRM_ESTATE, "null context");
    if (n < 0 || (n > 0 && (!x || !y || !exp_out || !hypot_out))) return fail(NRM_EINVAL, "bad arrays");
    if (n == 0) return NRM_OK;
    DeviceGuard g(c->device);
    NRM_CHECK(upload(c, c->pts, x, (size_t)n * sizeof(double)));
    NRM_CHECK(upload(c, c->probs, y, (size_t)n * sizeof(double)));
    NRM_CUDA(c->out_a.ensure((size_t)n * 2 * sizeof(double)));
    double* o = c->out_a.as<double>();
    NRM_CUDA(launch_selftest_libm(c->pts.as<double>(), c->probs.as<double>(), n, o, o + n, c->stream, &c->launches));
    NRM_CUDA(cudaMemcpyAsync(exp_out, o, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    NRM_CUDA(cudaMemcpyAsync(hypot_out, o + n, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    return NRM_OK;
}

int nrm_selftest_peak(nrm_ctx* c, int which, double* ops_per_s) {
    if (!c || !ops_per_s) return fail(NRM_EINVAL, "null argument");
    if (which != 0 && which != 1) return fail(NRM_EINVAL, "which: 0 = FP32 FFMA, 1 = MUFU.EX2");
    DeviceGuard g(c->device);
    NRM_CUDA(c->misc.ensure(256));
    const int iters = which == 0 ? 4096 : 1024;
    float ms = 0.f;
    NRM_CUDA(run_peak_probe(which, c->num_sms, iters, reinterpret_cast<float*>(c->misc.as<char>() + 64), c->stream,
                            &ms, &c->launches));
    const double ops = (double)c->num_sms * 8 * 256 * (double)iters * 16 * 8;  // lane-ops
    *ops_per_s = ops / (ms * 1e-3);
    return NRM_OK;
}

// ---- kernel timing -------------------------------------------------------------
int nrm_ctx_profile(nrm_ctx* c, int enable) {
    if (!c) return fail(NRM_ESTATE, "null context");
    DeviceGuard g(c->device);
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    c->prof.on = enable != 0;
    c->prof.used = 0;
    return NRM_OK;
}

int nrm_ctx_profile_read(nrm_ctx* c, char* names, int names_len, double* ms, int64_t* counts, int cap, int* n) {
    if (!c || !n) return fail(NRM_EINVAL, "null argument");
    DeviceGuard g(c->device);
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    std::vector<std::string> keys;
    std::vector<double> tot;
    std::vector<int64_t> cnt;
    Prof& p = c->prof;
    for (size_t i = 0; i + 1 < p.used; ++i) {
        if (!p.name[i]) continue;
        float dt = 0.f;
        NRM_CUDA(cudaEventElapsedTime(&dt, p.ev[i], p.ev[i + 1]));
        size_t k = 0;
        while (k < keys.size() && keys[k] != p.name[i]) ++k;
        if (k == keys.size()) {
            keys.emplace_back(p.name[i]);
            tot.push_back(0.0);
            cnt.push_back(0);
        }
        tot[k] += dt;
        cnt[k] += 1;
    }
    *n = (int)keys.size();
    std::string joined;
    for (size_t k = 0; k < keys.size(); ++k) {
        if (k < (size_t)cap) {
            if (ms) ms[k] = tot[k];
            if (counts) counts[k] = cnt[k];
        }
        joined += keys[k];
        joined += '\n';
    }
    if (names && names_len > 0) {
        std::strncpy(names, joined.c_str(), (size_t)names_len - 1);
        names[names_len - 1] = 0;
    }
    return NRM_OK;
}

// ---- pure host planning (no device needed) --------------------------------
int nrm_plan_ensure_contains(int64_t ox, int64_t oy, int w, int h, double x0, double y0, double x1, double y1,
                             int64_t* new_ox, int64_t* new_oy, int* new_w, int* new_h) {
    if (!new_ox || !new_oy || !new_w || !new_h) return fail(NRM_EINVAL, "null output");
    if (w < 0 || h < 0) return fail(NRM_EINVAL, "negative canvas size");
    int64_t a, b, c2, d;
    int grew;
    NRM_CHECK(plan_ensure_contains(ox, oy, w, h, x0, y0, x1, y1, &a, &b, &c2, &d, &grew));
    *new_ox = a;
    *new_oy = b;
    *new_w = (int)c2;
    *new_h = (int)d;
    return NRM_OK;
}

int nrm_plan_footprint(const double* poly, int npoly, int64_t origin_x, int64_t origin_y, int64_t* bbox4,
                       int64_t* footprint) {
    if (!bbox4 || !footprint) return fail(NRM_EINVAL, "null output");
    bbox4[0] = bbox4[1] = 0;
    bbox4[2] = bbox4[3] = -1;
    *footprint = 0;
    if (npoly < 3) return NRM_OK;
    if (!poly || !finite_all(poly, (size_t)npoly * 2)) return fail(NRM_EINVAL, "bad polygon");
    const Bbox bb = footprint_bbox(poly, npoly);
    const double orgx = (double)origin_x, orgy = (double)origin_y;  // mosaic.hpp:206-213
    bbox4[0] = (int64_t)std::floor(bb.x0 - orgx);
    bbox4[1] = (int64_t)std::floor(bb.y0 - orgy);
    bbox4[2] = (int64_t)std::ceil(bb.x1 - orgx);
    bbox4[3] = (int64_t)std::ceil(bb.y1 - orgy);
    const int64_t bw = bbox4[2] - bbox4[0] + 1, bh = bbox4[3] - bbox4[1] + 1;
    *footprint = bw > 0 && bh > 0 ? bw * bh : 0;
    return NRM_OK;
}

int nrm_band_owns_row(int64_t abs_row, int rank, int count) {
    if (count <= 1) return 1;
    int64_t s = abs_row / kStripeRows;
    if (abs_row % kStripeRows != 0 && abs_row < 0) --s;
    int64_t m = s % count;
    if (m < 0) m += count;
    return m == rank;
}

int nrm_ctx_exceptions(nrm_ctx* c, int64_t* blend_exceptions, int64_t* emdq_exact) {
    if (!c) return fail(NRM_ESTATE, "null context");
    DeviceGuard g(c->device);
    unsigned v[2] = {0, 0};
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    NRM_CUDA(cudaMemcpy(v, state_of(c).last_exc, sizeof(v), cudaMemcpyDeviceToHost));
    if (blend_exceptions) *blend_exceptions = v[0];
    if (emdq_exact) *emdq_exact = v[1];
    return NRM_OK;
}

int nrm_ctx_set_exception_capacity(nrm_ctx* c, int64_t slots) {
    if (!c) return fail(NRM_ESTATE, "null context");
    if (slots < 0) return fail(NRM_EINVAL, "exception capacity must be >= 0");
    c->exc_cap_override = slots;
    return NRM_OK;
}

int nrm_ctx_spilled_launches(nrm_ctx* c, int64_t* out) {
    if (!c || !out) return fail(NRM_EINVAL, "null argument");
    DeviceGuard g(c->device);
    unsigned v = 0;
    NRM_CUDA(cudaStreamSynchronize(c->stream));
    NRM_CUDA(cudaMemcpy(&v, state_of(c).overflow, sizeof(v), cudaMemcpyDeviceToHost));
    *out = v;
    return NRM_OK;
}

}  // extern "C"
