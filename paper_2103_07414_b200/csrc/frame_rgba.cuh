// K1's frame textures: ImageU8 frames with 3 or 4 channels converted to RGBA8
// rows so the fast tier's bilinear sample is three tex2Dgather calls. Used by
// k_frame_rgba (batched blends) and by the conversion CTAs of k_nf_plan.
#pragma once
#include <cstdint>

namespace nrm {

// ImageU8 -> RGBA8 (alpha 255), frame blockIdx.y into its pitched slot. The
// frame is a flat range of groups of 4 pixels (row-major); a thread converts
// 8 groups, blockDim.x * gridDim.x apart so each load and store instruction
// is coalesced across the warp, all loads before the stores (the pass is a
// 14 MB copy at 1080p): 12 (RGB) or 16 (RGBA) input bytes per group, one
// 16-byte store.
constexpr int RGBA_GROUPS = 8, RGBA_THREADS = 256;
__device__ __forceinline__ uint4 rgba_group(const uint8_t* src, int fch, int nvalid) {
    unsigned v[4];
    if (nvalid == 4 && (reinterpret_cast<uintptr_t>(src) & 3u) == 0) {
        const unsigned* w = reinterpret_cast<const unsigned*>(src);
        if (fch == 3) {
            const unsigned w0 = __ldg(w), w1 = __ldg(w + 1), w2 = __ldg(w + 2);
            v[0] = __byte_perm(w0, 0xffffffffu, 0x4210);       // R0 G0 B0 .
            v[1] = __byte_perm(w0, w1, 0x0543) | 0xff000000u;  // R1 G1 B1 .
            v[2] = __byte_perm(w1, w2, 0x0432) | 0xff000000u;  // R2 G2 B2 .
            v[3] = __byte_perm(w2, 0xffffffffu, 0x4321);       // R3 G3 B3 .
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = __ldg(w + k) | 0xff000000u;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[k] = 0xff000000u;
            if (k < nvalid) {
                const uint8_t* p = src + k * fch;
                v[k] |= (unsigned)__ldg(p) | ((unsigned)__ldg(p + 1) << 8) | ((unsigned)__ldg(p + 2) << 16);
            }
        }
    }
    return make_uint4(v[0], v[1], v[2], v[3]);
}

// Whole-thread fast path (every group full and 4-byte aligned: fw % 4 == 0
// and an aligned frame): the loads are unconditional on clamped group indices
// so none waits at a branch join (a per-group branch serialises the latency).
template <int FCH>
__device__ __forceinline__ void rgba_fast(const uint8_t* base, uint8_t* obase, int gpr, int total, size_t pitch,
                                          int g0, int stride) {
    unsigned w[RGBA_GROUPS][FCH];
#pragma unroll
    for (int u = 0; u < RGBA_GROUPS; ++u) {
        const int g = min(g0 + u * stride, total - 1);
        const unsigned* src = reinterpret_cast<const unsigned*>(base) + (size_t)g * FCH;
#pragma unroll
        for (int k = 0; k < FCH; ++k)  // volatile: the compiler would sink each load to its store
            asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(w[u][k]) : "l"(src + k));
    }
#pragma unroll
    for (int u = 0; u < RGBA_GROUPS; ++u) {
        const int g = g0 + u * stride;
        if (g >= total) continue;
        uint4 o;
        if (FCH == 3) {
            o.x = __byte_perm(w[u][0], 0xffffffffu, 0x4210);
            o.y = __byte_perm(w[u][0], w[u][1], 0x0543) | 0xff000000u;
            o.z = __byte_perm(w[u][1], w[u][2], 0x0432) | 0xff000000u;
            o.w = __byte_perm(w[u][2], 0xffffffffu, 0x4321);
        } else {
            o = make_uint4(w[u][0] | 0xff000000u, w[u][1] | 0xff000000u, w[u][2 % FCH] | 0xff000000u,
                           w[u][3 % FCH] | 0xff000000u);
        }
        const int y = g / gpr;
        *reinterpret_cast<uint4*>(obase + (size_t)y * pitch + 16 * (size_t)(g - y * gpr)) = o;
    }
}

// Converts the groups of CTA `cta` of `ncta` (blockDim.x threads each).
__device__ __forceinline__ void rgba_convert(const uint8_t* base, uint8_t* obase, int fw, int fh, int fch,
                                             size_t pitch, int cta, int ncta) {
    const int gpr = (fw + 3) >> 2, total = gpr * fh, stride = blockDim.x * ncta;
    const bool fast = (fw & 3) == 0 && (reinterpret_cast<uintptr_t>(base) & 3u) == 0;
    for (int g0 = cta * blockDim.x + threadIdx.x; g0 < total; g0 += stride * RGBA_GROUPS) {
        if (fast && fch == 3) {
            rgba_fast<3>(base, obase, gpr, total, pitch, g0, stride);
        } else if (fast && fch == 4) {
            rgba_fast<4>(base, obase, gpr, total, pitch, g0, stride);
        } else {
            for (int u = 0; u < RGBA_GROUPS; ++u) {
                const int g = g0 + u * stride;
                if (g >= total) break;
                const int y = g / gpr, x = 4 * (g - y * gpr);
                const uint4 o = rgba_group(base + ((size_t)y * fw + x) * fch, fch, min(4, fw - x));
                *reinterpret_cast<uint4*>(obase + (size_t)y * pitch + 4 * (size_t)x) = o;
            }
        }
    }
}

}  // namespace nrm
