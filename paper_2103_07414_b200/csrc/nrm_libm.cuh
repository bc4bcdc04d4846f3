// nrm_libm.cuh -- bit-exact device emulation of the host libm functions the
// reference calls on its decision paths (std::exp, std::hypot), so that the
// exact tier reproduces the reference's FP64 results to the last bit.
//
// Target: glibc 2.39 on x86-64 with FMA (the platform the reference is built
// and timed on here and on the GPU box; `ldd --version`, /proc/cpuinfo fma).
//   exp   -- the table-driven algorithm of glibc's dbl-64 exp (N = 128,
//            degree-5 polynomial), as its x86-64 FMA ifunc variant evaluates
//            it: every a*b+c of the main path fused, the subnormal/overflow
//            rescaling path unfused.
//   hypot -- glibc's correctly-rounded-by-correction hypot kernel (non-FMA
//            build): sqrt(ax^2 + ay^2) then one Newton-style correction.
// Both are checked bit for bit against the host libm on 4e5 random inputs per
// run (tests/test_gpu_libm.py; exp over [-800, 1] plus the special cases).
// The 2^(k/128) table is generated from first principles (gen_exp_table.py).
//
// Attribution: the exp algorithm -- its constants (InvLn2N, Shift,
// NegLn2hiN/loN, the C2..C5 polynomial), the special-case path and the
// 1009 / 1022 exponent rescaling -- is that of glibc's sysdeps/ieee754/dbl-64
// e_exp.c, which comes from ARM's optimized-routines (Szabolcs Nagy; MIT /
// Apache-2.0 WITH LLVM-exception in optimized-routines, LGPL-2.1+ in glibc).
// It is restated here, not copied, because matching the reference's results
// bit for bit requires the same operations in the same order; the hypot
// correction kernel likewise follows glibc's e_hypot.c (LGPL-2.1+).
#pragma once

#include <cstdint>

#include "libm_exp_table.h"

namespace nrm {

__device__ __forceinline__ uint64_t dbits(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ __forceinline__ double bitsd(uint64_t u) { return __longlong_as_double((long long)u); }

__device__ inline double xexp(double x) {
    constexpr double InvLn2N = 0x1.71547652b82fep7, Shift = 0x1.8p52;
    constexpr double NegLn2hiN = -0x1.62e42fefa0000p-8, NegLn2loN = -0x1.cf79abc9e3b3ap-47;
    constexpr double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3;
    constexpr double C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;
    uint32_t abstop = (uint32_t)(dbits(x) >> 52) & 0x7ff;
    if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {
        if (abstop - 0x3c9u >= 0x80000000u) return 1.0 + x;  // |x| < 2^-54
        if (abstop >= 0x409u) {                               // |x| >= 1024
            if (dbits(x) == 0xfff0000000000000ull) return 0.0;
            if (abstop >= 0x7ffu) return 1.0 + x;
            return (dbits(x) >> 63) ? 0.0 : __longlong_as_double(0x7ff0000000000000ll);
        }
        abstop = 0;  // large |x|: rescaled below
    }
    double kd = __fma_rn(InvLn2N, x, Shift);
    const uint64_t ki = dbits(kd);
    kd = __dsub_rn(kd, Shift);
    const double r = __fma_rn(kd, NegLn2loN, __fma_rn(kd, NegLn2hiN, x));
    const uint64_t idx = 2 * (ki % 128);
    const uint64_t top = ki << 45;
    const double tail = bitsd(__ldg(&kExpTab[idx]));
    uint64_t sbits = __ldg(&kExpTab[idx + 1]) + top;
    const double r2 = __dmul_rn(r, r);
    const double tmp = __fma_rn(__dmul_rn(r2, r2), __fma_rn(r, C5, C4),
                                __fma_rn(r2, __fma_rn(r, C3, C2), __dadd_rn(tail, r)));
    if (abstop == 0) {
        double scale, y;
        if ((ki & 0x80000000ull) == 0) {
            sbits -= 1009ull << 52;
            scale = bitsd(sbits);
            return __dmul_rn(0x1p1009, __dadd_rn(scale, __dmul_rn(scale, tmp)));
        }
        sbits += 1022ull << 52;
        scale = bitsd(sbits);
        y = __dadd_rn(scale, __dmul_rn(scale, tmp));
        if (y < 1.0) {
            double lo = __dadd_rn(__dsub_rn(scale, y), __dmul_rn(scale, tmp));
            const double hi = __dadd_rn(1.0, y);
            lo = __dadd_rn(__dadd_rn(__dsub_rn(1.0, hi), y), lo);
            y = __dsub_rn(__dadd_rn(hi, lo), 1.0);
            if (y == 0.0) y = 0.0;
        }
        return __dmul_rn(0x1p-1022, y);
    }
    const double scale = bitsd(sbits);
    return __fma_rn(scale, tmp, scale);
}

__device__ __forceinline__ double xhypot_kernel(double ax, double ay) {
    double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
    double t1, t2;
    if (h <= __dmul_rn(2.0, ay)) {
        const double delta = __dsub_rn(h, ay);
        t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
        t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
    } else {
        const double delta = __dsub_rn(h, ax);
        t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
        t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
    }
    return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}

__device__ inline double xhypot(double x, double y) {
    constexpr double SCALE = 0x1p-600, LARGE_VAL = 0x1p+511, TINY_VAL = 0x1p-511, EPS = 0x1p-54;
    if (!isfinite(x) || !isfinite(y)) {
        if (isinf(x) || isinf(y)) return __longlong_as_double(0x7ff0000000000000ll);
        return x + y;
    }
    x = fabs(x);
    y = fabs(y);
    double ax = x < y ? y : x, ay = x < y ? x : y;
    if (ax > LARGE_VAL) {
        if (ay <= __dmul_rn(ax, EPS)) return __dadd_rn(ax, ay);
        return __ddiv_rn(xhypot_kernel(__dmul_rn(ax, SCALE), __dmul_rn(ay, SCALE)), SCALE);
    }
    if (ay < TINY_VAL) {
        if (ax >= __ddiv_rn(ay, EPS)) return __dadd_rn(ax, ay);
        return __dmul_rn(xhypot_kernel(__ddiv_rn(ax, SCALE), __ddiv_rn(ay, SCALE)), SCALE);
    }
    if (ay <= __dmul_rn(ax, EPS)) return __dadd_rn(ax, ay);
    return xhypot_kernel(ax, ay);
}

}  // namespace nrm
