// tanh with the host libm's bits.
//
// The toy control environment (problems.hpp:149-241) chains 18 std::tanh per step over a whole episode, so the device
// evaluator follows the C library's own operation sequence: glibc's tanh (sysdeps/ieee754/dbl-64/s_tanh.c) on top of
// its expm1 (s_expm1.c), both the classic fdlibm algorithms (Sun Microsystems, freely redistributable): pure IEEE
// arithmetic, no tables. tanh itself has one build; expm1 is an IFUNC whose x86-64 FMA variant (the one every
// AVX2 + FMA host selects, like pow's: DESIGN.md section 5) contracts a fixed subset of its multiply-adds - the
// polynomial R1 / R2 / R3 / r1, t = 3 - r1 hfx, the divisor 6 - x t, and x e - hxs / x (e - c) - c. That pattern was
// read off the installed libm.so.6 (objdump of the function behind the expm1 resolver) and is spelled out with explicit
// fma calls below; every other line is one rounded operation (the device build uses --fmad=false).
// tests/test_pow_emulation.py checks the host twin against the live libm on random and special inputs.
#pragma once

#include <cstdint>
#include <cstring>

#include <cmath>

#ifdef __CUDACC__
#define TEMO_HD __host__ __device__ __forceinline__
#else
#define TEMO_HD inline
#endif
#ifdef __CUDA_ARCH__
#define TEMO_TFMA(a, b, c) __fma_rn((a), (b), (c))
#else
#define TEMO_TFMA(a, b, c) std::fma((a), (b), (c))
#endif

namespace temo_b200 {

TEMO_HD uint32_t tanh_high_word(double x) {
#ifdef __CUDA_ARCH__
    return (uint32_t)__double2hiint(x);
#else
    uint64_t u;
    std::memcpy(&u, &x, 8);
    return (uint32_t)(u >> 32);
#endif
}
TEMO_HD uint32_t tanh_low_word(double x) {
#ifdef __CUDA_ARCH__
    return (uint32_t)__double2loint(x);
#else
    uint64_t u;
    std::memcpy(&u, &x, 8);
    return (uint32_t)u;
#endif
}
TEMO_HD double tanh_with_high_word(double x, uint32_t hi) {
#ifdef __CUDA_ARCH__
    return __hiloint2double((int)hi, __double2loint(x));
#else
    uint64_t u;
    std::memcpy(&u, &x, 8);
    u = (u & 0xffffffffULL) | ((uint64_t)hi << 32);
    std::memcpy(&x, &u, 8);
    return x;
#endif
}

// expm1 (fdlibm / glibc s_expm1.c) for finite |x| < 709 (tanh only calls it with |x| < 44).
TEMO_HD double glibc_expm1(double x) {
    const double one = 1.0, huge = 1.0e+300, tiny = 1.0e-300;
    const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10, invln2 = 1.44269504088896338700e+00;
    const double Q1 = -3.33333333333331316428e-02, Q2 = 1.58730158725481460165e-03, Q3 = -7.93650757867487942473e-05,
                 Q4 = 4.00821782732936239552e-06, Q5 = -2.01099218183624371326e-07;
    double y, hi, lo, c = 0.0, t, e, hxs, hfx, r1, h2, h4, R1, R2, R3;
    int32_t k;
    uint32_t hx = tanh_high_word(x);
    const uint32_t xsb = hx & 0x80000000u;
    hx &= 0x7fffffffu;
    if (hx >= 0x4043687Au) {  // |x| >= 56 ln2
        if (xsb != 0) return tiny - one;  // x < -56 ln2
    }
    if (hx > 0x3fd62e42u) {  // |x| > 0.5 ln2
        if (hx < 0x3FF0A2B2u) {  // and |x| < 1.5 ln2
            if (xsb == 0) {
                hi = x - ln2_hi;
                lo = ln2_lo;
                k = 1;
            } else {
                hi = x + ln2_hi;
                lo = -ln2_lo;
                k = -1;
            }
        } else {
            k = (int32_t)(invln2 * x + ((xsb == 0) ? 0.5 : -0.5));
            t = (double)k;
            hi = TEMO_TFMA(-t, ln2_hi, x);  // t * ln2_hi is exact here
            lo = t * ln2_lo;
        }
        x = hi - lo;
        c = (hi - x) - lo;
    } else if (hx < 0x3c900000u) {  // |x| < 2^-54
        t = huge + x;
        return x - (t - (huge + x));
    } else {
        k = 0;
    }
    hfx = 0.5 * x;
    hxs = x * hfx;
    R1 = TEMO_TFMA(hxs, Q1, one);
    h2 = hxs * hxs;
    R2 = TEMO_TFMA(hxs, Q3, Q2);
    h4 = h2 * h2;
    R3 = TEMO_TFMA(hxs, Q5, Q4);
    r1 = TEMO_TFMA(h4, R3, TEMO_TFMA(h2, R2, R1));
    t = TEMO_TFMA(-r1, hfx, 3.0);
    e = hxs * ((r1 - t) / TEMO_TFMA(-x, t, 6.0));
    if (k == 0) return x - TEMO_TFMA(e, x, -hxs);
    e = TEMO_TFMA(e - c, x, -c);
    e -= hxs;
    if (k == -1) return 0.5 * (x - e) - 0.5;
    if (k == 1) {
        if (x < -0.25) return -2.0 * (e - (x + 0.5));
        return one + 2.0 * (x - e);
    }
    if (k <= -2 || k > 56) {  // suffice to return exp(x) - 1
        y = one - (e - x);
        y = tanh_with_high_word(y, tanh_high_word(y) + ((uint32_t)k << 20));
        return y - one;
    }
    t = one;
    if (k < 20) {
        t = tanh_with_high_word(t, 0x3ff00000u - (0x200000u >> k));  // 1 - 2^-k
        y = t - (e - x);
        y = tanh_with_high_word(y, tanh_high_word(y) + ((uint32_t)k << 20));
    } else {
        t = tanh_with_high_word(t, (uint32_t)((0x3ff - k) << 20));  // 2^-k
        y = x - (e + t);
        y += one;
        y = tanh_with_high_word(y, tanh_high_word(y) + ((uint32_t)k << 20));
    }
    return y;
}

// tanh (fdlibm / glibc s_tanh.c)
TEMO_HD double glibc_tanh(double x) {
    const double one = 1.0, two = 2.0, tiny = 1.0e-300;
    double t, z;
    const uint32_t jx = tanh_high_word(x), lx = tanh_low_word(x);
    const uint32_t ix = jx & 0x7fffffffu;
    const bool neg = (jx >> 31) != 0;
    if (ix >= 0x7ff00000u) return neg ? one / x - one : one / x + one;  // inf / NaN
    if (ix < 0x40360000u) {  // |x| < 22
        if ((ix | lx) == 0) return x;                 // +-0
        if (ix < 0x3c800000u) return x * (one + x);   // |x| < 2^-55
        const double ax = neg ? -x : x;
        if (ix >= 0x3ff00000u) {  // |x| >= 1
            t = glibc_expm1(two * ax);
            z = one - two / (t + two);
        } else {
            t = glibc_expm1(-two * ax);
            z = -t / (t + two);
        }
    } else {
        z = one - tiny;
    }
    return neg ? -z : z;
}

}  // namespace temo_b200
