// Device-side pieces of the objective evaluators, shared by the standalone evaluation
// kernel (evaluate.cu) and the evaluation epilogue fused into reproduction (reproduce.cu).
// reference: problems.hpp:24-92 (DTLZ1-4). LSMOP1 is an extension (parity unpinned).
#pragma once

#include "glibc_pow_dev.cuh"
#include "internal.h"

namespace temo_b200 {

// cos(a) for the bounded argument of the DTLZ1/3 term, |a| = |20 pi (x - 0.5)| <= 10 pi (valid far beyond: |a| < 2^30):
// one-step reduction a - n pi with a two-word pi (n <= 10: the first product is exact to the last bit of a), then the
// even Taylor polynomial of degree 24 on [-pi/2, pi/2]. Twenty instructions against the ~45 of the general routine (no
// quadrant table, no large-argument path); absolute error <= 2.8e-16 over 2e7 arguments against cosl (libm's cos:
// 0.6e-16, CUDA's cos: ~2e-16) - a term of the sum g carries t * t - cos(...) of magnitude O(1), so this is within one
// ulp of the term and far inside the 1e-12 relative tolerance of the objectives.
__device__ __forceinline__ double cos_bounded(double a) {
    const double kMagic = 6755399441055744.0;  // 1.5 * 2^52: rint through the adder
    const double z = a * 0.31830988618379067154 + kMagic;
    const double nf = z - kMagic;
    double r = fma(-nf, 3.141592653589793116, a);
    r = fma(-nf, 1.2246467991473532e-16, r);
    const double s = r * r;
    double p = 1.6117375710961184e-24;                 //  1 / 24!
    p = fma(p, s, -8.896791392450574e-22);           // -1 / 22!
    p = fma(p, s, 4.110317623312165e-19);            //  1 / 20!
    p = fma(p, s, -1.5619206968586225e-16);          // -1 / 18!
    p = fma(p, s, 4.779477332387385e-14);            //  1 / 16!
    p = fma(p, s, -1.1470745597729725e-11);          // -1 / 14!
    p = fma(p, s, 2.08767569878681e-09);             //  1 / 12!
    p = fma(p, s, -2.755731922398589e-07);           // -1 / 10!
    p = fma(p, s, 2.48015873015873e-05);             //  1 / 8!
    p = fma(p, s, -0.001388888888888889);            // -1 / 6!
    p = fma(p, s, 0.041666666666666664);             //  1 / 4!
    p = fma(p, s, -0.5);
    p = fma(p, s, 1.0);
    // odd n: cos(a) = -cos(r)
    return __hiloint2double(__double2hiint(p) ^ (__double2loint(z) << 31), __double2loint(p));
}

// Per-gene contribution of a tail gene (index >= m-1) to the distance function g.
//   DTLZ1/3 (problems.hpp:24-32): t*t - cos(20 pi t), t = x - 0.5
//   DTLZ2/4 (problems.hpp:34-41): t*t
template <int PID>
__device__ __forceinline__ double dtlz_term(double x) {
    const double t = x - 0.5;
    if (PID == kDtlz1 || PID == kDtlz3) {
        const double w = 20.0 * kPi;  // folded exactly like `20.0 * std::numbers::pi * t`
        return t * t - cos_bounded(w * t);
    }
    return t * t;
}

// Finishes one row: `sum` is the block-reduced tail sum, pos[0..m-2] the position genes.
// Thread-strided over the m objectives. problems.hpp:44-64,77-89.
template <int PID>
__device__ __forceinline__ void dtlz_finish(double sum, const double* pos, uint64_t m, uint64_t d,
                                            double* frow) {
    double g;
    if (PID == kDtlz1 || PID == kDtlz3)
        g = 100.0 * ((double)(d - m + 1) + sum);
    else
        g = sum;
    const double half_pi = kPi / 2.0;
    for (uint64_t j = threadIdx.x; j < m; j += blockDim.x) {
        double v;
        if (PID == kDtlz1) {
            v = 0.5 * (1.0 + g);
            for (uint64_t i = 0; i + j + 1 < m; ++i) v *= pos[i];
            if (j > 0) v *= 1.0 - pos[m - 1 - j];
        } else {
            v = 1.0 + g;
            for (uint64_t i = 0; i + j + 1 < m; ++i) {
                const double p = PID == kDtlz4 ? pow_like_host(pos[i], 100.0, pow_tables_global()) : pos[i];
                v *= cos(p * half_pi);
            }
            if (j > 0) {
                const double p = PID == kDtlz4 ? pow_like_host(pos[m - 1 - j], 100.0, pow_tables_global()) : pos[m - 1 - j];
                v *= sin(p * half_pi);
            }
        }
        frow[j] = v;
    }
}

}  // namespace temo_b200
