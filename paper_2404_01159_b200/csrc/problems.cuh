// Device-side pieces of the objective evaluators, shared by the standalone evaluation
// kernel (evaluate.cu) and the evaluation epilogue fused into reproduction (reproduce.cu).
// reference: problems.hpp:24-92 (DTLZ1-4). LSMOP1 is an extension (parity unpinned).
#pragma once

#include "glibc_pow_dev.cuh"
#include "internal.h"

namespace temo_b200 {

// Per-gene contribution of a tail gene (index >= m-1) to the distance function g.
//   DTLZ1/3 (problems.hpp:24-32): t*t - cos(20 pi t), t = x - 0.5
//   DTLZ2/4 (problems.hpp:34-41): t*t
template <int PID>
__device__ __forceinline__ double dtlz_term(double x) {
    const double t = x - 0.5;
    if (PID == kDtlz1 || PID == kDtlz3) {
        const double w = 20.0 * kPi;  // folded exactly like `20.0 * std::numbers::pi * t`
        return t * t - cos(w * t);
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
