// pow(x, y) with the exact operation sequence of glibc 2.39's x86-64 FMA variant (__pow_fma).
//
// Why: the reference's SBX / polynomial mutation call std::pow (operators.hpp:85-86,115-118).
// A child whose two parents are the same pool row (the pool is sampled with replacement,
// algorithms.hpp:218-220) equals that parent exactly on the CPU and then ties with it in the
// APD argmin (lowest row wins, selection.hpp:209-215). A pow that is off by one ulp breaks the
// tie the other way, so "survivor sets bit-exact" needs the C library's pow bit for bit — not
// merely an accurate one.
//
// What: glibc >= 2.28 implements pow with the algorithm of ARM Optimized Routines
// (math/pow.c, S. Nagy, MIT): log(x) = k ln2 + log(c_i) + log1p(z/c_i - 1) with a 128-entry
// table and a degree-7 polynomial evaluated in double-double (hi, lo); exp(y log x) with a
// 128-entry 2^(j/128) table and a degree-5 polynomial. The x86-64 multiarch build compiles it
// with -mfma, and GCC contracts a specific subset of the multiply-adds; the sequence below
// mirrors that build operation for operation (every line is one IEEE-754 operation: mul, add
// or fused multiply-add), so results are bit-identical wherever the host libm selects its FMA
// variant (every AVX2-class CPU). tests/test_pow_emulation.py pins it against the live libm.
//
// Scope: every finite x > 0 (subnormals included) with |y| in [2^-65, 2^63), including the
// under/overflow tails of exp. Callers get `false` for x = 0, negative x, inf/nan or extreme y
// and fall back to the platform pow (pow(0, y > 0) = 0 is exact in both).
#pragma once

#include <cmath>
#include <cstdint>

#include "glibc_pow_data.h"

namespace temo_b200 {

struct PowTables {
    const double* invc;      // [128]
    const double* logc;      // [128]
    const double* logctail;  // [128]
    const unsigned long long* exptab;  // [256] {tail, scale bits}
};

// The 17 scalar constants as one table: on the device it lives in constant memory, which lets the FP64
// instructions take them as c[bank][offset] operands (no register / uniform-register traffic).
#define TEMO_POW_SCALARS_INIT {TEMO_POW_LN2HI, TEMO_POW_LN2LO, TEMO_POW_A0, TEMO_POW_A1, TEMO_POW_A2, TEMO_POW_A3, \
                               TEMO_POW_A4, TEMO_POW_A5, TEMO_POW_A6, TEMO_POW_INVLN2N, TEMO_POW_SHIFT,           \
                               TEMO_POW_NEGLN2HIN, TEMO_POW_NEGLN2LON, TEMO_POW_C2, TEMO_POW_C3, TEMO_POW_C4,     \
                               TEMO_POW_C5}
#ifdef __CUDACC__
static __constant__ unsigned long long d_pow_scalars[17] = TEMO_POW_SCALARS_INIT;
#endif
static const unsigned long long h_pow_scalars[17] = TEMO_POW_SCALARS_INIT;

#ifdef __CUDA_ARCH__
#define TEMO_POW_K(i) __longlong_as_double((long long)d_pow_scalars[i])
#else
#define TEMO_POW_K(i) temo_as_double_host(h_pow_scalars[i])
#endif

#ifdef __CUDA_ARCH__
#define TEMO_FMA(a, b, c) __fma_rn((a), (b), (c))
#define TEMO_MUL(a, b) __dmul_rn((a), (b))
#define TEMO_ADD(a, b) __dadd_rn((a), (b))
#define TEMO_AS_DOUBLE(u) __longlong_as_double((long long)(u))
#define TEMO_AS_U64(d) ((unsigned long long)__double_as_longlong(d))
#else
#define TEMO_FMA(a, b, c) std::fma((a), (b), (c))
#define TEMO_MUL(a, b) ((a) * (b))
#define TEMO_ADD(a, b) ((a) + (b))
static inline double temo_as_double_host(unsigned long long u) {
    double d;
    __builtin_memcpy(&d, &u, 8);
    return d;
}
static inline unsigned long long temo_as_u64_host(double d) {
    unsigned long long u;
    __builtin_memcpy(&u, &d, 8);
    return u;
}
#define TEMO_AS_DOUBLE(u) temo_as_double_host(u)
#define TEMO_AS_U64(d) temo_as_u64_host(d)
#endif

// Returns true and writes *out when (x, y) is on a path restated here; false otherwise.
// NARROW = true is the caller's promise that x is positive and normal, |y| is ordinary and
// |y log x| < 512 (SBX: x in [2^-52, 2], |y| = 1/(eta+1)), which removes the range checks and the
// under/overflow tail; the arithmetic of the common path is the same instruction for instruction.
template <bool NARROW = false>
__host__ __device__ inline bool glibc_pow_main(double x, double y, const PowTables& T, double* out) {
    unsigned long long ix = TEMO_AS_U64(x);
    if (!NARROW) {
        const unsigned long long iy = TEMO_AS_U64(y);
        const unsigned topx = (unsigned)(ix >> 52), topy = (unsigned)(iy >> 52);
        if ((topy & 0x7ffu) - 0x3beu > 0x7fu) return false;  // |y| tiny or huge (or nan)
        if (topx - 1u > 0x7fdu) {
            if (topx != 0u || ix == 0ULL) return false;  // zero, negative, inf, nan
            // positive subnormal: normalise (x * 2^52, exponent corrected in the integer domain)
            ix = TEMO_AS_U64(TEMO_MUL(x, 4503599627370496.0)) - (52ULL << 52);
        }
    }

    // ---- log_inline: x = 2^k z, z in [OFF, 2 OFF), c_i near the centre of z's subinterval
    const unsigned long long tmp = ix - 0x3fe6955500000000ULL;
    const int i = (int)((tmp >> 45) & 127);
    const int k = (int)((long long)tmp >> 52);
    const double z = TEMO_AS_DOUBLE(ix - (tmp & 0xfff0000000000000ULL));
    const double kd = (double)k;
    const double ln2hi = TEMO_POW_K(0), ln2lo = TEMO_POW_K(1);
    const double A0 = TEMO_POW_K(2), A1 = TEMO_POW_K(3), A2 = TEMO_POW_K(4), A3 = TEMO_POW_K(5), A4 = TEMO_POW_K(6),
                 A5 = TEMO_POW_K(7), A6 = TEMO_POW_K(8);
    const double t1 = TEMO_FMA(kd, ln2hi, T.logc[i]);
    const double lo1 = TEMO_FMA(kd, ln2lo, T.logctail[i]);
    const double r = TEMO_FMA(z, T.invc[i], -1.0);
    const double ar = TEMO_MUL(r, A0);
    const double p12 = TEMO_FMA(r, A2, A1);
    const double p34 = TEMO_FMA(r, A4, A3);
    const double t2 = TEMO_ADD(r, t1);
    const double lo2 = TEMO_ADD(TEMO_ADD(t1, -t2), r);
    const double ar2 = TEMO_MUL(r, ar);
    const double ar3 = TEMO_MUL(r, ar2);
    const double lo3 = TEMO_FMA(ar, r, -ar2);
    const double hi = TEMO_ADD(t2, ar2);
    const double p56 = TEMO_FMA(r, A6, A5);
    const double lo4 = TEMO_ADD(TEMO_ADD(t2, -hi), ar2);
    const double q = TEMO_FMA(ar2, TEMO_FMA(p56, ar2, p34), p12);
    double lo = TEMO_ADD(lo1, lo2);
    lo = TEMO_ADD(lo, lo3);
    lo = TEMO_ADD(lo, lo4);
    lo = TEMO_FMA(ar3, q, lo);
    const double lg = TEMO_ADD(hi, lo);
    const double lgtail = TEMO_ADD(TEMO_ADD(hi, -lg), lo);

    // ---- y * log(x) in double-double
    const double ehi = TEMO_MUL(y, lg);
    const double elo = TEMO_FMA(y, lgtail, TEMO_FMA(lg, y, -ehi));

    // ---- exp_inline
    const unsigned abstop = (unsigned)(TEMO_AS_U64(ehi) >> 52) & 0x7ffu;
    bool special = false;
    if (abstop - 0x3c9u > 0x3eu) {
        if (abstop < 0x3c9u) {  // |y log x| < 2^-54: the result rounds from 1 + ehi
            *out = TEMO_ADD(ehi, 1.0);
            return true;
        }
        if (NARROW) return false;
        if (abstop > 0x408u) {  // |y log x| >= 1024: certain under/overflow (round to nearest)
            *out = (TEMO_AS_U64(ehi) >> 63) ? 0.0 : TEMO_AS_DOUBLE(0x7ff0000000000000ULL);
            return true;
        }
        special = true;  // 512 <= |y log x| < 1024: the scale may leave the normal range
    }
    const double invln2N = TEMO_POW_K(9), shift = TEMO_POW_K(10), negln2hiN = TEMO_POW_K(11),
                 negln2loN = TEMO_POW_K(12), C2 = TEMO_POW_K(13), C3 = TEMO_POW_K(14), C4 = TEMO_POW_K(15),
                 C5 = TEMO_POW_K(16);
    const double kds = TEMO_FMA(ehi, invln2N, shift);
    const unsigned long long ki = TEMO_AS_U64(kds);
    const double kdd = TEMO_ADD(kds, -shift);
    double rr = TEMO_FMA(kdd, negln2hiN, ehi);
    rr = TEMO_FMA(kdd, negln2loN, rr);
    rr = TEMO_ADD(elo, rr);
    const unsigned idx = 2u * (unsigned)(ki & 127);
    const unsigned long long sbits = T.exptab[idx + 1] + (ki << 45);
    const double tail = TEMO_AS_DOUBLE(T.exptab[idx]);
    const double c23 = TEMO_FMA(rr, C3, C2);
    const double tr = TEMO_ADD(rr, tail);
    const double r2 = TEMO_MUL(rr, rr);
    const double c45 = TEMO_FMA(rr, C5, C4);
    const double acc = TEMO_FMA(c23, r2, tr);
    const double r4 = TEMO_MUL(r2, r2);
    const double tmpv = TEMO_FMA(c45, r4, acc);
    if (!NARROW && special) {
        if ((ki & 0x80000000ULL) == 0) {  // k > 0: scale overflowed by <= 460 binades
            const double sc = TEMO_AS_DOUBLE(sbits - (1009ULL << 52));
            *out = TEMO_MUL(TEMO_FMA(sc, tmpv, sc), TEMO_AS_DOUBLE(0x7f00000000000000ULL));  // * 2^1009
            return true;
        }
        // k < 0: round once at the final (possibly subnormal) precision
        const unsigned long long sb = sbits + (1022ULL << 52);
        const double sc = TEMO_AS_DOUBLE(sb);
        const double st = TEMO_MUL(sc, tmpv);
        double yv = TEMO_ADD(sc, st);
        const double ay = yv < 0.0 ? -yv : yv;
        if (ay < 1.0) {
            const double one = yv < 0.0 ? -1.0 : 1.0;
            const double l0 = TEMO_ADD(TEMO_ADD(sc, -yv), st);
            const double h0 = TEMO_ADD(yv, one);
            double l1 = TEMO_ADD(TEMO_ADD(one, -h0), yv);
            l1 = TEMO_ADD(l1, l0);
            yv = TEMO_ADD(TEMO_ADD(l1, h0), -one);
            if (yv == 0.0) yv = TEMO_AS_DOUBLE(sb & 0x8000000000000000ULL);
        }
        *out = TEMO_MUL(yv, TEMO_AS_DOUBLE(0x0010000000000000ULL));  // * 2^-1022
        return true;
    }
    const double scale = TEMO_AS_DOUBLE(sbits);
    *out = TEMO_FMA(tmpv, scale, scale);
    return true;
}

// Branch-free form of the NARROW path for callers that evaluate several independent powers at once (the
// instruction streams interleave). Same operations, same bits; returns false when the result is not valid
// (|y log x| >= 512: never for the SBX spread factor) and the caller must fall back to the general routine.
// x must be positive and normal.
// STRICT: the |y log x| < 2^-54 case is reported as not valid as well (the caller's general routine handles it), which
// drops its add and select from the instruction stream.
template <bool STRICT = false>
__host__ __device__ __forceinline__ bool glibc_pow_narrow_flat(double x, double y, const PowTables& T, double* out) {
    const unsigned long long ix = TEMO_AS_U64(x);
    const unsigned long long tmp = ix - 0x3fe6955500000000ULL;
    const int i = (int)((tmp >> 45) & 127);
    const int k = (int)((long long)tmp >> 52);
    const double z = TEMO_AS_DOUBLE(ix - (tmp & 0xfff0000000000000ULL));
    const double kd = (double)k;
    const double ln2hi = TEMO_POW_K(0), ln2lo = TEMO_POW_K(1);
    const double A0 = TEMO_POW_K(2), A1 = TEMO_POW_K(3), A2 = TEMO_POW_K(4), A3 = TEMO_POW_K(5), A4 = TEMO_POW_K(6),
                 A5 = TEMO_POW_K(7), A6 = TEMO_POW_K(8);
    const double t1 = TEMO_FMA(kd, ln2hi, T.logc[i]);
    const double lo1 = TEMO_FMA(kd, ln2lo, T.logctail[i]);
    const double r = TEMO_FMA(z, T.invc[i], -1.0);
    const double ar = TEMO_MUL(r, A0);
    const double p12 = TEMO_FMA(r, A2, A1);
    const double p34 = TEMO_FMA(r, A4, A3);
    const double t2 = TEMO_ADD(r, t1);
    const double lo2 = TEMO_ADD(TEMO_ADD(t1, -t2), r);
    const double ar2 = TEMO_MUL(r, ar);
    const double ar3 = TEMO_MUL(r, ar2);
    const double lo3 = TEMO_FMA(ar, r, -ar2);
    const double hi = TEMO_ADD(t2, ar2);
    const double p56 = TEMO_FMA(r, A6, A5);
    const double lo4 = TEMO_ADD(TEMO_ADD(t2, -hi), ar2);
    const double q = TEMO_FMA(ar2, TEMO_FMA(p56, ar2, p34), p12);
    double lo = TEMO_ADD(lo1, lo2);
    lo = TEMO_ADD(lo, lo3);
    lo = TEMO_ADD(lo, lo4);
    lo = TEMO_FMA(ar3, q, lo);
    const double lg = TEMO_ADD(hi, lo);
    const double lgtail = TEMO_ADD(TEMO_ADD(hi, -lg), lo);
    const double ehi = TEMO_MUL(y, lg);
    const double elo = TEMO_FMA(y, lgtail, TEMO_FMA(lg, y, -ehi));
    const unsigned abstop = (unsigned)(TEMO_AS_U64(ehi) >> 52) & 0x7ffu;
    const bool tiny = abstop < 0x3c9u;              // |y log x| < 2^-54: the result rounds from 1 + ehi
    const bool valid = tiny || abstop - 0x3c9u <= 0x3eu;
    const double invln2N = TEMO_POW_K(9), shift = TEMO_POW_K(10), negln2hiN = TEMO_POW_K(11),
                 negln2loN = TEMO_POW_K(12), C2 = TEMO_POW_K(13), C3 = TEMO_POW_K(14), C4 = TEMO_POW_K(15),
                 C5 = TEMO_POW_K(16);
    const double kds = TEMO_FMA(ehi, invln2N, shift);
    const unsigned long long ki = TEMO_AS_U64(kds);
    const double kdd = TEMO_ADD(kds, -shift);
    double rr = TEMO_FMA(kdd, negln2hiN, ehi);
    rr = TEMO_FMA(kdd, negln2loN, rr);
    rr = TEMO_ADD(elo, rr);
    const unsigned idx = 2u * (unsigned)(ki & 127);
    const unsigned long long sbits = T.exptab[idx + 1] + (ki << 45);
    const double tail = TEMO_AS_DOUBLE(T.exptab[idx]);
    const double c23 = TEMO_FMA(rr, C3, C2);
    const double tr = TEMO_ADD(rr, tail);
    const double r2 = TEMO_MUL(rr, rr);
    const double c45 = TEMO_FMA(rr, C5, C4);
    const double acc = TEMO_FMA(c23, r2, tr);
    const double r4 = TEMO_MUL(r2, r2);
    const double tmpv = TEMO_FMA(c45, r4, acc);
    const double scale = TEMO_AS_DOUBLE(sbits);
    const double res = TEMO_FMA(tmpv, scale, scale);
    if (STRICT) {
        *out = res;
        return abstop - 0x3c9u <= 0x3eu;
    }
    *out = tiny ? TEMO_ADD(ehi, 1.0) : res;
    return valid;
}

// Host twin (used by the C-ABI self-test hook): tables straight from the generated header.
inline double glibc_pow_host(double x, double y) {
    static const unsigned long long invc[128] = TEMO_POW_INVC_INIT;
    static const unsigned long long logc[128] = TEMO_POW_LOGC_INIT;
    static const unsigned long long logctail[128] = TEMO_POW_LOGCTAIL_INIT;
    static const unsigned long long exptab[256] = TEMO_POW_EXPTAB_INIT;
    static const PowTables T{reinterpret_cast<const double*>(invc), reinterpret_cast<const double*>(logc),
                             reinterpret_cast<const double*>(logctail), exptab};
    double out;
    if (glibc_pow_main<false>(x, y, T, &out)) return out;
    return std::pow(x, y);
}

}  // namespace temo_b200
