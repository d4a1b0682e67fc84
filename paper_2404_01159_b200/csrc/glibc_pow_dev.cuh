// Device-side tables and wrappers for glibc_pow.cuh.
#pragma once

#include "glibc_pow.cuh"

namespace temo_b200 {

static __device__ const unsigned long long d_pow_invc[128] = TEMO_POW_INVC_INIT;
static __device__ const unsigned long long d_pow_logc[128] = TEMO_POW_LOGC_INIT;
static __device__ const unsigned long long d_pow_logctail[128] = TEMO_POW_LOGCTAIL_INIT;
static __device__ const unsigned long long d_pow_exptab[256] = TEMO_POW_EXPTAB_INIT;

// Shared-memory copy of the tables (5 KB): the lookups are lane-divergent, which shared memory
// serves at a few cycles per warp while constant memory would serialise them.
struct PowSmem {
    double invc[128];
    double logc[128];
    double logctail[128];
    unsigned long long exptab[256];
};

__device__ __forceinline__ void pow_smem_load(PowSmem& s) {
    for (int i = threadIdx.x; i < 128; i += blockDim.x) {
        s.invc[i] = __longlong_as_double((long long)d_pow_invc[i]);
        s.logc[i] = __longlong_as_double((long long)d_pow_logc[i]);
        s.logctail[i] = __longlong_as_double((long long)d_pow_logctail[i]);
    }
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s.exptab[i] = d_pow_exptab[i];
}

__device__ __forceinline__ PowTables pow_tables(const PowSmem& s) {
    return PowTables{s.invc, s.logc, s.logctail, s.exptab};
}

__device__ __forceinline__ PowTables pow_tables_global() {
    return PowTables{reinterpret_cast<const double*>(d_pow_invc), reinterpret_cast<const double*>(d_pow_logc),
                     reinterpret_cast<const double*>(d_pow_logctail), d_pow_exptab};
}

// pow with the host libm's bits on the main path, CUDA's pow elsewhere (x == 0, under/overflow).
__device__ __forceinline__ double pow_like_host(double x, double y, const PowTables& T) {
    double out;
    if (glibc_pow_main<false>(x, y, T, &out)) return out;
    return pow(x, y);
}

// Same bits, for callers that guarantee a positive normal x, an ordinary y and |y log x| < 512.
__device__ __forceinline__ double pow_like_host_narrow(double x, double y, const PowTables& T) {
    double out;
    if (glibc_pow_main<true>(x, y, T, &out)) return out;
    return pow_like_host(x, y, T);
}

}  // namespace temo_b200
