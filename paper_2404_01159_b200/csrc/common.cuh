// Shared device/host helpers for the temo_b200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace temo_b200 {

constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs
constexpr double kPi = 3.141592653589793238462643383279502884;

// ---- errors ---------------------------------------------------------------------------
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

// reference: detail::require (tensor.hpp:63-65)
inline void require(bool cond, const char* msg) {
    if (!cond) fail(1 /*EINVAL*/, msg);
}

#define TEMO_CUDA(expr)                                                                      \
    do {                                                                                     \
        cudaError_t err__ = (expr);                                                          \
        if (err__ != cudaSuccess)                                                            \
            ::temo_b200::fail(2, std::string(#expr) + ": " + cudaGetErrorString(err__));     \
    } while (0)

// ---- counter-based randomness -----------------------------------------------------------
// reference: rng.hpp:23-43. word(seed,k) = mix64(mix64(seed) + k*GOLDEN); uniform = top 53 bits.
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// High 32 bits of mix64(z) before the final xor-shift. Enough for every test that only looks at the top
// bits of the word — w = y ^ (y >> 31) leaves the top 31 bits of y untouched — and one multiply-add
// shorter than the full mix: the sign tests H(r - 0.5) (bit 63) and the quick reject of the mutation mask.
__host__ __device__ __forceinline__ uint32_t mix64_top32(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27;
    const uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
#ifdef __CUDA_ARCH__
    return __umulhi(lo, 0x133111ebu) + lo * 0x94d049bbu + hi * 0x133111ebu;
#else
    return (uint32_t)((z * 0x94d049bb133111ebULL) >> 32);
#endif
}

// Philox4x32-10 (Salmon et al. 2011), counter = (k >> 1, stream tag), key = seed; one call
// yields two 64-bit words, word (k & 1) is draw k. Not in the reference: parity unpinned.
__host__ __device__ __forceinline__ uint64_t philox_word(uint64_t seed, uint64_t k) {
    uint32_t c0 = (uint32_t)(k >> 1), c1 = (uint32_t)(k >> 33), c2 = 0x74656d6fu, c3 = 0x62323030u;
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return (k & 1) ? (((uint64_t)c3 << 32) | c2) : (((uint64_t)c1 << 32) | c0);
}

// RNG policy object passed by value into kernels. `base` is mix64(seed) for SplitMix64.
struct Rng {
    uint64_t seed;
    uint64_t base;
    int mode;  // 0 SplitMix64 (reference), 1 Philox4x32-10
};

inline Rng make_rng(uint64_t seed, int mode) { return Rng{seed, mix64(seed), mode}; }

template <int MODE>
__host__ __device__ __forceinline__ uint64_t draw_word(const Rng& g, uint64_t k) {
    if (MODE == 0) return mix64(g.base + k * kGolden);
    return philox_word(g.seed, k);
}

// Exact (double)(w >> 11) * 2^-53 without an integer->double conversion: the low 32 and the
// high 21 bits of the 53-bit integer are planted into the mantissas of 0.5 and 2^31 (whose
// ulps are 2^-53 and 2^-21); removing the offsets leaves lo*2^-53 and hi*2^-21, and their
// sum has at most 53 significant bits, so every step is exact.
__host__ __device__ __forceinline__ double word_to_unit(uint64_t w) {
#ifdef __CUDA_ARCH__
    const uint32_t w_hi = (uint32_t)(w >> 32), w_lo = (uint32_t)w;
    const uint32_t u_hi = w_hi >> 11;                     // top 21 of the 53 bits
    const uint32_t u_lo = (w_hi << 21) | (w_lo >> 11);    // low 32 of the 53 bits
    const double lo = __hiloint2double(0x3FE00000, (int)u_lo) - 0.5;
    const double hi = __hiloint2double(0x41E00000, (int)u_hi) - 2147483648.0;
    return hi + lo;
#else
    return (double)(w >> 11) * 0x1.0p-53;
#endif
}

// ---- scalar conventions (tensor.hpp:73-87) ------------------------------------------------
__host__ __device__ __forceinline__ double clampd(double x, double lo, double hi) {
    return x < lo ? lo : (x > hi ? hi : x);
}

// ---- block reductions with a fixed (launch-shape independent of the GPU count) order -------
// Canonical row mapping of every kernel that sums over a row (standalone and fused evaluation): the row is cut into
// blocks of 32 vectors (one per lane), warp w of the row's nw warps owns the cblk = ceil(blocks / nw) consecutive blocks
// [w * cblk, (w + 1) * cblk), and a lane adds the terms of its vectors in ascending order. (Consecutive blocks, not
// interleaved ones: a warp then streams one contiguous piece of the row, which is what lets a single warp of the pair
// kernel of reproduce.cu walk a whole row.) Then block_sum's tree: xor butterfly in the warp, warp totals ascending.
__host__ __device__ __forceinline__ uint32_t canon_chunk_blocks(uint32_t blocks, uint32_t nw) { return (blocks + nw - 1) / nw; }

// Sum over the block in a canonical tree: xor-shuffle butterfly inside each warp, then the
// warp totals are added in ascending warp order by every thread (all threads get the result).
template <int MAXW>
__device__ __forceinline__ double block_sum(double v, double* smem /* MAXW doubles */) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) smem[warp] = v;
    __syncthreads();
    double s = smem[0];
    for (int w = 1; w < nw; ++w) s += smem[w];
    return s;
}

}  // namespace temo_b200
