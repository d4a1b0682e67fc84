// K3 — APD environmental selection.
//
// reference: rv_select (selection.hpp:200-224) = detail::rv_core (selection.hpp:148-192:
// ideal-point translation, row norms, first-max-cosine association over the R reference
// vectors, one acos per row, angle-penalised distance) followed by the serial per-vector
// argmin with lowest-row tie-break (selection.hpp:206-217).
//
// Bit-exactness (compiled with --fmad=false): dot products
// accumulate in ascending k, the cosine is dot / (nf * vn[j]) with IEEE divide, strict `>`
// keeps the lowest j among equal cosines, and the elite of each vector is the lexicographic
// minimum of (apd, row) — implemented order-independently with two rounds of 64-bit/32-bit
// atomicMin, plus the reference's NaN rule (a NaN APD is never an improvement, but the first
// row of a subpopulation is taken unconditionally).
#include "compact.cuh"
#include "internal.h"
#include "vecindex.h"

namespace temo_b200 {

namespace {

// Total-order key of a double: monotone for all non-NaN values.
__device__ __forceinline__ unsigned long long order_key(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double key_value(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k;
    return __longlong_as_double((long long)b);
}
constexpr unsigned long long kKeyMax = 0xffffffffffffffffULL;

// ---- ideal point: column minima (tensor.hpp:211-219) --------------------------------------------
// grid (blocks, m): block-strided rows of one column; NaNs never win (strict <). The last CTA to finish decodes the keys
// (a NaN in row 0 sticks: the reference seeds the scan with row 0 and a NaN never compares smaller / greater) and clears
// the ticket. Scratch layout: m minimum keys, m maximum keys, one ticket word (col_minmax_scratch_words).
__global__ void colmin_kernel(const double* f, uint64_t n_rows, const uint32_t* n_rows_dev, uint64_t m,
                              unsigned long long* zkey_min, unsigned long long* zkey_max, unsigned long long* ticket,
                              bool want_max, double* zmin, double* zmax) {
    const uint64_t n = n_rows_dev ? (uint64_t)*n_rows_dev : n_rows;
    const uint64_t j = blockIdx.y;
    unsigned long long kmin = kKeyMax, kmax = 0ULL;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double v = f[i * m + j];
        if (v == v) {
            const unsigned long long k = order_key(v);
            kmin = k < kmin ? k : kmin;
            kmax = k > kmax ? k : kmax;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o1 = __shfl_xor_sync(0xffffffffu, kmin, off);
        const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, kmax, off);
        kmin = o1 < kmin ? o1 : kmin;
        kmax = o2 > kmax ? o2 : kmax;
    }
    if ((threadIdx.x & 31) == 0) {
        if (kmin != kKeyMax) atomicMin(&zkey_min[j], kmin);
        if (want_max && kmax != 0ULL) atomicMax(&zkey_max[j], kmax);
    }
    __shared__ bool s_last;
    __syncthreads();  // this CTA's atomics are issued
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(ticket, 1ULL) == (unsigned long long)gridDim.x * gridDim.y - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x < m) {
        const uint64_t c = threadIdx.x;
        const double first = f[c];
        if (zmin) zmin[c] = (first != first) ? first : key_value(*reinterpret_cast<volatile unsigned long long*>(&zkey_min[c]));
        if (zmax) zmax[c] = (first != first) ? first : key_value(*reinterpret_cast<volatile unsigned long long*>(&zkey_max[c]));
        zkey_min[c] = kKeyMax;  // the scratch is left as it was found: no reset launch (or memset) per call
        zkey_max[c] = 0ULL;
    }
    if (threadIdx.x == 0) *ticket = 0ULL;
}

// Start of a selection in one launch: gamma > 0 (selection.hpp:152), the per-vector minima reset, the column-key scratch reset.
__global__ void select_init_kernel(const double* gamma, uint64_t r, uint64_t m, uint32_t* err_flag, unsigned long long* best_key,
                                   uint32_t* best_row, uint32_t* first_row, unsigned long long* zkey) {
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j < r) {
        if (!(gamma[j] > 0.0)) atomicOr(err_flag, 1u);
        best_key[j] = kKeyMax;
        best_row[j] = 0xffffffffu;
        first_row[j] = 0xffffffffu;
    }
    if (j < m) {
        zkey[j] = kKeyMax;
        zkey[m + j] = 0ULL;
    }
    if (j == 0) zkey[2 * m] = 0ULL;
}

__global__ void row_norms_kernel(const double* v, uint64_t r, uint64_t m, double* vn) {
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j >= r) return;
    double s = 0.0;
    for (uint64_t k = 0; k < m; ++k) s += v[j * m + k] * v[j * m + k];  // tensor.hpp:171-182
    vn[j] = sqrt(s);
}


// ---- association + APD ------------------------------------------------------------------------------
constexpr int kAssocThreads = 128;
constexpr int kTileVecs = 512;

template <int M>
__global__ void __launch_bounds__(kAssocThreads) assoc_kernel(
    const double* __restrict__ f, uint64_t n_rows, const uint32_t* n_rows_dev, uint64_t m_rt,
    const double* __restrict__ z, const double* __restrict__ v, const double* __restrict__ vn,
    const double* __restrict__ gamma, uint64_t r, double penalty, uint32_t* __restrict__ assoc,
    double* __restrict__ theta_out, double* __restrict__ apd_out,
    unsigned long long* __restrict__ best_key, uint32_t* __restrict__ first_row) {
    constexpr int MM = M > 0 ? M : kMaxObj;
    const int m = M > 0 ? M : (int)m_rt;
    extern __shared__ double s_tile[];  // kTileVecs x (m + 1): v_j[0..m-1], vn_j
    const uint64_t n = n_rows_dev ? (uint64_t)*n_rows_dev : n_rows;
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const bool live = i < n;

    double fp[MM];
    double nf = 0.0;
    if (live) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < MM; ++k) {
            if (k < m) {
                fp[k] = f[i * m + k] - z[k];  // selection.hpp:155-157
                s += fp[k] * fp[k];
            }
        }
        nf = sqrt(s);
    }
    double best_cos = -INFINITY;
    uint32_t arg = 0;
    const int stride = m + 1;
    for (uint64_t j0 = 0; j0 < r; j0 += kTileVecs) {
        const int tile = (int)((r - j0) < (uint64_t)kTileVecs ? (r - j0) : kTileVecs);
        __syncthreads();
        for (int e = threadIdx.x; e < tile * stride; e += blockDim.x) {
            const int jj = e / stride, k = e - jj * stride;
            s_tile[e] = k < m ? v[(j0 + jj) * m + k] : vn[j0 + jj];
        }
        __syncthreads();
        if (live && nf != 0.0) {
            for (int jj = 0; jj < tile; ++jj) {
                const double* vr = s_tile + jj * stride;
                double dot = 0.0;
#pragma unroll
                for (int k = 0; k < MM; ++k)
                    if (k < m) dot += fp[k] * vr[k];
                const double c = dot / (nf * vr[m]);  // selection.hpp:178
                if (c > best_cos) {
                    best_cos = c;
                    arg = (uint32_t)(j0 + jj);
                }
            }
        }
    }
    if (!live) return;
    double theta = 0.0;  // a row at the ideal point: angle 0 to vector 0 (selection.hpp:167-169)
    if (nf != 0.0) {
        double c = best_cos;
        if (c > 1.0) c = 1.0;
        if (c < -1.0) c = -1.0;
        theta = acos(c);  // tensor.hpp:79-83
    }
    const double apd = (1.0 + penalty * (theta / gamma[arg])) * nf;  // selection.hpp:82-84
    assoc[i] = arg;
    theta_out[i] = theta;
    apd_out[i] = apd;
    const unsigned long long key = (apd != apd) ? kKeyMax : order_key(apd);
    atomicMin(&best_key[arg], key);
    atomicMin(&first_row[arg], (uint32_t)i);
}

// ---- exact association through a single-precision filter (many objectives) ---------------------------------------
// For m >= 5 the direction index prunes little (in 10 dimensions every patch of the lattice is wide) and the exact scan
// costs (rows x R) double-precision dots WITHOUT fused multiply-adds plus a divide per pair: 12 ms at BASELINE config #4
// (131072 rows x 48620 vectors x 10), which is the FP64 pipe's peak. Here every pair is first scored in fp32
// (cos32 = (u/|u|) . (v/|v|) with FFMA: 6.4e10 of them at config #4 = 1.7 ms at the FP32 peak); only a pair whose fp32
// score is within kFilterTol of the row's running fp32 maximum is re-evaluated with the reference's exact fp64 expression
// (selection.hpp:172-184), in ascending j with a strict >, so the result is the reference's first strict maximum.
// Why this is exact: for non-negative u and v all terms of the dot product are non-negative, so the fp32 score has
// relative error <= (m + 2) 2^-24 < 2.1e-6 (m <= 32: one rounding per input, one per FFMA); the running maximum never
// exceeds the final one, hence every j whose exact cosine could reach the final exact maximum satisfies
// cos32_j >= max32 (1 - 2 * 2.1e-6) > running32 (1 - kFilterTol) and is evaluated exactly. Rows or vector sets with a
// negative, non-finite or fp32-unrepresentable component take the exact expression for every j (threshold -inf).
// Shape of the scan (round 2): a thread keeps kFilterRows = 4 unit rows in registers and scores them against two vectors
// per step (eight independent FFMA chains, the vectors read once per step as 128-bit shared-memory broadcasts); the
// vectors are stored pre-normalised so that the score needs no scaling; the exact expression lives out of line and
// reloads its operands (it runs for a few dozen of the 48620 vectors of a row). With SELF the rows are the vectors
// themselves and j == row is skipped: the same scan gives gamma's max off-diagonal cosine (refvec.hpp:81-100).
constexpr float kFilterTol = 1e-5f;
constexpr float kFltMin = 1.17549435e-38f;
constexpr int kFilterTile = 512;      // vectors per shared-memory tile
constexpr int kFilterMaxChunks = 8;   // pieces the vector range is cut into (per-row winners merged afterwards)
constexpr int kFilterThreads = 128;
constexpr int kFilterRows = 4;        // rows per thread: 512 rows per CTA
#ifndef TEMO_FILTER_VECS
#define TEMO_FILTER_VECS 4
#endif
constexpr int kFilterVecs = TEMO_FILTER_VECS;  // vectors per step: kFilterRows x kFilterVecs independent FFMA chains per thread

// fp32 copy of the unit vectors: row j = v_j / |v_j| padded with zeros to a multiple of four floats (128-bit reads)
__host__ __device__ inline uint64_t v32_stride(uint64_t m) { return (m + 3) / 4 * 4; }

__global__ void v32_kernel(const double* __restrict__ v, const double* __restrict__ vn, uint64_t r, uint64_t m, float* __restrict__ v32,
                           uint32_t* __restrict__ flags) {
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j >= r) return;
    const uint64_t stride = v32_stride(m);
    const double nrm = vn[j];
    bool bad = !(nrm > 0.0) || !(nrm < INFINITY);
    for (uint64_t k = 0; k < m; ++k) {
        const double x = v[j * m + k];
        const double q = x / nrm;
        const float q32 = (float)q;
        v32[j * stride + k] = q32;
        if (!(x >= 0.0) || !(x < INFINITY)) bad = true;
        // outside fp32's normal range the relative-error bound of the filter does not hold (flushed or infinite terms)
        if (x != 0.0 && !(q32 >= kFltMin && q32 < INFINITY)) bad = true;
    }
    for (uint64_t k = m; k < stride; ++k) v32[j * stride + k] = 0.0f;
    if (bad) atomicOr(flags, 1u);
}

// the reference's expression for one (row, vector) pair (selection.hpp:172-178 / refvec.hpp:89-92): ascending-k dot of the
// translated row with v_j, divided by the product of the norms
__device__ __noinline__ double exact_cosine(const double* __restrict__ frow, const double* __restrict__ z, const double* __restrict__ vj,
                                            double nf, double vnj, int m) {
    double dot = 0.0;
    for (int k = 0; k < m; ++k) dot += (z ? frow[k] - z[k] : frow[k]) * vj[k];
    return dot / (nf * vnj);
}

// packed fp32 pairs (sm_100: FFMA2)
__device__ __forceinline__ uint64_t pack2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ float sum2(uint64_t a) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a));
    return x + y;
}

// Seed of the running threshold: the best fp32 score of a row over every kFilterSeedStep-th vector (6 % of the scan's
// work). Any real score is a lower bound of the final maximum, so starting from it is as exact as starting from zero,
// and with it only the handful of vectors that beat the subsample's best ever become candidates (a scan that starts
// from zero sees a new running maximum ~ln(R) times per chunk: 38 % of the warp steps took the candidate branch).
constexpr int kFilterSeedStep = 16;

constexpr int kSeedRows = 2;  // rows per thread of the seed scan: twice the CTAs of the main scan (it has no chunks)

template <int M, bool SELF>
__global__ void __launch_bounds__(kFilterThreads) filter_seed_kernel(const double* __restrict__ f, uint64_t n_rows, uint64_t m_rt,
                                                                     const double* __restrict__ z, const double* __restrict__ vn,
                                                                     const float* __restrict__ v32, uint64_t r, float* __restrict__ seed,
                                                                     const uint32_t* skip_flag) {
    if (skip_flag && *skip_flag) return;
    constexpr int MM = M > 0 ? M : kMaxObj;
    constexpr int R = kSeedRows;
    const int m = M > 0 ? M : (int)m_rt;
    constexpr int SS = (MM + 3) / 4 * 4;
    const int stride = M > 0 ? SS : (int)v32_stride(m);
    extern __shared__ __align__(16) float s_v32[];  // kFilterTile subsampled unit vectors
    constexpr int KP = (MM + 1) / 2;  // component pairs
    uint32_t row[R];
    float uf[R][MM], best[R];
    uint64_t uf2[R][KP];
#pragma unroll
    for (int t = 0; t < R; ++t) {
        row[t] = (uint32_t)(blockIdx.x * (uint64_t)(R * kFilterThreads) + t * kFilterThreads + threadIdx.x);
        const bool live = row[t] < n_rows;
        double fp[MM], s = 0.0;
#pragma unroll
        for (int k = 0; k < MM; ++k)
            if (k < m) {
                fp[k] = !live ? 0.0 : (SELF ? f[(uint64_t)row[t] * m + k] : f[(uint64_t)row[t] * m + k] - z[k]);
                s += fp[k] * fp[k];
            }
        const double nf = !live ? 0.0 : (SELF ? vn[row[t]] : sqrt(s));
#pragma unroll
        for (int k = 0; k < MM; ++k) uf[t][k] = (float)((k < m && nf != 0.0) ? fp[k] / nf : 0.0);  // the scan's own conversion
#pragma unroll
        for (int p = 0; p < KP; ++p) uf2[t][p] = pack2(uf[t][2 * p], 2 * p + 1 < MM ? uf[t][2 * p + 1 < MM ? 2 * p + 1 : 0] : 0.0f);
        best[t] = 0.0f;
    }
    const uint64_t n_sub = (r + kFilterSeedStep - 1) / kFilterSeedStep;  // vectors 0, 16, 32, ...
    for (uint64_t q0 = 0; q0 < n_sub; q0 += kFilterTile) {
        const int tile = (int)((n_sub - q0) < (uint64_t)kFilterTile ? (n_sub - q0) : kFilterTile);
        __syncthreads();
        for (int e = threadIdx.x; e < tile * stride / 4; e += blockDim.x) {
            const int jj = e / (stride / 4), part = e - jj * (stride / 4);
            reinterpret_cast<float4*>(s_v32)[e] = __ldg(reinterpret_cast<const float4*>(v32 + (q0 + jj) * kFilterSeedStep * stride) + part);
        }
        __syncthreads();
#pragma unroll 2
        for (int jj = 0; jj < tile; ++jj) {
            // packed multiply-adds, component pairs side by side (like the scan)
            const ulonglong2* p2 = reinterpret_cast<const ulonglong2*>(s_v32 + jj * stride);
            uint64_t vp[KP];
#pragma unroll
            for (int k4 = 0; k4 < SS / 4; ++k4)
                if (4 * k4 < m) {
                    const ulonglong2 t2 = p2[k4];
                    vp[2 * k4] = t2.x;
                    if (2 * k4 + 1 < KP) vp[2 * k4 + 1 < KP ? 2 * k4 + 1 : 0] = t2.y;
                }
            uint64_t acc[R];
#pragma unroll
            for (int t = 0; t < R; ++t) acc[t] = 0ull;
#pragma unroll
            for (int p = 0; p < KP; ++p)
                if (2 * p < m) {
#pragma unroll
                    for (int t = 0; t < R; ++t) acc[t] = ffma2(uf2[t][p], vp[p], acc[t]);
                }
            float sc[R];
#pragma unroll
            for (int t = 0; t < R; ++t) sc[t] = sum2(acc[t]);
            const uint32_t j = (uint32_t)((q0 + jj) * kFilterSeedStep);
#pragma unroll
            for (int t = 0; t < R; ++t)
                if (!(SELF && j == row[t])) best[t] = fmaxf(best[t], sc[t]);  // a NaN score (bad vector set: filter off) is ignored
        }
    }
#pragma unroll
    for (int t = 0; t < R; ++t)
        if (row[t] < n_rows) seed[row[t]] = best[t];
}

// Candidates of a row: vectors whose fp32 score reached the row's running threshold. Their exact evaluation is deferred
// to the end of the scan - the threshold only depends on the fp32 scores - when most of them have fallen below the final
// threshold and are dropped: a few exact evaluations per row remain instead of one per running-maximum record.
constexpr int kFilterCand = 6;  // candidate slots per row (pruned against the risen threshold when full)
constexpr int kFallbackItems = 8192;  // (row, vector range) items the fallback spreads its rows over (when there are fewer rows)

template <int M, bool SELF>
__global__ void __launch_bounds__(kFilterThreads, 4) assoc_filter_kernel(
    const double* __restrict__ f, uint64_t n_rows, uint64_t m_rt, const double* __restrict__ z, const double* __restrict__ v,
    const double* __restrict__ vn, const float* __restrict__ v32, const uint32_t* __restrict__ vflags, uint64_t r, uint64_t chunk_vecs,
    double* __restrict__ part_c, uint32_t* __restrict__ part_j, uint32_t* __restrict__ row_flag, uint32_t* __restrict__ flag_list,
    uint32_t* __restrict__ flag_count, const float* __restrict__ seed, const uint32_t* skip_flag) {
    // blockIdx.y = chunk of the vector range [y * chunk_vecs, (y + 1) * chunk_vecs): the per-row winners of the chunks are
    // merged in ascending chunk order afterwards (strict >: the first strict maximum overall)
    if (skip_flag && *skip_flag) return;
    constexpr int MM = M > 0 ? M : kMaxObj;
    constexpr int R = kFilterRows, CAP = kFilterCand, V = kFilterVecs;
    const int m = M > 0 ? M : (int)m_rt;
    extern __shared__ __align__(16) float s_v32[];  // (kFilterTile + V) x stride unit vectors in fp32, then the candidate slots
    constexpr int SS = (MM + 3) / 4 * 4;  // compile-time stride when M is known
    const int stride = M > 0 ? SS : (int)v32_stride(m);
    // candidate slot e of this thread's row t: index (t * CAP + e) * blockDim + tid (conflict-free)
    uint32_t* cand_j = reinterpret_cast<uint32_t*>(s_v32 + (kFilterTile + V) * stride);
    float* cand_s = reinterpret_cast<float*>(cand_j + R * CAP * kFilterThreads);
    const bool v_ok = (*vflags & 1u) == 0;
    constexpr int KP = (MM + 1) / 2;  // component pairs
    uint32_t row[R], cnt[R];
    float uf[R][MM], best32[R], thr[R];
    uint64_t uf2[R][KP];
    bool overflow[R], exact_only[R];
#pragma unroll
    for (int t = 0; t < R; ++t) {
        row[t] = (uint32_t)(blockIdx.x * (uint64_t)(R * kFilterThreads) + t * kFilterThreads + threadIdx.x);
        const bool live = row[t] < n_rows;
        cnt[t] = 0;
        overflow[t] = exact_only[t] = false;
        bool filter = v_ok && live;
        double fp[MM], nf = 0.0;
        if (live) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < MM; ++k)
                if (k < m) {
                    fp[k] = SELF ? f[(uint64_t)row[t] * m + k] : f[(uint64_t)row[t] * m + k] - z[k];  // selection.hpp:155-157
                    s += fp[k] * fp[k];
                    if (!(fp[k] >= 0.0)) filter = false;
                }
            nf = SELF ? vn[row[t]] : sqrt(s);  // refvec.hpp:84: the same row_norms the vectors' norms come from
            if (!(nf < INFINITY)) filter = false;  // inf or NaN
        }
#pragma unroll
        for (int k = 0; k < MM; ++k) {
            const double uk = (k < m && live && nf != 0.0) ? fp[k] / nf : 0.0;
            uf[t][k] = (float)uk;
            if (uk != 0.0 && !(uf[t][k] >= kFltMin)) filter = false;  // flushed component: no filter for this row
        }
#pragma unroll
        for (int p = 0; p < KP; ++p) uf2[t][p] = pack2(uf[t][2 * p], 2 * p + 1 < MM ? uf[t][2 * p + 1 < MM ? 2 * p + 1 : 0] : 0.0f);
        best32[t] = live ? seed[row[t]] : 0.0f;           // a real score of this row: a lower bound of its maximum
        thr[t] = best32[t] * (1.0f - kFilterTol);         // (0 when the subsample was empty: every score passes)
        if (!live || nf == 0.0) {
            thr[t] = INFINITY;  // nothing to do (selection.hpp:167-169: arg 0, theta 0)
        } else if (!filter) {   // the exact expression for every vector: filter_fallback_kernel
            thr[t] = INFINITY;
            overflow[t] = exact_only[t] = true;
        }
    }
    const uint64_t j_begin = blockIdx.y * chunk_vecs, j_end = j_begin + chunk_vecs < r ? j_begin + chunk_vecs : r;
    for (uint64_t j0 = j_begin; j0 < j_end; j0 += kFilterTile) {
        const int tile = (int)((j_end - j0) < (uint64_t)kFilterTile ? (j_end - j0) : kFilterTile);
        __syncthreads();
        {
            const float4* src = reinterpret_cast<const float4*>(v32 + j0 * stride);
            float4* dst = reinterpret_cast<float4*>(s_v32);
            for (int e = threadIdx.x; e < tile * stride / 4; e += blockDim.x) dst[e] = src[e];
            // a partial last step: its phantom vectors score zero
            if (threadIdx.x < (V - 1) * stride / 4) dst[tile * stride / 4 + threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncthreads();
#pragma unroll 1
        for (int jj = 0; jj < tile; jj += V) {
            // scores with the packed fp32 multiply-add (FFMA2: two lanes per instruction): components 2p and 2p + 1 of a
            // row / vector pair accumulate side by side and are added at the end - half the instructions of the scalar
            // form for the part of the kernel that is 3/4 of it. (Any summation order keeps the (m + 5) 2^-24 bound.)
            float sc[V][R];
#pragma unroll
            for (int u = 0; u < V; ++u) {
                const ulonglong2* p2 = reinterpret_cast<const ulonglong2*>(s_v32 + (jj + u) * stride);  // broadcast reads
                uint64_t vp[KP];
#pragma unroll
                for (int k4 = 0; k4 < SS / 4; ++k4)
                    if (4 * k4 < m) {
                        const ulonglong2 t2 = p2[k4];
                        vp[2 * k4] = t2.x;
                        if (2 * k4 + 1 < KP) vp[2 * k4 + 1 < KP ? 2 * k4 + 1 : 0] = t2.y;
                    }
                uint64_t acc[R];
#pragma unroll
                for (int t = 0; t < R; ++t) acc[t] = 0ull;
#pragma unroll
                for (int p = 0; p < KP; ++p)
                    if (2 * p < m) {
#pragma unroll
                        for (int t = 0; t < R; ++t) acc[t] = ffma2(uf2[t][p], vp[p], acc[t]);
                    }
#pragma unroll
                for (int t = 0; t < R; ++t) sc[u][t] = sum2(acc[t]);
            }
            bool any = false;
#pragma unroll
            for (int t = 0; t < R; ++t) {
                float mx = sc[0][t];
#pragma unroll
                for (int u = 1; u < V; ++u) mx = fmaxf(mx, sc[u][t]);
                any |= mx >= thr[t];
            }
            if (any) {  // a candidate: remember it, raise the threshold (ascending j)
#pragma unroll
                for (int u = 0; u < V; ++u) {
                    const uint32_t j = (uint32_t)(j0 + jj + u);
                    if (jj + u >= tile) continue;  // a phantom vector of the partial last step
#pragma unroll
                    for (int t = 0; t < R; ++t) {
                        const float s32 = sc[u][t];
                        if (!(s32 >= thr[t])) continue;
                        if (SELF && j == row[t]) continue;  // refvec.hpp:91
                        if (s32 > best32[t]) {
                            best32[t] = s32;
                            thr[t] = s32 * (1.0f - kFilterTol);
                        }
                        if (cnt[t] == CAP) {  // drop the candidates the threshold has left behind
                            uint32_t keep = 0;
                            for (uint32_t e = 0; e < CAP; ++e) {
                                const uint32_t at = (t * CAP + e) * kFilterThreads + threadIdx.x;
                                const float se = cand_s[at];
                                if (se >= thr[t]) {
                                    const uint32_t to = (t * CAP + keep) * kFilterThreads + threadIdx.x;
                                    cand_s[to] = se;
                                    cand_j[to] = cand_j[at];
                                    ++keep;
                                }
                            }
                            cnt[t] = keep;
                            if (keep == CAP) {  // more near-ties than slots: this row goes to the exact fallback
                                overflow[t] = true;
                                thr[t] = INFINITY;
                                continue;
                            }
                        }
                        const uint32_t at = (t * CAP + cnt[t]) * kFilterThreads + threadIdx.x;
                        cand_s[at] = s32;
                        cand_j[at] = j;
                        ++cnt[t];
                    }
                }
            }
        }
    }
    // the candidates that survive the final threshold, in ascending j, with the reference's exact expression
#pragma unroll
    for (int t = 0; t < R; ++t) {
        if (row[t] >= n_rows) continue;
        double best_c = -INFINITY;
        uint32_t arg = 0;
        if (overflow[t]) {
            // 2: a property of the row (every chunk says so); 1: more near-ties than slots. The first chunk to flag a row
            // appends it to the fallback's list.
            if (atomicExch(&row_flag[row[t]], exact_only[t] ? 2u : 1u) == 0u) flag_list[atomicAdd(flag_count, 1u)] = row[t];
        } else if (cnt[t]) {
            const double nf = SELF ? vn[row[t]] : [&] {
                double s = 0.0;
                for (int k = 0; k < m; ++k) {
                    const double x = f[(uint64_t)row[t] * m + k] - z[k];
                    s += x * x;
                }
                return sqrt(s);
            }();
            for (uint32_t e = 0; e < cnt[t]; ++e) {
                const uint32_t at = (t * CAP + e) * kFilterThreads + threadIdx.x;
                if (!(cand_s[at] >= thr[t])) continue;
                const uint32_t j = cand_j[at];
                const double c = exact_cosine(f + (uint64_t)row[t] * m, SELF ? nullptr : z, v + (uint64_t)j * m, nf, vn[j], m);
                if (c > best_c) {
                    best_c = c;
                    arg = j;
                }
            }
        }
        part_c[blockIdx.y * n_rows + row[t]] = best_c;
        part_j[blockIdx.y * n_rows + row[t]] = arg;
    }
}

// Rows the scan gave up on (a handful per generation, but a single warp needs 0.8 ms for the 48620 vectors of config #4:
// the latency of one serial scan used to be a fifth of the selection). The flagged rows are compacted by the scan; every
// row is cut into S vector ranges (S = kFallbackItems / rows, at most 64) and a warp takes one (row, range) item at a time;
// filter_fallback_merge_kernel then reduces the S partial winners of a row into chunk slot 0 (the chunk merge keeps the
// first strict maximum).
//   flag 1, more near-ties than candidate slots (rows with several near-zero components see many vectors of almost the
//     same cosine): the same filter without slots - a lane walks its vectors in ascending j, scores them in fp32 and
//     evaluates the reference's expression at once for every vector within kFilterTol of its running fp32 maximum (seeded
//     like the scan's). The argument of the scan carries over: the vector that attains the exact maximum scores within
//     2 * 2.1e-6 of the fp32 maximum, hence above every lane's running threshold.
//   flag 2, rows the filter does not apply to (a negative / non-finite / fp32-unrepresentable component, a bad vector
//     set): the reference's expression for every vector.
// Lexicographic reduction (max cosine, lowest j) across lanes and ranges = the first strict maximum.
__device__ __forceinline__ uint32_t fallback_split(uint32_t rows) {
    const uint32_t s = rows ? (uint32_t)kFallbackItems / rows : 1u;
    return s < 1u ? 1u : (s > 64u ? 64u : s);
}

template <int M, bool SELF>
__global__ void __launch_bounds__(128) filter_fallback_kernel(
    const double* __restrict__ f, uint64_t m_rt, const double* __restrict__ z, const double* __restrict__ v,
    const double* __restrict__ vn, const float* __restrict__ v32, const float* __restrict__ seed, uint64_t r,
    const uint32_t* __restrict__ row_flag, const uint32_t* __restrict__ flag_list, const uint32_t* __restrict__ flag_count,
    double* __restrict__ fb_c, uint32_t* __restrict__ fb_j, const uint32_t* skip_flag) {
    if (skip_flag && *skip_flag) return;
    constexpr int MM = M > 0 ? M : kMaxObj;
    constexpr int SS = (MM + 3) / 4 * 4;
    const int m = M > 0 ? M : (int)m_rt;
    const int stride = M > 0 ? SS : (int)v32_stride(m);
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t count = *flag_count, S = fallback_split(count);
    const uint64_t items = (uint64_t)count * S, warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t len = (r + S - 1) / S;  // vectors per range
    for (uint64_t item = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; item < items; item += warps) {
        const uint64_t row = flag_list[item / S], j_begin = (item % S) * len, j_end = j_begin + len < r ? j_begin + len : r;
        const unsigned flag = row_flag[row];
        double nf;
        if (SELF) {
            nf = vn[row];
        } else {
            double s = 0.0;
            for (int k = 0; k < m; ++k) {
                const double x = f[row * m + k] - z[k];
                s += x * x;
            }
            nf = sqrt(s);
        }
        double best_c = -INFINITY;
        uint32_t arg = 0xffffffffu;
        if (flag == 1) {
            float uf[MM];
#pragma unroll
            for (int k = 0; k < MM; ++k) {
                const double uk = (k < m && nf != 0.0) ? (SELF ? f[row * m + k] : f[row * m + k] - z[k]) / nf : 0.0;
                uf[k] = (float)uk;  // the scan's conversion
            }
            float best32 = seed[row], thr = best32 * (1.0f - kFilterTol);
            for (uint64_t j = j_begin + lane; j < j_end; j += 32) {
                const float4* p4 = reinterpret_cast<const float4*>(v32 + j * stride);
                float sc = 0.0f;
#pragma unroll
                for (int k4 = 0; k4 < SS / 4; ++k4)
                    if (4 * k4 < m) {
                        const float4 t4 = __ldg(p4 + k4);
                        sc = fmaf(uf[4 * k4], t4.x, sc);
                        if (4 * k4 + 1 < MM) sc = fmaf(uf[4 * k4 + 1 < MM ? 4 * k4 + 1 : 0], t4.y, sc);
                        if (4 * k4 + 2 < MM) sc = fmaf(uf[4 * k4 + 2 < MM ? 4 * k4 + 2 : 0], t4.z, sc);
                        if (4 * k4 + 3 < MM) sc = fmaf(uf[4 * k4 + 3 < MM ? 4 * k4 + 3 : 0], t4.w, sc);
                    }
                if (!(sc >= thr)) continue;
                if (SELF && j == row) continue;  // refvec.hpp:91
                if (sc > best32) {
                    best32 = sc;
                    thr = sc * (1.0f - kFilterTol);
                }
                const double c = exact_cosine(f + row * m, SELF ? nullptr : z, v + j * m, nf, vn[j], m);
                if (c > best_c) {
                    best_c = c;
                    arg = (uint32_t)j;
                }
            }
        } else {
            for (uint64_t j = j_begin + lane; j < j_end; j += 32) {
                if (SELF && j == row) continue;
                double dot = 0.0;
                for (int k = 0; k < m; ++k) dot += (SELF ? f[row * m + k] : f[row * m + k] - z[k]) * v[j * m + k];
                const double c = dot / (nf * vn[j]);
                if (c > best_c) {
                    best_c = c;
                    arg = (uint32_t)j;
                }
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double oc = __shfl_xor_sync(0xffffffffu, best_c, off);
            const uint32_t oj = __shfl_xor_sync(0xffffffffu, arg, off);
            if (oc > best_c || (oc == best_c && oj < arg)) {
                best_c = oc;
                arg = oj;
            }
        }
        if (lane == 0) {
            fb_c[item] = best_c;
            fb_j[item] = arg;
        }
    }
}

// the S partial winners of every flagged row -> chunk slot 0 of the scan's scratch
__global__ void filter_fallback_merge_kernel(const uint32_t* __restrict__ flag_list, const uint32_t* __restrict__ flag_count,
                                             const double* __restrict__ fb_c, const uint32_t* __restrict__ fb_j,
                                             double* __restrict__ part_c, uint32_t* __restrict__ part_j, const uint32_t* skip_flag) {
    if (skip_flag && *skip_flag) return;
    const uint32_t count = *flag_count, S = fallback_split(count);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
        double best_c = -INFINITY;
        uint32_t arg = 0xffffffffu;
        for (uint32_t k = 0; k < S; ++k) {
            const double c = fb_c[i * S + k];
            const uint32_t j = fb_j[i * S + k];
            if (c > best_c || (c == best_c && j < arg)) {
                best_c = c;
                arg = j;
            }
        }
        const uint32_t row = flag_list[i];
        part_c[row] = best_c;
        part_j[row] = arg == 0xffffffffu ? 0u : arg;
    }
}

// gamma_i = acos(max over the chunk winners) (refvec.hpp:93-98)
__global__ void gamma_filter_merge_kernel(uint64_t r, const double* __restrict__ part_c, uint32_t chunks, double* __restrict__ gamma,
                                          uint32_t* err_flag, const uint32_t* skip_flag) {
    if (skip_flag && *skip_flag) return;
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= r) return;
    double c = -INFINITY;
    for (uint32_t k = 0; k < chunks; ++k) {
        const double pc = part_c[k * r + i];
        if (pc > c) c = pc;
    }
    if (c > 1.0) c = 1.0;
    if (c < -1.0) c = -1.0;
    const double g = acos(c);  // tensor.hpp:79-83
    gamma[i] = g;
    if (!(g > 0.0)) atomicOr(err_flag, 1u);  // refvec.hpp:97-98
}

// merges the chunk winners of a row (ascending chunks = ascending j, strict >) and finishes theta / APD / per-vector minima
__global__ void assoc_filter_merge_kernel(const double* __restrict__ f, uint64_t n_rows, uint64_t m, const double* __restrict__ z,
                                          const double* __restrict__ part_c, const uint32_t* __restrict__ part_j, uint32_t chunks,
                                          const double* __restrict__ gamma, double penalty, uint32_t* __restrict__ assoc,
                                          double* __restrict__ theta_out, double* __restrict__ apd_out,
                                          unsigned long long* __restrict__ best_key, uint32_t* __restrict__ first_row, uint32_t row0) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n_rows) return;
    double s = 0.0;
    for (uint64_t k = 0; k < m; ++k) {
        const double u = f[i * m + k] - z[k];  // selection.hpp:155-157, same operations as in the scan
        s += u * u;
    }
    const double nf = sqrt(s);
    double best_c = -INFINITY;
    uint32_t arg = 0;
    for (uint32_t c = 0; c < chunks; ++c) {
        const double pc = part_c[c * n_rows + i];
        if (pc > best_c) {
            best_c = pc;
            arg = part_j[c * n_rows + i];
        }
    }
    double theta = 0.0;  // a row at the ideal point: angle 0 to vector 0 (selection.hpp:167-169)
    if (nf != 0.0) {
        double c = best_c;
        if (c > 1.0) c = 1.0;
        if (c < -1.0) c = -1.0;
        theta = acos(c);  // tensor.hpp:79-83
    } else {
        arg = 0;
    }
    const double apd = (1.0 + penalty * (theta / gamma[arg])) * nf;  // selection.hpp:82-84
    assoc[i] = arg;
    theta_out[i] = theta;
    apd_out[i] = apd;
    const unsigned long long key = (apd != apd) ? kKeyMax : order_key(apd);
    atomicMin(&best_key[arg], key);
    atomicMin(&first_row[arg], row0 + (uint32_t)i);
}

// lowest row among those that attain the minimal APD of their vector
__global__ void elite_rows_kernel(uint64_t n_rows, const uint32_t* n_rows_dev, const uint32_t* assoc,
                                  const double* apd, const unsigned long long* best_key,
                                  uint32_t* best_row, uint32_t row0) {
    const uint64_t n = n_rows_dev ? (uint64_t)*n_rows_dev : n_rows;
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double a = apd[i];
    const unsigned long long key = (a != a) ? kKeyMax : order_key(a);
    const uint32_t j = assoc[i];
    if (key == best_key[j]) atomicMin(&best_row[j], row0 + (uint32_t)i);
}

// validity + the elite of every valid vector (selection.hpp:209-217); compaction in ascending j follows
struct ElitePred {  // also records the validity of the vector (the compaction asks once per element)
    const uint32_t* first_row;
    unsigned char* valid;
    __device__ bool operator()(uint64_t j) const {
        const bool v = first_row[j] != 0xffffffffu;
        valid[j] = v ? 1 : 0;
        return v;
    }
};
struct EliteValPlain {  // sharded runs: objectives are finite, the NaN rule cannot trigger
    const uint32_t* best_row;
    __device__ uint32_t operator()(uint64_t j) const { return best_row[j]; }
};
struct EliteVal {
    const double* apd;
    const uint32_t* first_row;
    const uint32_t* best_row;
    // a NaN APD in the first row of a subpopulation is never displaced (selection.hpp:211)
    __device__ uint32_t operator()(uint64_t j) const {
        const uint32_t fr = first_row[j];
        const double a0 = apd[fr];
        return (a0 != a0) ? fr : best_row[j];
    }
};

template <int M>
void launch_assoc(const double* f, uint64_t n_rows, const uint32_t* n_rows_dev, uint64_t m,
                  const double* v, const double* gamma, uint64_t r, double penalty, SelectWorkspace& ws,
                  cudaStream_t s) {
    const unsigned grid = (unsigned)((n_rows + kAssocThreads - 1) / kAssocThreads);
    const size_t smem = (size_t)kTileVecs * (m + 1) * sizeof(double);
    if (smem > 48 * 1024) {
        static bool configured = false;
        if (!configured) {
            TEMO_CUDA(cudaFuncSetAttribute(assoc_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            configured = true;
        }
    }
    assoc_kernel<M><<<grid, kAssocThreads, smem, s>>>(f, n_rows, n_rows_dev, m, ws.z, v, ws.vn, gamma, r,
                                                     penalty, ws.assoc, ws.theta, ws.apd, ws.best_key,
                                                     ws.first_row);
}

}  // namespace

void SelectWorkspace::alloc(uint64_t rows_cap_, uint64_t r_, uint64_t m_) {
    rows_cap = rows_cap_;
    r = r_;
    m = m_;
    z = dev_alloc<double>(m);
    zkey = col_minmax_scratch_alloc(m);
    vn = dev_alloc<double>(r);
    assoc = dev_alloc<uint32_t>(rows_cap);
    theta = dev_alloc<double>(rows_cap);
    apd = dev_alloc<double>(rows_cap);
    best_key = dev_alloc<unsigned long long>(r);
    best_row = dev_alloc<uint32_t>(r);
    first_row = dev_alloc<uint32_t>(r);
    elite = dev_alloc<uint32_t>(r);
    valid = dev_alloc<unsigned char>(r);
    n_elite = dev_alloc<uint32_t>(1);
    err_flag = dev_alloc<uint32_t>(1);
    tile_scratch = compact_state_alloc(r);
    v32 = dev_alloc<float>(r * v32_stride(m));
    v32_flags = dev_alloc<uint32_t>(1);
    if (assoc_filter_preferred(m, r)) {
        part_c = dev_alloc<double>(rows_cap * kFilterMaxChunks);
        part_j = dev_alloc<uint32_t>(rows_cap * kFilterMaxChunks);
        row_flag = dev_alloc<uint32_t>(rows_cap);
        flag_list = dev_alloc<uint32_t>(rows_cap);
        flag_count = dev_alloc<uint32_t>(1);
        fb_c = dev_alloc<double>(rows_cap + kFallbackItems);
        fb_j = dev_alloc<uint32_t>(rows_cap + kFallbackItems);
        seed32 = dev_alloc<float>(rows_cap);
    }
    TEMO_CUDA(cudaMemset(err_flag, 0, sizeof(uint32_t)));
}

void SelectWorkspace::release() {
    cudaFree(z); cudaFree(zkey); cudaFree(vn); cudaFree(assoc); cudaFree(theta); cudaFree(apd);
    cudaFree(best_key); cudaFree(best_row); cudaFree(first_row); cudaFree(elite); cudaFree(valid);
    cudaFree(n_elite); cudaFree(err_flag); cudaFree(tile_scratch); cudaFree(v32); cudaFree(v32_flags); cudaFree(part_c); cudaFree(part_j); cudaFree(row_flag); cudaFree(seed32);
    cudaFree(flag_list); cudaFree(flag_count); cudaFree(fb_c); cudaFree(fb_j);
    *this = SelectWorkspace{};
}

void launch_row_norms(const double* v, uint64_t r, uint64_t m, double* vn, cudaStream_t s) {
    row_norms_kernel<<<(unsigned)((r + 255) / 256), 256, 0, s>>>(v, r, m, vn);
    TEMO_CUDA(cudaGetLastError());
}

// scratch of launch_col_minmax: m minimum keys (all ones), m maximum keys (zero), a ticket (zero); the kernel restores it
unsigned long long* col_minmax_scratch_alloc(uint64_t m) {
    unsigned long long* p = dev_alloc<unsigned long long>(2 * m + 1);
    TEMO_CUDA(cudaMemset(p, 0xff, m * sizeof(unsigned long long)));
    TEMO_CUDA(cudaMemset(p + m, 0x00, (m + 1) * sizeof(unsigned long long)));
    return p;
}

void launch_col_minmax(const double* f, uint64_t n_rows, const uint32_t* n_rows_dev, uint64_t m,
                       double* zmin, double* zmax, unsigned long long* scratch2m, cudaStream_t s) {
    uint64_t blocks = (n_rows + 255) / 256;
    if (blocks > (uint64_t)kSMs * 4) blocks = (uint64_t)kSMs * 4;
    if (blocks < 1) blocks = 1;
    colmin_kernel<<<dim3((unsigned)blocks, (unsigned)m), 256, 0, s>>>(f, n_rows, n_rows_dev, m, scratch2m, scratch2m + m,
                                                                     scratch2m + 2 * m, zmax != nullptr, zmin, zmax);
    TEMO_CUDA(cudaGetLastError());
}

void launch_select_prepare(const double* f, uint64_t n_rows, uint64_t m, const double* gamma, uint64_t r,
                           SelectWorkspace& ws, cudaStream_t s) {
    require(n_rows >= 1, "translate: empty objective tensor");
    require(m >= 1 && m <= (uint64_t)kMaxObj, "rv_select: unsupported objective count");
    require(n_rows <= ws.rows_cap && r <= ws.r, "rv_select: workspace too small");
    require(n_rows < 0xffffffffULL && r < 0xffffffffULL, "rv_select: index range");
    // one launch for the resets (a small population's selection is a chain of few-microsecond operations), one for the ideal point
    select_init_kernel<<<(unsigned)((std::max<uint64_t>(r, m) + 255) / 256), 256, 0, s>>>(gamma, r, m, ws.err_flag, ws.best_key,
                                                                                       ws.best_row, ws.first_row, ws.zkey);
    uint64_t blocks = (n_rows + 255) / 256;
    if (blocks > (uint64_t)kSMs * 4) blocks = (uint64_t)kSMs * 4;
    colmin_kernel<<<dim3((unsigned)blocks, (unsigned)m), 256, 0, s>>>(f, n_rows, nullptr, m, ws.zkey, ws.zkey + m, ws.zkey + 2 * m,
                                                                     false, ws.z, nullptr);
    TEMO_CUDA(cudaGetLastError());
}

void launch_elite_rows(uint64_t n_rows, const uint32_t* assoc, const double* apd, const unsigned long long* best_key,
                       uint32_t* best_row, uint32_t row0, cudaStream_t s) {
    elite_rows_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, s>>>(n_rows, nullptr, assoc, apd, best_key, best_row, row0);
    TEMO_CUDA(cudaGetLastError());
}

void launch_select_finish(uint64_t r, SelectWorkspace& ws, bool nan_rule, cudaStream_t s) {
    if (nan_rule)
        launch_compact(r, ElitePred{ws.first_row, ws.valid}, EliteVal{ws.apd, ws.first_row, ws.best_row}, ws.tile_scratch, r, ws.elite,
                       ws.n_elite, s);
    else
        launch_compact(r, ElitePred{ws.first_row, ws.valid}, EliteValPlain{ws.best_row}, ws.tile_scratch, r, ws.elite, ws.n_elite, s);
    TEMO_CUDA(cudaGetLastError());
}

bool assoc_filter_preferred(uint64_t m, uint64_t r) { return m >= 5 && r >= 256; }

namespace {
// the filtered scan over (rows x r): per-chunk winners into ws.part_c / ws.part_j; returns the number of chunks
template <bool SELF>
uint32_t launch_filter_scan(const double* rows, uint64_t n_rows, uint64_t m, const double* z, const double* v, uint64_t r,
                            SelectWorkspace& ws, const uint32_t* skip_flag, cudaStream_t s) {
    require(ws.v32 != nullptr && r <= ws.r && m == ws.m, "rv_select: workspace has no fp32 vector copy");
    TEMO_CUDA(cudaMemsetAsync(ws.v32_flags, 0, sizeof(uint32_t), s));
    v32_kernel<<<(unsigned)((r + 255) / 256), 256, 0, s>>>(v, ws.vn, r, m, ws.v32, ws.v32_flags);
    const uint64_t rows_per_cta = (uint64_t)kFilterRows * kFilterThreads;
    const unsigned row_blocks = (unsigned)((n_rows + rows_per_cta - 1) / rows_per_cta);
    // enough CTAs for several waves: the vector range is cut into chunks of whole tiles
    uint64_t chunks = (4ull * kSMs * 4 + row_blocks - 1) / row_blocks;
    const uint64_t tiles = (r + kFilterTile - 1) / kFilterTile;
    if (chunks > (uint64_t)kFilterMaxChunks) chunks = kFilterMaxChunks;
    if (chunks > tiles) chunks = tiles;
    if (chunks < 1) chunks = 1;
    const uint64_t chunk_vecs = (tiles + chunks - 1) / chunks * kFilterTile;
    chunks = (r + chunk_vecs - 1) / chunk_vecs;
    require(n_rows <= ws.rows_cap && ws.part_c != nullptr, "rv_select: workspace has no chunk scratch");
    const dim3 grid(row_blocks, (unsigned)chunks);
    const size_t smem = (size_t)(kFilterTile + kFilterVecs) * v32_stride(m) * sizeof(float) +
                        (size_t)kFilterRows * kFilterCand * kFilterThreads * (sizeof(uint32_t) + sizeof(float));
    require(ws.row_flag != nullptr, "rv_select: workspace has no row flags");
    TEMO_CUDA(cudaMemsetAsync(ws.row_flag, 0, n_rows * sizeof(uint32_t), s));
    TEMO_CUDA(cudaMemsetAsync(ws.flag_count, 0, sizeof(uint32_t), s));
    float* seed = ws.seed32;
#define CALL(MV)                                                                                                                  \
    {                                                                                                                             \
        static bool configured = false;                                                                                           \
        if (!configured && smem > 48 * 1024) {                                                                                    \
            TEMO_CUDA(cudaFuncSetAttribute(assoc_filter_kernel<MV, SELF>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024)); \
            configured = true;                                                                                                    \
        }                                                                                                                         \
        filter_seed_kernel<MV, SELF><<<(unsigned)((n_rows + kSeedRows * kFilterThreads - 1) / (kSeedRows * kFilterThreads)),     \
                                       kFilterThreads, (size_t)kFilterTile * v32_stride(m) * sizeof(float), s>>>(                \
            rows, n_rows, m, z, ws.vn, ws.v32, r, seed, skip_flag);                                                               \
        assoc_filter_kernel<MV, SELF><<<grid, kFilterThreads, smem, s>>>(rows, n_rows, m, z, v, ws.vn, ws.v32, ws.v32_flags, r,    \
                                                                         chunk_vecs, ws.part_c, ws.part_j, ws.row_flag, ws.flag_list, ws.flag_count, seed, \
                                                                         skip_flag);                                              \
        filter_fallback_kernel<MV, SELF><<<kSMs * 8, 128, 0, s>>>(rows, m, z, v, ws.vn, ws.v32, seed, r, ws.row_flag, ws.flag_list, \
                                                                  ws.flag_count, ws.fb_c, ws.fb_j, skip_flag);                      \
    }
    switch (m) {
    case 5: CALL(5); break;
    case 10: CALL(10); break;
    default: CALL(0); break;
    }
#undef CALL
    filter_fallback_merge_kernel<<<64, 256, 0, s>>>(ws.flag_list, ws.flag_count, ws.fb_c, ws.fb_j, ws.part_c, ws.part_j, skip_flag);
    TEMO_CUDA(cudaGetLastError());
    return (uint32_t)chunks;
}
}  // namespace

void launch_assoc_filter(const double* f, uint64_t n_rows, uint64_t m, const double* v, const double* gamma, uint64_t r, double penalty,
                         SelectWorkspace& ws, uint32_t* assoc, double* theta, double* apd, cudaStream_t s, uint32_t row0) {
    const uint32_t chunks = launch_filter_scan<false>(f, n_rows, m, ws.z, v, r, ws, nullptr, s);
    assoc_filter_merge_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, s>>>(f, n_rows, m, ws.z, ws.part_c, ws.part_j, chunks,
                                                                               gamma, penalty, assoc, theta, apd, ws.best_key,
                                                                               ws.first_row, row0);
    TEMO_CUDA(cudaGetLastError());
}

// min_vector_angles (refvec.hpp:81-100) through the same filtered scan (many objectives): ws.vn must hold the norms of v
void launch_gamma_filter(const double* v, uint64_t r, uint64_t m, SelectWorkspace& ws, double* gamma, uint32_t* err_flag,
                         const uint32_t* skip_flag, cudaStream_t s) {
    require(r >= 2, "min_vector_angles: needs at least two vectors");  // refvec.hpp:82
    const uint32_t chunks = launch_filter_scan<true>(v, r, m, nullptr, v, r, ws, skip_flag, s);
    gamma_filter_merge_kernel<<<(unsigned)((r + 255) / 256), 256, 0, s>>>(r, ws.part_c, chunks, gamma, err_flag, skip_flag);
    TEMO_CUDA(cudaGetLastError());
}

void launch_gamma_auto(const double* v, uint64_t r, uint64_t m, SelectWorkspace& ws, VecIndex* index, double* gamma,
                       uint32_t* err_flag, const uint32_t* skip_flag, cudaStream_t s) {
    if (assoc_filter_preferred(m, r) && ws.part_c != nullptr && r <= ws.rows_cap) {
        launch_gamma_filter(v, r, m, ws, gamma, err_flag, skip_flag, s);
    } else {
        require(index != nullptr && index->built, "min_vector_angles: no direction index");
        launch_gamma_indexed(v, ws.vn, r, m, *index, gamma, err_flag, skip_flag, s);
    }
}

void launch_select(const double* f, uint64_t n_rows, const uint32_t* n_rows_dev, uint64_t m,
                   const double* v, const double* gamma, uint64_t r, double penalty,
                   SelectWorkspace& ws, cudaStream_t s, VecIndex* index) {
    require(n_rows_dev == nullptr, "rv_select: device-side row counts are not supported here");
    launch_select_prepare(f, n_rows, m, gamma, r, ws, s);
    if (assoc_filter_preferred(m, r)) {
        launch_assoc_filter(f, n_rows, m, v, gamma, r, penalty, ws, ws.assoc, ws.theta, ws.apd, s, 0);
    } else if (index && index->built) {
        launch_assoc_indexed(f, n_rows, nullptr, m, ws.z, *index, gamma, penalty, ws.assoc, ws.theta, ws.apd,
                             ws.best_key, ws.first_row, s);
    } else {
        switch (m) {
        case 2: launch_assoc<2>(f, n_rows, nullptr, m, v, gamma, r, penalty, ws, s); break;
        case 3: launch_assoc<3>(f, n_rows, nullptr, m, v, gamma, r, penalty, ws, s); break;
        case 4: launch_assoc<4>(f, n_rows, nullptr, m, v, gamma, r, penalty, ws, s); break;
        case 5: launch_assoc<5>(f, n_rows, nullptr, m, v, gamma, r, penalty, ws, s); break;
        case 10: launch_assoc<10>(f, n_rows, nullptr, m, v, gamma, r, penalty, ws, s); break;
        default: launch_assoc<0>(f, n_rows, nullptr, m, v, gamma, r, penalty, ws, s); break;
        }
    }
    launch_elite_rows(n_rows, ws.assoc, ws.apd, ws.best_key, ws.best_row, 0, s);
    launch_select_finish(r, ws, /*nan_rule=*/true, s);
    TEMO_CUDA(cudaGetLastError());
}

}  // namespace temo_b200
