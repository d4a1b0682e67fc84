// The other reproduction operators of the reference behind the same boundary:
// DE/rand/1/bin, particle swarm and competitive swarm updates.
//
// reference: de_reproduce (operators.hpp:166-200), pso_reproduce (operators.hpp:205-240),
// cso_reproduce (operators.hpp:246-284), SwarmState / make_swarm_state (operators.hpp:46-60).
// All three are pure + - * / comparisons on fp64 (no libm): compiled with --fmad=false they are bit-identical to the
// reference, draw for draw (uniform_tensor addressing, rng.hpp:55-66: element (i, j) of a rows x cols tensor is draw
// base + i * cols + j). Random numbers are re-derived in registers; every kernel is one pass over its rows:
// HBM-bound elementwise work (one CTA per row, 128-bit accesses when d is even).
#include "internal.h"

namespace temo_b200 {

namespace {

template <int MODE>
__device__ __forceinline__ double unit_draw(const Rng& g, uint64_t k) {
    return word_to_unit(draw_word<MODE>(g, k));
}

// ---- DE/rand/1/bin -----------------------------------------------------------------------------------------
// draws: r_sel n x 3 at c, r_j n x 1 at c + 3n, r_cr n x d at c + 4n
template <int MODE>
__global__ void __launch_bounds__(256) de_kernel(const double* __restrict__ x, const uint32_t* __restrict__ src,
                                                  const uint32_t* __restrict__ dst, uint64_t n, uint64_t d, Rng rng, uint64_t c, double f,
                                                  double cr, const double* __restrict__ lower, const double* __restrict__ upper,
                                                  double* __restrict__ out) {
    const uint64_t i = blockIdx.x;
    const double nd = (double)n;
    // three mutually distinct donors, all != i (operators.hpp:177-187); every thread derives the same indices
    uint64_t r1 = (i + 1 + (uint64_t)(unit_draw<MODE>(rng, c + i * 3 + 0) * (nd - 1.0))) % n;
    const uint64_t excl_a = i < r1 ? i : r1, excl_b = i < r1 ? r1 : i;
    uint64_t r2 = (uint64_t)(unit_draw<MODE>(rng, c + i * 3 + 1) * (nd - 2.0));
    if (r2 >= excl_a) ++r2;
    if (r2 >= excl_b) ++r2;
    uint64_t e0 = i, e1 = r1, e2 = r2, t;  // sorted ascending
    if (e0 > e1) t = e0, e0 = e1, e1 = t;
    if (e1 > e2) t = e1, e1 = e2, e2 = t;
    if (e0 > e1) t = e0, e0 = e1, e1 = t;
    uint64_t r3 = (uint64_t)(unit_draw<MODE>(rng, c + i * 3 + 2) * (nd - 3.0));
    if (r3 >= e0) ++r3;
    if (r3 >= e1) ++r3;
    if (r3 >= e2) ++r3;
    const uint64_t j_rand = (uint64_t)(unit_draw<MODE>(rng, c + 3 * n + i) * (double)d);
    const uint64_t c_cr = c + 4 * n + i * d;
    // row i of the operand lives in storage row src[i], the child goes to storage row dst[i] (nullptr: i)
    const auto at = [&](uint64_t row) { return x + (src ? (uint64_t)src[row] : row) * d; };
    const double *xi = at(i), *x1 = at(r1), *x2 = at(r2), *x3 = at(r3);
    double* oi = out + (dst ? (uint64_t)dst[i] : i) * d;
    for (uint64_t j = threadIdx.x; j < d; j += blockDim.x) {
        double o;
        if (unit_draw<MODE>(rng, c_cr + j) < cr || j == j_rand) {
            const double trial = x1[j] + f * (x2[j] - x3[j]);  // operators.hpp:191
            o = clampd(trial, lower[j], upper[j]);
        } else {
            o = xi[j];
        }
        oi[j] = o;
    }
}

// ---- particle swarm ------------------------------------------------------------------------------------------
// personal bests refresh where the score improved (operators.hpp:213-219)
__global__ void __launch_bounds__(256) pso_pbest_kernel(const double* __restrict__ x, const uint32_t* __restrict__ src,
                                                         const double* __restrict__ scores, uint64_t d, double* __restrict__ pb_x,
                                                         double* __restrict__ pb_score) {
    const uint64_t i = blockIdx.x;
    if (!(scores[i] < pb_score[i])) return;  // CTA-uniform
    const double* xi = x + (src ? (uint64_t)src[i] : i) * d;
    for (uint64_t j = threadIdx.x; j < d; j += blockDim.x) pb_x[i * d + j] = xi[j];
    __syncthreads();
    if (threadIdx.x == 0) pb_score[i] = scores[i];
}

// best = the reference's scan `best = 0; for i: if (s[i] < s[best]) best = i` (operators.hpp:220-222): the first row with
// the smallest score; NaN scores never win, except that a NaN in row 0 is never displaced.
__global__ void __launch_bounds__(1024) argmin_first_kernel(const double* __restrict__ s, uint64_t n, uint32_t* out) {
    __shared__ double sv[32];
    __shared__ uint64_t si[32];
    double bv = 0.0;
    uint64_t bi = ~0ULL;  // none yet
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double v = s[i];
        if (v == v && (bi == ~0ULL || v < bv)) bv = v, bi = i;
    }
    auto take = [](double v, uint64_t i, double w, uint64_t k) {  // should (v, i) replace (w, k)? both NaN-free
        if (i == ~0ULL) return false;
        if (k == ~0ULL) return true;
        return v < w || (v == w && i < k);
    };
    for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const uint64_t oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (take(ov, oi, bv, bi)) bv = ov, bi = oi;
    }
    if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = bv, si[threadIdx.x >> 5] = bi;
    __syncthreads();
    if (threadIdx.x < 32) {
        bv = threadIdx.x < (blockDim.x >> 5) ? sv[threadIdx.x] : 0.0;
        bi = threadIdx.x < (blockDim.x >> 5) ? si[threadIdx.x] : ~0ULL;
        for (int off = 16; off > 0; off >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
            const uint64_t oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (take(ov, oi, bv, bi)) bv = ov, bi = oi;
        }
        if (threadIdx.x == 0) *out = (s[0] != s[0] || bi == ~0ULL) ? 0u : (uint32_t)bi;
    }
}

// draws: r1 n x d at c, r2 n x d at c + n d (operators.hpp:223-224); velocity and position update (:230-236)
template <int MODE>
__global__ void __launch_bounds__(256) pso_update_kernel(const double* __restrict__ x, const uint32_t* __restrict__ src,
                                                          const uint32_t* __restrict__ dst, uint64_t n, uint64_t d, Rng rng, uint64_t c,
                                                          double inertia, double c1, double c2, const double* __restrict__ pb_x,
                                                          const uint32_t* __restrict__ best, double* __restrict__ vel,
                                                          const double* __restrict__ lower, const double* __restrict__ upper,
                                                          double* __restrict__ out) {
    const uint64_t i = blockIdx.x;
    const double* gbest = pb_x + (uint64_t)*best * d;
    const uint64_t c_r1 = c + i * d, c_r2 = c + n * d + i * d;
    const double* xi = x + (src ? (uint64_t)src[i] : i) * d;
    double* oi = out + (dst ? (uint64_t)dst[i] : i) * d;
    for (uint64_t j = threadIdx.x; j < d; j += blockDim.x) {
        const double xv = xi[j];
        const double v = inertia * vel[i * d + j] + c1 * unit_draw<MODE>(rng, c_r1 + j) * (pb_x[i * d + j] - xv) +
                         c2 * unit_draw<MODE>(rng, c_r2 + j) * (gbest[j] - xv);
        vel[i * d + j] = v;
        oi[j] = clampd(xv + v, lower[j], upper[j]);
    }
}

// ---- competitive swarm ---------------------------------------------------------------------------------------
// column means in the reference's order: rows added one after the other, then one division (operators.hpp:257-260).
// The additions of a column are inherently sequential, the loads are not: a CTA owns kMeanCols columns, all its threads
// stream row tiles into a two-stage shared-memory ring with cp.async (LDGSTS) while kMeanCols threads add the previous
// tile in row order.
constexpr int kMeanCols = 8, kMeanRows = 128;
__global__ void __launch_bounds__(256) col_mean_kernel(const double* __restrict__ x, const uint32_t* __restrict__ src, uint64_t n, uint64_t d,
                                                        double* __restrict__ mean) {
    __shared__ double buf[2][kMeanRows][kMeanCols];
    const uint64_t j0 = blockIdx.x * (uint64_t)kMeanCols;
    const uint32_t cols = (uint32_t)(d - j0 < (uint64_t)kMeanCols ? d - j0 : (uint64_t)kMeanCols);
    const uint64_t tiles = (n + kMeanRows - 1) / kMeanRows;
    auto issue = [&](uint64_t tile, int b) {
        for (uint32_t e = threadIdx.x; e < kMeanRows * kMeanCols; e += blockDim.x) {
            const uint32_t r = e / kMeanCols, c = e % kMeanCols;
            const uint64_t row = tile * kMeanRows + r;
            if (row < n && c < cols) {
                const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&buf[b][r][c]);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(x + (src ? (uint64_t)src[row] : row) * d + j0 + c)
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double s = 0.0;
    if (tiles) issue(0, 0);
    for (uint64_t t = 0; t < tiles; ++t) {
        if (t + 1 < tiles) {
            issue(t + 1, (int)((t + 1) & 1));
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        if (threadIdx.x < cols) {
            const uint64_t rows = n - t * kMeanRows < (uint64_t)kMeanRows ? n - t * kMeanRows : (uint64_t)kMeanRows;
            for (uint64_t r = 0; r < rows; ++r) s += buf[t & 1][r][threadIdx.x];
        }
        __syncthreads();
    }
    if (threadIdx.x < cols) mean[j0 + threadIdx.x] = s / (double)n;
}

// one CTA per pair (perm[2q], perm[2q+1]); draws r1, r2, r3 (pairs x d each) at c, c + pairs d, c + 2 pairs d.
// The winner's row and velocity pass through bit-identically (operators.hpp:263-264: out = x, new_vel = velocities);
// CTA `pairs` copies the unpaired row of an odd population.
template <int MODE>
__global__ void __launch_bounds__(256) cso_kernel(const double* __restrict__ x, const uint32_t* __restrict__ src,
                                                   const uint32_t* __restrict__ dst, const double* __restrict__ scores, uint64_t n,
                                                   uint64_t pairs, uint64_t d, Rng rng, uint64_t c, double phi,
                                                   const uint32_t* __restrict__ perm, const double* __restrict__ mean,
                                                   const double* vel, const double* __restrict__ lower,
                                                   const double* __restrict__ upper, double* vel_out,
                                                   double* __restrict__ out) {
    const uint64_t q = blockIdx.x;
    if (q >= pairs) {  // odd n: the last row of the shuffled order is nobody's partner
        const uint64_t r = perm[n - 1];
        const double* xr = x + (src ? (uint64_t)src[r] : r) * d;
        double* orow = out + (dst ? (uint64_t)dst[r] : r) * d;
        for (uint64_t j = threadIdx.x; j < d; j += blockDim.x) {
            orow[j] = xr[j];
            if (vel_out != vel) vel_out[r * d + j] = vel[r * d + j];
        }
        return;
    }
    const uint64_t a = perm[2 * q], b = perm[2 * q + 1];
    uint64_t win = a, lose = b;
    if (scores[b] < scores[a] || (scores[b] == scores[a] && b < a)) win = b, lose = a;  // operators.hpp:267-271
    const uint64_t c1 = c + q * d, c2 = c + pairs * d + q * d, c3 = c + 2 * pairs * d + q * d;
    const double *xlose = x + (src ? (uint64_t)src[lose] : lose) * d, *xwin = x + (src ? (uint64_t)src[win] : win) * d;
    double *olose = out + (dst ? (uint64_t)dst[lose] : lose) * d, *owin = out + (dst ? (uint64_t)dst[win] : win) * d;
    for (uint64_t j = threadIdx.x; j < d; j += blockDim.x) {
        const double xl = xlose[j], xw = xwin[j];
        const double v = unit_draw<MODE>(rng, c1 + j) * vel[lose * d + j] + unit_draw<MODE>(rng, c2 + j) * (xw - xl) +
                         phi * unit_draw<MODE>(rng, c3 + j) * (mean[j] - xl);
        vel_out[lose * d + j] = v;
        olose[j] = clampd(xl + v, lower[j], upper[j]);
        owin[j] = xw;
        if (vel_out != vel) vel_out[win * d + j] = vel[win * d + j];  // in place (vel_out == vel): the winner's velocity stays
    }
}

}  // namespace

void launch_de(const double* x, uint64_t n, uint64_t d, Rng rng, uint64_t counter, double f, double cr, const double* lower,
               const double* upper, double* out, cudaStream_t s, const uint32_t* src, const uint32_t* dst) {
    require(n >= 4, "de_reproduce: needs at least four rows");  // operators.hpp:169
    require(n < 0xffffffffULL, "de_reproduce: too many rows");
    if (rng.mode == 0)
        de_kernel<0><<<(unsigned)n, 256, 0, s>>>(x, src, dst, n, d, rng, counter, f, cr, lower, upper, out);
    else
        de_kernel<1><<<(unsigned)n, 256, 0, s>>>(x, src, dst, n, d, rng, counter, f, cr, lower, upper, out);
    TEMO_CUDA(cudaGetLastError());
}

void launch_pso(const double* x, const double* scores, uint64_t n, uint64_t d, Rng rng, uint64_t counter, double inertia, double c1,
                double c2, double* vel, double* pb_x, double* pb_score, uint32_t* best_scratch, const double* lower,
                const double* upper, double* out, cudaStream_t s, const uint32_t* src, const uint32_t* dst) {
    require(n >= 1 && n < 0xffffffffULL, "pso_reproduce: bad row count");
    pso_pbest_kernel<<<(unsigned)n, 256, 0, s>>>(x, src, scores, d, pb_x, pb_score);
    argmin_first_kernel<<<1, 1024, 0, s>>>(pb_score, n, best_scratch);
    if (rng.mode == 0)
        pso_update_kernel<0><<<(unsigned)n, 256, 0, s>>>(x, src, dst, n, d, rng, counter, inertia, c1, c2, pb_x, best_scratch, vel, lower, upper, out);
    else
        pso_update_kernel<1><<<(unsigned)n, 256, 0, s>>>(x, src, dst, n, d, rng, counter, inertia, c1, c2, pb_x, best_scratch, vel, lower, upper, out);
    TEMO_CUDA(cudaGetLastError());
}

void launch_cso(const double* x, const double* scores, uint64_t n, uint64_t d, Rng rng, uint64_t counter, double phi,
                const uint32_t* perm, double* mean_scratch, const double* vel, double* vel_out, const double* lower,
                const double* upper, double* out, cudaStream_t s, const uint32_t* src, const uint32_t* dst) {
    require(n >= 1 && n < 0xffffffffULL, "cso_reproduce: bad row count");
    const uint64_t pairs = n / 2;
    col_mean_kernel<<<(unsigned)((d + kMeanCols - 1) / kMeanCols), 256, 0, s>>>(x, src, n, d, mean_scratch);
    const unsigned grid = (unsigned)(pairs + (n & 1));
    if (rng.mode == 0)
        cso_kernel<0><<<grid, 256, 0, s>>>(x, src, dst, scores, n, pairs, d, rng, counter, phi, perm, mean_scratch, vel, lower, upper, vel_out, out);
    else
        cso_kernel<1><<<grid, 256, 0, s>>>(x, src, dst, scores, n, pairs, d, rng, counter, phi, perm, mean_scratch, vel, lower, upper, vel_out, out);
    TEMO_CUDA(cudaGetLastError());
}

}  // namespace temo_b200
