// K1 — fused GA reproduction: mating gather + SBX crossover + polynomial mutation
// (+ optional objective evaluation of the children) in ONE pass over the population.
//
// reference: ga_reproduce (operators.hpp:153-161) = shuffle_indices -> row gather -> sbx
// (operators.hpp:65-102) -> polynomial_mutation (operators.hpp:126-149), which on the CPU is
// six full N x d passes plus five materialised N x d random tensors. Here every random
// number is re-derived in registers from its (seed, counter) address (rng.hpp:39-43; SURVEY.md
// Appendix A gives the counter map), the shuffled/pooled parent matrix is never built (the
// kernel reads parent rows through the `src` indirection) and children are written straight
// into free rows of the population pool (`dst`): algorithmic traffic = 16*N*d bytes.
//
// Mapping: one CTA per mating pair (rows p and half+p of the shuffled order); thread t owns
// gene vectors t, t+B, ... (VEC = 2 doubles = one 128-bit load/store when d is even), which
// is the canonical order the evaluation reductions share with evaluate.cu.
//
// Exactness (compiled with --fmad=false): all blends, clamps and copies are the reference's
// IEEE operations in the reference's order. Dead branches the reference multiplies by an
// exact 0.0 are skipped (verified bit-identical); the only inexact pieces are
// CUDA's pow (<= 2 ulp) on crossed/mutated genes.
#include "glibc_pow_dev.cuh"
#include "internal.h"
#include "problems.cuh"

namespace temo_b200 {

namespace {

struct ReproK {
    const double* pool;
    const uint32_t* src;
    double* out;
    const uint32_t* dst;
    uint64_t n, d, half;
    uint64_t g_unit0, g_half, g_n;  // position of this launch inside the global draw blocks (sharded runs)
    Rng rng;
    uint64_t c_mc, c_r1, c_r2, c_r3, c_mask, c_mut;
    // Draw addressing in stream units (SplitMix64: counter * GOLDEN added to mix64(seed); Philox: the counter
    // itself): element j of row u of a draw block sits at s_base + u * s_row + j * s_gene + (block delta). All
    // block deltas are launch constants, so one 64-bit value per CTA positions every stream.
    uint64_t s_base, s_row, s_gene, dl_r1, dl_r2, dl_mask_a, dl_mask_b, dl_mut_a, dl_mut_b;
    double pc, inv_exp, xi;
    uint64_t mask_thresh;  // mutate iff (word >> 11) <= mask_thresh
    uint32_t mask_top;     // = mask_thresh >> 32: necessary condition on the top 21 bits
    int mask_never;
    int narrow_pow;  // 1/(eta+1) in [2^-10, 1]: the SBX pow stays on the common path of the libm algorithm
    const double* lower;
    const double* upper;
    uint64_t m;
    double* f_out;
    uint64_t f_row0;
    const uint32_t* f_row0_dev;
};

// polynomial_delta (operators.hpp:106-121): both branches evaluated, blended by steps. Rare path (about one
// gene per row): tables are read from global memory so that no pointer into shared memory escapes the kernel.
__device__ __noinline__ double polynomial_delta_dev(double u, double x, double lo, double hi, double xi) {
    const PowTables T = pow_tables_global();
    const double range = hi - lo;
    const double e = xi + 1.0, inv_e = 1.0 / e;
    const double near_lo = 1.0 - (x - lo) / range;
    const double d_lo =
        range * (pow_like_host(2.0 * u + (1.0 - 2.0 * u) * pow_like_host(near_lo, e, T), inv_e, T) - 1.0);
    const double near_hi = 1.0 - (hi - x) / range;
    const double d_hi =
        range * (1.0 - pow_like_host(2.0 * (1.0 - u) + 2.0 * (u - 0.5) * pow_like_host(near_hi, e, T), inv_e, T));
    const double h_lo = (0.5 - u) >= 0.0 ? 1.0 : 0.0;
    const double h_hi = (u - 0.5) >= 0.0 ? 1.0 : 0.0;
    return d_lo * h_lo + d_hi * h_hi;
}

// Slow half of the mutation test (operators.hpp:136-145), entered only when the top 21 bits of the mask draw
// do not already exceed the threshold's (probability ~ pm/d): the full 53-bit comparison and, if the gene is
// really selected, the mutation itself. Kept out of line so that the hot loop carries only the top-word hash.
__device__ __noinline__ double mutate_if_selected(double x, uint64_t mask_word, uint64_t mut_word, uint64_t thresh,
                                                  double lo, double hi, double xi) {
    if ((mask_word >> 11) > thresh) return x;
    const double u = word_to_unit(mut_word);
    return clampd(x + polynomial_delta_dev(u, x, lo, hi, xi), lo, hi);
}

// Draw words of this CTA's rows. pos = s_base + row * s_row is computed once per CTA; a gene's stream
// positions are pos + j * s_gene + (launch-constant block delta), so a draw costs one 32x64-bit multiply-add
// per gene (shared by all of its streams), one 64-bit add per stream and the two mixing rounds.
template <int MODE>
struct Draws {
    uint64_t seed;
    __device__ __forceinline__ uint64_t gene(uint64_t pos, uint32_t j, uint64_t s_gene) const {
        return pos + (uint64_t)j * s_gene;
    }
    __device__ __forceinline__ uint64_t word(uint64_t at) const { return MODE == 0 ? mix64(at) : philox_word(seed, at); }
    // top 31 bits of word(at) (bit 0 of the result is not meaningful)
    __device__ __forceinline__ uint32_t top(uint64_t at) const {
        return MODE == 0 ? mix64_top32(at) : (uint32_t)(philox_word(seed, at) >> 32);
    }
};

#ifndef TEMO_REPRO_MIN_BLOCKS
#define TEMO_REPRO_MIN_BLOCKS 4
#endif
template <int MODE, bool SBX, bool PM, int EVAL, int VEC>
__global__ void __launch_bounds__(256, TEMO_REPRO_MIN_BLOCKS) reproduce_kernel(const ReproK a) {
    __shared__ double s_red[8];
    __shared__ double s_pos[2][kMaxObj];
    __shared__ PowSmem s_pow;
    __shared__ unsigned char s_list[8][64];  // per warp: compacted (lane, v) codes of the crossing genes
    __shared__ double s_beta[8][64];         // per warp: signed spread factor per (lane, v)
    pow_smem_load(s_pow);
    __syncthreads();
    const PowTables T = pow_tables(s_pow);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    const uint64_t unit = blockIdx.x;
    const bool paired = SBX && unit < a.half;
    // shuffled-order rows handled by this CTA
    const uint64_t row_a = SBX ? (paired ? unit : a.n - 1) : unit;
    const uint64_t row_b = a.half + unit;  // only meaningful when paired

    const uint64_t src_a = a.src ? a.src[row_a] : row_a;
    const uint64_t dst_a = a.dst ? a.dst[row_a] : row_a;
    const double* pa = a.pool + src_a * a.d;
    double* oa = a.out + dst_a * a.d;
    const double* pb = nullptr;
    double* ob = nullptr;
    if (paired) {
        const uint64_t src_b = a.src ? a.src[row_b] : row_b;
        const uint64_t dst_b = a.dst ? a.dst[row_b] : row_b;
        pb = a.pool + src_b * a.d;
        ob = a.out + dst_b * a.d;
    }

    // draw streams of this CTA's rows: SBX blocks are half x d, PM blocks n x d
    // (global numbering: a shard of a multi-GPU run draws exactly what the single-GPU run draws for its rows)
    const uint64_t g_unit = a.g_unit0 + unit;
    const uint64_t g_row_a = SBX ? (paired ? g_unit : a.g_n - 1) : g_unit;
    const Draws<MODE> rnd{a.rng.seed};
    const uint64_t pos = a.s_base + g_row_a * a.s_row;  // Mc block position of row g_row_a; the others are offsets

    // pair-level crossover switch: hc = H(r3 - pc) (operators.hpp:82)
    bool pair_cross = false;
    if (paired) {
        const double r3 = word_to_unit(draw_word<MODE>(a.rng, a.c_r3 + g_unit));
        pair_cross = !(r3 - a.pc >= 0.0);
    }

    double acc_a = 0.0, acc_b = 0.0;
    const uint32_t nvec = (uint32_t)(a.d / VEC);
    const uint32_t nvec_ceil = (nvec + blockDim.x - 1) / blockDim.x * blockDim.x;

    for (uint32_t q = threadIdx.x; q < nvec_ceil; q += blockDim.x) {  // whole warps stay in the loop
        const bool in_range = q < nvec;
        const uint32_t j0 = q * VEC;
        double xa[VEC], xb[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) xa[v] = xb[v] = 0.0;
        if (in_range) {
            if (VEC == 2) {
                const double2 t = *reinterpret_cast<const double2*>(pa + j0);
                xa[0] = t.x;
                xa[VEC - 1] = t.y;
                if (paired) {
                    const double2 w = *reinterpret_cast<const double2*>(pb + j0);
                    xb[0] = w.x;
                    xb[VEC - 1] = w.y;
                }
            } else {
                xa[0] = pa[j0];
                if (paired) xb[0] = pb[j0];
            }
        }
        double beta[VEC];
        bool crosses[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
            beta[v] = 1.0;
            crosses[v] = false;
        }
        if (SBX && paired && pair_cross) {  // CTA-uniform
            // hr = H(r2 - 0.5): the top bit of the word; a gene crosses iff it is clear (operators.hpp:90-91)
#pragma unroll
            for (int v = 0; v < VEC; ++v)
                crosses[v] = in_range && (rnd.top(rnd.gene(pos, j0 + v, a.s_gene) + a.dl_r2) >> 31) == 0;
            // The spread factor (two draws + one pow) is needed by ~half of the genes only: compact the
            // crossing genes of the warp so that the expensive part runs with full lanes.
            const unsigned b0 = __ballot_sync(0xffffffffu, crosses[0]);
            const unsigned b1 = VEC == 2 ? __ballot_sync(0xffffffffu, crosses[VEC - 1]) : 0u;
            const unsigned lt = (1u << lane) - 1u;
            const int n0 = __popc(b0), total = n0 + __popc(b1);
            if (crosses[0]) s_list[warp][__popc(b0 & lt)] = (unsigned char)(lane * 2);
            if (VEC == 2 && crosses[VEC - 1]) s_list[warp][n0 + __popc(b1 & lt)] = (unsigned char)(lane * 2 + 1);
            __syncwarp();
            const uint32_t q_warp = q - lane;  // vector index handled by lane 0 of this warp
            for (int t = lane; t < total; t += 32) {
                const int code = s_list[warp][t];
                const uint32_t j = (q_warp + (code >> 1)) * VEC + (code & 1);
                const uint64_t at = rnd.gene(pos, j, a.s_gene);
                const double mc = word_to_unit(rnd.word(at));
                const bool up = (rnd.top(at + a.dl_r1) >> 31) != 0;  // sgn(r1 - 0.5)
                // live spread branch only (hm = H(0.5 - mc)); the other one is multiplied by exactly 0.0
                const bool low = 0.5 - mc >= 0.0;
                const double base = low ? 2.0 * mc : 2.0 - 2.0 * mc;
                // base is 0 (mc == 0) or in [2^-52, 2]; |y log base| < 2 for any eta >= 0
                const double yexp = low ? a.inv_exp : -a.inv_exp;
                const double spread = (base > 0.0 && a.narrow_pow) ? pow_like_host_narrow(base, yexp, T) : pow_like_host(base, yexp, T);
                s_beta[warp][code] = up ? spread : -spread;
            }
            __syncwarp();
#pragma unroll
            for (int v = 0; v < VEC; ++v)
                if (crosses[v]) beta[v] = s_beta[warp][lane * 2 + v];
            __syncwarp();
        }
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
            const uint32_t j = j0 + v;
            if (!in_range) continue;
            const double lo = a.lower[j], hi = a.upper[j];
            double ca = xa[v], cb = xb[v];
            if (SBX && paired) {
                // operators.hpp:92-95 as written: a gene that does not cross has beta = 1 exactly (hr = 1 or hc = 1),
                // and the blend then returns the parents through the same arithmetic as on the CPU
                const double b = beta[v];
                ca = clampd(((1.0 + b) * xa[v] + (1.0 - b) * xb[v]) / 2.0, lo, hi);
                cb = clampd(((1.0 - b) * xa[v] + (1.0 + b) * xb[v]) / 2.0, lo, hi);
            }
            if (PM && !a.mask_never) {
                const bool live = !(hi - lo <= 0.0);
                // (word >> 11) <= T can only hold if the top 21 bits do not exceed T's: decided from the top word
                const uint64_t at = rnd.gene(pos, j, a.s_gene);
                if (live && (rnd.top(at + a.dl_mask_a) >> 11) <= a.mask_top)
                    ca = mutate_if_selected(ca, rnd.word(at + a.dl_mask_a), rnd.word(at + a.dl_mut_a), a.mask_thresh, lo, hi, a.xi);
                if (paired && live && (rnd.top(at + a.dl_mask_b) >> 11) <= a.mask_top)
                    cb = mutate_if_selected(cb, rnd.word(at + a.dl_mask_b), rnd.word(at + a.dl_mut_b), a.mask_thresh, lo, hi, a.xi);
            }
            if (EVAL != 0) {
                if (j + 1 >= a.m) {
                    acc_a += dtlz_term<EVAL>(ca);
                    if (paired) acc_b += dtlz_term<EVAL>(cb);
                } else {
                    s_pos[0][j] = ca;
                    if (paired) s_pos[1][j] = cb;
                }
            }
            xa[v] = ca;
            xb[v] = cb;
        }
        if (in_range) {
            if (VEC == 2) {
                *reinterpret_cast<double2*>(oa + j0) = make_double2(xa[0], xa[VEC - 1]);
                if (paired) *reinterpret_cast<double2*>(ob + j0) = make_double2(xb[0], xb[VEC - 1]);
            } else {
                oa[j0] = xa[0];
                if (paired) ob[j0] = xb[0];
            }
        }
    }

    if (EVAL != 0) {
        const uint64_t f0 = a.f_row0 + (a.f_row0_dev ? (uint64_t)*a.f_row0_dev : 0);
        // leave {tail sum, position genes} in the objective rows; launch_dtlz_finish turns them into objectives
        // (keeps the cos/sin/pow latency chain out of the tail of every CTA)
        const double ga = block_sum<8>(acc_a, s_red);
        double* fa = a.f_out + (f0 + row_a) * a.m;
        if (threadIdx.x == 0) fa[0] = ga;
        if (threadIdx.x >= 1 && threadIdx.x < a.m) fa[threadIdx.x] = s_pos[0][threadIdx.x - 1];
        if (paired) {
            const double gb = block_sum<8>(acc_b, s_red);
            double* fb = a.f_out + (f0 + row_b) * a.m;
            if (threadIdx.x == 0) fb[0] = gb;
            if (threadIdx.x >= 1 && threadIdx.x < a.m) fb[threadIdx.x] = s_pos[1][threadIdx.x - 1];
        }
    }
}

template <int MODE, bool SBX, bool PM, int EVAL>
void launch_vec(const ReproK& k, uint64_t units, int block, int vec, cudaStream_t s) {
    if (units == 0) return;
    if (vec == 2)
        reproduce_kernel<MODE, SBX, PM, EVAL, 2><<<(unsigned)units, block, 0, s>>>(k);
    else
        reproduce_kernel<MODE, SBX, PM, EVAL, 1><<<(unsigned)units, block, 0, s>>>(k);
}

template <int MODE, bool SBX, bool PM>
void launch_eval(const ReproK& k, uint64_t units, int block, int vec, int eval, cudaStream_t s) {
    switch (eval) {
    case 0: launch_vec<MODE, SBX, PM, 0>(k, units, block, vec, s); break;
    case kDtlz1: launch_vec<MODE, SBX, PM, kDtlz1>(k, units, block, vec, s); break;
    case kDtlz2: launch_vec<MODE, SBX, PM, kDtlz2>(k, units, block, vec, s); break;
    case kDtlz3: launch_vec<MODE, SBX, PM, kDtlz3>(k, units, block, vec, s); break;
    case kDtlz4: launch_vec<MODE, SBX, PM, kDtlz4>(k, units, block, vec, s); break;
    default: fail(1, "reproduce: fused evaluation supports DTLZ1-4 only");
    }
}

template <int MODE>
void launch_mode(const ReproK& k, bool sbx, bool pm, uint64_t units, int block, int vec, int eval,
                 cudaStream_t s) {
    if (sbx && pm) launch_eval<MODE, true, true>(k, units, block, vec, eval, s);
    else if (sbx) launch_eval<MODE, true, false>(k, units, block, vec, eval, s);
    else if (pm) launch_eval<MODE, false, true>(k, units, block, vec, eval, s);
    else fail(1, "reproduce: nothing to do");
}

template <int MODE>
__global__ void random_reproduce_kernel(double* out, const uint32_t* dst, uint64_t n, uint64_t d,
                                        Rng rng, uint64_t counter, const double* lower,
                                        const double* upper) {
    const uint64_t total = n * d;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = e / d, j = e - i * d;
        const double u = word_to_unit(draw_word<MODE>(rng, counter + e));
        const uint64_t row = dst ? dst[i] : i;
        out[row * d + j] = lower[j] + u * (upper[j] - lower[j]);  // operators.hpp:293
    }
}

template <int MODE>
__global__ void uniform_fill_kernel(double* out, uint64_t count, Rng rng, uint64_t counter) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < count;
         e += (uint64_t)gridDim.x * blockDim.x)
        out[e] = word_to_unit(draw_word<MODE>(rng, counter + e));
}

__global__ void pow_batch_kernel(const double* x, const double* y, uint64_t n, double* out) {
    __shared__ PowSmem s_pow;
    pow_smem_load(s_pow);
    __syncthreads();
    const PowTables T = pow_tables(s_pow);
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x)
        out[e] = pow_like_host(x[e], y[e], T);
}

inline unsigned stream_grid(uint64_t total, int block) {
    uint64_t g = (total + block - 1) / block;
    const uint64_t cap = (uint64_t)kSMs * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

}  // namespace

void launch_reproduce(const ReproArgs& a, cudaStream_t s) {
    require(a.n >= 1 && a.d >= 1, "reproduce: empty population");
    require(a.d < 0xffffffffULL, "reproduce: decision dimension exceeds 32 bits");
    if (a.do_sbx) require(a.n >= 2, "sbx: needs at least two rows");  // operators.hpp:67
    require(a.eval_problem == 0 || (a.m >= 2 && a.m <= (uint64_t)kMaxObj && a.d >= a.m),
            "reproduce: bad objective count for fused evaluation");
    ReproK k{};
    k.pool = a.pool;
    k.src = a.src;
    k.out = a.out;
    k.dst = a.dst;
    k.n = a.n;
    k.d = a.d;
    k.half = a.n / 2;
    k.g_n = a.global_n ? a.global_n : a.n;
    k.g_half = k.g_n / 2;
    k.g_unit0 = a.global_unit0;
    if (a.global_n) require(a.n % 2 == 0 && a.global_n % 2 == 0, "reproduce: sharded launches need an even row count");
    k.rng = a.rng;
    const uint64_t hd = k.g_half * a.d;
    k.c_mc = a.c_sbx;
    k.c_r1 = a.c_sbx + hd;
    k.c_r2 = a.c_sbx + 2 * hd;
    k.c_r3 = a.c_sbx + 3 * hd;
    k.c_mask = a.c_pm;
    k.c_mut = a.c_pm + k.g_n * a.d;
    {
        // stream units: SplitMix64 positions are (counter * GOLDEN) added to mix64(seed); Philox uses the counter
        const uint64_t u = a.rng.mode == 0 ? kGolden : 1ULL;
        const uint64_t c_ref = a.do_sbx ? k.c_mc : k.c_mask;  // block the CTA position refers to
        k.s_base = (a.rng.mode == 0 ? a.rng.base : 0ULL) + c_ref * u;
        k.s_row = a.d * u;
        k.s_gene = u;
        k.dl_r1 = (k.c_r1 - c_ref) * u;
        k.dl_r2 = (k.c_r2 - c_ref) * u;
        k.dl_mask_a = (k.c_mask - c_ref) * u;
        k.dl_mask_b = k.dl_mask_a + k.g_half * a.d * u;  // row half + p of the mask block
        k.dl_mut_a = (k.c_mut - c_ref) * u;
        k.dl_mut_b = k.dl_mut_a + k.g_half * a.d * u;
    }
    k.pc = a.ga.pc;
    k.inv_exp = 1.0 / (a.ga.eta + 1.0);  // operators.hpp:75
    k.xi = a.ga.xi;
    k.narrow_pow = (k.inv_exp >= 0x1.0p-10 && k.inv_exp <= 1.0) ? 1 : 0;
    // H(rate - r4) == 1  <=>  r4 <= rate  <=>  (word >> 11) <= floor(rate * 2^53)   (r4 = k * 2^-53)
    const double rate = a.ga.pm / (double)a.d;  // operators.hpp:133
    k.mask_never = !(rate >= 0.0);
    if (!k.mask_never) {
        const double scaled = rate * 0x1.0p53;
        k.mask_thresh = scaled >= 0x1.0p53 ? ((1ULL << 53) - 1) : (uint64_t)scaled;
        k.mask_top = (uint32_t)(k.mask_thresh >> 32);
    }
    k.lower = a.lower;
    k.upper = a.upper;
    k.m = a.m;
    k.f_out = a.f_out;
    k.f_row0 = a.f_row0;
    k.f_row0_dev = a.f_row0_dev;
    const uint64_t units = a.do_sbx ? k.half + (a.n & 1) : a.n;
    const int vec = row_vec(a.d), block = row_block(a.d);
    if (a.rng.mode == 0)
        launch_mode<0>(k, a.do_sbx, a.do_pm, units, block, vec, a.eval_problem, s);
    else
        launch_mode<1>(k, a.do_sbx, a.do_pm, units, block, vec, a.eval_problem, s);
    TEMO_CUDA(cudaGetLastError());
    if (a.eval_problem != 0) {
        require(a.f_row0_dev == nullptr, "reproduce: device-side row offsets are not supported with fused evaluation");
        launch_dtlz_finish(a.eval_problem, a.f_out, a.n, a.m, a.d, a.f_row0, s);
    }
}

void launch_pow_batch(const double* x, const double* y, uint64_t n, double* out, cudaStream_t s) {
    pow_batch_kernel<<<stream_grid(n, 256), 256, 0, s>>>(x, y, n, out);
    TEMO_CUDA(cudaGetLastError());
}

void launch_random_reproduce(double* out, const uint32_t* dst, uint64_t n, uint64_t d, Rng rng,
                             uint64_t counter, const double* lower, const double* upper,
                             cudaStream_t s) {
    const unsigned g = stream_grid(n * d, 256);
    if (rng.mode == 0)
        random_reproduce_kernel<0><<<g, 256, 0, s>>>(out, dst, n, d, rng, counter, lower, upper);
    else
        random_reproduce_kernel<1><<<g, 256, 0, s>>>(out, dst, n, d, rng, counter, lower, upper);
    TEMO_CUDA(cudaGetLastError());
}

void launch_uniform_fill(double* out, uint64_t count, Rng rng, uint64_t counter, cudaStream_t s) {
    const unsigned g = stream_grid(count, 256);
    if (rng.mode == 0)
        uniform_fill_kernel<0><<<g, 256, 0, s>>>(out, count, rng, counter);
    else
        uniform_fill_kernel<1><<<g, 256, 0, s>>>(out, count, rng, counter);
    TEMO_CUDA(cudaGetLastError());
}

}  // namespace temo_b200
