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
#include <algorithm>
#include <cstdlib>

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
    uint64_t unit0;  // first mating unit of this launch (grid block 0)
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
    int cand_cap;    // pair kernel: mutation-candidate slots per warp and tile (<= kPairCand)
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

// Shared memory of the generic unit (also carved out of the pair kernel's tile for its redo path).
struct GenericSmem {
    double red[8];
    double pos[2][kMaxObj];
    PowSmem pow;
    unsigned char list[8][64];  // per warp: compacted (lane, v) codes of the crossing genes
    double beta[8][64];         // per warp: signed spread factor per (lane, v)
};

// One mating unit (a pair, or the unpaired last row of an odd population) by the whole CTA.
template <int MODE, bool SBX, bool PM, int EVAL, int VEC>
__device__ __forceinline__ void reproduce_unit(const ReproK& a, const uint64_t unit, GenericSmem& G) {
    double* const s_red = G.red;
    double (*const s_pos)[kMaxObj] = G.pos;
    unsigned char (*const s_list)[64] = G.list;
    double (*const s_beta)[64] = G.beta;
    pow_smem_load(G.pow);
    __syncthreads();
    const PowTables T = pow_tables(G.pow);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

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

#ifndef TEMO_REPRO_MIN_BLOCKS
#define TEMO_REPRO_MIN_BLOCKS 4
#endif
template <int MODE, bool SBX, bool PM, int EVAL, int VEC>
__global__ void __launch_bounds__(256, TEMO_REPRO_MIN_BLOCKS) reproduce_kernel(const ReproK a) {
    __shared__ GenericSmem G;
    reproduce_unit<MODE, SBX, PM, EVAL, VEC>(a, a.unit0 + blockIdx.x, G);
}


// ------------------------------------------------------------------------------------------------
// Fast path: SBX + PM over full mating pairs, 128-bit vectors (d even), 256 threads per pair.
//
// Same arithmetic, same draws, same thread->gene map (warp w owns the 64-gene blocks w, w+8, ... of the
// row; lane l the vector l of a block) as reproduce_unit above, reorganised so that the expensive parts
// run dense and branch-free. Every warp walks its blocks of a row tile in four passes of its own (no CTA
// barrier between them, so the warps of an SM drift apart and their passes overlap):
//   A  hashes only. hr = H(r2 - 0.5) for every gene (operators.hpp:90-91): the crossing genes (about half)
//      are appended to the warp's list in shared memory and beta = 1 is planted for everybody. The quick
//      reject of the mutation mask H(pm/d - r4) (operators.hpp:136) for both children: the few genes that
//      survive it (about one per row) go to the warp's candidate list.
//   B  the crossing list is consumed 32 genes at a time with all lanes busy: Mc, sgn(R1 - 0.5) and the
//      libm-exact pow give the signed spread factor, stored by gene into the beta tile (operators.hpp:85-89).
//   M  the candidate list (rare): exact 53-bit mask test, SBX children of that gene, polynomial mutation
//      (operators.hpp:106-145); the final pair of children is parked in shared memory and the gene's beta is
//      replaced by a tagged NaN pointing at it.
//   C  the streaming pass: 128-bit loads of both parents, blend + clamp (operators.hpp:92-95), a tagged beta
//      swaps in the parked children, fused objective partial sums, 128-bit stores of both children.
// The parent rows are pulled into L2 by the bulk-copy engine (cp.async.bulk.prefetch.L2, SASS UBLKPF) when
// the CTA starts, so HBM streams while passes A and B compute and pass C reads L2 hits.
// A warp with more than kPairCand mutation candidates in one tile (probability ~1e-15 at pm = 1) raises a
// flag and the CTA redoes the pair through reproduce_unit: the result is exact in every case.
constexpr int kPairWarps = 8;
constexpr int kPairBlocks = 10;                              // 64-gene blocks per warp and tile
constexpr int kPairTile = kPairWarps * kPairBlocks * 64;     // genes per tile (5120)
constexpr int kPairCand = 16;                                // mutation candidates per warp and tile
constexpr uint32_t kBetaTagHi = 0x7ff80000u;                 // high word of the tagged NaN

struct PairSmem {
    PowSmem pow;
    double beta[kPairTile];
    unsigned short list[kPairTile];
    double2 side[kPairWarps][kPairCand];  // final children {a, b} of a candidate gene
    unsigned short cand[kPairWarps][kPairCand];
    uint32_t ncand[kPairWarps];
    uint32_t overflow;
    double red[8];
    double pos[2][kMaxObj];
};
static_assert(sizeof(GenericSmem) <= sizeof(double) * kPairTile, "redo path aliases the beta tile");

__device__ __forceinline__ void l2_prefetch_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// mix64 (rng.hpp:23-30) on 32-bit halves; a 64-bit product costs one wide multiply and two multiply-adds.
struct Hash64 {
    uint32_t lo, hi;
};
__device__ __forceinline__ Hash64 mix_round1(uint64_t z) {
    const uint32_t zl = (uint32_t)z, zh = (uint32_t)(z >> 32);
    const uint32_t xl = zl ^ __funnelshift_r(zl, zh, 30), xh = zh ^ (zh >> 30);
    uint32_t pl, ph;
    asm("{\n\t.reg .u64 p;\n\tmul.wide.u32 p, %2, 0x1ce4e5b9;\n\tmov.b64 {%0, %1}, p;\n\t"
        "mad.lo.u32 %1, %3, 0x1ce4e5b9, %1;\n\tmad.lo.u32 %1, %2, 0xbf58476d, %1;\n\t}"
        : "=r"(pl), "=&r"(ph)
        : "r"(xl), "r"(xh));
    Hash64 y;
    y.lo = pl ^ __funnelshift_r(pl, ph, 27);
    y.hi = ph ^ (ph >> 27);
    return y;
}
// top 32 bits of mix64(z) before the last xor-shift (bits 31..1 are those of the word: w = y ^ (y >> 31))
__device__ __forceinline__ uint32_t mix_top(uint64_t z) {
    const Hash64 y = mix_round1(z);
    uint32_t t;
    asm("{\n\tmul.hi.u32 %0, %1, 0x133111eb;\n\tmad.lo.u32 %0, %1, 0x94d049bb, %0;\n\tmad.lo.u32 %0, %2, 0x133111eb, %0;\n\t}"
        : "=&r"(t)
        : "r"(y.lo), "r"(y.hi));
    return t;
}
__device__ __forceinline__ uint64_t mix_full(uint64_t z) {
    const Hash64 y = mix_round1(z);
    uint32_t pl, ph;
    asm("{\n\t.reg .u64 p;\n\tmul.wide.u32 p, %2, 0x133111eb;\n\tmov.b64 {%0, %1}, p;\n\t"
        "mad.lo.u32 %1, %3, 0x133111eb, %1;\n\tmad.lo.u32 %1, %2, 0x94d049bb, %1;\n\t}"
        : "=r"(pl), "=&r"(ph)
        : "r"(y.lo), "r"(y.hi));
    const uint32_t wl = pl ^ __funnelshift_r(pl, ph, 31), wh = ph ^ (ph >> 31);
    return ((uint64_t)wh << 32) | wl;
}
template <int MODE>
__device__ __forceinline__ uint32_t draw_top(uint64_t seed, uint64_t at) {
    return MODE == 0 ? mix_top(at) : (uint32_t)(philox_word(seed, at) >> 32);
}
template <int MODE>
__device__ __forceinline__ uint64_t draw_full(uint64_t seed, uint64_t at) {
    return MODE == 0 ? mix_full(at) : philox_word(seed, at);
}

// SBX blend of one gene (operators.hpp:92-95 as written); beta = 1 returns the parents through the same
// arithmetic as on the CPU. Shared by passes M and C so that both produce the same bits.
__device__ __forceinline__ void sbx_children(double xa, double xb, double beta, double lo, double hi, double& ca,
                                             double& cb) {
    const double p = 1.0 + beta, m = 1.0 - beta;
    ca = clampd((p * xa + m * xb) / 2.0, lo, hi);
    cb = clampd((m * xa + p * xb) / 2.0, lo, hi);
}

// pow for the spread factor outside the narrow fast path (never taken for ordinary eta)
__device__ __noinline__ double pow_spread_slow(double x, double y) { return pow_like_host(x, y, pow_tables_global()); }

// Pass M for one candidate gene (rare, out of line): exact mask tests, live range, mutation of either child.
template <int MODE>
__device__ __noinline__ void mutate_candidate(uint64_t seed, uint64_t pos_ma, uint64_t pos_mb, uint64_t d_mut, uint64_t thresh,
                                              double xi, uint32_t entry, uint32_t j, double xa, double xb, double lo, double hi,
                                              double* beta_slot, double2* side_slot, uint32_t slot) {
    constexpr uint64_t SG = MODE == 0 ? kGolden : 1ULL;
    double ca, cb;
    sbx_children(xa, xb, *beta_slot, lo, hi, ca, cb);
    if (!(hi - lo <= 0.0)) {  // operators.hpp:137
        if (entry & 0x2000u) {
            const uint64_t at = pos_ma + (uint64_t)j * SG;
            ca = mutate_if_selected(ca, draw_full<MODE>(seed, at), draw_full<MODE>(seed, at + d_mut), thresh, lo, hi, xi);
        }
        if (entry & 0x4000u) {
            const uint64_t at = pos_mb + (uint64_t)j * SG;
            cb = mutate_if_selected(cb, draw_full<MODE>(seed, at), draw_full<MODE>(seed, at + d_mut), thresh, lo, hi, xi);
        }
    }
    *side_slot = make_double2(ca, cb);
    *beta_slot = __hiloint2double((int)kBetaTagHi, (int)slot);
}

template <int MODE, int EVAL>
__device__ __noinline__ void redo_pair(const ReproK a, uint64_t unit, GenericSmem& G) {
    reproduce_unit<MODE, true, true, EVAL, 2>(a, unit, G);
}

#ifndef TEMO_PAIR_MIN_BLOCKS
#define TEMO_PAIR_MIN_BLOCKS 3
#endif
// Shared-memory accesses of the pair kernel go through explicit 32-bit shared addresses, and the per-thread
// constants are made opaque to the compiler once: both keep ptxas from re-deriving them (special-register reads,
// window-base arithmetic, 64-bit multiplies) inside the hot loops.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t opaque(uint32_t v) {
    asm volatile("" : "+r"(v));
    return v;
}
template <class P>
__device__ __forceinline__ P* opaque_ptr(P* p) {
    asm volatile("" : "+l"(p));
    return p;
}
__device__ __forceinline__ void sts_f64x2(uint32_t addr, double a, double b) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(a), "d"(b) : "memory");
}
__device__ __forceinline__ void sts_f64(uint32_t addr, double a) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(a) : "memory");
}
__device__ __forceinline__ void sts_u16(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ double2 lds_f64x2(uint32_t addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}

template <int MODE, int EVAL>
__global__ void __launch_bounds__(256, TEMO_PAIR_MIN_BLOCKS) reproduce_pairs_kernel(const ReproK a) {
    extern __shared__ __align__(16) unsigned char pair_smem_raw[];
    PairSmem& S = *reinterpret_cast<PairSmem*>(pair_smem_raw);
    constexpr uint64_t SG = MODE == 0 ? kGolden : 1ULL;  // stream distance of neighbouring genes
    constexpr uint64_t STEP = SG * (uint64_t)(kPairWarps * 64);  // ... of a lane's consecutive blocks
    constexpr uint32_t kBlockBytes = kPairWarps * 64 * 8;  // beta-tile distance of a lane's consecutive blocks
    const uint32_t lane = opaque(threadIdx.x & 31), warp = opaque(threadIdx.x >> 5);

    const uint64_t unit = a.unit0 + blockIdx.x;  // < a.half: always a full pair
    const uint64_t row_a = unit, row_b = a.half + unit;
    const double* pa = a.pool + (a.src ? (uint64_t)a.src[row_a] : row_a) * a.d;
    const double* pb = a.pool + (a.src ? (uint64_t)a.src[row_b] : row_b) * a.d;
    double* oa = a.out + (a.dst ? (uint64_t)a.dst[row_a] : row_a) * a.d;
    double* ob = a.out + (a.dst ? (uint64_t)a.dst[row_b] : row_b) * a.d;
    if (threadIdx.x == 0) {
        l2_prefetch_bulk(pa, (uint32_t)(a.d * 8));
        l2_prefetch_bulk(pb, (uint32_t)(a.d * 8));
        S.overflow = 0;
    }
    pow_smem_load(S.pow);
    __syncthreads();
    const PowTables T = pow_tables(S.pow);

    const uint64_t g_unit = a.g_unit0 + unit;
    const uint64_t seed = a.rng.seed;
    const uint64_t pos = a.s_base + g_unit * a.s_row;  // Mc block position of gene 0 of this pair
    const bool pair_cross = !(word_to_unit(draw_word<MODE>(a.rng, a.c_r3 + g_unit)) - a.pc >= 0.0);  // operators.hpp:82

    const uint32_t nvec = (uint32_t)(a.d >> 1);
    const uint32_t nblk = (nvec + 31) >> 5;  // 64-gene blocks in a row
    const uint32_t lt = opaque((1u << lane) - 1u);
    const uint32_t top_thr = a.mask_never ? 0u : ((a.mask_top << 11) | 0x7ffu);  // (top >> 11) <= mask_top
    // this thread's slots: its vector of the warp's first block in the beta tile, the warp's crossing list
    const uint32_t sm_beta0 = opaque(smem_u32(S.beta) + (warp * 64 + lane * 2) * 8);
    const uint32_t sm_beta_tile = opaque(smem_u32(S.beta));
    const uint32_t sm_list = opaque(smem_u32(S.list) + warp * (kPairBlocks * 64 * 2));
    double acc_a = 0.0, acc_b = 0.0;

    for (uint32_t blk0 = 0; blk0 < nblk; blk0 += kPairWarps * kPairBlocks) {
        const uint32_t q_first = (blk0 + warp) * 32 + lane;  // this lane's vector in the warp's first block
        // blocks of this warp in this tile (warp-uniform)
        const uint32_t left = nblk - blk0 > warp ? (nblk - blk0 - warp + kPairWarps - 1) / kPairWarps : 0u;
        const uint32_t kmax = opaque(min(left, (uint32_t)kPairBlocks));
        // ---- pass A: crossing genes and mutation candidates (hashes only)
        uint32_t total = 0;
        {
            if (lane == 0) S.ncand[warp] = 0;
            __syncwarp();
            const uint64_t first = pos + (uint64_t)(2 * q_first) * SG;
            uint64_t p_r2 = first + a.dl_r2, p_ma = first + a.dl_mask_a, p_mb = first + a.dl_mask_b;
            uint32_t q = q_first, goff = (warp * 64 + lane * 2), sm_b = sm_beta0;
            for (uint32_t k = 0; k < kmax; ++k, p_r2 += STEP, p_ma += STEP, p_mb += STEP, q += kPairWarps * 32,
                          goff += kPairWarps * 64, sm_b += kBlockBytes) {
                const bool valid = q < nvec;
                const bool vc = valid && pair_cross;
                // hr = H(r2 - 0.5) = 0 <=> top bit clear
                const bool c0 = vc & ((int)draw_top<MODE>(seed, p_r2) >= 0);
                const bool c1 = vc & ((int)draw_top<MODE>(seed, p_r2 + SG) >= 0);
                const unsigned b0 = __ballot_sync(0xffffffffu, c0), b1 = __ballot_sync(0xffffffffu, c1);
                sts_f64x2(sm_b, 1.0, 1.0);
                const uint32_t n0 = __popc(b0);
                const uint32_t i0 = total + __popc(b0 & lt), i1 = total + n0 + __popc(b1 & lt);
                if (c0) sts_u16(sm_list + 2 * i0, goff);
                if (c1) sts_u16(sm_list + 2 * i1, goff + 1);
                total += n0 + __popc(b1);
                if (!a.mask_never) {
                    const uint32_t ta0 = draw_top<MODE>(seed, p_ma), ta1 = draw_top<MODE>(seed, p_ma + SG);
                    const uint32_t tb0 = draw_top<MODE>(seed, p_mb), tb1 = draw_top<MODE>(seed, p_mb + SG);
                    if (valid && min(min(ta0, ta1), min(tb0, tb1)) <= top_thr) {  // ~ 4 pm/d of the vectors
                        if (min(ta0, tb0) <= top_thr) {
                            const uint32_t slot = atomicAdd(&S.ncand[warp], 1u);
                            if (slot < (uint32_t)a.cand_cap)
                                S.cand[warp][slot] = (unsigned short)(goff | (ta0 <= top_thr ? 0x2000u : 0u) | (tb0 <= top_thr ? 0x4000u : 0u));
                            else
                                S.overflow = 1;
                        }
                        if (min(ta1, tb1) <= top_thr) {
                            const uint32_t slot = atomicAdd(&S.ncand[warp], 1u);
                            if (slot < (uint32_t)a.cand_cap)
                                S.cand[warp][slot] = (unsigned short)((goff + 1) | (ta1 <= top_thr ? 0x2000u : 0u) | (tb1 <= top_thr ? 0x4000u : 0u));
                            else
                                S.overflow = 1;
                        }
                    }
                }
            }
        }
        __syncwarp();
        // ---- pass B: signed spread factor of the crossing genes, 32 at a time
        {
            const uint64_t pos_tile = pos + (uint64_t)(blk0 * 64) * SG;
            for (uint32_t t = lane; t < total; t += 32) {
                const uint32_t goff = lds_u16(sm_list + 2 * t);
                const uint64_t at = pos_tile + (uint64_t)goff * SG;
                const double mc = word_to_unit(draw_full<MODE>(seed, at));
                const bool up = (int)draw_top<MODE>(seed, at + a.dl_r1) < 0;  // sgn(r1 - 0.5)
                // live spread branch only (hm = H(0.5 - mc)); the other one is multiplied by exactly 0.0
                const bool low = 0.5 - mc >= 0.0;
                const double base = low ? 2.0 * mc : 2.0 - 2.0 * mc;
                const double yexp = low ? a.inv_exp : -a.inv_exp;
                // base is 0 (mc == 0) or in [2^-52, 2]; |y log base| < 2 for any eta >= 0
                double spread;
                if (!(base > 0.0 && a.narrow_pow) || !glibc_pow_main<true>(base, yexp, T, &spread))
                    spread = pow_spread_slow(base, yexp);
                sts_f64(sm_beta_tile + 8 * goff, up ? spread : -spread);
            }
        }
        __syncwarp();
        // ---- pass M: the mutation candidates of this warp (usually none)
        {
            const uint32_t nc = min(S.ncand[warp], (uint32_t)a.cand_cap);
#pragma unroll 1
            for (uint32_t t = lane; t < nc; t += 32) {
                const uint32_t entry = S.cand[warp][t], goff = entry & 0x1fffu, j = blk0 * 64 + goff;
                mutate_candidate<MODE>(seed, pos + a.dl_mask_a, pos + a.dl_mask_b, a.dl_mut_a - a.dl_mask_a, a.mask_thresh, a.xi,
                                       entry, j, pa[j], pb[j], a.lower[j], a.upper[j], &S.beta[goff], &S.side[warp][t], t);
            }
        }
        __syncwarp();
        // ---- pass C: stream the rows
        {
            const uint32_t m1 = (uint32_t)a.m - 1;  // first tail gene (fused evaluation)
            const double2* __restrict__ pa2 = opaque_ptr(reinterpret_cast<const double2*>(pa));
            const double2* __restrict__ pb2 = opaque_ptr(reinterpret_cast<const double2*>(pb));
            double2* __restrict__ oa2 = opaque_ptr(reinterpret_cast<double2*>(oa));
            double2* __restrict__ ob2 = opaque_ptr(reinterpret_cast<double2*>(ob));
            const double2* __restrict__ lo2 = reinterpret_cast<const double2*>(a.lower);
            const double2* __restrict__ hi2 = reinterpret_cast<const double2*>(a.upper);
            const uint32_t sm_side = smem_u32(S.side[warp]);
            uint32_t q = q_first, sm_b = sm_beta0;
#pragma unroll 2
            for (uint32_t k = 0; k < kmax; ++k, q += kPairWarps * 32, sm_b += kBlockBytes) {
                if (q >= nvec) break;  // only in the last block of the row
                const double2 va = pa2[q];
                const double2 vb = pb2[q];
                const double2 vlo = __ldg(lo2 + q);
                const double2 vhi = __ldg(hi2 + q);
                const double2 vbeta = lds_f64x2(sm_b);
                double ca0, cb0, ca1, cb1;
                sbx_children(va.x, vb.x, vbeta.x, vlo.x, vhi.x, ca0, cb0);
                sbx_children(va.y, vb.y, vbeta.y, vlo.y, vhi.y, ca1, cb1);
                if (max(__double2hiint(vbeta.x), __double2hiint(vbeta.y)) >= (int)kBetaTagHi) {  // rare: parked children
                    if (__double2hiint(vbeta.x) >= (int)kBetaTagHi) {
                        const double2 e = lds_f64x2(sm_side + 16 * __double2loint(vbeta.x));
                        ca0 = e.x;
                        cb0 = e.y;
                    }
                    if (__double2hiint(vbeta.y) >= (int)kBetaTagHi) {
                        const double2 e = lds_f64x2(sm_side + 16 * __double2loint(vbeta.y));
                        ca1 = e.x;
                        cb1 = e.y;
                    }
                }
                if (EVAL != 0) {
                    const uint32_t j0 = 2 * q;
                    if (j0 >= m1) {
                        acc_a += dtlz_term<EVAL>(ca0);
                        acc_b += dtlz_term<EVAL>(cb0);
                        acc_a += dtlz_term<EVAL>(ca1);
                        acc_b += dtlz_term<EVAL>(cb1);
                    } else {  // the vector holds a position gene (first block of the row only)
                        S.pos[0][j0] = ca0;
                        S.pos[1][j0] = cb0;
                        if (j0 + 1 >= m1) {
                            acc_a += dtlz_term<EVAL>(ca1);
                            acc_b += dtlz_term<EVAL>(cb1);
                        } else {
                            S.pos[0][j0 + 1] = ca1;
                            S.pos[1][j0 + 1] = cb1;
                        }
                    }
                }
                oa2[q] = make_double2(ca0, ca1);
                ob2[q] = make_double2(cb0, cb1);
            }
        }
        __syncwarp();
    }

    __syncthreads();
    if (S.overflow) {  // a warp ran out of candidate slots: redo the pair the plain way (exact, practically never)
        __syncthreads();
        redo_pair<MODE, EVAL>(a, unit, *reinterpret_cast<GenericSmem*>(S.beta));
        return;
    }
    if (EVAL != 0) {
        const uint64_t f0 = a.f_row0 + (a.f_row0_dev ? (uint64_t)*a.f_row0_dev : 0);
        const double ga = block_sum<8>(acc_a, S.red);
        double* fa = a.f_out + (f0 + row_a) * a.m;
        if (threadIdx.x == 0) fa[0] = ga;
        if (threadIdx.x >= 1 && threadIdx.x < a.m) fa[threadIdx.x] = S.pos[0][threadIdx.x - 1];
        const double gb = block_sum<8>(acc_b, S.red);
        double* fb = a.f_out + (f0 + row_b) * a.m;
        if (threadIdx.x == 0) fb[0] = gb;
        if (threadIdx.x >= 1 && threadIdx.x < a.m) fb[threadIdx.x] = S.pos[1][threadIdx.x - 1];
    }
}

template <int MODE, int EVAL>
void launch_pairs_eval(const ReproK& k, uint64_t units, cudaStream_t s) {
    static bool configured = false;  // per instantiation
    if (!configured) {
        TEMO_CUDA(cudaFuncSetAttribute(reproduce_pairs_kernel<MODE, EVAL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(PairSmem)));
        configured = true;
    }
    reproduce_pairs_kernel<MODE, EVAL><<<(unsigned)units, 256, sizeof(PairSmem), s>>>(k);
}

template <int MODE>
void launch_pairs(const ReproK& k, uint64_t units, int eval, cudaStream_t s) {
    switch (eval) {
    case 0: launch_pairs_eval<MODE, 0>(k, units, s); break;
    case kDtlz1: launch_pairs_eval<MODE, kDtlz1>(k, units, s); break;
    case kDtlz2: launch_pairs_eval<MODE, kDtlz2>(k, units, s); break;
    case kDtlz3: launch_pairs_eval<MODE, kDtlz3>(k, units, s); break;
    case kDtlz4: launch_pairs_eval<MODE, kDtlz4>(k, units, s); break;
    default: fail(1, "reproduce: fused evaluation supports DTLZ1-4 only");
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

// TEMO_B200_GENERIC_K1=1 routes everything through the generic kernel (A/B checks of the two K1 paths)
inline bool force_generic_kernel() {
    static const bool v = [] { const char* e = getenv("TEMO_B200_GENERIC_K1"); return e && e[0] == '1'; }();
    return v;
}

// TEMO_B200_K1_CAND_CAP=<n> shrinks the candidate slots of the pair kernel (0 forces its redo path; tests)
inline int pair_cand_cap() {
    static const int v = [] {
        const char* e = getenv("TEMO_B200_K1_CAND_CAP");
        const int c = e ? atoi(e) : kPairCand;
        return c < 0 ? 0 : (c > kPairCand ? kPairCand : c);
    }();
    return v;
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
    uint64_t units = a.do_sbx ? k.half + (a.n & 1) : a.n;
    const int vec = row_vec(a.d), block = row_block(a.d);
    const auto aligned16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    // Full pairs of wide even rows go through the phased pair kernel when mutation candidates are rare (expected
    // number per warp and tile <= 1); what is left (an odd last row) and every other shape through the generic one.
    const double cand_rate = k.mask_never ? 0.0 : ((double)k.mask_top + 1.0) * 0x1.0p-21;  // P(quick reject passes)
    const double cand_per_warp = 2.0 * (double)std::min<uint64_t>(a.d, kPairTile) / kPairWarps * cand_rate;
    k.cand_cap = pair_cand_cap();
    if (a.do_sbx && a.do_pm && vec == 2 && block == 256 && k.half > 0 && a.d * 8 < (1ULL << 32) && cand_per_warp <= 1.0 &&
        aligned16(a.pool) && aligned16(a.out) && aligned16(a.lower) && aligned16(a.upper) && !force_generic_kernel()) {
        if (a.rng.mode == 0)
            launch_pairs<0>(k, k.half, a.eval_problem, s);
        else
            launch_pairs<1>(k, k.half, a.eval_problem, s);
        TEMO_CUDA(cudaGetLastError());
        k.unit0 = k.half;
        units -= k.half;
    }
    if (units > 0) {
        if (a.rng.mode == 0)
            launch_mode<0>(k, a.do_sbx, a.do_pm, units, block, vec, a.eval_problem, s);
        else
            launch_mode<1>(k, a.do_sbx, a.do_pm, units, block, vec, a.eval_problem, s);
    }
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
