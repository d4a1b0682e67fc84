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
#include <atomic>
#include <cstddef>
#include <mutex>
#include <cstdlib>

#include "glibc_pow_dev.cuh"
#include <type_traits>

#include "internal.h"
#include "problems.cuh"

namespace temo_b200 {

namespace {

struct ReproK {
    const double* pool;
    const double* const* src_ptr;  // optional: address of mating row i's parent (rows of other GPUs' pools: sharded runs)
    const uint32_t* src;
    double* out;
    const uint32_t* dst;
    uint64_t n, d, half;
    uint64_t unit0;     // first mating unit of this launch (grid block 0)
    uint64_t unit_end;  // pair kernel: one past its last unit (<= half)
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
    uint32_t seg_split;          // pair kernel, SEG variant: genes < seg_split have bounds [0], the others [1]
    double seg_lo[2], seg_hi[2];
    // SEG == 1 standing in for two NESTED segments (LSMOP: [0, 1] for the first m - 1 genes inside [0, 10]): pass C clamps
    // every gene to the outer box and the genes below fix_split (all in a row's first block) are clamped again to the inner
    // one afterwards - clamp(clamp(x, outer), inner) = clamp(x, inner) bit for bit. 0: nothing to fix.
    uint32_t fix_split;
    double fix_lo, fix_hi;
    uint64_t m;
    double* f_out;
    uint64_t f_row0;
    const uint32_t* f_row0_dev;
    uint32_t* work_counter;  // pair kernel: pairs handed out beyond the first one of every team (nullptr: static round-robin)
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
    const double* pa = a.src_ptr ? a.src_ptr[row_a] : a.pool + src_a * a.d;
    double* oa = a.out + dst_a * a.d;
    const double* pb = nullptr;
    double* ob = nullptr;
    if (paired) {
        const uint64_t src_b = a.src ? a.src[row_b] : row_b;
        const uint64_t dst_b = a.dst ? a.dst[row_b] : row_b;
        pb = a.src_ptr ? a.src_ptr[row_b] : a.pool + src_b * a.d;
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
    // canonical row mapping (common.cuh): this warp's consecutive blocks
    const uint32_t cblk = canon_chunk_blocks((nvec + 31) >> 5, blockDim.x >> 5), q_first = (uint32_t)warp * cblk * 32 + lane;

    for (uint32_t it = 0; it < cblk; ++it) {  // whole warps stay in the loop
        const uint32_t q = q_first + it * 32;
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
// Fast path: SBX + PM over full mating pairs of even rows — persistent warps, a pair per warp (TEAM = 1: whenever the
// launch has a pair for every resident warp) or per team of eight warps (TEAM = 8: small populations of wide rows).
//
// Same arithmetic, same draws, same thread->gene map (virtual warp w owns the consecutive 64-gene blocks
// [w * cblk, (w + 1) * cblk) of the row, lane l the vector l of a block: common.cuh) and the same reduction order as
// reproduce_unit above, reorganised so that the expensive parts run dense and branch-free and no warp ever waits for
// another one: a warp works through its blocks in tiles of up to kPairBlocks (a single warp walks the eight virtual
// warps of a pair one after the other), each tile in four passes:
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
// There is no CTA barrier after start-up. In a team a warp that finishes its share of a pair leaves its partial sums in
// one of kPairSlots per-pair slots and moves on to the next pair; the last warp to arrive adds the eight
// partials in ascending warp order (the order of block_sum) and writes the objective rows. A single warp flushes the
// sums of each virtual warp into its own slot and writes the rows after the eighth. The warps of an SM
// therefore drift apart and their compute and memory passes overlap. At the start of a tile every warp asks for
// its own parent blocks to be pulled into L2 (prefetch.global.L2; about half of those hints are honoured under
// load), and pass C keeps the parents of the next two blocks in flight in registers.
// A tile with more than kPairCand mutation candidates (probability ~1e-15 at pm = 1) is recomputed by
// tile_plain(), the literal per-gene formulation: the result is exact in every case.
constexpr int kVirtWarps = 8;                                // warps of the canonical row mapping = warps of a team
#ifndef TEMO_PAIR_BLOCKS
#define TEMO_PAIR_BLOCKS 10
#endif
constexpr int kPairBlocks = TEMO_PAIR_BLOCKS;                // 64-gene blocks per warp and tile
constexpr int kTileGenes = kPairBlocks * 64;                 // genes of one warp tile
constexpr int kPairCand = 8;                                 // mutation candidates per warp tile
#ifndef TEMO_PAIR_SLOTS
#define TEMO_PAIR_SLOTS 3
#endif
constexpr int kPairSlots = TEMO_PAIR_SLOTS;                  // pairs a team can have in flight
constexpr uint32_t kBetaTagHi = 0x7ff80000u;                 // high word of the tagged NaN
#ifndef TEMO_PAIR_MIN_BLOCKS
#define TEMO_PAIR_MIN_BLOCKS 3                               // teams per SM
#endif


// Everything a warp needs to know about its current pair (kept in shared memory, not in registers).
struct PairCtx {
    const double* pa;
    const double* pb;
    double* oa;
    double* ob;
    uint64_t pos;    // stream position of (Mc block, gene 0) of this pair
    uint32_t cross;  // pair-level crossover switch hc = H(r3 - pc) == 0 (operators.hpp:82)
    uint32_t pad;
};
#ifndef TEMO_PAIR_SETS
#define TEMO_PAIR_SETS 3                                     // pass C: parent register sets = blocks in flight; 3 applies without fused sums only
#endif
#ifndef TEMO_PAIR_SLEEP
#define TEMO_PAIR_SLEEP 200                                  // ns between two polls of a pair slot that is still in use
#endif
struct WarpSmem {
    double beta[kTileGenes];
    unsigned short list[kTileGenes];
    double2 side[kPairCand];  // final children {a, b} of a candidate gene
    unsigned short cand[kPairCand];
};
struct PairSlot {
    double part[2][kVirtWarps];  // per-warp totals of the two children
    uint32_t arrived;            // warps that have delivered their partials
    uint32_t done;               // pairs completed through this slot
};
#ifndef TEMO_PAIR_RING
#define TEMO_PAIR_RING 4
#endif
constexpr int kUnitRing = TEMO_PAIR_RING;                    // pairs a team's warps may be apart
// CTA geometry of the single-warp pairs (TEAM == 1): warps per CTA and CTAs per SM (the register budget follows)
#ifndef TEMO_SOLO_WARPS
#define TEMO_SOLO_WARPS 8
#endif
#ifndef TEMO_SOLO_CTAS
#define TEMO_SOLO_CTAS 3
#endif
constexpr int kSoloWarps = TEMO_SOLO_WARPS, kSoloCtas = TEMO_SOLO_CTAS;
template <int NW>
struct PairSmemT {
    PowSmem pow;
    WarpSmem w[NW];
    PairSlot slot[kPairSlots];
    // pair hand-out: turn T of this team works on pair ring[T % kUnitRing], described by ringctx[T % kUnitRing] (filled once
    // per pair by the warp that fetched it)
    uint32_t ring[kUnitRing];
    PairCtx ringctx[kUnitRing];
    PairCtx warpctx[NW];    // single-warp pairs (TEAM == 1): every warp describes its own
    PairSlot warpslot[NW];  // ... and collects its own totals
    uint32_t progress[NW];  // turns every warp has finished
    uint32_t claiming, published;   // highest turn being fetched / already published
};

using PairSmem = PairSmemT<kVirtWarps>;
static_assert(sizeof(PairSmem) + 1024 <= (228 * 1024) / TEMO_PAIR_MIN_BLOCKS, "the teams of an SM must fit its shared memory");
static_assert(sizeof(PairSmemT<kSoloWarps>) + 1024 <= (228 * 1024) / kSoloCtas, "the single-warp CTAs of an SM must fit its shared memory");
template <int N> struct ShowSize;
#ifdef TEMO_SHOW_SMEM
ShowSize<sizeof(PairSmem)> show_pair_smem;
#endif

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
// arithmetic as on the CPU. Shared by every pass so that all of them produce the same bits.
__device__ __forceinline__ void sbx_children(double xa, double xb, double beta, double lo, double hi, double& ca,
                                             double& cb) {
    const double p = 1.0 + beta, m = 1.0 - beta;
    ca = clampd((p * xa + m * xb) / 2.0, lo, hi);
    cb = clampd((m * xa + p * xb) / 2.0, lo, hi);
}

// pow for the spread factor outside the narrow fast path (never taken for ordinary eta)
__device__ __noinline__ double pow_spread_slow(double x, double y) { return pow_like_host(x, y, pow_tables_global()); }

// Signed SBX spread factor of a crossing gene: Mc at stream position `at`, R1 at `at + dl_r1` (operators.hpp:85-89).
// Branch-free on the common path so that several genes can be evaluated side by side.
struct SpreadIn {
    double base, yexp;
    bool up;
};
template <int MODE>
__device__ __forceinline__ SpreadIn spread_inputs(uint64_t seed, uint64_t at, uint64_t dl_r1, double inv_exp) {
    SpreadIn s;
    const double mc = word_to_unit(draw_full<MODE>(seed, at));
    s.up = (int)draw_top<MODE>(seed, at + dl_r1) < 0;  // sgn(r1 - 0.5)
    // live spread branch only (hm = H(0.5 - mc)); the other one is multiplied by exactly 0.0
    const bool low = 0.5 - mc >= 0.0;
    s.base = low ? 2.0 * mc : 2.0 - 2.0 * mc;  // 0 (mc == 0) or in [2^-52, 2]; |y log base| < 2 for any eta >= 0
    s.yexp = low ? inv_exp : -inv_exp;
    return s;
}
template <int MODE>
__device__ __forceinline__ double signed_spread(uint64_t seed, uint64_t at, uint64_t dl_r1, double inv_exp, int narrow,
                                                const PowTables& T) {
    const SpreadIn s = spread_inputs<MODE>(seed, at, dl_r1, inv_exp);
    double spread;
    const bool fast = s.base > 0.0 && narrow;
    if (!glibc_pow_narrow_flat(fast ? s.base : 1.0, s.yexp, T, &spread) || !fast) spread = pow_spread_slow(s.base, s.yexp);
    return s.up ? spread : -spread;
}

// Both children of one gene with the mutation applied where the full 53-bit mask test selects it
// (operators.hpp:133-145). hit_a / hit_b: the quick reject let that child through.
template <int MODE>
__device__ __noinline__ double2 mutated_children(uint64_t seed, uint64_t at_ma, uint64_t at_mb, uint64_t d_mut, uint64_t thresh,
                                                 double xi, bool hit_a, bool hit_b, double xa, double xb, double beta,
                                                 double lo, double hi) {
    double ca, cb;
    sbx_children(xa, xb, beta, lo, hi, ca, cb);
    if (!(hi - lo <= 0.0)) {  // operators.hpp:137
        if (hit_a) ca = mutate_if_selected(ca, draw_full<MODE>(seed, at_ma), draw_full<MODE>(seed, at_ma + d_mut), thresh, lo, hi, xi);
        if (hit_b) cb = mutate_if_selected(cb, draw_full<MODE>(seed, at_mb), draw_full<MODE>(seed, at_mb + d_mut), thresh, lo, hi, xi);
    }
    return make_double2(ca, cb);
}

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
__device__ __forceinline__ double lds_f64(uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// Fused evaluation terms of one vector (two genes of both children); the position genes (the first m - 1 of a row) carry
// no term - they are read back from the children's rows when the objective rows are written.
template <int EVAL>
__device__ __forceinline__ void accumulate_vector(uint32_t j0, uint32_t m1, double ca0, double cb0, double ca1, double cb1,
                                                  double& acc_a, double& acc_b) {
    if (EVAL == 0) return;
    if (j0 + 1 >= m1) {
        if (j0 >= m1) {
            acc_a += dtlz_term<EVAL>(ca0);
            acc_b += dtlz_term<EVAL>(cb0);
        }
        acc_a += dtlz_term<EVAL>(ca1);
        acc_b += dtlz_term<EVAL>(cb1);
    }
}

// Pass B of a tile with the general pow (base 0, or an exponent outside the narrow path's range): same list, same stores.
template <int MODE>
__device__ __noinline__ void pass_b_general(const ReproK& a, uint64_t pos_tile, uint32_t total, uint32_t sm_w, uint32_t lane) {
    constexpr uint64_t SG = MODE == 0 ? kGolden : 1ULL;
    constexpr uint32_t kOffList = offsetof(WarpSmem, list);
    for (uint32_t t = lane; t < total; t += 32) {
        const uint32_t e = lds_u16(sm_w + kOffList + 2 * t);
        const uint32_t j = e;
        const SpreadIn s = spread_inputs<MODE>(a.rng.seed, pos_tile + (uint64_t)j * SG, a.dl_r1, a.inv_exp);
        const double p = pow_spread_slow(s.base, s.yexp);
        sts_f64(sm_w + 8 * e, s.up ? p : -p);
    }
}

// Everything the warps of a team need to know about pair `unit`: computed once per pair by the warp that fetched it.
template <int MODE>
__device__ __forceinline__ void fill_pair_ctx(PairCtx& c, const ReproK& a, uint64_t unit) {
    const uint64_t row_a = unit, row_b = a.half + unit, g_unit = a.g_unit0 + unit;
    c.pa = a.src_ptr ? a.src_ptr[row_a] : a.pool + (a.src ? (uint64_t)a.src[row_a] : row_a) * a.d;
    c.pb = a.src_ptr ? a.src_ptr[row_b] : a.pool + (a.src ? (uint64_t)a.src[row_b] : row_b) * a.d;
    c.oa = a.out + (a.dst ? (uint64_t)a.dst[row_a] : row_a) * a.d;
    c.ob = a.out + (a.dst ? (uint64_t)a.dst[row_b] : row_b) * a.d;
    c.pos = a.s_base + g_unit * a.s_row;
    c.cross = !(word_to_unit(draw_word<MODE>(a.rng, a.c_r3 + g_unit)) - a.pc >= 0.0) ? 1u : 0u;  // operators.hpp:82
}

// The literal per-gene formulation of one warp tile (blocks v + 8k of the row tile starting at blk0): used when
// the candidate slots of the phased passes overflow. Same bits, same accumulation order.
template <int MODE, int EVAL>
__device__ __noinline__ void tile_plain(const ReproK& a, uint32_t blk0, uint32_t v, uint32_t kmax, double* acc, const PairCtx* ctx) {
    const PairCtx c = *ctx;
    constexpr uint64_t SG = MODE == 0 ? kGolden : 1ULL;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nvec = (uint32_t)(a.d >> 1), m1 = (uint32_t)a.m - 1;
    const uint32_t top_thr = a.mask_never ? 0u : ((a.mask_top << 11) | 0x7ffu);
    const PowTables T = pow_tables_global();
    double acc_a = acc[0], acc_b = acc[1];
    for (uint32_t k = 0; k < kmax; ++k) {
        const uint32_t q = (blk0 + v + k) * 32 + lane;
        if (q >= nvec) break;
        double xa[2], xb[2], lo[2], hi[2], ca[2], cb[2];
        const double2 va = reinterpret_cast<const double2*>(c.pa)[q], vb = reinterpret_cast<const double2*>(c.pb)[q];
        const double2 vlo = reinterpret_cast<const double2*>(a.lower)[q], vhi = reinterpret_cast<const double2*>(a.upper)[q];
        xa[0] = va.x, xa[1] = va.y, xb[0] = vb.x, xb[1] = vb.y, lo[0] = vlo.x, lo[1] = vlo.y, hi[0] = vhi.x, hi[1] = vhi.y;
        for (int g = 0; g < 2; ++g) {
            const uint64_t at = c.pos + (uint64_t)(2 * q + g) * SG;
            double beta = 1.0;
            if (c.cross && (int)draw_top<MODE>(a.rng.seed, at + a.dl_r2) >= 0)
                beta = signed_spread<MODE>(a.rng.seed, at, a.dl_r1, a.inv_exp, a.narrow_pow, T);
            const bool hit_a = !a.mask_never && draw_top<MODE>(a.rng.seed, at + a.dl_mask_a) <= top_thr;
            const bool hit_b = !a.mask_never && draw_top<MODE>(a.rng.seed, at + a.dl_mask_b) <= top_thr;
            const double2 ch = mutated_children<MODE>(a.rng.seed, at + a.dl_mask_a, at + a.dl_mask_b, a.dl_mut_a - a.dl_mask_a,
                                                      a.mask_thresh, a.xi, hit_a, hit_b, xa[g], xb[g], beta, lo[g], hi[g]);
            ca[g] = ch.x, cb[g] = ch.y;
        }
        accumulate_vector<EVAL>(2 * q, m1, ca[0], cb[0], ca[1], cb[1], acc_a, acc_b);
        reinterpret_cast<double2*>(c.oa)[q] = make_double2(ca[0], ca[1]);
        reinterpret_cast<double2*>(c.ob)[q] = make_double2(cb[0], cb[1]);
    }
    acc[0] = acc_a, acc[1] = acc_b;
}

// TEAM: warps that share a pair. 8: the team of the description above (wide rows). 1: narrow rows - every warp takes whole
// pairs on its own and walks the row's blocks consecutively (a row of d = 1000 is 16 blocks: two per warp of a team, and the
// per-pair and per-tile work of eight warps for them; one warp makes a ten- and a six-block tile of it). Without the fused
// sums only: their canonical order is that of the eight-warp mapping.
template <int MODE, int EVAL, int SEG, int TEAM>  // SEG: 0 bound arrays, 1 one constant segment, 2 two constant segments
__global__ void __launch_bounds__((TEAM == 1 ? kSoloWarps : kVirtWarps) * 32, TEAM == 1 ? kSoloCtas : TEMO_PAIR_MIN_BLOCKS)
    reproduce_pairs_kernel(const __grid_constant__ ReproK a) {
    static_assert(TEAM == kVirtWarps || TEAM == 1, "a pair belongs to a team of eight warps or to one warp");
    constexpr int NW = TEAM == 1 ? kSoloWarps : kVirtWarps;  // warps of the CTA
    extern __shared__ __align__(16) unsigned char pair_smem_raw[];
    PairSmemT<NW>& S = *reinterpret_cast<PairSmemT<NW>*>(pair_smem_raw);
    constexpr uint32_t kVPerWarp = TEAM == 1 && EVAL != 0 ? kVirtWarps : 1;  // virtual warps a warp walks through
    constexpr uint64_t SG = MODE == 0 ? kGolden : 1ULL;            // stream distance of neighbouring genes
    constexpr uint64_t STEP = SG * 64ULL;                           // ... of a lane's consecutive blocks
    constexpr uint32_t kOffList = offsetof(WarpSmem, list), kOffSide = offsetof(WarpSmem, side);
    const uint32_t lane = opaque(threadIdx.x & 31), warp = opaque(threadIdx.x >> 5);
    WarpSmem& W = S.w[warp];

    pow_smem_load(S.pow);
    if (threadIdx.x < kPairSlots) {
        S.slot[threadIdx.x].arrived = 0;
        S.slot[threadIdx.x].done = 0;
    }
    if (threadIdx.x < NW) S.progress[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        S.claiming = S.published = 0;
        if (TEAM != 1 && a.unit0 + blockIdx.x < a.unit_end) fill_pair_ctx<MODE>(S.ringctx[0], a, a.unit0 + blockIdx.x);  // the team's first pair
    }
    __syncthreads();  // the only CTA barrier: from here on every warp is on its own
    const PowTables T = pow_tables(S.pow);

    const uint64_t seed = a.rng.seed;
    const uint32_t nvec = (uint32_t)(a.d >> 1);
    const uint32_t nblk = (nvec + 31) >> 5;  // 64-gene blocks in a row
    // blocks per virtual warp of the canonical row mapping (internal.h); one warp without fused sums takes the row in one go
    const uint32_t cblk = TEAM == 1 && EVAL == 0 ? nblk : canon_chunk_blocks(nblk, kVirtWarps);
    uint32_t lt;  // lanes below this one (kept in a register: an asm volatile result cannot be rematerialised in the loops)
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    const uint32_t top_thr = a.mask_never ? 0u : ((a.mask_top << 11) | 0x7ffu);  // (top >> 11) <= mask_top
    const uint32_t sm_w = opaque(smem_u32(&W)), sm_lane = opaque(smem_u32(&W) + lane * 16);  // beta tile is first in WarpSmem

    uint32_t turn = 0;   // pairs this team has started
    // Pairs are handed out dynamically: the hardware arbiter favours one of the three teams of an SM, so with a fixed
    // share per team the favoured one would leave early and the SM would finish the launch with 16, then 8 warps.
    // A team's first pair is its block index; for every later turn the first warp to get there draws the next pair
    // from a global counter and publishes it to the team through a small ring (the warps of a team are never more
    // than kUnitRing turns apart).
    for (uint64_t unit = a.unit0 + (TEAM == 1 ? blockIdx.x * NW + warp : blockIdx.x); unit < a.unit_end; ++turn) {
        PairSlot& slot = TEAM == 1 ? S.warpslot[warp] : S.slot[turn % kPairSlots];
        const PairCtx& C = TEAM == 1 ? S.warpctx[warp] : S.ringctx[turn % kUnitRing];
        if (TEAM == 1 && lane == 0) fill_pair_ctx<MODE>(S.warpctx[warp], a, unit);
        if (EVAL != 0 && TEAM != 1 && lane == 0)  // the slot is free once the pair that used it kPairSlots turns ago has been written out
            while (*reinterpret_cast<volatile uint32_t*>(&slot.done) < turn / kPairSlots) __nanosleep(TEMO_PAIR_SLEEP);
        __syncwarp();  // also orders the reads of the pair's context behind lane 0's look at the hand-out ring

#pragma unroll 1
        for (uint32_t vv = 0; vv < kVPerWarp; ++vv) {
        const uint32_t v = TEAM == 1 ? vv : warp;
        double acc_a = 0.0, acc_b = 0.0;
        // virtual warp v owns the blocks [v * cblk, (v + 1) * cblk) of the row: a tile is up to kPairBlocks of them
        const uint32_t blk_end = min(nblk, (v + 1) * cblk);
        for (uint32_t blk0 = v * cblk; blk0 < blk_end; blk0 += kPairBlocks) {
            const uint32_t kmax = opaque(min(blk_end - blk0, (uint32_t)kPairBlocks));
            const uint32_t q_first = blk0 * 32 + lane;  // this lane's vector in the tile's first block
            const uint64_t pos = C.pos;
            {   // this warp's parent blocks of this tile into L2 (they are read in pass C)
                const uint32_t kk = lane & 15, blk = blk0 + kk;
                if (kk < kmax && blk < nblk) {
                    const char* p = reinterpret_cast<const char*>(lane < 16 ? C.pa : C.pb) + (uint64_t)blk * 512;
#pragma unroll
                    for (int o = 0; o < 512; o += 128) prefetch_l2(p + o);
                }
            }
            // ---- pass A: crossing genes and mutation candidates (hashes only)
            uint32_t total = 0, ncand = 0;
            {
                const bool cross = C.cross != 0;
                const uint64_t first = pos + (uint64_t)(2 * q_first) * SG;
                uint64_t p_r2 = first + a.dl_r2, p_ma = first + a.dl_mask_a, p_mb = first + a.dl_mask_b;
                uint32_t q = q_first, e = lane * 2, sm_b = sm_lane;
                for (uint32_t k = 0; k < kmax; ++k, p_r2 += STEP, p_ma += STEP, p_mb += STEP, q += 32, e += 64, sm_b += 512) {
                    const bool valid = q < nvec;
                    const bool vc = valid && cross;
                    // hr = H(r2 - 0.5) = 0 <=> top bit clear
                    const bool c0 = vc & ((int)draw_top<MODE>(seed, p_r2) >= 0);
                    const bool c1 = vc & ((int)draw_top<MODE>(seed, p_r2 + SG) >= 0);
                    const unsigned b0 = __ballot_sync(0xffffffffu, c0), b1 = __ballot_sync(0xffffffffu, c1);
                    sts_f64x2(sm_b, 1.0, 1.0);
                    const uint32_t n0 = __popc(b0);
                    const uint32_t i0 = total + __popc(b0 & lt), i1 = total + n0 + __popc(b1 & lt);
                    if (c0) sts_u16(sm_w + kOffList + 2 * i0, e);
                    if (c1) sts_u16(sm_w + kOffList + 2 * i1, e + 1);
                    total += n0 + __popc(b1);
                    if (!a.mask_never) {
                        const uint32_t ta0 = draw_top<MODE>(seed, p_ma), ta1 = draw_top<MODE>(seed, p_ma + SG);
                        const uint32_t tb0 = draw_top<MODE>(seed, p_mb), tb1 = draw_top<MODE>(seed, p_mb + SG);
                        const bool hit = valid && min(min(ta0, ta1), min(tb0, tb1)) <= top_thr;
                        if (__any_sync(0xffffffffu, hit)) {  // ~ 128 pm/d of the blocks
                            const bool h0 = hit && min(ta0, tb0) <= top_thr, h1 = hit && min(ta1, tb1) <= top_thr;
                            const unsigned m0 = __ballot_sync(0xffffffffu, h0), mm1 = __ballot_sync(0xffffffffu, h1);
                            const uint32_t s0 = ncand + __popc(m0 & lt), s1 = ncand + __popc(m0) + __popc(mm1 & lt);
                            if (h0 && s0 < (uint32_t)a.cand_cap)
                                W.cand[s0] = (unsigned short)(e | (ta0 <= top_thr ? 0x2000u : 0u) | (tb0 <= top_thr ? 0x4000u : 0u));
                            if (h1 && s1 < (uint32_t)a.cand_cap)
                                W.cand[s1] = (unsigned short)((e + 1) | (ta1 <= top_thr ? 0x2000u : 0u) | (tb1 <= top_thr ? 0x4000u : 0u));
                            ncand += __popc(m0) + __popc(mm1);
                        }
                    }
                }
            }
            __syncwarp();
            if (ncand > (uint32_t)a.cand_cap) {  // practically never: the literal formulation of this tile
                double acc[2] = {acc_a, acc_b};
                tile_plain<MODE, EVAL>(a, blk0, 0, kmax, acc, &C);
                acc_a = acc[0], acc_b = acc[1];
                __syncwarp();
                continue;
            }
            // ---- pass B: signed spread factor of the crossing genes, 64 at a time
            {
                const uint64_t pos_tile = pos + (uint64_t)(blk0 * 64) * SG;  // gene blk0 * 64
                // Anything off the common path (a base of exactly 0, a result within 2^-54 of 1, an exponent outside the narrow
                // range) only raises `redo`: the general routine then recomputes the tile's list after the loop, so the loop
                // itself carries no call, no fallback selects and no per-iteration look at the launch constants.
                bool redo = !a.narrow_pow;
                const uint32_t inv_hi = (uint32_t)__double2hiint(a.inv_exp), inv_lo = (uint32_t)__double2loint(a.inv_exp);
                for (uint32_t t = lane; t < total; t += 64) {  // two genes per lane: their pow chains interleave
                    const bool two = t + 32 < total;
                    const uint32_t e0 = lds_u16(sm_w + kOffList + 2 * t), e1 = two ? lds_u16(sm_w + kOffList + 2 * t + 64) : e0;
                    // gene index relative to the tile's first gene
                    const uint32_t j0 = e0, j1 = e1;
                    const uint64_t at0 = pos_tile + (uint64_t)j0 * SG, at1 = pos_tile + (uint64_t)j1 * SG;
                    const double mc0 = word_to_unit(draw_full<MODE>(seed, at0)), mc1 = word_to_unit(draw_full<MODE>(seed, at1));
                    const uint32_t r10 = draw_top<MODE>(seed, at0 + a.dl_r1), r11 = draw_top<MODE>(seed, at1 + a.dl_r1);
                    // live spread branch only (hm = H(0.5 - mc)): base 2 mc with exponent 1 / (eta + 1), or 2 - 2 mc with its negative
                    const bool low0 = 0.5 - mc0 >= 0.0, low1 = 0.5 - mc1 >= 0.0;
                    const double b0 = low0 ? 2.0 * mc0 : 2.0 - 2.0 * mc0, b1 = low1 ? 2.0 * mc1 : 2.0 - 2.0 * mc1;
                    const double y0 = __hiloint2double((int)(inv_hi ^ (low0 ? 0u : 0x80000000u)), (int)inv_lo);
                    const double y1 = __hiloint2double((int)(inv_hi ^ (low1 ? 0u : 0x80000000u)), (int)inv_lo);
                    double p0, p1;
                    const bool ok0 = glibc_pow_narrow_flat<true>(b0, y0, T, &p0);
                    const bool ok1 = glibc_pow_narrow_flat<true>(b1, y1, T, &p1);
                    redo |= !(ok0 && ok1) || !(b0 > 0.0) || !(b1 > 0.0);
                    // sgn(r1 - 0.5): the spread factor is positive, so its sign is planted from the draw's top bit
                    const double q0 = __hiloint2double(__double2hiint(p0) ^ (int)(~r10 & 0x80000000u), __double2loint(p0));
                    const double q1 = __hiloint2double(__double2hiint(p1) ^ (int)(~r11 & 0x80000000u), __double2loint(p1));
                    sts_f64(sm_w + 8 * e0, q0);
                    if (two) sts_f64(sm_w + 8 * e1, q1);
                }
                if (__any_sync(0xffffffffu, redo)) pass_b_general<MODE>(a, pos_tile, total, sm_w, lane);
            }
            __syncwarp();
            // ---- pass M: the mutation candidates of this tile (usually none)
#pragma unroll 1
            for (uint32_t t = lane; t < ncand; t += 32) {
                const uint32_t entry = W.cand[t], e = entry & 0x1fffu;
                const uint32_t j = blk0 * 64 + e;
                const uint64_t at = pos + (uint64_t)j * SG;
                const double2 ch = mutated_children<MODE>(seed, at + a.dl_mask_a, at + a.dl_mask_b, a.dl_mut_a - a.dl_mask_a,
                                                          a.mask_thresh, a.xi, (entry & 0x2000u) != 0, (entry & 0x4000u) != 0,
                                                          C.pa[j], C.pb[j], W.beta[e], a.lower[j], a.upper[j]);
                W.side[t] = ch;
                W.beta[e] = __hiloint2double((int)kBetaTagHi, (int)t);
            }
            __syncwarp();
            // ---- pass C: stream the rows
            {
                const uint32_t m1 = (uint32_t)a.m - 1;  // first tail gene (fused evaluation)
                double2* __restrict__ oa2 = reinterpret_cast<double2*>(C.oa);
                double2* __restrict__ ob2 = reinterpret_cast<double2*>(C.ob);
                const double2* __restrict__ lo2 = reinterpret_cast<const double2*>(a.lower);
                const double2* __restrict__ hi2 = reinterpret_cast<const double2*>(a.upper);
                // piecewise-constant bounds from the launch constants (SEG): one side of the split for the whole tile,
                // unless the tile's blocks straddle it
                const uint32_t tile_g0 = blk0 * 64, tile_g1 = (blk0 + kmax) * 64;
                const bool seg_hi_side = tile_g0 >= a.seg_split, seg_mixed = SEG != 0 && !seg_hi_side && tile_g1 > a.seg_split;
                const double seg_lo = a.seg_lo[seg_hi_side ? 1 : 0], seg_hi = a.seg_hi[seg_hi_side ? 1 : 0];
                const double2* __restrict__ pa2 = reinterpret_cast<const double2*>(C.pa);
                const double2* __restrict__ pb2 = reinterpret_cast<const double2*>(C.pb);
                // Two register sets for the parents, used alternately by a loop unrolled by two: block k is blended out of
                // set k & 1, and as soon as its children exist the same registers receive block k + 2 — two blocks are
                // always in flight and no value is ever moved between registers (the rotating three-set form of the earlier
                // kernel spent ~30 of its ~135 instructions per block on moves). One instance of the loop only: a second
                // copy for the tile that holds the bounds split cost more in instruction fetch than the moves it saved
                // (no_instruction stalls 0.2 -> 1.1 per issue), so two-segment bounds (SEG == 2) are selected per gene, behind a
                // warp-uniform branch, in the one tile of a row that holds the split.
                {
                    uint32_t q = q_first, sm_b = sm_lane;
                    const double2 zero2 = make_double2(0.0, 0.0);
                    double2 a0 = q < nvec ? __ldcs(pa2 + q) : zero2, b0 = q < nvec ? __ldcs(pb2 + q) : zero2;
                    double2 a1 = zero2, b1 = zero2;
                    if (kmax > 1 && q + 32 < nvec) {
                        a1 = __ldcs(pa2 + q + 32);
                        b1 = __ldcs(pb2 + q + 32);
                    }
                    // three sets (three blocks in flight) pay without the fused sums only: with them the larger loop body costs
                    // more in instruction fetch than the extra block in flight saves (3.32 vs 3.05 ms)
                    #ifndef TEMO_PAIR_SETS_FUSED
#define TEMO_PAIR_SETS_FUSED 2
#endif
                    constexpr int kSets = EVAL == 0 ? TEMO_PAIR_SETS : TEMO_PAIR_SETS_FUSED;
                    double2 a2 = zero2, b2 = zero2;
                    if constexpr (kSets == 3) {
                        if (kmax > 2 && q + 2 * 32 < nvec) {
                            a2 = __ldcs(pa2 + q + 2 * 32);
                            b2 = __ldcs(pb2 + q + 2 * 32);
                        }
                    }
                    auto block = [&](uint32_t k, double2& pa_v, double2& pb_v) {
                        double lo_x, lo_y, hi_x, hi_y;
                        if (SEG == 1) {
                            lo_x = lo_y = seg_lo, hi_x = hi_y = seg_hi;
                        } else if (SEG == 2) {
                            lo_x = lo_y = seg_lo, hi_x = hi_y = seg_hi;
                            if (seg_mixed) {  // the one tile of a row that holds the split (warp-uniform)
                                const bool sx = 2 * q >= a.seg_split, sy = 2 * q + 1 >= a.seg_split;
                                lo_x = sx ? a.seg_lo[1] : a.seg_lo[0], lo_y = sy ? a.seg_lo[1] : a.seg_lo[0];
                                hi_x = sx ? a.seg_hi[1] : a.seg_hi[0], hi_y = sy ? a.seg_hi[1] : a.seg_hi[0];
                            }
                        } else {
                            const double2 vlo = __ldg(lo2 + q), vhi = __ldg(hi2 + q);
                            lo_x = vlo.x, lo_y = vlo.y, hi_x = vhi.x, hi_y = vhi.y;
                        }
                        const double2 vbeta = lds_f64x2(sm_b);
                        double ca0, cb0, ca1, cb1;
                        sbx_children(pa_v.x, pb_v.x, vbeta.x, lo_x, hi_x, ca0, cb0);
                        sbx_children(pa_v.y, pb_v.y, vbeta.y, lo_y, hi_y, ca1, cb1);
                        {   // the set is free: block k + kSets goes into it
                            const uint32_t qf = q + kSets * 32;
                            if (k + kSets < kmax && qf < nvec) {
                                pa_v = __ldcs(pa2 + qf);
                                pb_v = __ldcs(pb2 + qf);
                            }
                        }
                        if (max(__double2hiint(vbeta.x), __double2hiint(vbeta.y)) >= (int)kBetaTagHi) {  // rare: parked children
                            if (__double2hiint(vbeta.x) >= (int)kBetaTagHi) {
                                const double2 ch = lds_f64x2(sm_w + kOffSide + 16 * __double2loint(vbeta.x));
                                ca0 = ch.x;
                                cb0 = ch.y;
                            }
                            if (__double2hiint(vbeta.y) >= (int)kBetaTagHi) {
                                const double2 ch = lds_f64x2(sm_w + kOffSide + 16 * __double2loint(vbeta.y));
                                ca1 = ch.x;
                                cb1 = ch.y;
                            }
                        }
                        accumulate_vector<EVAL>(2 * q, m1, ca0, cb0, ca1, cb1, acc_a, acc_b);
                        __stcs(oa2 + q, make_double2(ca0, ca1));
                        __stcs(ob2 + q, make_double2(cb0, cb1));
                        q += 32;
                        sm_b += 512;
                    };
                    for (uint32_t k = 0; k < kmax; k += kSets) {
                        if (q >= nvec) break;  // only in the last block of the row
                        block(k, a0, b0);
                        if (k + 1 >= kmax || q >= nvec) break;
                        block(k + 1, a1, b1);
                        if constexpr (kSets == 3) {
                            if (k + 2 >= kmax || q >= nvec) break;
                            block(k + 2, a2, b2);
                        }
                    }
                    if (SEG == 1 && EVAL == 0 && a.fix_split && blk0 == 0 && 2 * lane < a.fix_split) {
                        // the row's first genes belong to the inner box: this lane's own stores of block 0, clamped again
                        double2 ca = oa2[lane], cb = ob2[lane];
                        ca.x = clampd(ca.x, a.fix_lo, a.fix_hi), cb.x = clampd(cb.x, a.fix_lo, a.fix_hi);
                        if (2 * lane + 1 < a.fix_split) ca.y = clampd(ca.y, a.fix_lo, a.fix_hi), cb.y = clampd(cb.y, a.fix_lo, a.fix_hi);
                        oa2[lane] = ca;
                        ob2[lane] = cb;
                    }
                }
            }
            __syncwarp();
        }
        if (EVAL != 0) {
            // this warp's totals (the xor butterfly of block_sum) go into the pair's slot; the last warp to arrive adds
            // the eight totals in ascending warp order and writes the two objective rows
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                acc_a += __shfl_xor_sync(0xffffffffu, acc_a, off);
                acc_b += __shfl_xor_sync(0xffffffffu, acc_b, off);
            }
            uint32_t before = 0;
            if (lane == 0) {
                slot.part[0][v] = acc_a;
                slot.part[1][v] = acc_b;
                if (TEAM != 1) {
                    __threadfence_block();
                    before = atomicAdd(&slot.arrived, 1u);
                }
            }
            if (TEAM == 1) {
                __syncwarp();
                before = v;  // the last virtual warp writes the rows out
            } else {
                before = __shfl_sync(0xffffffffu, before, 0);
            }
            if (before == kVirtWarps - 1) {
                __threadfence_block();
                const uint64_t f0 = a.f_row0 + (a.f_row0_dev ? (uint64_t)*a.f_row0_dev : 0);
                double* fa = a.f_out + (f0 + unit) * a.m;
                double* fb = a.f_out + (f0 + a.half + unit) * a.m;
                if (lane < 2) {
                    const volatile double* part = slot.part[lane];
                    double g = part[0];
#pragma unroll
                    for (int w = 1; w < kVirtWarps; ++w) g += part[w];
                    (lane == 0 ? fa : fb)[0] = g;
                }
                for (uint32_t i = lane + 1; i < a.m; i += 32) {  // the children's position genes, as written by pass C
                    fa[i] = __ldcg(C.oa + (i - 1));
                    fb[i] = __ldcg(C.ob + (i - 1));
                }
                __syncwarp();
                if (TEAM != 1 && lane == 0) {
                    slot.arrived = 0;
                    __threadfence_block();
                    *reinterpret_cast<volatile uint32_t*>(&slot.done) = turn / kPairSlots + 1;
                }
            }
        }
        }  // virtual warps
        __syncwarp();
        if constexpr (TEAM == 1) {  // this warp's next pair
            uint32_t next = 0;
            if (lane == 0) next = a.work_counter ? atomicAdd(a.work_counter, 1u) : turn * gridDim.x * NW + blockIdx.x * NW + warp;
            next = __shfl_sync(0xffffffffu, next, 0);
            unit = a.unit0 + (uint64_t)gridDim.x * NW + next;
            continue;
        }
        // ---- the team's next pair (round-robin over the grid without a work counter)
        uint32_t next = 0;
        if (lane == 0) {
            const uint32_t T = turn + 1;
            *reinterpret_cast<volatile uint32_t*>(&S.progress[warp]) = T;
            for (;;) {
                if (*reinterpret_cast<volatile uint32_t*>(&S.published) >= T) {
                    next = *reinterpret_cast<volatile uint32_t*>(&S.ring[T % kUnitRing]);
                    break;
                }
                if (atomicCAS(&S.claiming, T - 1, T) == T - 1) {  // this warp fetches turn T for the team
                    if (T >= (uint32_t)kUnitRing)                 // the ring entry is free once everybody has finished turn T - kUnitRing
                        for (int w = 0; w < kVirtWarps; ++w)
                            while (*reinterpret_cast<volatile uint32_t*>(&S.progress[w]) + kUnitRing <= T) __nanosleep(100);
                    next = a.work_counter ? atomicAdd(a.work_counter, 1u) : (T - 1) * gridDim.x + blockIdx.x;
                    if (a.unit0 + gridDim.x + next < a.unit_end) fill_pair_ctx<MODE>(S.ringctx[T % kUnitRing], a, a.unit0 + gridDim.x + next);
                    *reinterpret_cast<volatile uint32_t*>(&S.ring[T % kUnitRing]) = next;
                    __threadfence_block();
                    *reinterpret_cast<volatile uint32_t*>(&S.published) = T;
                    break;
                }
                __nanosleep(100);
            }
        }
        next = __shfl_sync(0xffffffffu, next, 0);
        unit = a.unit0 + gridDim.x + next;
    }
}

struct K1Options {
    int generic, bound_arrays, cand_cap;
    int dynamic_pairs;  // pair kernel: pairs handed out through a global counter (1, default) or round-robin (0)
    int single_warp;    // pair kernel, one warp per pair: -1 when the launch has a pair for every resident warp (default), 0 never
                        // (teams of eight warps), 1 always
    int nested_bounds;  // two nested bound segments through the one-segment kernel + fix-up (1, default) or per-gene selects (0)
};
inline int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}
inline K1Options& k1_options() {
    static K1Options o{env_int("TEMO_B200_GENERIC_K1", 0), env_int("TEMO_B200_K1_BOUND_ARRAYS", 0),
                       std::max(0, std::min(kPairCand, env_int("TEMO_B200_K1_CAND_CAP", kPairCand))),
                       env_int("TEMO_B200_K1_DYNAMIC_PAIRS", 1), env_int("TEMO_B200_K1_SINGLE_WARP", -1),
                       env_int("TEMO_B200_K1_NESTED_BOUNDS", 1)};
    return o;
}
inline bool force_generic_kernel() { return k1_options().generic != 0; }
inline bool no_bound_segments() { return k1_options().bound_arrays != 0; }
inline int pair_cand_cap() { return k1_options().cand_cap; }

inline uint32_t* next_work_counter() {
    constexpr unsigned kCounters = 256;
    static std::once_flag once;
    static uint32_t* counters = nullptr;
    static std::atomic<unsigned> next{0};
    std::call_once(once, [] { counters = dev_alloc<uint32_t>(kCounters); });
    return counters + (next.fetch_add(1) % kCounters);
}

template <int MODE, int EVAL, int SEG, int TEAM = kVirtWarps>
void launch_pairs_seg(const ReproK& k, uint64_t units, cudaStream_t s) {
    constexpr int NW = TEAM == 1 ? kSoloWarps : kVirtWarps;
    constexpr int kCtas = TEAM == 1 ? kSoloCtas : TEMO_PAIR_MIN_BLOCKS;
    static int grid = 0;  // per instantiation
    static std::once_flag configured;  // shards of one process may launch concurrently
    std::call_once(configured, [] {
        TEMO_CUDA(cudaFuncSetAttribute(reproduce_pairs_kernel<MODE, EVAL, SEG, TEAM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(PairSmemT<NW>)));
        int dev = 0, sms = 0;
        TEMO_CUDA(cudaGetDevice(&dev));
        TEMO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        grid = (sms > 0 ? sms : kSMs) * kCtas;
    });
    ReproK kk = k;
    kk.work_counter = nullptr;
    if (k1_options().dynamic_pairs) {
        // one zeroed counter per launch out of a small ring (launches of different streams may overlap)
        // (shared by every instantiation and thread of the process: shards of one process launch concurrently)
        kk.work_counter = next_work_counter();
        TEMO_CUDA(cudaMemsetAsync(kk.work_counter, 0, sizeof(uint32_t), s));
    }
    const uint64_t pairs_per_cta = TEAM == 1 ? NW : 1;
    reproduce_pairs_kernel<MODE, EVAL, SEG, TEAM>
        <<<(unsigned)std::min<uint64_t>((units + pairs_per_cta - 1) / pairs_per_cta, (uint64_t)grid), NW * 32, sizeof(PairSmemT<NW>), s>>>(kk);
}

template <int MODE, int EVAL>
void launch_pairs_eval(const ReproK& k, uint64_t units, int seg, int team, cudaStream_t s) {
    if (team == 1) {  // one warp per pair
        switch (seg) {
        case 1: launch_pairs_seg<MODE, EVAL, 1, 1>(k, units, s); break;
        case 2: launch_pairs_seg<MODE, EVAL, 2, 1>(k, units, s); break;
        default: launch_pairs_seg<MODE, EVAL, 0, 1>(k, units, s); break;
        }
        return;
    }
    switch (seg) {
    case 1: launch_pairs_seg<MODE, EVAL, 1>(k, units, s); break;
    case 2: launch_pairs_seg<MODE, EVAL, 2>(k, units, s); break;
    default: launch_pairs_seg<MODE, EVAL, 0>(k, units, s); break;
    }
}

template <int MODE>
void launch_pairs(const ReproK& k, uint64_t units, int eval, int seg, int team, cudaStream_t s) {
    switch (eval) {
    case 0: launch_pairs_eval<MODE, 0>(k, units, seg, team, s); break;
    case kDtlz1: launch_pairs_eval<MODE, kDtlz1>(k, units, seg, team, s); break;
    case kDtlz2: launch_pairs_eval<MODE, kDtlz2>(k, units, seg, team, s); break;
    case kDtlz3: launch_pairs_eval<MODE, kDtlz3>(k, units, seg, team, s); break;
    case kDtlz4: launch_pairs_eval<MODE, kDtlz4>(k, units, seg, team, s); break;
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

// Path-selection knobs of K1 (tests and A/B measurements; temo_b200_set_option, or the environment at start-up):
//   k1_generic       1: everything goes through the generic kernel        TEMO_B200_GENERIC_K1
//   k1_bound_arrays  1: the pair kernel reads the bound arrays even when
//                       they are piecewise constant                       TEMO_B200_K1_BOUND_ARRAYS
//   k1_cand_cap      mutation-candidate slots per warp tile of the pair
//                    kernel, 0..kPairCand (0 forces its plain-tile path)  TEMO_B200_K1_CAND_CAP
//   k1_single_warp   pair kernel with one warp per pair: -1 when the launch
//                    has a pair per resident warp, 0 never, 1 always      TEMO_B200_K1_SINGLE_WARP
//   k1_nested_bounds 1: two nested bound segments go through the
//                    one-segment kernel + fix-up, 0: per-gene selects     TEMO_B200_K1_NESTED_BOUNDS
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
    k.src_ptr = a.src_ptr;
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
    const uint64_t units_all = a.do_sbx ? k.half + (a.n & 1) : a.n;
    require(a.unit_begin <= units_all && a.unit_count <= units_all - a.unit_begin, "reproduce: bad unit range");
    const uint64_t unit_lo = a.unit_begin, unit_hi = a.unit_count ? a.unit_begin + a.unit_count : units_all;
    const int vec = row_vec(a.d), block = row_block(a.d);
    const auto aligned16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    // Full pairs of wide even rows go through the phased pair kernel when mutation candidates are rare (expected
    // number per warp and tile <= 1); what is left (an odd last row) and every other shape through the generic one.
    const double cand_rate = k.mask_never ? 0.0 : ((double)k.mask_top + 1.0) * 0x1.0p-21;  // P(quick reject passes)
    // One warp per pair (narrow rows, no fused sums): when the launch has enough pairs to give every resident warp its own.
    const uint64_t pairs_launched = std::min(unit_hi, k.half) > unit_lo ? std::min(unit_hi, k.half) - unit_lo : 0;
    const bool enough_pairs = pairs_launched >= (uint64_t)kSMs * kSoloCtas * kSoloWarps;
    const int sw = k1_options().single_warp;
    const bool single_warp = sw > 0 || (sw < 0 && enough_pairs);
    const int team = single_warp ? 1 : kVirtWarps;
    // expected mutation candidates per warp tile (the tile's slots overflow into its literal formulation: P(more than 8) is
    // 2e-4 at an expectation of 2, the most a single warp's tile of consecutive blocks can see at pm = 1)
    const double cand_per_warp = 2.0 * (double)std::min<uint64_t>(single_warp && a.eval_problem == 0 ? a.d : (a.d + kVirtWarps - 1) / kVirtWarps + 64, kTileGenes) * cand_rate;
    const double cand_limit = single_warp ? 2.1 : 1.0;
    k.cand_cap = pair_cand_cap();
    uint64_t next = unit_lo;  // first unit not yet launched
    if (a.do_sbx && a.do_pm && vec == 2 && (block == 256 || single_warp) && unit_lo < std::min(unit_hi, k.half) && a.d * 8 < (1ULL << 32) &&
        cand_per_warp <= cand_limit && (a.src_ptr != nullptr || aligned16(a.pool)) && aligned16(a.out) && aligned16(a.lower) && aligned16(a.upper) &&
        !force_generic_kernel()) {
        // bounds as launch constants: 0 arrays, 1 one constant segment (DTLZ), 2 two constant segments (LSMOP)
        int seg = 0;
        if (a.seg.valid && a.seg.split <= a.d && !no_bound_segments()) {
            seg = a.seg.split == 0 || a.seg.split >= a.d ? 1 : 2;
            k.seg_split = (uint32_t)a.seg.split;
            for (int i = 0; i < 2; ++i) {
                const int from = seg == 1 ? (a.seg.split == 0 ? 1 : 0) : i;  // one segment: both entries hold it
                k.seg_lo[i] = a.seg.lo[from], k.seg_hi[i] = a.seg.hi[from];
            }
            // two nested segments whose split lies in the first block, no fused sums: the one-segment kernel + a fix-up
            if (seg == 2 && a.eval_problem == 0 && a.seg.split <= 64 && a.seg.lo[0] >= a.seg.lo[1] && a.seg.hi[0] <= a.seg.hi[1] &&
                k1_options().nested_bounds) {
                seg = 1;
                k.fix_split = (uint32_t)a.seg.split;
                k.fix_lo = a.seg.lo[0], k.fix_hi = a.seg.hi[0];
                k.seg_lo[0] = k.seg_lo[1] = a.seg.lo[1];
                k.seg_hi[0] = k.seg_hi[1] = a.seg.hi[1];
                k.seg_split = 0;
            }
        }
        k.unit0 = unit_lo;
        k.unit_end = std::min(unit_hi, k.half);
        if (a.rng.mode == 0)
            launch_pairs<0>(k, k.unit_end - k.unit0, a.eval_problem, seg, team, s);
        else
            launch_pairs<1>(k, k.unit_end - k.unit0, a.eval_problem, seg, team, s);
        TEMO_CUDA(cudaGetLastError());
        next = k.unit_end;
    }
    if (next < unit_hi) {
        k.unit0 = next;
        const uint64_t units = unit_hi - next;
        if (a.rng.mode == 0)
            launch_mode<0>(k, a.do_sbx, a.do_pm, units, block, vec, a.eval_problem, s);
        else
            launch_mode<1>(k, a.do_sbx, a.do_pm, units, block, vec, a.eval_problem, s);
    }
    TEMO_CUDA(cudaGetLastError());
    if (a.eval_problem != 0) {
        require(a.f_row0_dev == nullptr, "reproduce: device-side row offsets are not supported with fused evaluation");
        if (unit_lo == 0 && unit_hi == units_all) {
            launch_dtlz_finish(a.eval_problem, a.f_out, a.n, a.m, a.d, a.f_row0, s);
        } else if (a.do_sbx) {  // rows p and half + p of the units launched (the unpaired last row is unit `half`)
            const uint64_t pairs_hi = std::min(unit_hi, k.half);
            if (pairs_hi > unit_lo) {
                launch_dtlz_finish(a.eval_problem, a.f_out, pairs_hi - unit_lo, a.m, a.d, a.f_row0 + unit_lo, s);
                launch_dtlz_finish(a.eval_problem, a.f_out, pairs_hi - unit_lo, a.m, a.d, a.f_row0 + k.half + unit_lo, s);
            }
            if (unit_hi > k.half) launch_dtlz_finish(a.eval_problem, a.f_out, 1, a.m, a.d, a.f_row0 + a.n - 1, s);
        } else {
            launch_dtlz_finish(a.eval_problem, a.f_out, unit_hi - unit_lo, a.m, a.d, a.f_row0 + unit_lo, s);
        }
    }
}

bool set_k1_option(const char* name, long value) {
    const std::string key(name ? name : "");
    K1Options& o = k1_options();
    if (key == "k1_generic") o.generic = value != 0;
    else if (key == "k1_bound_arrays") o.bound_arrays = value != 0;
    else if (key == "k1_cand_cap") o.cand_cap = (int)std::max(0L, std::min((long)kPairCand, value));
    else if (key == "k1_dynamic_pairs") o.dynamic_pairs = value != 0;
    else if (key == "k1_single_warp") o.single_warp = value < 0 ? -1 : (value != 0);
    else if (key == "k1_nested_bounds") o.nested_bounds = value != 0;
    else return false;
    return true;
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
