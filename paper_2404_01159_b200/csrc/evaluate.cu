// K2 — objective evaluation as bandwidth-bound row reductions.
//
// reference: dtlz_eval (problems.hpp:69-92) behind ProblemInstance::evaluate
// (problems.hpp:252); LSMOP1 is an extension (not in the reference: parity unpinned).
// Algorithmic traffic: 8*n*d bytes read + 8*n*m written.
//
// Two DTLZ paths with bit-identical results (same thread->gene mapping, same reduction tree
// as the epilogue fused into reproduce.cu: common.cuh, canon_chunk_blocks):
//   eval_tma_kernel  persistent CTAs; every warp streams its consecutive blocks of the CTA's rows
//                    through its own shared-memory ring with cp.async.bulk (TMA, SASS UBLKCP) +
//                    mbarrier complete_tx; needs 16-byte aligned rows (d even).
//   eval_ldg_kernel  one CTA per row with plain (128-bit when d is even) loads; any shape.
#include <map>
#include <mutex>

#include "internal.h"
#include "problems.cuh"

namespace temo_b200 {

namespace {

struct EvalK {
    const double* x;
    const uint32_t* rows;
    uint64_t n, d, m;
    double* f;
    uint64_t f_row0;
    const uint32_t* f_row0_dev;
};

template <int PID, int VEC>
__global__ void __launch_bounds__(256) eval_ldg_kernel(const EvalK a) {
    __shared__ double s_red[8];
    __shared__ double s_pos[kMaxObj];
    const uint64_t i = blockIdx.x;
    const uint64_t row = a.rows ? a.rows[i] : i;
    const double* p = a.x + row * a.d;
    double acc = 0.0;
    const uint32_t nvec = (uint32_t)(a.d / VEC);
    const uint32_t cblk = canon_chunk_blocks((nvec + 31) >> 5, blockDim.x >> 5), q_first = (threadIdx.x >> 5) * cblk * 32 + (threadIdx.x & 31);
    for (uint32_t it = 0; it < cblk; ++it) {  // canonical mapping: this warp's consecutive blocks
        const uint32_t q = q_first + it * 32;
        if (q >= nvec) break;
        const uint64_t j0 = (uint64_t)q * VEC;
        double xv[VEC];
        if (VEC == 2) {
            const double2 t = *reinterpret_cast<const double2*>(p + j0);
            xv[0] = t.x;
            xv[VEC - 1] = t.y;
        } else {
            xv[0] = p[j0];
        }
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
            const uint64_t j = j0 + v;
            if (j + 1 >= a.m)
                acc += dtlz_term<PID>(xv[v]);
            else
                s_pos[j] = xv[v];
        }
    }
    const double sum = block_sum<8>(acc, s_red);
    const uint64_t f0 = a.f_row0 + (a.f_row0_dev ? (uint64_t)*a.f_row0_dev : 0);
    dtlz_finish<PID>(sum, s_pos, a.m, a.d, a.f + (f0 + i) * a.m);
}

// ---- TMA path ---------------------------------------------------------------------------------
constexpr int kWarpStageGenes = 640;  // 5 KB per warp and stage: ten 64-gene blocks, the tile of the pair kernel
#ifndef TEMO_EVAL_STAGES
#define TEMO_EVAL_STAGES 2
#endif
#ifndef TEMO_EVAL_CTAS
#define TEMO_EVAL_CTAS 2
#endif
constexpr int kStages = TEMO_EVAL_STAGES;  // per warp; 8 warps x kStages x 5 KB per CTA
constexpr int kEvalSlots = 4;              // rows a CTA's warps may be apart

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_LOOP:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE;\n"
        "bra WAIT_LOOP;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D bulk async copy global -> shared, completion signalled on the mbarrier (TMA unit).
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

struct EvalRowSlot {
    double part[8];        // per-warp totals of the row
    double pos[kMaxObj];   // its position genes
    uint32_t arrived;      // warps that have delivered their total
    uint32_t done;         // rows completed through this slot
};
struct EvalTmaSmem {
    double tile[8][kStages][kWarpStageGenes];
    uint64_t full_bar[8][kStages];
    EvalRowSlot slot[kEvalSlots];
};

// Persistent: CTA c handles rows c, c + grid, ... Every warp streams ITS blocks of those rows (the canonical mapping:
// warp w owns the consecutive blocks [w * cblk, (w + 1) * cblk) of a row) through its own ring of kStages bulk copies
// with its own mbarriers - no CTA barrier anywhere: lane 0 issues the warp's next copy as soon as the warp has drained
// a stage, the warps of a CTA drift apart, and the last of the eight to deliver a row's total adds the totals in
// ascending warp order and leaves {sum, position genes} for eval_finish_kernel. d must be even (16-byte rows).
template <int PID>
__global__ void __launch_bounds__(256) eval_tma_kernel(const EvalK a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    EvalTmaSmem& S = *reinterpret_cast<EvalTmaSmem*>(smem_raw);
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;

    if (threadIdx.x < 8 * kStages) mbar_init(&S.full_bar[threadIdx.x / kStages][threadIdx.x % kStages], 1);
    if (threadIdx.x < kEvalSlots) S.slot[threadIdx.x].arrived = S.slot[threadIdx.x].done = 0;
    if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();  // the only one

    const uint32_t nvec = (uint32_t)(a.d >> 1), nblk = (nvec + 31) >> 5, cblk = canon_chunk_blocks(nblk, 8);
    const uint32_t g_begin = min(w * cblk * 64u, (uint32_t)a.d), g_end = min((w + 1) * cblk * 64u, (uint32_t)a.d);
    const uint32_t nsub = (g_end - g_begin + kWarpStageGenes - 1) / kWarpStageGenes;  // copies per row (0: nothing of the row is ours)
    const uint64_t my_rows = a.n > blockIdx.x ? (a.n - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const uint64_t total = my_rows * nsub;
    const uint32_t m1 = (uint32_t)a.m - 1;
    double* const ring = &S.tile[w][0][0];
    uint64_t* const bars = &S.full_bar[w][0];

    auto issue = [&](uint64_t c) {  // lane 0: start this warp's c-th copy
        const uint64_t local_row = c / nsub;
        const uint32_t sub = (uint32_t)(c - local_row * nsub);
        const uint64_t i = blockIdx.x + local_row * gridDim.x;
        const uint64_t row = a.rows ? a.rows[i] : i;
        const uint32_t g0 = g_begin + sub * kWarpStageGenes;
        const uint32_t genes = min((uint32_t)kWarpStageGenes, g_end - g0);
        const int st = (int)(c % kStages);
        mbar_expect_tx(&bars[st], genes * 8u);
        tma_load_1d(ring + (size_t)st * kWarpStageGenes, a.x + row * a.d + g0, genes * 8u, &bars[st]);
    };
    if (lane == 0)
        for (uint64_t c = 0; c < total && c < (uint64_t)kStages; ++c) issue(c);

    const uint64_t f0 = a.f_row0 + (a.f_row0_dev ? (uint64_t)*a.f_row0_dev : 0);
    uint64_t c = 0;
    for (uint64_t r = 0; r < my_rows; ++r) {
        EvalRowSlot& slot = S.slot[r % kEvalSlots];
        if (lane == 0)  // the slot is free once the row that used it kEvalSlots rows ago has been written out
            while (*reinterpret_cast<volatile uint32_t*>(&slot.done) < (uint32_t)(r / kEvalSlots)) __nanosleep(100);
        __syncwarp();
        double acc = 0.0;
        for (uint32_t sub = 0; sub < nsub; ++sub, ++c) {
            const int st = (int)(c % kStages);
            mbar_wait(&bars[st], (uint32_t)((c / kStages) & 1));
            const uint32_t g0 = g_begin + sub * kWarpStageGenes;
            const uint32_t genes = min((uint32_t)kWarpStageGenes, g_end - g0);
            const double2* tile = reinterpret_cast<const double2*>(ring + (size_t)st * kWarpStageGenes);
            // canonical order: this lane's vectors of the warp's blocks in ascending order
            for (uint32_t t = lane; t < genes / 2; t += 32) {
                const double2 v = tile[t];
                const uint32_t j = g0 + 2 * t;
                if (j >= m1) acc += dtlz_term<PID>(v.x); else slot.pos[j] = v.x;
                if (j + 1 >= m1) acc += dtlz_term<PID>(v.y); else slot.pos[j + 1] = v.y;
            }
            __syncwarp();  // stage drained by the warp
            if (lane == 0 && c + kStages < total) issue(c + kStages);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        uint32_t before = 0;
        if (lane == 0) {
            slot.part[w] = acc;
            __threadfence_block();
            before = atomicAdd(&slot.arrived, 1u);
        }
        before = __shfl_sync(0xffffffffu, before, 0);
        if (before == 7) {  // row complete: leave {sum, position genes} for eval_finish_kernel
            __threadfence_block();
            const uint64_t i = blockIdx.x + r * gridDim.x;
            double* frow = a.f + (f0 + i) * a.m;
            if (lane == 0) {
                const volatile double* part = slot.part;
                double sum = part[0];
#pragma unroll
                for (int k = 1; k < 8; ++k) sum += part[k];
                frow[0] = sum;
            }
            for (uint32_t o = lane + 1; o < a.m; o += 32) frow[o] = *reinterpret_cast<volatile double*>(&slot.pos[o - 1]);
            __syncwarp();
            if (lane == 0) {
                slot.arrived = 0;
                __threadfence_block();
                *reinterpret_cast<volatile uint32_t*>(&slot.done) = (uint32_t)(r / kEvalSlots) + 1;
            }
        }
    }
}

// Narrow rows (450 <= d <= kRowWarpGenes): with eight warps on a row of 8 KB every warp would spend its time on the
// per-row hand-shake. Here a warp takes whole rows: one bulk copy per row into the warp's own ring, the lane walks the
// eight virtual warps' blocks (same canonical order: eight per-lane accumulators, eight butterflies side by side, totals
// added in ascending order), no slot, no atomic, no CTA barrier.
constexpr int kRowWarpGenes = 1536;  // 12 KB rows: still eight warps' rings per SM
constexpr int kRowWarps = 4;         // warps per CTA

template <int PID>
__global__ void __launch_bounds__(kRowWarps * 32) eval_tma_rows_kernel(const EvalK a, uint32_t stage_genes) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* const tiles = reinterpret_cast<double*>(smem_raw);  // kRowWarps x kStages x stage_genes
    __shared__ __align__(8) uint64_t full_bar[kRowWarps][kStages];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x < kRowWarps * kStages) mbar_init(&full_bar[threadIdx.x / kStages][threadIdx.x % kStages], 1);
    if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();  // the only one

    const uint32_t d = (uint32_t)a.d, nvec = d >> 1, nblk = (nvec + 31) >> 5, cblk = canon_chunk_blocks(nblk, 8);
    const uint32_t m1 = (uint32_t)a.m - 1;
    const uint64_t gw = (uint64_t)blockIdx.x * kRowWarps + w, nw = (uint64_t)gridDim.x * kRowWarps;
    const uint64_t my_rows = a.n > gw ? (a.n - gw + nw - 1) / nw : 0;
    double* const ring = tiles + (size_t)w * kStages * stage_genes;
    uint64_t* const bars = &full_bar[w][0];
    auto issue = [&](uint64_t c) {  // lane 0: start the copy of this warp's c-th row
        const uint64_t i = gw + c * nw;
        const uint64_t row = a.rows ? a.rows[i] : i;
        const int st = (int)(c % kStages);
        mbar_expect_tx(&bars[st], d * 8u);
        tma_load_1d(ring + (size_t)st * stage_genes, a.x + row * a.d, d * 8u, &bars[st]);
    };
    if (lane == 0)
        for (uint64_t c = 0; c < my_rows && c < (uint64_t)kStages; ++c) issue(c);
    const uint64_t f0 = a.f_row0 + (a.f_row0_dev ? (uint64_t)*a.f_row0_dev : 0);
    for (uint64_t c = 0; c < my_rows; ++c) {
        const int st = (int)(c % kStages);
        mbar_wait(&bars[st], (uint32_t)((c / kStages) & 1));
        const double* row = ring + (size_t)st * stage_genes;
        const double2* tile = reinterpret_cast<const double2*>(row);
        double acc[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) {  // virtual warp v: blocks [v * cblk, (v + 1) * cblk)
            acc[v] = 0.0;
            for (uint32_t k = 0; k < cblk; ++k) {
                const uint32_t t = (v * cblk + k) * 32 + lane;
                if (t < nvec) {
                    const double2 x = tile[t];
                    const uint32_t j = 2 * t;
                    if (j >= m1) acc[v] += dtlz_term<PID>(x.x);
                    if (j + 1 >= m1) acc[v] += dtlz_term<PID>(x.y);
                }
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
            for (int v = 0; v < 8; ++v) acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], off);
        double sum = acc[0];
#pragma unroll
        for (int v = 1; v < 8; ++v) sum += acc[v];
        double* frow = a.f + (f0 + gw + c * nw) * a.m;  // {sum, position genes} for eval_finish_kernel
        if (lane == 0) frow[0] = sum;
        for (uint32_t o = lane + 1; o < a.m; o += 32) frow[o] = row[o - 1];
        __syncwarp();  // stage drained by the warp
        if (lane == 0 && c + kStages < my_rows) issue(c + kStages);
    }
}

// ---- LSMOP1 --------------------------------------------------------------------------------------
// y_j = (1 + (j + 1) / d) x_j - 10 x_0 over the tail genes, g_i = mean of y^2 over group i (m consecutive groups of
// nk * sublen_i tail genes), objectives like DTLZ1's linear front without the 0.5. The linkage coefficients come from
// a table (lsmop1_coef: one correctly rounded division per gene, done once per d on the host). Reduction order = the
// canonical one of this library (common.cuh), per group: a lane adds its genes of a group in ascending order; xor
// butterfly inside a warp; warp totals in ascending order.
// Measured at n = 2^17, d = 5000 (round 2): 1.19 ms = 4.4 TB/s (the round-1 kernel with scalar loads and a division per
// gene: 1.66 ms). Two alternatives were built, verified bit-identical and dropped: the same sums through the
// cp.async.bulk ring of eval_tma_kernel (2.9 ms: m block reductions and ten CTA barriers per 40 KB row), and the sums
// fused into the pair kernel of reproduce.cu (child gene 0 recomputed per warp, per-group slots): 5.2 ms against
// 2.8 + 1.2 unfused - the extra code pushed the kernel out of the instruction cache (no_instruction stalls 0.2 -> 3.4
// per issue) and over its register budget.
template <int VEC>
__global__ void __launch_bounds__(256) eval_lsmop1_kernel(const EvalK a, const LsmopLayout lay, const double* __restrict__ coef) {
    extern __shared__ __align__(16) unsigned char lsmop_raw[];
    double* part = reinterpret_cast<double*>(lsmop_raw);  // m x blockDim: per-thread partial of every group
    __shared__ double s_red[8];
    __shared__ double s_g[kMaxObj];
    __shared__ uint32_t s_end[kMaxObj + 1];
    const uint32_t m = (uint32_t)a.m, m1 = m - 1, B = blockDim.x;
    for (uint32_t g = threadIdx.x; g < m; g += B) s_end[g] = m1 + lay.start[g + 1];  // first gene after group g
    for (uint32_t g = 0; g < m; ++g) part[g * B + threadIdx.x] = 0.0;
    __syncthreads();
    const uint64_t i = blockIdx.x;
    const uint64_t row = a.rows ? a.rows[i] : i;
    const double* p = a.x + row * a.d;
    const double t0 = 10.0 * p[0];
    uint32_t cur = 0;
    double acc = 0.0;
    const uint32_t nvec = (uint32_t)(a.d / VEC);
    const uint32_t cblk = canon_chunk_blocks((nvec + 31) >> 5, B >> 5), q_first = (threadIdx.x >> 5) * cblk * 32 + (threadIdx.x & 31);
    for (uint32_t it = 0; it < cblk; ++it) {  // canonical mapping: this warp's consecutive blocks
        const uint32_t q = q_first + it * 32;
        if (q >= nvec) break;
        double xv[VEC], cv[VEC];
        if (VEC == 2) {
            const double2 t = *reinterpret_cast<const double2*>(p + 2 * (uint64_t)q);
            const double2 c = __ldg(reinterpret_cast<const double2*>(coef) + q);
            xv[0] = t.x, xv[VEC - 1] = t.y, cv[0] = c.x, cv[VEC - 1] = c.y;
        } else {
            xv[0] = p[q];
            cv[0] = __ldg(coef + q);
        }
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
            const uint32_t j = q * VEC + v;
            if (j < m1) continue;  // position gene
            while (cur < m && j >= s_end[cur]) {
                part[cur * B + threadIdx.x] = acc;
                acc = 0.0;
                ++cur;
            }
            if (cur < m) {
                const double y = cv[v] * xv[v] - t0;
                acc += y * y;
            }
        }
    }
    if (cur < m) part[cur * B + threadIdx.x] = acc;
    for (uint32_t g = 0; g < m; ++g) {
        const double sum = block_sum<8>(part[g * B + threadIdx.x], s_red);
        if (threadIdx.x == 0) s_g[g] = lay.sublen[g] ? sum / (double)lay.sublen[g] / (double)kLsmopNk : 0.0;
    }
    __syncthreads();
    const uint64_t f0 = a.f_row0 + (a.f_row0_dev ? (uint64_t)*a.f_row0_dev : 0);
    double* frow = a.f + (f0 + i) * a.m;
    for (uint64_t o = threadIdx.x; o < a.m; o += blockDim.x) {
        double v = 1.0 + s_g[o];
        for (uint64_t k = 0; k + o + 1 < a.m; ++k) v *= p[k];
        if (o > 0) v *= 1.0 - p[a.m - 1 - o];
        frow[o] = v;
    }
}

// LSMOP1 through per-warp bulk-copy rings (the structure of eval_tma_kernel) for rows of up to 8 x 640 genes: a warp's
// blocks of a row are the same genes in every row, so the group of each of a lane's twenty genes is decided once per
// launch (one bit mask per group the warp touches: the inner loop is branch-free, one predicated add per candidate
// group), and the lane's linkage coefficients stay in registers. x_0 of the next row (it scales the linkage term) is fetched a row ahead. The last warp to deliver
// its group totals adds them in ascending warp order (warps that do not touch a group deliver 0.0, like the idle
// threads of the plain kernel) and writes the objectives. Same bits as the plain kernel. Needs at most kLsmopTouch
// groups per warp (lsmop_tma_touch); everything else goes through the plain kernel.
constexpr int kLsmopTouch = 4;
constexpr int kLsmopVecs = kWarpStageGenes / 64;  // vectors per lane and row
struct LsmopRowSlot {
    double part[kMaxObj][8];  // per-group, per-warp totals
    double pos[kMaxObj];
    uint32_t arrived, done;
};
struct LsmopTmaSmem {
    double tile[8][kStages][kWarpStageGenes];
    uint64_t full_bar[8][kStages];
    LsmopRowSlot slot[kEvalSlots];
    uint32_t end[kMaxObj + 1];
};

template <int TOUCH>  // accumulators per lane = groups a warp's genes may touch (2 or kLsmopTouch)
__global__ void __launch_bounds__(256) eval_lsmop1_tma_kernel(const EvalK a, const LsmopLayout lay, const double* __restrict__ coef) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    LsmopTmaSmem& S = *reinterpret_cast<LsmopTmaSmem*>(smem_raw);
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t m = (uint32_t)a.m, m1 = m - 1;

    if (threadIdx.x < 8 * kStages) mbar_init(&S.full_bar[threadIdx.x / kStages][threadIdx.x % kStages], 1);
    if (threadIdx.x < kEvalSlots) S.slot[threadIdx.x].arrived = S.slot[threadIdx.x].done = 0;
    if (threadIdx.x < m) S.end[threadIdx.x] = m1 + lay.start[threadIdx.x + 1];  // first gene after the group
    if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();  // the only one

    const uint32_t nvec = (uint32_t)(a.d >> 1), nblk = (nvec + 31) >> 5, cblk = canon_chunk_blocks(nblk, 8);
    const uint32_t g_begin = min(w * cblk * 64u, (uint32_t)a.d), g_end = min((w + 1) * cblk * 64u, (uint32_t)a.d);
    const uint32_t genes = g_end - g_begin;  // <= kWarpStageGenes; 0: nothing of the row is ours
    const uint64_t my_rows = a.n > blockIdx.x ? (a.n - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const uint64_t total = genes ? my_rows : 0;
    double* const ring = &S.tile[w][0][0];
    uint64_t* const bars = &S.full_bar[w][0];
    auto group_of = [&](uint32_t j) {  // first group whose end lies beyond gene j (m: beyond the last group)
        uint32_t g = 0;
        while (g < m && j >= S.end[g]) ++g;
        return g;
    };
    const uint32_t grp_lo = group_of(max(g_begin, m1)), grp_hi = genes ? min(group_of(g_end - 1) + 1, m) : grp_lo;
    // this lane's genes: coefficients, and for each accumulator (= group among the groups of this warp) the genes that go
    // into it (bit 2k + v: gene v of the lane's k-th vector); position genes, genes beyond the last group and vectors
    // beyond the row are in no mask
    double2 cf[kLsmopVecs];
    uint32_t in_group[TOUCH];
#pragma unroll
    for (int i = 0; i < TOUCH; ++i) in_group[i] = 0;
    {
        uint32_t cur = group_of(max(g_begin + 2 * lane, m1));
#pragma unroll
        for (int k = 0; k < kLsmopVecs; ++k) {
            const uint32_t t = lane + 32 * k, j = g_begin + 2 * t;
            const bool valid = t < genes / 2;
            cf[k] = valid ? __ldg(reinterpret_cast<const double2*>(coef) + (j >> 1)) : make_double2(0.0, 0.0);
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const uint32_t jj = j + v;
                if (valid && jj >= m1) {
                    while (cur < m && jj >= S.end[cur]) ++cur;
#pragma unroll
                    for (int i = 0; i < TOUCH; ++i)
                        if (cur < m && cur - grp_lo == (uint32_t)i) in_group[i] |= 1u << (2 * k + v);
                }
            }
        }
    }
    const uint32_t ntouch = grp_hi - grp_lo;  // <= TOUCH
    const bool has_pos = g_begin == 0 && 2 * lane < m1;  // this lane's first vector holds position genes

    auto row_of = [&](uint64_t r) {
        const uint64_t i = blockIdx.x + r * gridDim.x;
        return a.rows ? (uint64_t)a.rows[i] : i;
    };
    auto issue = [&](uint64_t c) {  // lane 0: start the copy of this warp's genes of its c-th row
        const int st = (int)(c % kStages);
        mbar_expect_tx(&bars[st], genes * 8u);
        tma_load_1d(ring + (size_t)st * kWarpStageGenes, a.x + row_of(c) * a.d + g_begin, genes * 8u, &bars[st]);
    };
    if (lane == 0)
        for (uint64_t c = 0; c < total && c < (uint64_t)kStages; ++c) issue(c);

    const uint64_t f0 = a.f_row0 + (a.f_row0_dev ? (uint64_t)*a.f_row0_dev : 0);
    double x0_next = my_rows ? a.x[row_of(0) * a.d] : 0.0;
    for (uint64_t r = 0; r < my_rows; ++r) {
        LsmopRowSlot& slot = S.slot[r % kEvalSlots];
        const double t0 = 10.0 * x0_next;
        if (r + 1 < my_rows) x0_next = a.x[row_of(r + 1) * a.d];
        if (lane == 0)
            while (*reinterpret_cast<volatile uint32_t*>(&slot.done) < (uint32_t)(r / kEvalSlots)) __nanosleep(100);
        __syncwarp();
        double acc[TOUCH];
#pragma unroll
        for (int i = 0; i < TOUCH; ++i) acc[i] = 0.0;
        if (genes) {
            const int st = (int)(r % kStages);
            mbar_wait(&bars[st], (uint32_t)((r / kStages) & 1));
            const double2* tile = reinterpret_cast<const double2*>(ring + (size_t)st * kWarpStageGenes);
            if (has_pos) {
                const double2 xv = tile[lane];
                slot.pos[2 * lane] = xv.x;
                if (2 * lane + 1 < m1) slot.pos[2 * lane + 1] = xv.y;
            }
            // branch-free: a predicated add per accumulator (a plain `if` becomes a jump table); a vector beyond the row reads
            // stale shared memory and is in no mask
#pragma unroll
            for (int k = 0; k < kLsmopVecs; ++k) {
                const double2 xv = tile[lane + 32 * k];
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const double y = (v ? cf[k].y : cf[k].x) * (v ? xv.y : xv.x) - t0;
                    const double yy = y * y;
#pragma unroll
                    for (int i = 0; i < TOUCH; ++i)
                        asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %1, %2;\n\tsetp.ne.u32 p, t, 0;\n\t@p add.rn.f64 %0, %0, %3;\n\t}"
                            : "+d"(acc[i])
                            : "r"(in_group[i]), "r"(1u << (2 * k + v)), "d"(yy));
                }
            }
            __syncwarp();  // stage drained by the warp
            if (lane == 0 && r + kStages < total) issue(r + kStages);
        }
        // the warp's total of every group it touches (xor butterfly), 0.0 for the others
        double mine = 0.0;  // lane g keeps the total of group g
#pragma unroll
        for (int i = 0; i < TOUCH; ++i) {
            if ((uint32_t)i < ntouch) {  // warp-uniform
                double v = acc[i];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                if (lane == grp_lo + i) mine = v;
            }
        }
        if (lane < m) slot.part[lane][w] = mine;
        __syncwarp();
        uint32_t before = 0;
        if (lane == 0) {
            __threadfence_block();
            before = atomicAdd(&slot.arrived, 1u);
        }
        before = __shfl_sync(0xffffffffu, before, 0);
        if (before == 7) {  // row complete
            __threadfence_block();
            const uint64_t i = blockIdx.x + r * gridDim.x;
            double* frow = a.f + (f0 + i) * a.m;
            if (lane < m) {
                const volatile double* part = slot.part[lane];
                double sum = part[0];
#pragma unroll
                for (int k = 1; k < 8; ++k) sum += part[k];
                const double gval = lay.sublen[lane] ? sum / (double)lay.sublen[lane] / (double)kLsmopNk : 0.0;
                const volatile double* pos = slot.pos;
                double v = 1.0 + gval;
                for (uint32_t k = 0; k + lane + 1 < m; ++k) v *= pos[k];
                if (lane > 0) v *= 1.0 - pos[m - 1 - lane];
                frow[lane] = v;
            }
            __syncwarp();
            if (lane == 0) {
                slot.arrived = 0;
                __threadfence_block();
                *reinterpret_cast<volatile uint32_t*>(&slot.done) = (uint32_t)(r / kEvalSlots) + 1;
            }
        }
    }
}

// the conditions of eval_lsmop1_tma_kernel: 0 if they do not hold, else the most groups a warp's genes touch
int lsmop_tma_touch(const LsmopLayout& lay, uint64_t d, uint64_t m) {
    const uint32_t nvec = (uint32_t)(d >> 1), nblk = (nvec + 31) >> 5, cblk = canon_chunk_blocks(nblk, 8), m1 = (uint32_t)m - 1;
    if (cblk * 64u > (uint32_t)kWarpStageGenes) return 0;
    uint32_t touch = 1;
    for (uint32_t w = 0; w < 8; ++w) {
        const uint32_t g_begin = std::min<uint32_t>(w * cblk * 64u, (uint32_t)d), g_end = std::min<uint32_t>((w + 1) * cblk * 64u, (uint32_t)d);
        if (g_end <= g_begin) continue;
        auto group_of = [&](uint32_t j) {
            uint32_t g = 0;
            while (g < m && j >= m1 + lay.start[g + 1]) ++g;
            return g;
        };
        const uint32_t lo = group_of(std::max(g_begin, m1)), hi = std::min<uint32_t>(group_of(g_end - 1) + 1, (uint32_t)m);
        if (hi > lo) touch = std::max(touch, hi - lo);
    }
    return touch <= (uint32_t)kLsmopTouch ? (int)touch : 0;
}

// Second half of the TMA path: the streaming kernel leaves {tail sum, position genes} in each objective
// row; one thread per row turns them into objectives. Keeping the cos/sin/pow latency chain out of the
// streaming CTAs is what lets them run at HBM speed.
template <int PID>
__global__ void eval_finish_kernel(double* f, uint64_t n, uint64_t m, uint64_t d, uint64_t f_row0,
                                   const uint32_t* f_row0_dev) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t f0 = f_row0 + (f_row0_dev ? (uint64_t)*f_row0_dev : 0);
    double* frow = f + (f0 + i) * m;
    double pos[kMaxObj];
    const double sum = frow[0];
    for (uint64_t k = 0; k + 1 < m; ++k) pos[k] = frow[1 + k];
    double g;
    if (PID == kDtlz1 || PID == kDtlz3)
        g = 100.0 * ((double)(d - m + 1) + sum);
    else
        g = sum;
    const double half_pi = kPi / 2.0;
    const PowTables T = pow_tables_global();
    for (uint64_t j = 0; j < m; ++j) {  // same arithmetic as dtlz_finish (problems.cuh)
        double v;
        if (PID == kDtlz1) {
            v = 0.5 * (1.0 + g);
            for (uint64_t q = 0; q + j + 1 < m; ++q) v *= pos[q];
            if (j > 0) v *= 1.0 - pos[m - 1 - j];
        } else {
            v = 1.0 + g;
            for (uint64_t q = 0; q + j + 1 < m; ++q) {
                const double p = PID == kDtlz4 ? pow_like_host(pos[q], 100.0, T) : pos[q];
                v *= cos(p * half_pi);
            }
            if (j > 0) {
                const double p = PID == kDtlz4 ? pow_like_host(pos[m - 1 - j], 100.0, T) : pos[m - 1 - j];
                v *= sin(p * half_pi);
            }
        }
        frow[j] = v;
    }
}

int g_eval_tma = 1;  // set_option("eval_tma", 0) sends everything through the one-CTA-per-row kernels (tests)
bool eval_tma_enabled() { return g_eval_tma != 0; }

template <int PID>
void launch_dtlz(const EvalK& k, bool tma, cudaStream_t s) {
    const int vec = row_vec(k.d), block = row_block(k.d);
    if (tma && eval_tma_enabled() && vec == 2 && block == 256 && k.d <= (uint64_t)kRowWarpGenes) {  // one warp per row
        const uint32_t stage_genes = (uint32_t)((k.d + 15) / 16 * 16);
        const size_t smem = (size_t)kRowWarps * kStages * stage_genes * sizeof(double);
        static std::once_flag configured;  // per instantiation; shards of one process may launch concurrently
        std::call_once(configured, [] {
            TEMO_CUDA(cudaFuncSetAttribute(eval_tma_rows_kernel<PID>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(kRowWarps * kStages * kRowWarpGenes * sizeof(double))));
        });
        const uint64_t ctas_per_sm = std::max<uint64_t>(1, std::min<uint64_t>(16, (200u * 1024u) / (smem + 1024)));
        const uint64_t grid = std::min<uint64_t>((uint64_t)kSMs * ctas_per_sm, (k.n + kRowWarps - 1) / kRowWarps);
        eval_tma_rows_kernel<PID><<<(unsigned)grid, kRowWarps * 32, smem, s>>>(k, stage_genes);
        eval_finish_kernel<PID><<<(unsigned)((k.n + 127) / 128), 128, 0, s>>>(k.f, k.n, k.m, k.d, k.f_row0, k.f_row0_dev);
    } else if (tma && eval_tma_enabled() && vec == 2 && block == 256) {
        const size_t smem = sizeof(EvalTmaSmem);
        static std::once_flag configured;
        std::call_once(configured, [] {
            TEMO_CUDA(cudaFuncSetAttribute(eval_tma_kernel<PID>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(EvalTmaSmem)));
        });
        uint64_t grid = (uint64_t)kSMs * TEMO_EVAL_CTAS;
        if (grid > k.n) grid = k.n;
        eval_tma_kernel<PID><<<(unsigned)grid, 256, smem, s>>>(k);
        eval_finish_kernel<PID><<<(unsigned)((k.n + 127) / 128), 128, 0, s>>>(k.f, k.n, k.m, k.d, k.f_row0, k.f_row0_dev);
    } else if (vec == 2) {
        eval_ldg_kernel<PID, 2><<<(unsigned)k.n, block, 0, s>>>(k);
    } else {
        eval_ldg_kernel<PID, 1><<<(unsigned)k.n, block, 0, s>>>(k);
    }
}

}  // namespace

bool set_eval_option(const char* name, long value) {
    if (std::string(name ? name : "") != "eval_tma") return false;
    g_eval_tma = value != 0;
    return true;
}

LsmopLayout lsmop1_layout(uint64_t d, uint64_t m) {
    // LSMOP suite (Cheng et al. 2017): logistic-map group sizes, nk = 5 sub-components.
    LsmopLayout lay{};
    double c[kMaxObj];
    double sum = 0.0;
    c[0] = 3.8 * 0.1 * (1.0 - 0.1);
    for (uint64_t i = 1; i < m; ++i) c[i] = 3.8 * c[i - 1] * (1.0 - c[i - 1]);
    for (uint64_t i = 0; i < m; ++i) sum += c[i];
    lay.start[0] = 0;
    for (uint64_t i = 0; i < m; ++i) {
        lay.sublen[i] = (uint32_t)std::floor(c[i] / sum * (double)(d - m + 1) / (double)kLsmopNk);
        lay.start[i + 1] = lay.start[i] + lay.sublen[i] * kLsmopNk;
    }
    return lay;
}

// Linkage coefficients of LSMOP1, 1 + (j + 1) / d for j < d, as a device table (cached per d; one IEEE division per gene
// on the host, the same expression the CPU restatement evaluates inline).
const double* lsmop1_coef(uint64_t d, cudaStream_t s) {
    static std::mutex mu;
    static std::map<uint64_t, double*> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(d);
    if (it != cache.end()) return it->second;
    std::vector<double> host(d + (d & 1));
    const double dd = (double)d;
    for (uint64_t j = 0; j < d; ++j) host[j] = 1.0 + (double)(j + 1) / dd;
    double* dev = dev_alloc<double>(host.size());
    TEMO_CUDA(cudaMemcpyAsync(dev, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    TEMO_CUDA(cudaStreamSynchronize(s));  // the host vector goes away; once per d
    cache[d] = dev;
    return dev;
}

// {tail sum, position genes} left in the objective rows by a streaming kernel -> objectives (DTLZ1-4)
void launch_dtlz_finish(int problem, double* f, uint64_t n, uint64_t m, uint64_t d, uint64_t f_row0, cudaStream_t s) {
    if (n == 0) return;
    const unsigned grid = (unsigned)((n + 127) / 128);
    switch (problem) {
    case kDtlz1: eval_finish_kernel<kDtlz1><<<grid, 128, 0, s>>>(f, n, m, d, f_row0, nullptr); break;
    case kDtlz2: eval_finish_kernel<kDtlz2><<<grid, 128, 0, s>>>(f, n, m, d, f_row0, nullptr); break;
    case kDtlz3: eval_finish_kernel<kDtlz3><<<grid, 128, 0, s>>>(f, n, m, d, f_row0, nullptr); break;
    case kDtlz4: eval_finish_kernel<kDtlz4><<<grid, 128, 0, s>>>(f, n, m, d, f_row0, nullptr); break;
    default: fail(1, "dtlz finish: not a DTLZ problem");
    }
    TEMO_CUDA(cudaGetLastError());
}

void launch_evaluate(const EvalArgs& a, cudaStream_t s) {
    require(problem_known(a.problem), "evaluate: unknown problem");
    if (a.problem == kToy2 || a.problem == kToy3) {  // make_problem's toy evaluators (problems.hpp:279-294): negated returns
        require(a.m == (a.problem == kToy2 ? 2u : 3u), "make_problem: toy2 has 2 objectives, toy3 has 3");
        launch_env_rollout(a.x, a.rows, a.n, a.d, kToyHidden, a.horizon, a.m, /*negate=*/true, a.f, a.f_row0, a.f_row0_dev, s);
        return;
    }
    if (a.problem <= kDtlz4) require(a.problem >= 1, "dtlz_eval: id must be in 1..4");  // problems.hpp:70
    require(a.m >= 2, "dtlz_eval: m must be at least 2");                                // problems.hpp:71
    require(a.d >= a.m, "dtlz_eval: d must be at least m");                              // problems.hpp:72
    require(a.m <= (uint64_t)kMaxObj, "evaluate: more than 32 objectives are not supported");
    if (a.n == 0) return;
    EvalK k{a.x, a.rows, a.n, a.d, a.m, a.f, a.f_row0, a.f_row0_dev};
    switch (a.problem) {
    case kDtlz1: launch_dtlz<kDtlz1>(k, a.allow_tma, s); break;
    case kDtlz2: launch_dtlz<kDtlz2>(k, a.allow_tma, s); break;
    case kDtlz3: launch_dtlz<kDtlz3>(k, a.allow_tma, s); break;
    case kDtlz4: launch_dtlz<kDtlz4>(k, a.allow_tma, s); break;
    case kLsmop1: {
        const int block = row_block(a.d);
        const size_t smem = (size_t)a.m * block * sizeof(double);
        const double* coef = lsmop1_coef(a.d, s);
        const LsmopLayout lay = lsmop1_layout(a.d, a.m);
        const int touch = a.allow_tma && eval_tma_enabled() && row_vec(a.d) == 2 && block == 256 ? lsmop_tma_touch(lay, a.d, a.m) : 0;
        if (touch) {
            static std::once_flag configured;
            std::call_once(configured, [] {
                TEMO_CUDA(cudaFuncSetAttribute(eval_lsmop1_tma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LsmopTmaSmem)));
                TEMO_CUDA(cudaFuncSetAttribute(eval_lsmop1_tma_kernel<kLsmopTouch>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LsmopTmaSmem)));
            });
            const uint64_t grid = std::min<uint64_t>((uint64_t)kSMs * TEMO_EVAL_CTAS, a.n);
            if (touch <= 2)
                eval_lsmop1_tma_kernel<2><<<(unsigned)grid, 256, sizeof(LsmopTmaSmem), s>>>(k, lay, coef);
            else
                eval_lsmop1_tma_kernel<kLsmopTouch><<<(unsigned)grid, 256, sizeof(LsmopTmaSmem), s>>>(k, lay, coef);
        } else if (smem > 48 * 1024 && ([&] {  // m x block partials beyond the default dynamic shared memory (m > 24)
                       static std::once_flag configured;
                       std::call_once(configured, [] {
                           const int most = kMaxObj * 256 * (int)sizeof(double);
                           TEMO_CUDA(cudaFuncSetAttribute(eval_lsmop1_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, most));
                           TEMO_CUDA(cudaFuncSetAttribute(eval_lsmop1_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, most));
                       });
                       return false;
                   })()) {
        } else if (row_vec(a.d) == 2)
            eval_lsmop1_kernel<2><<<(unsigned)a.n, block, smem, s>>>(k, lsmop1_layout(a.d, a.m), coef);
        else
            eval_lsmop1_kernel<1><<<(unsigned)a.n, block, smem, s>>>(k, lsmop1_layout(a.d, a.m), coef);
        break;
    }
    }
    TEMO_CUDA(cudaGetLastError());
}

}  // namespace temo_b200
