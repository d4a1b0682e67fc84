// Order-preserving stream compaction across many CTAs (three tiny launches): count per tile of
// 1024 elements -> exclusive scan of the tile counts (one CTA) -> scatter. Used for the elite list
// (valid reference vectors in ascending vector index, selection.hpp:216-217) and the free-slot list.
#pragma once

#include "internal.h"

namespace temo_b200 {

constexpr int kCompactTile = 1024;

// Pred: __device__ bool operator()(uint64_t i) ; Val: __device__ uint32_t operator()(uint64_t i)
template <class Pred>
__global__ void __launch_bounds__(kCompactTile) compact_count_kernel(uint64_t n, Pred pred, uint32_t* tile_count) {
    const uint64_t i = blockIdx.x * (uint64_t)kCompactTile + threadIdx.x;
    const int c = __syncthreads_count(i < n && pred(i));
    if (threadIdx.x == 0) tile_count[blockIdx.x] = (uint32_t)c;
}

// exclusive scan in place over `tiles` counts (tiles <= 1024 * 1024); writes the total to *total
static __global__ void __launch_bounds__(1024) compact_scan_kernel(uint32_t* tile_count, uint64_t tiles, uint32_t* total) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t base = 0; base < tiles; base += 1024) {
        const uint64_t i = base + threadIdx.x;
        const uint32_t v = i < tiles ? tile_count[i] : 0;
        uint32_t incl = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += o;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = s_warp[lane];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, w, off);
                if (lane >= off) w += o;
            }
            s_warp[lane] = w;
        }
        __syncthreads();
        const uint32_t carry = s_carry;
        if (i < tiles) tile_count[i] = carry + incl - v + (warp ? s_warp[warp - 1] : 0);
        __syncthreads();
        if (threadIdx.x == 1023) s_carry = carry + incl + (warp ? s_warp[warp - 1] : 0);
        __syncthreads();
    }
    if (threadIdx.x == 0 && total) *total = s_carry;
}

template <class Pred, class Val>
__global__ void __launch_bounds__(kCompactTile) compact_scatter_kernel(uint64_t n, Pred pred, Val val,
                                                                      const uint32_t* tile_offset, uint64_t limit,
                                                                      uint32_t* out) {
    __shared__ uint32_t s_warp[32];
    const uint64_t i = blockIdx.x * (uint64_t)kCompactTile + threadIdx.x;
    const bool p = i < n && pred(i);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned bal = __ballot_sync(0xffffffffu, p);
    if (lane == 0) s_warp[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
        uint32_t w = s_warp[lane], incl = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += o;
        }
        s_warp[lane] = incl - w;  // exclusive
    }
    __syncthreads();
    if (p) {
        const uint64_t pos = (uint64_t)tile_offset[blockIdx.x] + s_warp[warp] + __popc(bal & ((1u << lane) - 1u));
        if (pos < limit) out[pos] = val(i);
    }
}

// tile_scratch: >= ceil(n / 1024) uint32. total (optional) receives the number of kept elements.
template <class Pred, class Val>
void launch_compact(uint64_t n, Pred pred, Val val, uint32_t* tile_scratch, uint64_t limit, uint32_t* out, uint32_t* total,
                    cudaStream_t s) {
    const uint64_t tiles = (n + kCompactTile - 1) / kCompactTile;
    compact_count_kernel<<<(unsigned)tiles, kCompactTile, 0, s>>>(n, pred, tile_scratch);
    compact_scan_kernel<<<1, 1024, 0, s>>>(tile_scratch, tiles, total);
    compact_scatter_kernel<<<(unsigned)tiles, kCompactTile, 0, s>>>(n, pred, val, tile_scratch, limit, out);
}

}  // namespace temo_b200
