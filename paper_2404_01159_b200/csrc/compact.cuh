// Order-preserving stream compaction across many CTAs in ONE launch: a CTA draws its tile number from a ticket counter
// (so that every tile it has to wait for belongs to a CTA that already runs), counts its tile of 1024 elements, publishes
// the count, adds up the published counts of the tiles before it and scatters. The last CTA to finish clears the state for
// the next launch. Used for the elite list (valid reference vectors in ascending vector index, selection.hpp:216-217), the
// free-slot list and the archive. (Three launches - count, scan, scatter - before: the selection of a small population is
// a chain of such few-microsecond kernels.)
#pragma once

#include "internal.h"

namespace temo_b200 {

constexpr int kCompactTile = 1024;
constexpr uint32_t kCompactReady = 0x80000000u;

// uint32 words of state for n elements; must be zero before the first launch (compact_state_alloc)
inline size_t compact_state_words(uint64_t n) { return (size_t)((n + kCompactTile - 1) / kCompactTile) + 2; }
inline uint32_t* compact_state_alloc(uint64_t n) {
    uint32_t* p = dev_alloc<uint32_t>(compact_state_words(n));
    TEMO_CUDA(cudaMemset(p, 0, compact_state_words(n) * sizeof(uint32_t)));
    return p;
}

// Pred: __device__ bool operator()(uint64_t i) ; Val: __device__ uint32_t operator()(uint64_t i)
// state: [0] ticket counter, [1] finished CTAs, [2 + t] count of tile t | kCompactReady
template <class Pred, class Val>
__global__ void __launch_bounds__(kCompactTile) compact_kernel(uint64_t n, Pred pred, Val val, uint32_t* state, uint64_t limit,
                                                               uint32_t* out, uint32_t* total) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_tile, s_before, s_count;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        s_tile = atomicAdd(&state[0], 1u);
        s_before = 0;
    }
    __syncthreads();
    const uint32_t tile = s_tile, tiles = gridDim.x;
    const uint64_t i = (uint64_t)tile * kCompactTile + threadIdx.x;
    const bool p = i < n && pred(i);
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
        if (lane == 31) {
            s_count = incl;
            __threadfence();
            atomicExch(&state[2 + tile], incl | kCompactReady);  // publish this tile's count
        }
    }
    // the tiles before this one (all of them belong to CTAs that hold an earlier ticket, i.e. that run or have finished)
    uint32_t before = 0;
    for (uint32_t t = threadIdx.x; t < tile; t += kCompactTile) {
        uint32_t v;
        while (!((v = *reinterpret_cast<volatile uint32_t*>(&state[2 + t])) & kCompactReady)) __nanosleep(20);
        before += v & ~kCompactReady;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) before += __shfl_xor_sync(0xffffffffu, before, off);
    if (lane == 0 && before) atomicAdd(&s_before, before);
    __syncthreads();
    if (p) {
        const uint64_t pos = (uint64_t)s_before + s_warp[warp] + __popc(bal & ((1u << lane) - 1u));
        if (pos < limit) out[pos] = val(i);
    }
    if (threadIdx.x == 0) {
        if (total && tile == tiles - 1) *total = s_before + s_count;
        __threadfence();
        s_tile = atomicAdd(&state[1], 1u);  // finished CTAs before this one
    }
    __syncthreads();
    if (s_tile == tiles - 1) {  // everybody has read what it needed: clear the state for the next launch
        for (uint32_t t = threadIdx.x; t < tiles + 2; t += kCompactTile) state[t] = 0;
    }
}

// state: compact_state_alloc(n' >= n). total (optional) receives the number of kept elements.
template <class Pred, class Val>
void launch_compact(uint64_t n, Pred pred, Val val, uint32_t* state, uint64_t limit, uint32_t* out, uint32_t* total,
                    cudaStream_t s) {
    const uint64_t tiles = (n + kCompactTile - 1) / kCompactTile;
    if (tiles == 0) {
        if (total) TEMO_CUDA(cudaMemsetAsync(total, 0, sizeof(uint32_t), s));
        return;
    }
    compact_kernel<<<(unsigned)tiles, kCompactTile, 0, s>>>(n, pred, val, state, limit, out, total);
}

}  // namespace temo_b200
