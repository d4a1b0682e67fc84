// Quality indicators on the device: igd and the Monte-Carlo hypervolume of
// metrics.hpp, evaluated on objective matrices that already live in HBM so that a run can report its IGD / HV
// trajectory without copying F to the host every generation (fill_metrics, algorithms.hpp:161-180).
//
// Both are exact restatements: igd takes the minimum of squared distances (order independent) whose terms are added
// in ascending objective order without contraction, the square roots are summed in ascending reference-point order
// on the host (metrics.hpp:40-43); hv_mc counts dominated samples, an integer (metrics.hpp:92-113).
#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"

namespace temo_b200 {

namespace {

// metrics.hpp:25-38: one CTA per reference-front point, threads stride the solutions.
__global__ void __launch_bounds__(256) igd_nearest_kernel(const double* __restrict__ f, const uint32_t* __restrict__ n_dev, uint64_t n,
                                                           uint64_t m, const double* __restrict__ f_ref, double* __restrict__ nearest2) {
    __shared__ double part[8];
    const uint64_t i = blockIdx.x;
    if (n_dev) n = *n_dev;
    double ref[kMaxObj];
    for (uint64_t k = 0; k < m; ++k) ref[k] = f_ref[i * m + k];
    double best = INFINITY;
    for (uint64_t j = threadIdx.x; j < n; j += blockDim.x) {
        double s = 0.0;
        for (uint64_t k = 0; k < m; ++k) {
            const double diff = f[j * m + k] - ref[k];
            s += diff * diff;
        }
        if (s < best) best = s;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, best, off);
        if (o < best) best = o;
    }
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w)
            if (part[w] < best) best = part[w];
        nearest2[i] = best;
    }
}

// metrics.hpp:92-113: one warp per sample; sample s uses draws s*m .. s*m+m-1 of RngStream{seed}; a row dominates the
// sample when every objective is <= the sample's. The objectives are divided by `scale` first (fill_metrics,
// algorithms.hpp:171-172); scale == 1 leaves them untouched.
__global__ void __launch_bounds__(256) hv_mc_kernel(const double* __restrict__ f, const uint32_t* __restrict__ n_dev, uint64_t n, uint64_t m,
                                                     const double* __restrict__ lo, const double* __restrict__ ref, double scale,
                                                     int lo_scaled, uint64_t samples, uint64_t base, unsigned long long* __restrict__ hits) {
    const uint64_t s = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31;
    if (s >= samples) return;
    if (n_dev) n = *n_dev;
    double pt[kMaxObj];
    for (uint64_t k = 0; k < m; ++k) {
        const double u = word_to_unit(mix64(base + (s * m + k) * kGolden));
        const double l = lo_scaled ? lo[k] / scale : lo[k];
        pt[k] = l + u * (ref[k] - l);
    }
    bool dominated = false;
    for (uint64_t i0 = 0; i0 < n; i0 += 32) {
        const uint64_t i = i0 + lane;
        bool all_le = i < n;
        if (all_le) {
            for (uint64_t k = 0; k < m; ++k) {
                const double v = scale != 1.0 ? f[i * m + k] / scale : f[i * m + k];
                if (v > pt[k]) {
                    all_le = false;
                    break;
                }
            }
        }
        if (__any_sync(0xffffffffu, all_le)) {
            dominated = true;
            break;
        }
    }
    if (dominated && lane == 0) atomicAdd(hits, 1ULL);
}


// ---- Archive::insert (algorithms.hpp:72-122): the O(n^2) dominance filter ------------------------------------
// a dominates b: a <= b everywhere and a < b somewhere (selection.hpp:240-247)
__device__ __forceinline__ bool dominates_dev(const double* a, const double* b, uint64_t m) {
    bool strict = false;
    for (uint64_t k = 0; k < m; ++k) {
        if (a[k] > b[k]) return false;
        if (a[k] < b[k]) strict = true;
    }
    return strict;
}
__device__ __forceinline__ bool equal_rows(const double* a, const double* b, uint64_t m) {
    for (uint64_t k = 0; k < m; ++k)
        if (!(a[k] == b[k])) return false;
    return true;
}

// One warp per row. Rows [0, n_old) are the archive, [n_old, n_old + n_new) the inserted rows.
//   new row i is dropped when an archive row equals or dominates it, a new row dominates it, or an earlier new row
//   equals it (algorithms.hpp:76-90); an archive row is dropped when a new row dominates it (:91-100).
__global__ void __launch_bounds__(256) archive_filter_kernel(const double* __restrict__ f_old, uint64_t n_old, const double* __restrict__ f_new,
                                                              uint64_t n_new, uint64_t m, unsigned char* __restrict__ keep_old,
                                                              unsigned char* __restrict__ keep_new) {
    const uint64_t row = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31;
    if (row >= n_old + n_new) return;
    double mine[kMaxObj];
    const bool is_new = row >= n_old;
    const uint64_t i = is_new ? row - n_old : row;
    const double* me = (is_new ? f_new : f_old) + i * m;
    for (uint64_t k = 0; k < m; ++k) mine[k] = me[k];
    bool drop = false;
    if (is_new) {
        for (uint64_t j0 = 0; j0 < n_old && !drop; j0 += 32) {
            const uint64_t j = j0 + lane;
            const bool hit = j < n_old && (equal_rows(mine, f_old + j * m, m) || dominates_dev(f_old + j * m, mine, m));
            drop = __any_sync(0xffffffffu, hit);
        }
    }
    for (uint64_t k0 = 0; k0 < n_new && !drop; k0 += 32) {
        const uint64_t k = k0 + lane;
        bool hit = false;
        if (k < n_new && !(is_new && k == i)) {
            const double* fk = f_new + k * m;
            hit = dominates_dev(fk, mine, m) || (is_new && k < i && equal_rows(mine, fk, m));
        }
        drop = __any_sync(0xffffffffu, hit);
    }
    if (lane == 0) (is_new ? keep_new : keep_old)[i] = drop ? 0 : 1;
}

}  // namespace

void launch_archive_filter(const double* f_old, uint64_t n_old, const double* f_new, uint64_t n_new, uint64_t m, unsigned char* keep_old,
                           unsigned char* keep_new, cudaStream_t s) {
    require(m >= 1 && m <= (uint64_t)kMaxObj, "Archive::insert: unsupported objective count");
    const uint64_t rows = n_old + n_new;
    if (rows == 0) return;
    archive_filter_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(f_old, n_old, f_new, n_new, m, keep_old, keep_new);
    TEMO_CUDA(cudaGetLastError());
}

double device_igd(const double* f, const uint32_t* n_dev, uint64_t n, uint64_t m, const double* f_ref, uint64_t n_ref,
                  double* nearest_scratch, cudaStream_t s) {
    require(n >= 1 && n_ref >= 1, "igd: empty set");  // metrics.hpp:22
    require(m >= 1 && m <= (uint64_t)kMaxObj, "igd: unsupported objective count");
    require(n_ref < 0x7fffffffULL, "igd: too many reference points");
    igd_nearest_kernel<<<(unsigned)n_ref, 256, 0, s>>>(f, n_dev, n, m, f_ref, nearest_scratch);
    TEMO_CUDA(cudaGetLastError());
    std::vector<double> nearest(n_ref);
    TEMO_CUDA(cudaMemcpyAsync(nearest.data(), nearest_scratch, n_ref * sizeof(double), cudaMemcpyDeviceToHost, s));
    TEMO_CUDA(cudaStreamSynchronize(s));
    double sum = 0.0;
    for (uint64_t i = 0; i < n_ref; ++i) sum += std::sqrt(nearest[i]);  // metrics.hpp:38-42
    return sum / (double)n_ref;
}

void device_hv_mc_box(const double* f, const uint32_t* n_dev, uint64_t n, uint64_t m, const double* lo_dev, const double* lo_host,
                      bool lo_scaled, const double* ref_dev, const double* ref_host, double scale, uint64_t samples, uint64_t seed,
                      unsigned long long* hits_scratch, double* value, double* std_error, cudaStream_t s) {
    require(samples >= 1, "hv_mc: needs at least one sample");  // metrics.hpp:78
    require(n >= 1, "hv_mc: bad shapes");
    require(m >= 1 && m <= (uint64_t)kMaxObj, "hv_mc: unsupported objective count");
    double volume = 1.0;
    for (uint64_t k = 0; k < m; ++k) {  // metrics.hpp:82-87
        const double l = lo_scaled ? lo_host[k] / scale : lo_host[k];
        const double side = ref_host[k] - l;
        if (side <= 0.0) {
            *value = 0.0;
            if (std_error) *std_error = 0.0;
            return;
        }
        volume *= side;
    }
    TEMO_CUDA(cudaMemsetAsync(hits_scratch, 0, sizeof(unsigned long long), s));
    const unsigned warps = 8;
    hv_mc_kernel<<<(unsigned)((samples + warps - 1) / warps), warps * 32, 0, s>>>(f, n_dev, n, m, lo_dev, ref_dev, scale, lo_scaled ? 1 : 0,
                                                                                samples, mix64(seed), hits_scratch);
    TEMO_CUDA(cudaGetLastError());
    unsigned long long hits = 0;
    TEMO_CUDA(cudaMemcpyAsync(&hits, hits_scratch, sizeof(hits), cudaMemcpyDeviceToHost, s));
    TEMO_CUDA(cudaStreamSynchronize(s));
    const double p = (double)hits / (double)samples;  // metrics.hpp:114-116
    *value = volume * p;
    if (std_error) *std_error = volume * std::sqrt(p * (1.0 - p) / (double)samples);
}

// metrics.hpp:48-66 on a host copy (a sort-based sweep over n x 2 values).
double host_hv_exact_2d(const double* f, uint64_t n, const double* ref, double scale) {
    std::vector<std::pair<double, double>> pts;
    pts.reserve(n);
    for (uint64_t i = 0; i < n; ++i) {
        const double a = scale != 1.0 ? f[2 * i] / scale : f[2 * i], b = scale != 1.0 ? f[2 * i + 1] / scale : f[2 * i + 1];
        if (a <= ref[0] && b <= ref[1]) pts.emplace_back(a, b);
    }
    std::sort(pts.begin(), pts.end());
    double area = 0.0, prev = ref[1];
    for (const auto& [x, y] : pts) {
        if (y < prev) {
            area += (ref[0] - x) * (prev - y);
            prev = y;
        }
    }
    return area;
}

}  // namespace temo_b200
