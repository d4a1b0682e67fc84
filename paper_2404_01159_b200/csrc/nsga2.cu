// NSGA-II baseline: nondominated_sort / nsga2_select (selection.hpp:251-346) and the
// generational loop nsga2_run (algorithms.hpp:301-369), the comparison algorithm of the paper.
//
// The population stays in HBM (three n x d buffers: parents, offspring, next parents); reproduction is K1 with the
// tournament winners as its row indirection (no take_rows copy), evaluation is K2 or K1's fused epilogue. The O(n^2 m)
// part of the fast nondominated sort runs on the device: dominator counts once, then fronts are peeled level by level,
// each level testing only (front member, unranked row) pairs, so the total work is the n^2 pair tests of the reference.
// Ranks are integers and dominance is an exact comparison: bit-exact by construction. The crowding distance is a
// sort-based O(n log n) pass over n x m objectives and stays on the host (host_ops.cu: crowding_distance_host).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <vector>

#include "internal.h"
#include "nsga2.h"

namespace temo_b200 {

namespace {

constexpr uint32_t kUnranked = 0xffffffffu;

__device__ __forceinline__ bool dominates_row(const double* a, const double* b, uint64_t m) {  // selection.hpp:240-247
    bool strict = false;
    for (uint64_t k = 0; k < m; ++k) {
        if (a[k] > b[k]) return false;
        if (a[k] < b[k]) strict = true;
    }
    return strict;
}

// count[i] = rows dominating row i (the reference's dom_count, selection.hpp:256-266); one warp per row.
__global__ void __launch_bounds__(256) dom_count_kernel(const double* __restrict__ f, uint64_t n, uint64_t m, uint32_t* __restrict__ count,
                                                         uint32_t* __restrict__ rank) {
    const uint64_t i = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31;
    if (i >= n) return;
    double mine[kMaxObj];
    for (uint64_t k = 0; k < m; ++k) mine[k] = f[i * m + k];
    uint32_t c = 0;
    for (uint64_t j = lane; j < n; j += 32)
        if (j != i && dominates_row(f + j * m, mine, m)) ++c;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    if (lane == 0) {
        count[i] = c;
        rank[i] = kUnranked;
    }
}

// the unranked rows nobody unranked dominates form the next front (selection.hpp:269-281)
__global__ void front_kernel(const uint32_t* __restrict__ count, uint32_t* __restrict__ rank, uint64_t n, uint32_t level,
                             uint32_t* __restrict__ front, uint32_t* __restrict__ n_front) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n || rank[i] != kUnranked || count[i] != 0) return;
    rank[i] = level;
    front[atomicAdd(n_front, 1u)] = (uint32_t)i;
}

// every still unranked row loses the dominators that have just been ranked; one warp per row
__global__ void __launch_bounds__(256) peel_kernel(const double* __restrict__ f, uint64_t n, uint64_t m, const uint32_t* __restrict__ rank,
                                                    const uint32_t* __restrict__ front, const uint32_t* __restrict__ n_front,
                                                    uint32_t* __restrict__ count) {
    const uint64_t j = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31;
    if (j >= n || rank[j] != kUnranked) return;
    double mine[kMaxObj];
    for (uint64_t k = 0; k < m; ++k) mine[k] = f[j * m + k];
    const uint32_t nf = *n_front;
    uint32_t c = 0;
    for (uint32_t a = lane; a < nf; a += 32)
        if (dominates_row(f + (uint64_t)front[a] * m, mine, m)) ++c;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    if (lane == 0 && c) count[j] -= c;
}

__global__ void gather_merged_rows_kernel(const double* __restrict__ parents, const double* __restrict__ offspring, const uint32_t* __restrict__ sel,
                                          uint64_t n, uint64_t d, double* __restrict__ out) {
    const uint64_t k = blockIdx.x;
    const uint32_t e = sel[k];
    const double* p = e < n ? parents + (uint64_t)e * d : offspring + (uint64_t)(e - n) * d;
    for (uint64_t j = threadIdx.x; j < d; j += blockDim.x) out[k * d + j] = p[j];
}

}  // namespace

void SortScratch::alloc(uint64_t rows) {
    release();
    cap = rows;
    count = dev_alloc<uint32_t>(rows);
    rank = dev_alloc<uint32_t>(rows);
    front = dev_alloc<uint32_t>(rows);
    n_front = dev_alloc<uint32_t>(1);
}
void SortScratch::release() {
    cudaFree(count); cudaFree(rank); cudaFree(front); cudaFree(n_front);
    count = rank = front = n_front = nullptr;
    cap = 0;
}

// nondominated_sort (selection.hpp:251-283) of device-resident objectives; ranks go to rank_host.
uint64_t device_nondominated_sort(const double* f, uint64_t n, uint64_t m, SortScratch& sc, uint32_t* rank_host, cudaStream_t s) {
    require(n <= sc.cap, "nondominated_sort: scratch too small");
    require(m >= 1 && m <= (uint64_t)kMaxObj, "nondominated_sort: unsupported objective count");
    require(n < 0xffffffffULL, "nondominated_sort: too many rows");
    if (n == 0) return 0;
    const unsigned warp_grid = (unsigned)((n + 7) / 8), thread_grid = (unsigned)((n + 255) / 256);
    dom_count_kernel<<<warp_grid, 256, 0, s>>>(f, n, m, sc.count, sc.rank);
    uint64_t left = n;
    uint32_t level = 0;
    while (left) {
        TEMO_CUDA(cudaMemsetAsync(sc.n_front, 0, sizeof(uint32_t), s));
        front_kernel<<<thread_grid, 256, 0, s>>>(sc.count, sc.rank, n, level, sc.front, sc.n_front);
        uint32_t nf = 0;
        TEMO_CUDA(cudaMemcpyAsync(&nf, sc.n_front, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        TEMO_CUDA(cudaStreamSynchronize(s));
        require(nf >= 1 && nf <= left, "nondominated_sort: objectives are not comparable (NaN?)");
        left -= nf;
        ++level;
        if (left) peel_kernel<<<warp_grid, 256, 0, s>>>(f, n, m, sc.rank, sc.front, sc.n_front, sc.count);
    }
    TEMO_CUDA(cudaGetLastError());
    TEMO_CUDA(cudaMemcpyAsync(rank_host, sc.rank, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    TEMO_CUDA(cudaStreamSynchronize(s));
    return level;
}

// nsga2_select (selection.hpp:316-346) from the ranks and a host copy of the objectives.
void nsga2_select_host(const double* f, const uint32_t* rank, uint64_t n, uint64_t m, uint64_t target, uint32_t* selected) {
    require(target <= n, "nsga2_select: target exceeds population");
    // rows of every level in ascending row order (a counting sort by rank)
    uint32_t levels = 0;
    for (uint64_t i = 0; i < n; ++i) levels = std::max(levels, rank[i] + 1);
    std::vector<uint64_t> start(levels + 1, 0);
    for (uint64_t i = 0; i < n; ++i) ++start[rank[i] + 1];
    for (uint32_t l = 0; l < levels; ++l) start[l + 1] += start[l];
    std::vector<uint32_t> by_level(n);
    {
        std::vector<uint64_t> at(start.begin(), start.end() - 1);
        for (uint64_t i = 0; i < n; ++i) by_level[at[rank[i]]++] = (uint32_t)i;
    }
    uint64_t cnt = 0;
    for (uint32_t l = 0; l < levels && cnt < target; ++l) {
        const uint32_t* rows = by_level.data() + start[l];
        const uint64_t k = start[l + 1] - start[l];
        if (cnt + k <= target) {
            for (uint64_t a = 0; a < k; ++a) selected[cnt++] = rows[a];
            continue;
        }
        std::vector<double> front(k * m), crowd(k);
        for (uint64_t a = 0; a < k; ++a) std::copy_n(f + (uint64_t)rows[a] * m, m, front.data() + a * m);
        crowding_distance_host(front.data(), k, m, crowd.data());
        std::vector<uint64_t> by(k);
        for (uint64_t a = 0; a < k; ++a) by[a] = a;
        std::sort(by.begin(), by.end(), [&](uint64_t a, uint64_t b) {
            if (crowd[a] != crowd[b]) return crowd[a] > crowd[b];
            return rows[a] < rows[b];
        });
        for (uint64_t a = 0; cnt < target; ++a) selected[cnt++] = rows[by[a]];
    }
}

Nsga2Run::Nsga2Run(const RunConfig& c) : cfg(c) {
    require(cfg.pop >= 2 && cfg.generations >= 1, "nsga2_run: bad config");  // algorithms.hpp:303
    require(problem_known(cfg.problem), "make_problem: unknown problem");
    require(cfg.obj >= 2 && cfg.obj <= (uint64_t)kMaxObj, "nsga2_run: objective count out of range");
    n = cfg.pop;
    m = cfg.obj;
    if (cfg.problem == kToy2 || cfg.problem == kToy3) {  // problems.hpp:279-287: the environment fixes m and d
        m = cfg.problem == kToy2 ? 2 : 3;
        require(cfg.dim == 0 || cfg.dim == problem_default_dim(cfg.problem, m), "make_problem: toy env dimension is fixed");
    }
    d = cfg.dim ? cfg.dim : problem_default_dim(cfg.problem, m);
    require(d >= m, "make_problem: DTLZ needs d >= m");
    require(2 * n < 0xffffffffULL, "nsga2_run: population too large");
    rng = make_rng(cfg.seed, cfg.rng_mode);
    stream = ctx().stream;
    for (int b = 0; b < 2; ++b) x[b] = dev_alloc<double>(n * d);
    off = dev_alloc<double>(n * d);
    fm = dev_alloc<double>(2 * n * m);
    lower = dev_alloc<double>(d);
    upper = dev_alloc<double>(d);
    idx_dev = dev_alloc<uint32_t>(n);
    sort.alloc(2 * n);
    f_host.resize(2 * n * m);
    rank_host.resize(2 * n);
    sel_host.resize(n);
    pool_idx.resize(n);
    std::vector<double> lo(d), hi(d);
    problem_bounds(cfg.problem, d, m, lo.data(), hi.data());
    bound_seg = find_bound_segments(lo.data(), hi.data(), d);
    TEMO_CUDA(cudaMemcpyAsync(lower, lo.data(), d * sizeof(double), cudaMemcpyHostToDevice, stream));
    TEMO_CUDA(cudaMemcpyAsync(upper, hi.data(), d * sizeof(double), cudaMemcpyHostToDevice, stream));
    TEMO_CUDA(cudaStreamSynchronize(stream));
    // initial population (algorithms.hpp:309-310)
    launch_random_reproduce(x[0], nullptr, n, d, rng, 0, lower, upper, stream);
    counter = n * d;
    EvalArgs ea;
    ea.problem = cfg.problem;
    ea.x = x[0];
    ea.n = n;
    ea.d = d;
    ea.m = m;
    ea.horizon = cfg.horizon;
    ea.f = fm;
    launch_evaluate(ea, stream);
    TEMO_CUDA(cudaMemcpyAsync(f_host.data(), fm, n * m * sizeof(double), cudaMemcpyDeviceToHost, stream));
    TEMO_CUDA(cudaStreamSynchronize(stream));
}

Nsga2Run::~Nsga2Run() {
    cudaStreamSynchronize(stream);
    cudaFree(x[0]); cudaFree(x[1]); cudaFree(off); cudaFree(fm); cudaFree(lower); cudaFree(upper); cudaFree(idx_dev);
    sort.release();
}

void Nsga2Run::inject(const double* x_in, const double* f_in, uint64_t counter_in, uint64_t t_in) {
    TEMO_CUDA(cudaStreamSynchronize(stream));
    if (x_in) TEMO_CUDA(cudaMemcpy(x[cur], x_in, n * d * sizeof(double), cudaMemcpyHostToDevice));
    if (f_in) {
        TEMO_CUDA(cudaMemcpy(fm, f_in, n * m * sizeof(double), cudaMemcpyHostToDevice));
        std::copy_n(f_in, n * m, f_host.data());
    }
    counter = counter_in;
    t = t_in;
}

void Nsga2Run::download(double* x_out, double* f_out) {
    TEMO_CUDA(cudaStreamSynchronize(stream));
    if (x_out) TEMO_CUDA(cudaMemcpy(x_out, x[cur], n * d * sizeof(double), cudaMemcpyDeviceToHost));
    if (f_out) std::copy_n(f_host.data(), n * m, f_out);
}

void Nsga2Run::last_generation(double* offspring, double* f_off, uint64_t* sel, uint64_t* pool) {
    require(t >= 1, "last_generation: no generation has run");
    TEMO_CUDA(cudaStreamSynchronize(stream));
    if (offspring) TEMO_CUDA(cudaMemcpy(offspring, off, n * d * sizeof(double), cudaMemcpyDeviceToHost));
    if (f_off) std::copy_n(f_off_device.data(), n * m, f_off);
    if (sel)
        for (uint64_t k = 0; k < n; ++k) sel[k] = sel_host[k];
    if (pool)
        for (uint64_t k = 0; k < n; ++k) pool[k] = pool_idx[k];
}

// One generation (algorithms.hpp:314-356). f_off_inject (optional, host n x m): the objectives selection runs on instead of
// the device's (lock-step testing); the device's own are kept for last_generation either way.
void Nsga2Run::step(const double* f_off_inject) {
    require(t < cfg.generations, "nsga2_run: all generations already done");
    // rank and crowding distance of the parents (:315-329)
    const uint64_t levels = device_nondominated_sort(fm, n, m, sort, rank_host.data(), stream);
    std::vector<double> crowd(n, 0.0);
    {
        std::vector<std::vector<uint32_t>> members(levels);
        for (uint64_t i = 0; i < n; ++i) members[rank_host[i]].push_back((uint32_t)i);
        std::vector<double> front, cd;
        for (const auto& rows : members) {
            if (rows.empty()) continue;
            front.resize(rows.size() * m);
            cd.resize(rows.size());
            for (size_t a = 0; a < rows.size(); ++a) std::copy_n(f_host.data() + (uint64_t)rows[a] * m, m, front.data() + a * m);
            crowding_distance_host(front.data(), rows.size(), m, cd.data());
            for (size_t a = 0; a < rows.size(); ++a) crowd[rows[a]] = cd[a];
        }
    }
    // binary tournament: 2n draws (:332-345)
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t wa = rng.mode == 0 ? draw_word<0>(rng, counter + 2 * i) : draw_word<1>(rng, counter + 2 * i);
        const uint64_t wb = rng.mode == 0 ? draw_word<0>(rng, counter + 2 * i + 1) : draw_word<1>(rng, counter + 2 * i + 1);
        const uint64_t a = (uint64_t)(word_to_unit(wa) * (double)n), b = (uint64_t)(word_to_unit(wb) * (double)n);
        bool a_wins;
        if (rank_host[a] != rank_host[b])
            a_wins = rank_host[a] < rank_host[b];
        else if (crowd[a] != crowd[b])
            a_wins = crowd[a] > crowd[b];
        else
            a_wins = a <= b;
        pool_idx[i] = (uint32_t)(a_wins ? a : b);
    }
    counter += 2 * n;
    TEMO_CUDA(cudaMemcpyAsync(idx_dev, pool_idx.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
    // sbx + polynomial_mutation on the tournament winners, addressed in place (:346-349); children evaluated in the same
    // kernel where the problem allows it
    const uint64_t h = n / 2;
    ReproArgs ra;
    ra.pool = x[cur];
    ra.src = idx_dev;
    ra.out = off;
    ra.n = n;
    ra.d = d;
    ra.rng = rng;
    ra.c_sbx = counter;
    ra.c_pm = counter + 3 * h * d + h;
    ra.ga = cfg.ga;
    ra.lower = lower;
    ra.upper = upper;
    ra.seg = bound_seg;
    const bool fused = fuse_offspring_eval(cfg.fuse_eval, cfg.problem, d);
    if (fused) {
        ra.eval_problem = cfg.problem;
        ra.m = m;
        ra.f_out = fm;
        ra.f_row0 = n;
    }
    launch_reproduce(ra, stream);
    counter = ra.c_pm + 2 * n * d;
    if (!fused) {
        EvalArgs ea;
        ea.problem = cfg.problem;
        ea.x = off;
        ea.n = n;
        ea.d = d;
        ea.m = m;
        ea.horizon = cfg.horizon;
        ea.f = fm;
        ea.f_row0 = n;
        launch_evaluate(ea, stream);
    }
    f_off_device.resize(n * m);
    TEMO_CUDA(cudaMemcpyAsync(f_off_device.data(), fm + n * m, n * m * sizeof(double), cudaMemcpyDeviceToHost, stream));
    if (f_off_inject) TEMO_CUDA(cudaMemcpyAsync(fm + n * m, f_off_inject, n * m * sizeof(double), cudaMemcpyHostToDevice, stream));
    TEMO_CUDA(cudaStreamSynchronize(stream));
    std::copy_n(f_off_inject ? f_off_inject : f_off_device.data(), n * m, f_host.data() + n * m);
    // environmental selection over parents + offspring (:350-355)
    device_nondominated_sort(fm, 2 * n, m, sort, rank_host.data(), stream);
    nsga2_select_host(f_host.data(), rank_host.data(), 2 * n, m, n, sel_host.data());
    TEMO_CUDA(cudaMemcpyAsync(idx_dev, sel_host.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
    gather_merged_rows_kernel<<<(unsigned)n, 256, 0, stream>>>(x[cur], off, idx_dev, n, d, x[cur ^ 1]);
    TEMO_CUDA(cudaGetLastError());
    std::vector<double> nf(n * m);
    for (uint64_t k = 0; k < n; ++k) std::copy_n(f_host.data() + (uint64_t)sel_host[k] * m, m, nf.data() + k * m);
    std::copy_n(nf.data(), n * m, f_host.data());
    TEMO_CUDA(cudaMemcpyAsync(fm, f_host.data(), n * m * sizeof(double), cudaMemcpyHostToDevice, stream));
    TEMO_CUDA(cudaStreamSynchronize(stream));
    cur ^= 1;
    ++t;
}

}  // namespace temo_b200
