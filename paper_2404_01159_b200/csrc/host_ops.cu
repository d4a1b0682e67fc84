// Host-side pieces of the path that stay C++ (SURVEY.md §8b "host-side responsibilities"):
// the Das-Dennis lattice (run once), the sequential Fisher-Yates mating permutation, the
// scalar APD penalty (glibc pow, bit-identical to the reference), problem registry data, and
// the per-process device context.
#include <cmath>
#include <cstring>
#include <mutex>

#include <algorithm>
#include <limits>
#include <vector>
#include "internal.h"

namespace temo_b200 {

// refvec.hpp:15-19
uint64_t lattice_count(uint64_t m, uint64_t H) {
    uint64_t c = 1;
    for (uint64_t i = 1; i < m; ++i) c = c * (H + i) / i;
    return c;
}

// refvec.hpp:22-35: lattice size closest to the target, ties -> smaller H.
uint64_t lattice_density_for(uint64_t m, uint64_t target) {
    uint64_t best_h = 1, best_gap = ~0ULL;
    for (uint64_t h = 1; h < 100000; ++h) {
        const uint64_t c = lattice_count(m, h);
        const uint64_t gap = c > target ? c - target : target - c;
        if (gap < best_gap) {
            best_gap = gap;
            best_h = h;
        }
        if (c >= target) break;
    }
    return best_h;
}

// refvec.hpp:40-62: compositions of H into m parts / H, lexicographic with every part counting
// down from what is left. Iterative successor instead of the reference's recursion.
std::vector<double> simplex_lattice(uint64_t m, uint64_t H) {
    require(m >= 2, "simplex_lattice: m must be at least 2");
    require(H >= 1, "simplex_lattice: H must be at least 1");
    const uint64_t r = lattice_count(m, H);
    std::vector<double> out(r * m);
    std::vector<uint64_t> part(m, 0);
    part[0] = H;
    for (uint64_t row = 0;; ++row) {
        for (uint64_t j = 0; j < m; ++j) out[row * m + j] = (double)part[j] / (double)H;
        const uint64_t tail = part[m - 1];
        part[m - 1] = 0;
        uint64_t k = m - 1;
        while (k > 0 && part[k - 1] == 0) --k;
        if (k == 0) break;
        part[k - 1] -= 1;
        part[k] = tail + 1;
    }
    return out;
}

// refvec.hpp:65-75
std::vector<double> normalize_to_unit(const std::vector<double>& v, uint64_t r, uint64_t m) {
    std::vector<double> out(r * m);
    for (uint64_t i = 0; i < r; ++i) {
        double s = 0.0;
        for (uint64_t k = 0; k < m; ++k) s += v[i * m + k] * v[i * m + k];
        const double norm = std::sqrt(s);
        require(norm > 0.0, "normalize_to_unit: zero row");
        for (uint64_t k = 0; k < m; ++k) out[i * m + k] = v[i * m + k] / norm;
    }
    return out;
}

// rng.hpp:69-78: n-1 dependent swaps, draw k used at i = n-1-k. 32-bit indices (n < 2^32).
void shuffle_indices(uint64_t seed, uint64_t& counter, uint64_t n, uint32_t* perm) {
    require(n >= 1, "shuffle_indices: n must be positive");
    for (uint64_t i = 0; i < n; ++i) perm[i] = (uint32_t)i;
    const uint64_t base = mix64(seed);
    uint64_t z = base + counter * kGolden;
    for (uint64_t i = n - 1; i >= 1; --i) {
        const double u = (double)(mix64(z) >> 11) * 0x1.0p-53;
        z += kGolden;
        const uint64_t j = (uint64_t)(u * (double)(i + 1));
        const uint32_t t = perm[i];
        perm[i] = perm[j];
        perm[j] = t;
    }
    counter += n - 1;
}

// selection.hpp:86-89 (host scalar; glibc pow as in the reference)
double apd_penalty(uint64_t m, uint64_t t, uint64_t t_max, double alpha) {
    return (double)m * std::pow((double)t / (double)t_max, alpha);
}

bool problem_known(int problem) {
    return (problem >= kDtlz1 && problem <= kDtlz4) || problem == kLsmop1 || problem == kToy2 || problem == kToy3;
}

// problems.hpp:266-272 (DTLZ: [0,1]^d); LSMOP1: position genes [0,1], tail genes [0,10].
void problem_bounds(int problem, uint64_t d, uint64_t m, double* lower, double* upper) {
    require(problem_known(problem), "make_problem: unknown problem");
    if (problem == kToy2 || problem == kToy3) {  // problems.hpp:285-286: MLP parameters in [-1, 1]
        for (uint64_t j = 0; j < d; ++j) lower[j] = -1.0, upper[j] = 1.0;
        return;
    }
    for (uint64_t j = 0; j < d; ++j) {
        lower[j] = 0.0;
        upper[j] = (problem == kLsmop1 && j + 1 >= m) ? 10.0 : 1.0;
    }
}

// problems.hpp:268 (DTLZ1: 7, DTLZ2-4: 12); LSMOP default 100*m.
uint64_t problem_default_dim(int problem, uint64_t m) {
    if (problem == kDtlz1) return 7;
    if (problem >= kDtlz2 && problem <= kDtlz4) return 12;
    if (problem == kToy2 || problem == kToy3) return mlp_param_count(kToyHidden);  // problems.hpp:283
    return 100 * m;
}

// ---- device context ---------------------------------------------------------------------------------
namespace {
Context g_ctx;
std::mutex g_ctx_mutex;
}  // namespace

void init_context(int device) {
    std::lock_guard<std::mutex> lock(g_ctx_mutex);
    if (g_ctx.device == device && g_ctx.stream) return;
    // Kernels that a run launches for the first time in the middle of its loop (the first adaptation of the reference
    // vectors) would be loaded there under CUDA's lazy module loading: 0.4 ... 13 ms measured for two small kernels, inside
    // somebody's timed region. A run loads them at creation (preload_adapt_kernels); TEMO_B200_EAGER_MODULES=1 asks for eager
    // loading of everything instead (process-wide, and only if this is the process' first CUDA call).
    if (getenv("TEMO_B200_EAGER_MODULES")) setenv("CUDA_MODULE_LOADING", "EAGER", 0);
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        fail(3, std::string("no CUDA device available (the temo_b200 path has no CPU fallback): ") +
                    (e != cudaSuccess ? cudaGetErrorString(e) : "device count is 0"));
    if (device < 0 || device >= count) fail(1, "temo_b200_init: device index out of range");
    TEMO_CUDA(cudaSetDevice(device));
    if (g_ctx.stream) {
        cudaStreamDestroy(g_ctx.stream);
        cudaStreamDestroy(g_ctx.copy_stream);
        if (g_ctx.flush_buf) cudaFree(g_ctx.flush_buf);
        g_ctx = Context{};
    }
    TEMO_CUDA(cudaStreamCreateWithFlags(&g_ctx.stream, cudaStreamNonBlocking));
    TEMO_CUDA(cudaStreamCreateWithFlags(&g_ctx.copy_stream, cudaStreamNonBlocking));
    g_ctx.device = device;
}

Context& ctx() {
    if (!g_ctx.stream) init_context(0);
    return g_ctx;
}

// Bounds that are constant on [0, split) and on [split, d) (bit patterns compared, so -0.0 != 0.0 and NaNs
// never match: anything unusual simply stays on the array path).
BoundSegments find_bound_segments(const double* lower, const double* upper, uint64_t d) {
    BoundSegments g;
    if (!lower || !upper || d == 0) return g;
    const auto same = [](double x, double y) { return std::memcmp(&x, &y, sizeof(double)) == 0; };
    uint64_t split = d;
    for (uint64_t j = 1; j < d; ++j)
        if (!same(lower[j], lower[0]) || !same(upper[j], upper[0])) {
            split = j;
            break;
        }
    for (uint64_t j = split; j < d; ++j)
        if (!same(lower[j], lower[split]) || !same(upper[j], upper[split])) return g;
    g.valid = true;
    g.split = split;
    g.lo[0] = lower[0];
    g.hi[0] = upper[0];
    g.lo[1] = split < d ? lower[split] : lower[0];
    g.hi[1] = split < d ? upper[split] : upper[0];
    return g;
}

// crowding_distance (selection.hpp:289-312): per objective a (value, index)-ordered sort; the boundary rows get
// infinity, the inner rows accumulate (next - previous) / range in objective order.
void crowding_distance_host(const double* front, uint64_t k, uint64_t m, double* dist) {
    require(k >= 1, "crowding_distance: empty front");
    const double inf = std::numeric_limits<double>::infinity();
    if (k <= 2) {
        for (uint64_t i = 0; i < k; ++i) dist[i] = inf;
        return;
    }
    for (uint64_t i = 0; i < k; ++i) dist[i] = 0.0;
    std::vector<uint64_t> order(k);
    for (uint64_t obj = 0; obj < m; ++obj) {
        for (uint64_t i = 0; i < k; ++i) order[i] = i;
        std::sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) {
            const double fa = front[a * m + obj], fb = front[b * m + obj];
            if (fa != fb) return fa < fb;
            return a < b;
        });
        const double range = front[order[k - 1] * m + obj] - front[order[0] * m + obj];
        if (range <= 0.0) continue;
        dist[order[0]] = inf;
        dist[order[k - 1]] = inf;
        for (uint64_t i = 1; i + 1 < k; ++i)
            dist[order[i]] += (front[order[i + 1] * m + obj] - front[order[i - 1] * m + obj]) / range;
    }
}

}  // namespace temo_b200
