// Sharded generation loop: the stage-level pieces one rank (one process, one GPU) runs between the
// collectives that paper_2404_01159_b200/dist.py issues with torch.distributed.
//
// reference: the same rvea_run loop (algorithms.hpp:227-296); the reference itself is single-process.
// Sharding: rank g owns the mating pairs [g*h_loc, (g+1)*h_loc) of the shuffled order (h_loc = n/2/G),
// i.e. the children with global rows p and n/2+p; a survivor stays in the pool of the rank where it was
// born. Replicated on every rank (a few MB): the merged objective matrix, the reference set with its
// direction index, and the survivor -> (owner, slot) tables (kept by the host orchestration).
// Exchanges per generation: parents of a rank's pairs (all-to-all of rows), offspring objectives and
// free-slot lists (all-gather), per-vector minima (two min-allreduces). Everything else is rank-local and
// draws/evaluates/selects exactly what the single-GPU run does for the same rows (global draw addressing).
#include <cstring>
#include <numeric>
#include <thread>

#include "../../include/temo_b200.h"
#include "compact.cuh"
#include "internal.h"
#include "run.h"
#include "vecindex.h"

namespace temo_b200 {

namespace {

__global__ void gather_slots_kernel(const double* pool, const uint32_t* slot, uint64_t rows, uint64_t d, double* out) {
    const uint64_t i = blockIdx.x;
    if (i >= rows) return;
    const double2* p = reinterpret_cast<const double2*>(pool + (uint64_t)slot[i] * d);
    double2* o = reinterpret_cast<double2*>(out + i * d);
    if (d % 2 == 0) {
        for (uint64_t j = threadIdx.x; j < d / 2; j += blockDim.x) o[j] = p[j];
    } else {
        for (uint64_t j = threadIdx.x; j < d; j += blockDim.x) out[i * d + j] = pool[(uint64_t)slot[i] * d + j];
    }
}

// gathered[rank][local child j][m] -> merged rows P + global child row
__global__ void scatter_offspring_f_kernel(const double* gathered, uint64_t world, uint64_t h_loc, uint64_t half,
                                           uint64_t m, uint64_t P, double* fm) {
    const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t n_loc = 2 * h_loc;
    if (e >= world * n_loc) return;
    const uint64_t rk = e / n_loc, j = e - rk * n_loc;
    const uint64_t g = j < h_loc ? rk * h_loc + j : half + rk * h_loc + (j - h_loc);
    for (uint64_t k = 0; k < m; ++k) fm[(P + g) * m + k] = gathered[e * m + k];
}

__global__ void compact_f_kernel(const uint32_t* elite, uint64_t cnt, uint64_t m, const double* f_merged, double* f_next) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= cnt) return;
    const uint64_t e = elite[k];
    for (uint64_t j = 0; j < m; ++j) f_next[k * m + j] = f_merged[e * m + j];
}

__global__ void mark_used_kernel(const uint32_t* slots, uint64_t cnt, unsigned char* used) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k < cnt) used[slots[k]] = 1;
}

// order-preserving signed view of the unsigned APD keys, so that an int64 min-allreduce merges them
__global__ void flip_keys_kernel(unsigned long long* keys, uint64_t r) {
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j < r) keys[j] ^= 0x8000000000000000ULL;
}

// same for the 32-bit row indices (0xffffffff = "none" must stay the maximum in the signed view)
__global__ void flip_rows_kernel(uint32_t* rows, uint64_t r) {
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j < r) rows[j] ^= 0x80000000u;
}

struct FreePredS {
    const unsigned char* used;
    __device__ bool operator()(uint64_t i) const { return used[i] == 0; }
};
struct IdentityValS {
    __device__ uint32_t operator()(uint64_t i) const { return (uint32_t)i; }
};

}  // namespace

// Speculative mating permutation: the Fisher-Yates shuffle of generation t+1 only depends on the draw
// counter, so a host thread computes it while the GPU is busy with generation t (rng.hpp:69-78).
struct PermCache {
    std::thread worker;
    std::vector<uint32_t> perm;
    uint64_t seed = 0, c_shuffle = 0, n = 0;
    bool valid = false;
    void start(uint64_t seed_, uint64_t c_shuffle_, uint64_t n_) {
        join();
        seed = seed_;
        c_shuffle = c_shuffle_;
        n = n_;
        valid = true;
        worker = std::thread([this] {
            perm.resize(n);
            uint64_t c = c_shuffle;
            shuffle_indices(seed, c, n, perm.data());
        });
    }
    void join() {
        if (worker.joinable()) worker.join();
    }
    bool take(uint64_t seed_, uint64_t c_shuffle_, uint64_t n_, std::vector<uint32_t>& out) {
        join();
        if (!valid || seed != seed_ || c_shuffle != c_shuffle_ || n != n_) return false;
        out.swap(perm);
        valid = false;
        return true;
    }
    ~PermCache() { join(); }
};
static PermCache g_perm_cache;

// Host-side exchange plan of one generation (pure host code; exercised on CPU by the gloo tests).
// Inputs: the replicated survivor tables and the draw counter at the top of the generation.
// Outputs (for `rank`): the local slots to send, grouped by destination rank and ordered by the
// destination's local mating row; send/recv row counts per peer; for every local mating row its row in
// the receive buffer; and the draw counters of the generation.
// The exchange is cut into `chunks` pieces by local mating pair (pair p of a rank belongs to chunk p / ceil(h_loc / chunks)):
// piece c carries the parents of the pairs of chunk c, so K1 can start on chunk c while piece c + 1 is still on the
// wire. Layout: send_slots ordered by (chunk, destination), counts indexed [chunk * world + peer], the receive buffer
// filled chunk after chunk and, inside a chunk, source after source (the order all_to_all delivers).
void shard_plan(uint64_t seed, uint64_t counter, uint64_t P, uint64_t n, int rank, int world, int chunks, const int32_t* surv_owner,
                const uint32_t* surv_slot, std::vector<uint32_t>& send_slots, std::vector<uint64_t>& send_counts,
                std::vector<uint64_t>& recv_counts, std::vector<uint32_t>& recv_pos, uint64_t counters_out[3]) {
    require(world >= 1 && rank >= 0 && rank < world, "shard_plan: bad rank");
    require(chunks >= 1, "shard_plan: at least one chunk");
    require(n % (2 * (uint64_t)world) == 0, "shard_plan: population must be divisible by 2 * world size");
    const uint64_t half = n / 2, h_loc = half / world, n_loc = 2 * h_loc;
    const uint64_t per_chunk = (h_loc + (uint64_t)chunks - 1) / (uint64_t)chunks;  // pairs per chunk
    uint64_t c = counter;
    const uint64_t c_pool = c;
    if (P != n) c += n;  // algorithms.hpp:211-221
    std::vector<uint32_t> perm;
    if (g_perm_cache.take(seed, c, n, perm)) {
        c += n - 1;  // computed ahead of time by the speculation thread
    } else {
        perm.resize(n);
        shuffle_indices(seed, c, n, perm.data());  // advances c by n - 1
    }
    counters_out[0] = c;                       // c_sbx: first draw after the shuffle
    const uint64_t base = mix64(seed);
    auto pool_idx = [&](uint64_t q) -> uint64_t {
        if (P == n) return q;
        const double u = (double)(mix64(base + (c_pool + q) * kGolden) >> 11) * 0x1.0p-53;
        return (uint64_t)(u * (double)P);
    };
    // mating row i of the shuffled order is handled by rank (i mod half) / h_loc, local row
    // (i < half ? i - dest*h_loc : h_loc + (i - half) - dest*h_loc)
    const size_t cells = (size_t)chunks * (size_t)world;
    send_counts.assign(cells, 0);
    recv_counts.assign(cells, 0);
    recv_pos.assign(n_loc, 0);
    std::vector<std::vector<uint32_t>> send_cell(cells);  // [chunk * world + dest]: my slots to send
    std::vector<std::vector<uint32_t>> recv_cell(cells);  // [chunk * world + src]: my local mating rows fed by src
    // every destination is independent (its own cells; only dest == rank fills the receive cells): one host thread
    // per destination keeps this O(n) bookkeeping at O(n / world) wall time on every rank
    auto plan_dest = [&](int dest) {
        for (uint64_t j = 0; j < n_loc; ++j) {
            const uint64_t pair = j < h_loc ? j : j - h_loc;
            const size_t chunk = (size_t)(pair / per_chunk);
            const uint64_t i = j < h_loc ? dest * h_loc + j : half + dest * h_loc + (j - h_loc);
            const uint64_t k = pool_idx(perm[i]);
            const int owner = surv_owner[k];
            if (owner == rank) send_cell[chunk * world + dest].push_back(surv_slot[k]);
            if (dest == rank) recv_cell[chunk * world + owner].push_back((uint32_t)j);
        }
    };
    if (world > 1 && n_loc >= 4096) {
        std::vector<std::thread> workers;
        for (int dest = 1; dest < world; ++dest) workers.emplace_back(plan_dest, dest);
        plan_dest(0);
        for (auto& w : workers) w.join();
    } else {
        for (int dest = 0; dest < world; ++dest) plan_dest(dest);
    }
    send_slots.clear();
    uint32_t pos = 0;
    for (size_t cell = 0; cell < cells; ++cell) {
        send_counts[cell] = send_cell[cell].size();
        send_slots.insert(send_slots.end(), send_cell[cell].begin(), send_cell[cell].end());
        recv_counts[cell] = recv_cell[cell].size();
        for (const uint32_t j : recv_cell[cell]) recv_pos[j] = pos++;
    }
    counters_out[1] = counters_out[2] = 0;  // filled by the caller (needs d)
}

struct Shard {
    RunConfig cfg;
    int rank = 0, world = 1;
    uint64_t n = 0, d = 0, m = 0, r = 0, H = 0, adapt_every = 1;
    uint64_t h_loc = 0, n_loc = 0, pcap = 0, cap_loc = 0, send_cap = 0;
    Rng rng{};
    cudaStream_t stream = nullptr;
    double* pool = nullptr;       // cap_loc x d (local rows only)
    double* send_buf = nullptr;   // send_cap x d
    double* recv_buf = nullptr;   // n_loc x d
    uint32_t* send_slots = nullptr;  // send_cap
    uint32_t* recv_pos = nullptr;    // n_loc
    uint32_t* free_slot = nullptr;   // n_loc
    uint32_t* surv_slots_dev = nullptr;  // pcap (local slots owned by this rank)
    unsigned char* used = nullptr;
    uint32_t* free_scratch = nullptr;
    double* fm[2] = {nullptr, nullptr};  // replicated merged objectives, (pcap + n) x m
    int cur = 0;
    double* f_off_loc = nullptr;  // n_loc x m
    double* f_gather = nullptr;   // world x n_loc x m
    double *v0 = nullptr, *v = nullptr, *gamma = nullptr, *lower = nullptr, *upper = nullptr;
    BoundSegments bound_seg;
    double *zmin = nullptr, *zmax = nullptr;
    unsigned long long* zscratch = nullptr;
    uint32_t* skip_flag = nullptr;
    SelectWorkspace ws;
    VecIndex vindex;

    Shard(const RunConfig& c, int rank_, int world_) : cfg(c), rank(rank_), world(world_) {
        require(world >= 1 && rank >= 0 && rank < world, "shard: bad rank");
        require(problem_known(cfg.problem), "make_problem: unknown problem");
        n = cfg.pop;
        m = cfg.obj;
        if (cfg.problem == kToy2 || cfg.problem == kToy3) m = cfg.problem == kToy2 ? 2 : 3;  // problems.hpp:279-287
        d = cfg.dim ? cfg.dim : problem_default_dim(cfg.problem, m);
        require(n % (2 * (uint64_t)world) == 0, "shard: population must be divisible by 2 * world size");
        require(d >= m && m >= 2 && m <= (uint64_t)kMaxObj, "shard: bad problem shape");
        H = cfg.lattice_h ? cfg.lattice_h : lattice_density_for(m, n);
        r = lattice_count(m, H);
        const double ae = std::ceil(cfg.fr * (double)cfg.generations);
        adapt_every = ae < 1.0 ? 1 : (uint64_t)ae;
        rng = make_rng(cfg.seed, cfg.rng_mode);
        h_loc = n / 2 / world;
        n_loc = 2 * h_loc;
        pcap = n > r ? n : r;
        // survivors are spread over the ranks like their births (uniformly): 60 % head-room over the mean
        const uint64_t own_cap = world == 1 ? pcap : std::min<uint64_t>(pcap, (pcap * 8) / (5 * (uint64_t)world) + 1024);
        cap_loc = own_cap + n_loc;
        send_cap = world == 1 ? n_loc : std::min<uint64_t>(n, 2 * n_loc + 1024);
        stream = ctx().stream;
        pool = dev_alloc<double>(cap_loc * d);
        send_buf = dev_alloc<double>(send_cap * d);
        recv_buf = dev_alloc<double>(n_loc * d);
        send_slots = dev_alloc<uint32_t>(send_cap);
        recv_pos = dev_alloc<uint32_t>(n_loc);
        free_slot = dev_alloc<uint32_t>(n_loc);
        surv_slots_dev = dev_alloc<uint32_t>(pcap);
        used = dev_alloc<unsigned char>(cap_loc);
        free_scratch = dev_alloc<uint32_t>((cap_loc + kCompactTile - 1) / kCompactTile + 1);
        for (int b = 0; b < 2; ++b) fm[b] = dev_alloc<double>((pcap + n) * m);
        f_off_loc = dev_alloc<double>(n_loc * m);
        f_gather = dev_alloc<double>((uint64_t)world * n_loc * m);
        v0 = dev_alloc<double>(r * m);
        v = dev_alloc<double>(r * m);
        gamma = dev_alloc<double>(r);
        lower = dev_alloc<double>(d);
        upper = dev_alloc<double>(d);
        zmin = dev_alloc<double>(m);
        zmax = dev_alloc<double>(m);
        zscratch = dev_alloc<unsigned long long>(2 * m);
        skip_flag = dev_alloc<uint32_t>(1);
        ws.alloc(pcap + n, r, m);
        const std::vector<double> unit = normalize_to_unit(simplex_lattice(m, H), r, m);
        TEMO_CUDA(cudaMemcpyAsync(v0, unit.data(), r * m * sizeof(double), cudaMemcpyHostToDevice, stream));
        TEMO_CUDA(cudaMemcpyAsync(v, v0, r * m * sizeof(double), cudaMemcpyDeviceToDevice, stream));
        launch_row_norms(v, r, m, ws.vn, stream);
        vindex.alloc(r, m);
        vindex.set_order(unit.data(), stream);
        if (!assoc_filter_preferred(m, r)) vindex.build(v, ws.vn, stream);  // m >= 5: the fp32-filtered scans need no index
        launch_gamma_auto(v, r, m, ws, &vindex, gamma, ws.err_flag, nullptr, stream);
        std::vector<double> lo(d), hi(d);
        problem_bounds(cfg.problem, d, m, lo.data(), hi.data());
        bound_seg = find_bound_segments(lo.data(), hi.data(), d);
        TEMO_CUDA(cudaMemcpyAsync(lower, lo.data(), d * sizeof(double), cudaMemcpyHostToDevice, stream));
        TEMO_CUDA(cudaMemcpyAsync(upper, hi.data(), d * sizeof(double), cudaMemcpyHostToDevice, stream));
        // initial population (algorithms.hpp:241-242): global rows [rank*n/world, (rank+1)*n/world) in local
        // slots 0.., drawn at their global counters; objectives of the local block
        const uint64_t rows0 = n / world;
        launch_random_reproduce(pool, nullptr, rows0, d, rng, (uint64_t)rank * rows0 * d, lower, upper, stream);
        EvalArgs ea;
        ea.problem = cfg.problem;
        ea.x = pool;
        ea.n = rows0;
        ea.d = d;
        ea.m = m;
        ea.horizon = cfg.horizon;
        ea.f = f_off_loc;  // n/world = n_loc rows
        launch_evaluate(ea, stream);
        TEMO_CUDA(cudaMemsetAsync(used, 0, cap_loc, stream));
        std::vector<uint32_t> own(rows0);
        std::iota(own.begin(), own.end(), 0u);
        TEMO_CUDA(cudaMemcpyAsync(surv_slots_dev, own.data(), rows0 * sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
        mark_used_kernel<<<(unsigned)((rows0 + 255) / 256), 256, 0, stream>>>(surv_slots_dev, rows0, used);
        launch_compact(cap_loc, FreePredS{used}, IdentityValS{}, free_scratch, n_loc, free_slot, nullptr, stream);
        TEMO_CUDA(cudaStreamSynchronize(stream));
        check();
    }

    ~Shard() {
        cudaStreamSynchronize(stream);
        cudaFree(pool); cudaFree(send_buf); cudaFree(recv_buf); cudaFree(send_slots); cudaFree(recv_pos);
        cudaFree(free_slot); cudaFree(surv_slots_dev); cudaFree(used); cudaFree(free_scratch);
        cudaFree(fm[0]); cudaFree(fm[1]); cudaFree(f_off_loc); cudaFree(f_gather);
        cudaFree(v0); cudaFree(v); cudaFree(gamma); cudaFree(lower); cudaFree(upper);
        cudaFree(zmin); cudaFree(zmax); cudaFree(zscratch); cudaFree(skip_flag);
        ws.release();
        vindex.release();
    }

    void check() {
        uint32_t flag = 0;
        TEMO_CUDA(cudaMemcpyAsync(&flag, ws.err_flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, stream));
        TEMO_CUDA(cudaStreamSynchronize(stream));
        if (flag & 1u) fail(1, "min_vector_angles: duplicate reference vectors / rv_select: gamma must be positive");
        if (flag & 2u) fail(1, "normalize_to_unit: zero row");
    }

    // rows of the send buffer <- local pool rows (slots given by the plan)
    // (rows [row0, row0 + count) of the send buffer: one piece of a chunked exchange)
    void pack(const uint32_t* slots_host, uint64_t count, uint64_t row0) {
        require(row0 <= send_cap && count <= send_cap - row0, "shard: send buffer too small (ownership imbalance)");
        if (count == 0) return;
        TEMO_CUDA(cudaMemcpyAsync(send_slots + row0, slots_host, count * sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
        gather_slots_kernel<<<(unsigned)count, 256, 0, stream>>>(pool, send_slots + row0, count, d, send_buf + row0 * d);
        TEMO_CUDA(cudaGetLastError());
    }

    // K1 (+ fused evaluation) on this rank's pairs; parents in recv_buf at recv_pos_host[]
    // (pairs [unit_begin, unit_begin + unit_count) only; unit_count = 0: all of them)
    void reproduce(const uint32_t* recv_pos_host, uint64_t c_sbx, uint64_t c_pm, uint64_t unit_begin, uint64_t unit_count) {
        require(unit_begin <= h_loc && unit_count <= h_loc - unit_begin, "shard: bad pair range");
        if (unit_begin == 0)
            TEMO_CUDA(cudaMemcpyAsync(recv_pos, recv_pos_host, n_loc * sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
        ReproArgs ra;
        ra.pool = recv_buf;
        ra.src = recv_pos;
        ra.out = pool;
        ra.dst = free_slot;
        ra.n = n_loc;
        ra.d = d;
        ra.rng = rng;
        ra.c_sbx = c_sbx;
        ra.c_pm = c_pm;
        ra.ga = cfg.ga;
        ra.lower = lower;
        ra.upper = upper;
        ra.seg = bound_seg;
        ra.global_n = n;
        ra.global_unit0 = (uint64_t)rank * h_loc;
        ra.unit_begin = unit_begin;
        ra.unit_count = unit_count;
        const bool fused = cfg.fuse_eval && cfg.problem >= kDtlz1 && cfg.problem <= kDtlz4;
        if (fused) {
            ra.eval_problem = cfg.problem;
            ra.m = m;
            ra.f_out = f_off_loc;
            ra.f_row0 = 0;
        }
        launch_reproduce(ra, stream);
        const bool last = unit_count == 0 || unit_begin + unit_count == h_loc;
        if (!fused && last) {  // unfused problems are evaluated once every child exists
            EvalArgs ea;
            ea.problem = cfg.problem;
            ea.x = pool;
            ea.rows = free_slot;
            ea.n = n_loc;
            ea.d = d;
            ea.m = m;
            ea.horizon = cfg.horizon;
            ea.f = f_off_loc;
            launch_evaluate(ea, stream);
        }
    }

    // f_gather (all-gathered offspring objectives) -> merged rows [P, P + n); P = 0 with `initial` puts the
    // gathered blocks of the initial population into rows [0, n) in global order
    void place_offspring_f(uint64_t P, bool initial) {
        if (initial) {
            TEMO_CUDA(cudaMemcpyAsync(fm[cur], f_gather, n * m * sizeof(double), cudaMemcpyDeviceToDevice, stream));
        } else {
            const uint64_t total = (uint64_t)world * n_loc;
            scatter_offspring_f_kernel<<<(unsigned)((total + 255) / 256), 256, 0, stream>>>(f_gather, world, h_loc, n / 2, m, P, fm[cur]);
        }
        TEMO_CUDA(cudaGetLastError());
    }

    // ideal point + association/APD for merged rows [lo, hi) + this rank's per-vector minima
    void select_local(uint64_t P, uint64_t lo, uint64_t hi, uint64_t t) {
        const uint64_t rows = P + n;
        require(lo <= hi && hi <= rows, "shard: bad row slice");
        const double penalty = apd_penalty(m, t, cfg.generations, cfg.alpha);
        launch_select_prepare(fm[cur], rows, m, gamma, r, ws, stream);
        if (hi > lo) {
            if (assoc_filter_preferred(m, r))
                launch_assoc_filter(fm[cur] + lo * m, hi - lo, m, v, gamma, r, penalty, ws, ws.assoc + lo, ws.theta + lo, ws.apd + lo,
                                    stream, (uint32_t)lo);
            else
                launch_assoc_indexed(fm[cur] + lo * m, hi - lo, nullptr, m, ws.z, vindex, gamma, penalty, ws.assoc + lo,
                                     ws.theta + lo, ws.apd + lo, ws.best_key, ws.first_row, stream, (uint32_t)lo);
        }
        flip_keys_kernel<<<(unsigned)((r + 255) / 256), 256, 0, stream>>>(ws.best_key, r);
        flip_rows_kernel<<<(unsigned)((r + 255) / 256), 256, 0, stream>>>(ws.first_row, r);
    }

    // after the min-allreduce of best_key / first_row: lowest row attaining the minimum, own slice
    void select_rows(uint64_t lo, uint64_t hi) {
        flip_keys_kernel<<<(unsigned)((r + 255) / 256), 256, 0, stream>>>(ws.best_key, r);
        flip_rows_kernel<<<(unsigned)((r + 255) / 256), 256, 0, stream>>>(ws.first_row, r);
        if (hi > lo) launch_elite_rows(hi - lo, ws.assoc + lo, ws.apd + lo, ws.best_key, ws.best_row, (uint32_t)lo, stream);
        flip_rows_kernel<<<(unsigned)((r + 255) / 256), 256, 0, stream>>>(ws.best_row, r);
    }

    // after the min-allreduce of best_row: validity + compaction; returns the survivor count
    uint64_t select_finish(uint32_t* elite_host) {
        flip_rows_kernel<<<(unsigned)((r + 255) / 256), 256, 0, stream>>>(ws.best_row, r);
        launch_select_finish(r, ws, /*nan_rule=*/false, stream);
        uint32_t cnt = 0;
        TEMO_CUDA(cudaMemcpyAsync(&cnt, ws.n_elite, sizeof(uint32_t), cudaMemcpyDeviceToHost, stream));
        TEMO_CUDA(cudaStreamSynchronize(stream));
        if (elite_host && cnt) TEMO_CUDA(cudaMemcpy(elite_host, ws.elite, cnt * sizeof(uint32_t), cudaMemcpyDeviceToHost));
        return cnt;
    }

    // survivors' objectives compacted (replicated); slots owned by this rank re-marked; free list rebuilt
    void commit(uint64_t cnt, const uint32_t* own_slots_host, uint64_t own_count, uint64_t t) {
        require(own_count + n_loc <= cap_loc, "shard: local pool too small (ownership imbalance)");
        compact_f_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, stream>>>(ws.elite, cnt, m, fm[cur], fm[cur ^ 1]);
        cur ^= 1;
        TEMO_CUDA(cudaMemsetAsync(used, 0, cap_loc, stream));
        if (own_count) {
            TEMO_CUDA(cudaMemcpyAsync(surv_slots_dev, own_slots_host, own_count * sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
            mark_used_kernel<<<(unsigned)((own_count + 255) / 256), 256, 0, stream>>>(surv_slots_dev, own_count, used);
        }
        launch_compact(cap_loc, FreePredS{used}, IdentityValS{}, free_scratch, n_loc, free_slot, nullptr, stream);
        if ((t + 1) % adapt_every == 0) {  // algorithms.hpp:281 (replicated: every rank adapts identically)
            launch_col_minmax(fm[cur], cnt, nullptr, m, zmin, zmax, zscratch, stream);
            launch_adapt_vectors(v0, v, ws.vn, r, m, zmin, zmax, skip_flag, ws.err_flag, stream);
            if (!assoc_filter_preferred(m, r)) vindex.build(v, ws.vn, stream);  // m >= 5: the fp32-filtered scans need no index
            launch_gamma_auto(v, r, m, ws, &vindex, gamma, ws.err_flag, skip_flag, stream);
        }
        TEMO_CUDA(cudaStreamSynchronize(stream));  // host staging arrays may go away
        check();
    }
};

}  // namespace temo_b200

// ---------------------------------------------------------------------------------------------- C ABI
using namespace temo_b200;

namespace {
thread_local std::string g_shard_error;
template <class F>
int guarded_shard(F&& body) {
    try {
        body();
        return TEMO_B200_OK;
    } catch (const Error& e) {
        g_shard_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_shard_error = e.what();
        return TEMO_B200_ERUNTIME;
    }
}
}  // namespace

struct temo_b200_shard {
    Shard* impl;
};

extern "C" {

const char* temo_b200_shard_last_error(void) { return g_shard_error.c_str(); }

int temo_b200_shard_plan(uint64_t seed, uint64_t counter, uint64_t P, uint64_t n, uint64_t d, int rank, int world, int chunks,
                         const int32_t* surv_owner, const uint32_t* surv_slot, uint32_t* send_slots,
                         uint64_t send_slots_cap, uint64_t* send_counts, uint64_t* recv_counts, uint32_t* recv_pos,
                         uint64_t* counters3) {
    return guarded_shard([&] {
        require(surv_owner && surv_slot && send_slots && send_counts && recv_counts && recv_pos && counters3,
                "shard_plan: null argument");
        std::vector<uint32_t> ss, rp;
        std::vector<uint64_t> sc, rc;
        uint64_t cs[3];
        shard_plan(seed, counter, P, n, rank, world, chunks, surv_owner, surv_slot, ss, sc, rc, rp, cs);
        require(ss.size() <= send_slots_cap, "shard_plan: send list exceeds the caller's capacity");
        std::memcpy(send_slots, ss.data(), ss.size() * sizeof(uint32_t));
        std::memcpy(send_counts, sc.data(), sc.size() * sizeof(uint64_t));
        std::memcpy(recv_counts, rc.data(), rc.size() * sizeof(uint64_t));
        std::memcpy(recv_pos, rp.data(), rp.size() * sizeof(uint32_t));
        // draw counters: [pool n] + shuffle n-1, then SBX 3*h*d + h, then PM 2*n*d
        const uint64_t half = n / 2;
        counters3[0] = cs[0];                              // c_sbx
        counters3[1] = cs[0] + 3 * half * d + half;        // c_pm
        counters3[2] = counters3[1] + 2 * n * d;           // counter after the generation
    });
}

// Starts the Fisher-Yates shuffle of a future generation on a host thread (consumed by the next
// temo_b200_shard_plan with the same seed / shuffle counter / n; ignored otherwise).
int temo_b200_shard_perm_prefetch(uint64_t seed, uint64_t c_shuffle, uint64_t n) {
    return guarded_shard([&] {
        require(n >= 1 && n < 0xffffffffULL, "shuffle_indices: n must be positive");
        g_perm_cache.start(seed, c_shuffle, n);
    });
}

// Pure host code: survivor tables after selection. Survivor k takes over merged row elite[k]: a parent keeps
// its (owner, slot); child i = elite[k] - P lives on the rank that produced it, in that rank's free slot
// (free_all[rank * n_loc + local child index]). Also lists the slots owned by `rank`.
int temo_b200_shard_update_tables(const uint32_t* elite, uint64_t count, uint64_t P, uint64_t n, int rank, int world,
                                  const uint32_t* free_all, int32_t* surv_owner, uint32_t* surv_slot,
                                  uint32_t* own_slots, uint64_t* own_count) {
    return guarded_shard([&] {
        require(elite && free_all && surv_owner && surv_slot && own_slots && own_count, "update_tables: null argument");
        const uint64_t half = n / 2, h_loc = half / world, n_loc = 2 * h_loc;
        std::vector<int32_t> no(count);
        std::vector<uint32_t> ns(count);
        // ranges of survivors in parallel; the slots owned by `rank` are concatenated in survivor order afterwards
        const unsigned parts = count >= 65536 ? std::min<unsigned>(8u, std::max(1u, std::thread::hardware_concurrency() / 2)) : 1u;
        std::vector<std::vector<uint32_t>> mine_part(parts);
        auto work = [&](unsigned part) {
            const uint64_t k0 = count * part / parts, k1 = count * (part + 1) / parts;
            for (uint64_t k = k0; k < k1; ++k) {
                const uint64_t e = elite[k];
                if (e < P) {
                    no[k] = surv_owner[e];
                    ns[k] = surv_slot[e];
                } else {
                    const uint64_t i = e - P, p = i < half ? i : i - half;
                    const uint64_t rk = p / h_loc;
                    const uint64_t j = i < half ? p - rk * h_loc : h_loc + p - rk * h_loc;
                    no[k] = (int32_t)rk;
                    ns[k] = free_all[rk * n_loc + j];
                }
                if (no[k] == rank) mine_part[part].push_back(ns[k]);
            }
        };
        {
            std::vector<std::thread> workers;
            for (unsigned part = 1; part < parts; ++part) workers.emplace_back(work, part);
            work(0);
            for (auto& w : workers) w.join();
        }
        uint64_t mine = 0;
        for (const auto& v : mine_part) {
            std::memcpy(own_slots + mine, v.data(), v.size() * sizeof(uint32_t));
            mine += v.size();
        }
        std::memcpy(surv_owner, no.data(), count * sizeof(int32_t));
        std::memcpy(surv_slot, ns.data(), count * sizeof(uint32_t));
        *own_count = mine;
    });
}

int temo_b200_shard_create(const temo_b200_run_config* cfg, int rank, int world, temo_b200_shard** out) {
    return guarded_shard([&] {
        require(cfg && out, "shard_create: null argument");
        RunConfig rc;
        rc.problem = cfg->problem;
        rc.rng_mode = cfg->rng_mode;
        rc.pop = cfg->pop;
        rc.lattice_h = cfg->lattice_h;
        rc.generations = cfg->generations;
        rc.seed = cfg->seed;
        rc.dim = cfg->dim;
        rc.obj = cfg->obj;
        rc.alpha = cfg->alpha;
        rc.fr = cfg->fr;
        rc.ga.pc = cfg->ga.pc;
        rc.ga.eta = cfg->ga.eta;
        rc.ga.pm = cfg->ga.pm;
        rc.ga.xi = cfg->ga.xi;
        rc.fuse_eval = cfg->fuse_eval;
        rc.horizon = cfg->horizon ? cfg->horizon : 100;
        *out = new temo_b200_shard{new Shard(rc, rank, world)};
    });
}

int temo_b200_shard_destroy(temo_b200_shard* s) {
    return guarded_shard([&] {
        if (s) {
            delete s->impl;
            delete s;
        }
    });
}

// sizes: [0] n_loc, [1] d, [2] m, [3] r, [4] send_cap, [5] pcap, [6] cap_loc, [7] adapt_every
int temo_b200_shard_info(temo_b200_shard* s, uint64_t* info8) {
    return guarded_shard([&] {
        require(s && s->impl && info8, "shard_info: null argument");
        const Shard& S = *s->impl;
        const uint64_t v[8] = {S.n_loc, S.d, S.m, S.r, S.send_cap, S.pcap, S.cap_loc, S.adapt_every};
        std::memcpy(info8, v, sizeof(v));
    });
}

// device pointers the collectives operate on: which = 0 send_buf, 1 recv_buf, 2 f_off_loc, 3 f_gather,
// 4 best_key (int64 view, R), 5 first_row (int32 view, R), 6 best_row (int32 view, R), 7 free_slot (int32 view, n_loc)
void* temo_b200_shard_buffer(temo_b200_shard* s, int which) {
    if (!s || !s->impl) return nullptr;
    Shard& S = *s->impl;
    switch (which) {
    case 0: return S.send_buf;
    case 1: return S.recv_buf;
    case 2: return S.f_off_loc;
    case 3: return S.f_gather;
    case 4: return S.ws.best_key;
    case 5: return S.ws.first_row;
    case 6: return S.ws.best_row;
    case 7: return S.free_slot;
    default: return nullptr;
    }
}

int temo_b200_shard_pack(temo_b200_shard* s, const uint32_t* slots, uint64_t count) {
    return guarded_shard([&] { s->impl->pack(slots, count, 0); TEMO_CUDA(cudaStreamSynchronize(s->impl->stream)); });
}
int temo_b200_shard_reproduce(temo_b200_shard* s, const uint32_t* recv_pos, uint64_t c_sbx, uint64_t c_pm) {
    return guarded_shard([&] { s->impl->reproduce(recv_pos, c_sbx, c_pm, 0, 0); TEMO_CUDA(cudaStreamSynchronize(s->impl->stream)); });
}
// Pieces of a chunked exchange; both only enqueue work on the shard's stream (temo_b200_shard_stream) and return.
int temo_b200_shard_pack_at(temo_b200_shard* s, const uint32_t* slots, uint64_t count, uint64_t row0) {
    return guarded_shard([&] { s->impl->pack(slots, count, row0); });
}
int temo_b200_shard_reproduce_range(temo_b200_shard* s, const uint32_t* recv_pos, uint64_t c_sbx, uint64_t c_pm,
                                    uint64_t unit_begin, uint64_t unit_count) {
    return guarded_shard([&] { s->impl->reproduce(recv_pos, c_sbx, c_pm, unit_begin, unit_count); });
}
// The CUDA stream (cudaStream_t) every stage of this shard is enqueued on: a caller that issues collectives on it
// (or on a stream ordered against it) needs no device-wide synchronisation between stages.
void* temo_b200_shard_stream(temo_b200_shard* s) { return (s && s->impl) ? (void*)s->impl->stream : nullptr; }
int temo_b200_shard_place_f(temo_b200_shard* s, uint64_t P, int initial) {
    return guarded_shard([&] { s->impl->place_offspring_f(P, initial != 0); });
}
int temo_b200_shard_select_local(temo_b200_shard* s, uint64_t P, uint64_t lo, uint64_t hi, uint64_t t) {
    return guarded_shard([&] { s->impl->select_local(P, lo, hi, t); TEMO_CUDA(cudaStreamSynchronize(s->impl->stream)); });
}
int temo_b200_shard_select_rows(temo_b200_shard* s, uint64_t lo, uint64_t hi) {
    return guarded_shard([&] { s->impl->select_rows(lo, hi); TEMO_CUDA(cudaStreamSynchronize(s->impl->stream)); });
}
int temo_b200_shard_select_finish(temo_b200_shard* s, uint32_t* elite, uint64_t* count) {
    return guarded_shard([&] { *count = s->impl->select_finish(elite); });
}
int temo_b200_shard_commit(temo_b200_shard* s, uint64_t count, const uint32_t* own_slots, uint64_t own_count, uint64_t t) {
    return guarded_shard([&] { s->impl->commit(count, own_slots, own_count, t); });
}
// copies out this rank's rows: x of the given local slots (rows x d) and the replicated f / v / gamma
int temo_b200_shard_download(temo_b200_shard* s, const uint32_t* slots, uint64_t rows, double* x, uint64_t f_rows,
                             double* f, double* v, double* gamma) {
    return guarded_shard([&] {
        Shard& S = *s->impl;
        if (x && rows) {
            double* tmp = dev_alloc<double>(rows * S.d);
            uint32_t* ds = dev_alloc<uint32_t>(rows);
            TEMO_CUDA(cudaMemcpy(ds, slots, rows * sizeof(uint32_t), cudaMemcpyHostToDevice));
            gather_slots_kernel<<<(unsigned)rows, 256, 0, S.stream>>>(S.pool, ds, rows, S.d, tmp);
            const cudaError_t e = cudaMemcpyAsync(x, tmp, rows * S.d * sizeof(double), cudaMemcpyDeviceToHost, S.stream);
            cudaStreamSynchronize(S.stream);
            cudaFree(tmp);
            cudaFree(ds);
            TEMO_CUDA(e);
        }
        if (f && f_rows) TEMO_CUDA(cudaMemcpy(f, S.fm[S.cur], f_rows * S.m * sizeof(double), cudaMemcpyDeviceToHost));
        if (v) TEMO_CUDA(cudaMemcpy(v, S.v, S.r * S.m * sizeof(double), cudaMemcpyDeviceToHost));
        if (gamma) TEMO_CUDA(cudaMemcpy(gamma, S.gamma, S.r * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"
