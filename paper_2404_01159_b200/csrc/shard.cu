// Sharded generation loop: the stage-level pieces one rank (one process, one GPU) runs between the
// collectives that paper_2404_01159_b200/dist.py issues with torch.distributed.
//
// reference: the same rvea_run loop (algorithms.hpp:227-296); the reference itself is single-process.
// Sharding: rank g owns the mating pairs [g*h_loc, (g+1)*h_loc) of the shuffled order (h_loc = n/2/G),
// i.e. the children with global rows p and n/2+p; a survivor stays in the pool of the rank where it was
// born. Replicated on every rank, IN DEVICE MEMORY (a few MB): the merged objective matrix, the reference
// set with its direction index, and the survivor -> (owner rank, pool slot) tables.
//
// Parents: the mating shuffle pairs arbitrary rows, so a rank's pairs need parents from every rank's pool.
// They are not copied: every rank maps its peers' pools into its address space once (CUDA IPC over
// NVLink / NVSwitch), a kernel turns the replicated tables into one parent ADDRESS per local mating row,
// and K1 streams the remote rows directly (40 KB contiguous each, 128-bit loads: NVLink peer loads inside the
// kernel, overlapped tile by tile with its arithmetic and its local stores). No pack kernel, no all-to-all,
// no receive buffer, no host-side exchange plan. (The first round's design - host plan + pack + NCCL all-to-all of
// rows, pipelined in chunks - cost 11.0 ms per generation at world size 1 against 3.9 ms for the monolithic loop.)
// Exchanges per generation (NCCL, small): offspring objectives and free-slot lists (all-gather), per-vector
// minima (two min-allreduces). The host reads one word per generation (the survivor count, which decides the
// next generation's draw counters: algorithms.hpp:211-221) and ships the mating permutation (4 n bytes).
//
// Why remote reads are ordered without extra synchronisation: a rank's K1 of generation t+1 is enqueued behind
// its collectives of generation t on the same stream; those complete only after every peer has contributed,
// and a peer contributes behind its own K1 of generation t. So (i) every row a rank reads was written before
// the reader's K1 starts, and (ii) a slot freed by selection t is overwritten by its owner's K1 of t+1 only after
// every reader's K1 of generation t has finished (free slots never hold a current survivor).
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
    for (uint64_t j = threadIdx.x; j < d; j += blockDim.x) out[i * d + j] = pool[(uint64_t)slot[i] * d + j];
}

// initial tables: global row i lives on rank i / n_loc in slot i % n_loc (contiguous blocks of the initial population)
__global__ void init_tables_kernel(uint64_t n, uint64_t n_loc, uint32_t* owner, uint32_t* slot) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    owner[i] = (uint32_t)(i / n_loc);
    slot[i] = (uint32_t)(i % n_loc);
}

// Address of the parent of every local mating row: local row j is global mating row i (first halves of the pairs, then
// second halves); its parent is survivor k = pool_idx[perm[i]] (algorithms.hpp:211-221, operators.hpp:155-158), which
// lives in pool `owner[k]` at slot `slot[k]`.
template <int MODE>
__global__ void parent_ptr_kernel(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ owner, const uint32_t* __restrict__ slot,
                                  uint64_t n, uint64_t h_loc, uint64_t rank, uint64_t P, Rng rng, uint64_t c_pool, uint64_t d,
                                  const double* const* __restrict__ peer_pool, const double** __restrict__ parent) {
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j >= 2 * h_loc) return;
    const uint64_t i = j < h_loc ? rank * h_loc + j : n / 2 + rank * h_loc + (j - h_loc);
    const uint64_t q = perm[i];
    uint64_t k = q;
    if (P != n) k = (uint64_t)(word_to_unit(draw_word<MODE>(rng, c_pool + q)) * (double)P);
    parent[j] = peer_pool[owner[k]] + (uint64_t)slot[k] * d;
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

// Survivor k takes over merged row elite[k] (algorithms.hpp:278-279 in sharded form): a parent keeps its (owner, slot);
// child i = elite[k] - P lives on the rank that produced it, in that rank's free slot free_all[rank * n_loc + local
// child index]. Also: objectives compacted, the slots this rank owns marked used, the survivor count published.
__global__ void update_tables_kernel(const uint32_t* __restrict__ elite, const uint32_t* __restrict__ n_elite, uint64_t P, uint64_t n,
                                     uint64_t h_loc, uint32_t rank, const uint32_t* __restrict__ free_all,
                                     const uint32_t* __restrict__ owner, const uint32_t* __restrict__ slot,
                                     uint32_t* __restrict__ owner_next, uint32_t* __restrict__ slot_next, uint64_t m,
                                     const double* __restrict__ f_merged, double* __restrict__ f_next, unsigned char* __restrict__ used,
                                     uint32_t* d_P, uint32_t* own_count) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint32_t cnt = *n_elite;
    if (k == 0) *d_P = cnt;
    if (k >= cnt) return;
    const uint64_t e = elite[k];
    uint32_t o, s;
    if (e < P) {
        o = owner[e];
        s = slot[e];
    } else {
        const uint64_t i = e - P, half = n / 2, p = i < half ? i : i - half;
        const uint64_t rk = p / h_loc, j = i < half ? p - rk * h_loc : h_loc + p - rk * h_loc;
        o = (uint32_t)rk;
        s = free_all[rk * 2 * h_loc + j];
    }
    owner_next[k] = o;
    slot_next[k] = s;
    if (o == rank) {
        used[s] = 1;
        atomicAdd(own_count, 1u);
    }
    for (uint64_t j = 0; j < m; ++j) f_next[k * m + j] = f_merged[e * m + j];
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

struct Shard {
    RunConfig cfg;
    int rank = 0, world = 1;
    uint64_t n = 0, d = 0, m = 0, r = 0, H = 0, adapt_every = 1;
    uint64_t h_loc = 0, n_loc = 0, pcap = 0, cap_loc = 0;
    Rng rng{};
    cudaStream_t stream = nullptr;
    // population
    double* pool = nullptr;                  // cap_loc x d (the rows born on this rank)
    std::vector<void*> peer_host;            // pools of all ranks as seen from this process
    std::vector<bool> peer_opened;           // mapped through cudaIpcOpenMemHandle (to be closed)
    const double** peer_pool = nullptr;      // device copy of peer_host
    const double** parent = nullptr;         // [n_loc] parent address of every local mating row
    uint32_t* free_slot = nullptr;           // [n_loc] where this rank's children go
    uint32_t* free_all = nullptr;            // [world x n_loc] all ranks' free-slot lists (all-gathered)
    unsigned char* used = nullptr;
    uint32_t* free_scratch = nullptr;
    uint32_t *owner[2] = {nullptr, nullptr}, *slot[2] = {nullptr, nullptr};  // replicated survivor tables [pcap]
    int tcur = 0;
    uint32_t* perm_dev = nullptr;            // [n] mating permutation of the current generation
    uint32_t* h_perm[2] = {nullptr, nullptr};  // pinned; [hp] current, [hp ^ 1] being shuffled for the next generation
    int hp = 0;
    std::thread perm_worker;
    uint64_t spec_c_shuffle = 0;
    bool spec_valid = false;
    // objectives, reference set, selection
    double* fm[2] = {nullptr, nullptr};      // replicated merged objectives, (pcap + n) x m
    int cur = 0;
    double* f_off_loc = nullptr;             // n_loc x m
    double* f_gather = nullptr;              // world x n_loc x m
    double *v0 = nullptr, *v = nullptr, *gamma = nullptr, *lower = nullptr, *upper = nullptr;
    BoundSegments bound_seg;
    double *zmin = nullptr, *zmax = nullptr;
    unsigned long long* zscratch = nullptr;
    uint32_t* skip_flag = nullptr;
    uint32_t* d_P = nullptr;                 // [2]: survivor count, survivors owned by this rank
    uint32_t* h_status = nullptr;            // pinned: [0] error flags, [1] survivor count, [2] own count
    SelectWorkspace ws;
    VecIndex vindex;
    // loop state (host)
    uint64_t P = 0, counter = 0, t = 0, lo = 0, hi = 0;
    uint64_t c_sbx = 0, c_pm = 0, c_end = 0;
    uint64_t launches = 0;                   // kernels + copies enqueued by this shard so far

    Shard(const RunConfig& c, int rank_, int world_) : cfg(c), rank(rank_), world(world_) {
        preload_adapt_kernels();  // first used at the first adaptation: not in the middle of the loop
        require(world >= 1 && rank >= 0 && rank < world, "shard: bad rank");
        require(problem_known(cfg.problem), "make_problem: unknown problem");
        require(cfg.op == kOpGa, "shard: the sharded loop runs the ga operator");
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
        require(cap_loc < 0xffffffffULL && pcap + n < 0xffffffffULL, "shard: population too large for 32-bit slots");
        stream = ctx().stream;
        pool = dev_alloc<double>(cap_loc * d);
        peer_host.assign(world, nullptr);
        peer_opened.assign(world, false);
        peer_host[rank] = pool;
        peer_pool = reinterpret_cast<const double**>(reinterpret_cast<void*>(dev_alloc<void*>(world)));
        parent = reinterpret_cast<const double**>(reinterpret_cast<void*>(dev_alloc<void*>(n_loc)));
        free_slot = dev_alloc<uint32_t>(n_loc);
        free_all = dev_alloc<uint32_t>((uint64_t)world * n_loc);
        used = dev_alloc<unsigned char>(cap_loc);
        free_scratch = compact_state_alloc(cap_loc);
        for (int b = 0; b < 2; ++b) {
            owner[b] = dev_alloc<uint32_t>(pcap);
            slot[b] = dev_alloc<uint32_t>(pcap);
            fm[b] = dev_alloc<double>((pcap + n) * m);
            TEMO_CUDA(cudaHostAlloc(&h_perm[b], n * sizeof(uint32_t), cudaHostAllocDefault));
        }
        TEMO_CUDA(cudaHostAlloc(&h_status, 4 * sizeof(uint32_t), cudaHostAllocDefault));
        perm_dev = dev_alloc<uint32_t>(n);
        f_off_loc = dev_alloc<double>(n_loc * m);
        f_gather = dev_alloc<double>((uint64_t)world * n_loc * m);
        v0 = dev_alloc<double>(r * m);
        v = dev_alloc<double>(r * m);
        gamma = dev_alloc<double>(r);
        lower = dev_alloc<double>(d);
        upper = dev_alloc<double>(d);
        zmin = dev_alloc<double>(m);
        zmax = dev_alloc<double>(m);
        zscratch = col_minmax_scratch_alloc(m);
        skip_flag = dev_alloc<uint32_t>(1);
        d_P = dev_alloc<uint32_t>(2);
        ws.alloc(pcap + n, r, m);
        if (world == 1) set_peers_direct(peer_host.data());
        const std::vector<double> unit = normalize_to_unit(simplex_lattice(m, H), r, m);
        TEMO_CUDA(cudaMemcpyAsync(v0, unit.data(), r * m * sizeof(double), cudaMemcpyHostToDevice, stream));
        TEMO_CUDA(cudaMemcpyAsync(v, v0, r * m * sizeof(double), cudaMemcpyDeviceToDevice, stream));
        launch_row_norms(v, r, m, ws.vn, stream);
        vindex.alloc(r, m);
        vindex.set_order(unit.data(), stream);
        if (!assoc_filter_preferred(m, r)) vindex.build(v, ws.vn, stream);  // m >= 5: the fp32-filtered scans need no index
        launch_gamma_auto(v, r, m, ws, &vindex, gamma, ws.err_flag, nullptr, stream);
        std::vector<double> blo(d), bhi(d);
        problem_bounds(cfg.problem, d, m, blo.data(), bhi.data());
        bound_seg = find_bound_segments(blo.data(), bhi.data(), d);
        TEMO_CUDA(cudaMemcpyAsync(lower, blo.data(), d * sizeof(double), cudaMemcpyHostToDevice, stream));
        TEMO_CUDA(cudaMemcpyAsync(upper, bhi.data(), d * sizeof(double), cudaMemcpyHostToDevice, stream));
        // initial population (algorithms.hpp:241-242): global rows [rank*n/world, (rank+1)*n/world) in local
        // slots 0.., drawn at their global counters; objectives of the local block
        launch_random_reproduce(pool, nullptr, n_loc, d, rng, (uint64_t)rank * n_loc * d, lower, upper, stream);
        EvalArgs ea;
        ea.problem = cfg.problem;
        ea.x = pool;
        ea.n = n_loc;
        ea.d = d;
        ea.m = m;
        ea.horizon = cfg.horizon;
        ea.f = f_off_loc;
        launch_evaluate(ea, stream);
        init_tables_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(n, n_loc, owner[tcur], slot[tcur]);
        TEMO_CUDA(cudaMemsetAsync(used, 0, cap_loc, stream));
        TEMO_CUDA(cudaMemsetAsync(used, 1, n_loc, stream));  // slots 0 .. n_loc - 1 hold the initial block
        launch_compact(cap_loc, FreePredS{used}, IdentityValS{}, free_scratch, n_loc, free_slot, nullptr, stream);
        TEMO_CUDA(cudaStreamSynchronize(stream));
        check();
        P = n;
        counter = n * d;  // operators.hpp:287-296: n*d draws for the initial population
    }

    ~Shard() {
        if (perm_worker.joinable()) perm_worker.join();
        cudaStreamSynchronize(stream);
        for (int g = 0; g < world; ++g)
            if (peer_opened[g]) cudaIpcCloseMemHandle(peer_host[g]);
        cudaFree(pool); cudaFree(peer_pool); cudaFree(parent); cudaFree(free_slot); cudaFree(free_all); cudaFree(used);
        cudaFree(free_scratch); cudaFree(perm_dev); cudaFree(f_off_loc); cudaFree(f_gather);
        for (int b = 0; b < 2; ++b) {
            cudaFree(owner[b]); cudaFree(slot[b]); cudaFree(fm[b]);
            cudaFreeHost(h_perm[b]);
        }
        cudaFreeHost(h_status);
        cudaFree(v0); cudaFree(v); cudaFree(gamma); cudaFree(lower); cudaFree(upper);
        cudaFree(zmin); cudaFree(zmax); cudaFree(zscratch); cudaFree(skip_flag); cudaFree(d_P);
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

    // ---- peer pools
    void ipc_handle(unsigned char* out64) {
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handles are 64 bytes");
        cudaIpcMemHandle_t h;
        TEMO_CUDA(cudaIpcGetMemHandle(&h, pool));
        std::memcpy(out64, &h, sizeof(h));
    }
    void open_peers(const unsigned char* handles) {  // world x 64 bytes, all-gathered by the caller
        for (int g = 0; g < world; ++g) {
            if (g == rank) continue;
            cudaIpcMemHandle_t h;
            std::memcpy(&h, handles + 64 * (size_t)g, sizeof(h));
            void* p = nullptr;
            TEMO_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            peer_host[g] = p;
            peer_opened[g] = true;
        }
        set_peers_direct(peer_host.data());
    }
    void set_peers_direct(void* const* ptrs) {  // pools already addressable from this process
        for (int g = 0; g < world; ++g) {
            require(ptrs[g] != nullptr && (reinterpret_cast<uintptr_t>(ptrs[g]) & 15u) == 0, "shard: bad peer pool pointer");
            peer_host[g] = ptrs[g];
        }
        TEMO_CUDA(cudaMemcpyAsync(peer_pool, peer_host.data(), world * sizeof(void*), cudaMemcpyHostToDevice, stream));
        TEMO_CUDA(cudaStreamSynchronize(stream));
    }

    // ---- the mating permutation: shuffled on a host thread for the next generation while the GPU works on this one
    void shuffle_into(uint32_t* dst, uint64_t c_shuffle) {
        uint64_t c = c_shuffle;
        shuffle_indices(cfg.seed, c, n, dst);
    }
    void ensure_permutation(uint64_t c_shuffle) {
        if (perm_worker.joinable()) perm_worker.join();
        if (spec_valid && spec_c_shuffle == c_shuffle) {
            hp ^= 1;  // the speculation was right
        } else {
            shuffle_into(h_perm[hp], c_shuffle);
        }
        spec_valid = false;
    }
    void prefetch_permutation(uint64_t c_shuffle) {
        spec_c_shuffle = c_shuffle;
        spec_valid = true;
        uint32_t* dst = h_perm[hp ^ 1];
        perm_worker = std::thread([this, dst, c_shuffle] { shuffle_into(dst, c_shuffle); });
    }

    // ---- stage 1: draw counters of the generation, permutation, parent addresses
    void begin() {
        require(t < cfg.generations, "rvea_run: all generations already done");
        uint64_t c = counter;
        const uint64_t c_pool = c;
        if (P != n) c += n;  // algorithms.hpp:211-221
        ensure_permutation(c);
        c += n - 1;
        c_sbx = c;
        c_pm = c_sbx + 3 * (n / 2) * d + n / 2;
        c_end = c_pm + 2 * n * d;
        TEMO_CUDA(cudaMemcpyAsync(perm_dev, h_perm[hp], n * sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
        const unsigned g = (unsigned)((n_loc + 255) / 256);
        if (rng.mode == 0)
            parent_ptr_kernel<0><<<g, 256, 0, stream>>>(perm_dev, owner[tcur], slot[tcur], n, h_loc, (uint64_t)rank, P, rng, c_pool, d,
                                                        peer_pool, parent);
        else
            parent_ptr_kernel<1><<<g, 256, 0, stream>>>(perm_dev, owner[tcur], slot[tcur], n, h_loc, (uint64_t)rank, P, rng, c_pool, d,
                                                        peer_pool, parent);
        TEMO_CUDA(cudaGetLastError());
        launches += 2;
        // the next generation's shuffle (its counter assumes a survivor count != n; redone in the rare other case)
        if (t + 1 < cfg.generations) prefetch_permutation(c_end + n);
        const uint64_t rows = P + n;
        lo = rows * (uint64_t)rank / (uint64_t)world;
        hi = rows * (uint64_t)(rank + 1) / (uint64_t)world;
    }

    // ---- stage 2: K1 (+ fused evaluation) on this rank's pairs; parents streamed from wherever they live
    void reproduce() {
        ReproArgs ra;
        ra.src_ptr = parent;
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
        const bool fused = fuse_offspring_eval(cfg.fuse_eval, cfg.problem, d);
        if (fused) {
            ra.eval_problem = cfg.problem;
            ra.m = m;
            ra.f_out = f_off_loc;
            ra.f_row0 = 0;
        }
        launch_reproduce(ra, stream);
        launches += fused ? 3 : 1;
        if (!fused) {
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
            launches += 2;
        }
    }

    // f_gather (all-gathered objectives) -> rows [0, n) in global order (initial population)
    void place_initial_f() {
        TEMO_CUDA(cudaMemcpyAsync(fm[cur], f_gather, n * m * sizeof(double), cudaMemcpyDeviceToDevice, stream));
        ++launches;
    }

    // ---- stage 3 (after the all-gathers): merged objectives, ideal point, association / APD of this rank's slice of
    // merged rows, local per-vector minima in the order-preserving signed views the min-allreduces need
    void select_local() {
        const uint64_t total = (uint64_t)world * n_loc, rows = P + n;
        scatter_offspring_f_kernel<<<(unsigned)((total + 255) / 256), 256, 0, stream>>>(f_gather, world, h_loc, n / 2, m, P, fm[cur]);
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
        TEMO_CUDA(cudaGetLastError());
        launches += 11;
    }

    // ---- stage 4 (after the min-allreduce of best_key / first_row): lowest row attaining the minimum, own slice
    void select_rows() {
        flip_keys_kernel<<<(unsigned)((r + 255) / 256), 256, 0, stream>>>(ws.best_key, r);
        flip_rows_kernel<<<(unsigned)((r + 255) / 256), 256, 0, stream>>>(ws.first_row, r);
        if (hi > lo) launch_elite_rows(hi - lo, ws.assoc + lo, ws.apd + lo, ws.best_key, ws.best_row, (uint32_t)lo, stream);
        flip_rows_kernel<<<(unsigned)((r + 255) / 256), 256, 0, stream>>>(ws.best_row, r);
        TEMO_CUDA(cudaGetLastError());
        launches += 4;
    }

    // ---- stage 5 (after the min-allreduce of best_row): compaction, survivor tables, free list, adaptation; the one
    // host synchronisation of the generation reads the survivor count back
    uint64_t finish() {
        flip_rows_kernel<<<(unsigned)((r + 255) / 256), 256, 0, stream>>>(ws.best_row, r);
        launch_select_finish(r, ws, /*nan_rule=*/false, stream);
        TEMO_CUDA(cudaMemsetAsync(used, 0, cap_loc, stream));
        TEMO_CUDA(cudaMemsetAsync(d_P + 1, 0, sizeof(uint32_t), stream));
        const uint64_t kmax = r < P + n ? r : P + n;
        update_tables_kernel<<<(unsigned)((kmax + 255) / 256), 256, 0, stream>>>(ws.elite, ws.n_elite, P, n, h_loc, (uint32_t)rank, free_all,
                                                                               owner[tcur], slot[tcur], owner[tcur ^ 1], slot[tcur ^ 1], m,
                                                                               fm[cur], fm[cur ^ 1], used, d_P, d_P + 1);
        launch_compact(cap_loc, FreePredS{used}, IdentityValS{}, free_scratch, n_loc, free_slot, nullptr, stream);
        launches += 11;
        if ((t + 1) % adapt_every == 0) {  // algorithms.hpp:281 (replicated: every rank adapts identically)
            launch_col_minmax(fm[cur ^ 1], pcap, d_P, m, zmin, zmax, zscratch, stream);
            launch_adapt_vectors(v0, v, ws.vn, r, m, zmin, zmax, skip_flag, ws.err_flag, stream);
            if (!assoc_filter_preferred(m, r)) vindex.build(v, ws.vn, stream);
            launch_gamma_auto(v, r, m, ws, &vindex, gamma, ws.err_flag, skip_flag, stream);
            launches += 8 + vindex.levels;
        }
        TEMO_CUDA(cudaMemcpyAsync(h_status, ws.err_flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, stream));
        TEMO_CUDA(cudaMemcpyAsync(h_status + 1, d_P, 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, stream));
        TEMO_CUDA(cudaGetLastError());
        TEMO_CUDA(cudaStreamSynchronize(stream));
        if (h_status[0] & 1u) fail(1, "rv_select: gamma must be positive");
        if (h_status[0] & 2u) fail(1, "normalize_to_unit: zero row");
        const uint64_t cnt = h_status[1];
        // this rank's share of the survivors plus its next children must fit its pool (births are spread uniformly)
        require((uint64_t)h_status[2] + n_loc <= cap_loc, "shard: local pool too small (ownership imbalance)");
        cur ^= 1;
        tcur ^= 1;
        P = cnt;
        counter = c_end;
        ++t;
        return cnt;
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
        rc.op = cfg->op;
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

// sizes: [0] n_loc, [1] d, [2] m, [3] r, [4] pcap, [5] cap_loc, [6] adapt_every, [7] kernels / copies enqueued so far
int temo_b200_shard_info(temo_b200_shard* s, uint64_t* info8) {
    return guarded_shard([&] {
        require(s && s->impl && info8, "shard_info: null argument");
        const Shard& S = *s->impl;
        const uint64_t v[8] = {S.n_loc, S.d, S.m, S.r, S.pcap, S.cap_loc, S.adapt_every, S.launches};
        std::memcpy(info8, v, sizeof(v));
    });
}

// loop state: [0] survivor count, [1] draw counter, [2] generations done, [3] lo, [4] hi (this rank's slice of the merged rows
// of the generation begun last)
int temo_b200_shard_state(temo_b200_shard* s, uint64_t* state5) {
    return guarded_shard([&] {
        require(s && s->impl && state5, "shard_state: null argument");
        const Shard& S = *s->impl;
        const uint64_t v[5] = {S.P, S.counter, S.t, S.lo, S.hi};
        std::memcpy(state5, v, sizeof(v));
    });
}

// device pointers the collectives operate on: which = 0 f_off_loc (n_loc x m), 1 f_gather (world x n_loc x m),
// 2 best_key (int64 view, R), 3 first_row (int32 view, R), 4 best_row (int32 view, R), 5 free_slot (int32 view, n_loc),
// 6 free_all (int32 view, world x n_loc), 7 pool (cap_loc x d)
void* temo_b200_shard_buffer(temo_b200_shard* s, int which) {
    if (!s || !s->impl) return nullptr;
    Shard& S = *s->impl;
    switch (which) {
    case 0: return S.f_off_loc;
    case 1: return S.f_gather;
    case 2: return S.ws.best_key;
    case 3: return S.ws.first_row;
    case 4: return S.ws.best_row;
    case 5: return S.free_slot;
    case 6: return S.free_all;
    case 7: return S.pool;
    default: return nullptr;
    }
}

// The CUDA stream (cudaStream_t) every stage of this shard is enqueued on: a caller that issues collectives on it
// (or on a stream ordered against it) needs no device-wide synchronisation between stages.
void* temo_b200_shard_stream(temo_b200_shard* s) { return (s && s->impl) ? (void*)s->impl->stream : nullptr; }

int temo_b200_shard_ipc_handle(temo_b200_shard* s, unsigned char* handle64) {
    return guarded_shard([&] {
        require(s && s->impl && handle64, "shard_ipc_handle: null argument");
        s->impl->ipc_handle(handle64);
    });
}
int temo_b200_shard_open_peers(temo_b200_shard* s, const unsigned char* handles) {
    return guarded_shard([&] {
        require(s && s->impl && handles, "shard_open_peers: null argument");
        s->impl->open_peers(handles);
    });
}
int temo_b200_shard_set_peer_pointers(temo_b200_shard* s, void* const* pools) {
    return guarded_shard([&] {
        require(s && s->impl && pools, "shard_set_peer_pointers: null argument");
        s->impl->set_peers_direct(pools);
    });
}

int temo_b200_shard_begin(temo_b200_shard* s) {
    return guarded_shard([&] { s->impl->begin(); });
}
int temo_b200_shard_reproduce(temo_b200_shard* s) {
    return guarded_shard([&] { s->impl->reproduce(); });
}
int temo_b200_shard_place_initial_f(temo_b200_shard* s) {
    return guarded_shard([&] { s->impl->place_initial_f(); });
}
int temo_b200_shard_select_local(temo_b200_shard* s) {
    return guarded_shard([&] { s->impl->select_local(); });
}
int temo_b200_shard_select_rows(temo_b200_shard* s) {
    return guarded_shard([&] { s->impl->select_rows(); });
}
int temo_b200_shard_finish(temo_b200_shard* s, uint64_t* count) {
    return guarded_shard([&] {
        require(count != nullptr, "shard_finish: null argument");
        *count = s->impl->finish();
    });
}

// Copies out the replicated state and this rank's rows: owner / slot tables (P entries each), x of the survivors this
// rank owns (in survivor order, own_rows x d; own_index receives their survivor indices), f (P x m), v, gamma. Any may be NULL.
int temo_b200_shard_download(temo_b200_shard* s, uint32_t* owner, uint32_t* slot, uint64_t* own_rows, uint64_t* own_index, double* x,
                             double* f, double* v, double* gamma) {
    return guarded_shard([&] {
        Shard& S = *s->impl;
        TEMO_CUDA(cudaStreamSynchronize(S.stream));
        std::vector<uint32_t> o(S.P), sl(S.P);
        TEMO_CUDA(cudaMemcpy(o.data(), S.owner[S.tcur], S.P * sizeof(uint32_t), cudaMemcpyDeviceToHost));
        TEMO_CUDA(cudaMemcpy(sl.data(), S.slot[S.tcur], S.P * sizeof(uint32_t), cudaMemcpyDeviceToHost));
        if (owner) std::memcpy(owner, o.data(), S.P * sizeof(uint32_t));
        if (slot) std::memcpy(slot, sl.data(), S.P * sizeof(uint32_t));
        std::vector<uint32_t> mine;
        std::vector<uint64_t> idx;
        for (uint64_t k = 0; k < S.P; ++k)
            if (o[k] == (uint32_t)S.rank) {
                mine.push_back(sl[k]);
                idx.push_back(k);
            }
        if (own_rows) *own_rows = mine.size();
        if (own_index) std::memcpy(own_index, idx.data(), idx.size() * sizeof(uint64_t));
        if (x && !mine.empty()) {
            double* tmp = dev_alloc<double>(mine.size() * S.d);
            uint32_t* ds = dev_alloc<uint32_t>(mine.size());
            TEMO_CUDA(cudaMemcpy(ds, mine.data(), mine.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
            gather_slots_kernel<<<(unsigned)mine.size(), 256, 0, S.stream>>>(S.pool, ds, mine.size(), S.d, tmp);
            const cudaError_t e = cudaMemcpyAsync(x, tmp, mine.size() * S.d * sizeof(double), cudaMemcpyDeviceToHost, S.stream);
            cudaStreamSynchronize(S.stream);
            cudaFree(tmp);
            cudaFree(ds);
            TEMO_CUDA(e);
        }
        if (f && S.P) TEMO_CUDA(cudaMemcpy(f, S.fm[S.cur], S.P * S.m * sizeof(double), cudaMemcpyDeviceToHost));
        if (v) TEMO_CUDA(cudaMemcpy(v, S.v, S.r * S.m * sizeof(double), cudaMemcpyDeviceToHost));
        if (gamma) TEMO_CUDA(cudaMemcpy(gamma, S.gamma, S.r * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"
