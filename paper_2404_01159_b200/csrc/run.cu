// Device-resident generation loop.
//
// reference: rvea_run (algorithms.hpp:227-296) with op = "ga", track_archive = false.
// The CPU loop copies the whole population four times per generation (take_rows x3, vconcat,
// plus the shuffle gather); here X never moves: the population lives in a pool of
// max(n,R)+n rows in HBM, survivors are addressed through a slot table, children are written
// into free slots, and the merged objective matrix (parents first, algorithms.hpp:274-275) is
// the only thing that is compacted (it is (|P|+n) x m, a few MB).
//
// Host work per generation: the sequential Fisher-Yates permutation (rng.hpp:69-78), computed
// speculatively for generation t+1 while the GPU runs generation t (the draw counters depend on
// the survivor count only through "|P| == n ? 0 : n" extra draws, algorithms.hpp:211-221 — the
// speculation assumes |P| != n and is redone in the rare other case), one 4*n-byte H2D of the
// permutation, and one 8-byte D2H of the survivor count + error flags.
#include <chrono>
#include <cmath>
#include <cstring>

#include <algorithm>

#include "compact.cuh"
#include "internal.h"
#include "run.h"

namespace temo_b200 {

namespace {

// src[i] = storage slot of the i-th row of the shuffled mating pool:
// pool_idx = identity when |P| == n, else floor(u * |P|) with u the draw at c_pool + q
// (algorithms.hpp:211-221); mating row i is pool row perm[i] (operators.hpp:155-158).
template <int MODE>
__global__ void build_src_kernel(const uint32_t* perm, const uint32_t* parent_slot, uint64_t n, uint64_t P,
                                 Rng rng, uint64_t c_pool, uint32_t* src, uint32_t* pool_idx_out) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t q = perm ? perm[i] : i;  // no mating shuffle for de / pso / cso: pool order
    uint64_t k = q;
    if (P != n) k = (uint64_t)(word_to_unit(draw_word<MODE>(rng, c_pool + q)) * (double)P);
    src[i] = parent_slot[k];
    if (pool_idx_out) pool_idx_out[i] = (uint32_t)k;  // survivor index of pool row i (its objective row)
}

// pool_f = take_rows(f, pool_idx) (algorithms.hpp:257,263)
__global__ void gather_f_kernel(const double* f, const uint32_t* idx, uint64_t n, uint64_t m, double* out) {
    const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (e >= n * m) return;
    const uint64_t i = e / m, j = e - i * m;
    out[e] = f[(uint64_t)idx[i] * m + j];
}

// Survivor k takes over the storage slot and the objective row of merged row elite[k]
// (detail::take_rows on merged_x / merged_f, algorithms.hpp:278-279).
__global__ void commit_survivors_kernel(const uint32_t* elite, const uint32_t* n_elite, uint64_t P, uint64_t m,
                                        const uint32_t* parent_slot, const uint32_t* free_slot,
                                        uint32_t* parent_slot_next, const double* f_merged, double* f_next,
                                        unsigned char* used, uint32_t* d_P) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint32_t cnt = *n_elite;
    if (k == 0) *d_P = cnt;
    if (k >= cnt) return;
    const uint32_t e = elite[k];
    const uint32_t slot = e < P ? parent_slot[e] : free_slot[e - P];
    parent_slot_next[k] = slot;
    used[slot] = 1;
    for (uint64_t j = 0; j < m; ++j) f_next[k * m + j] = f_merged[(uint64_t)e * m + j];
}

// The first `want` unused slots in ascending order become the next free list.
struct FreePred {
    const unsigned char* used;
    __device__ bool operator()(uint64_t i) const { return used[i] == 0; }
};
struct IdentityVal {
    __device__ uint32_t operator()(uint64_t i) const { return (uint32_t)i; }
};

__global__ void iota_kernel(uint32_t* p, uint64_t n, uint32_t first) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = first + (uint32_t)i;
}

__global__ void gather_rows_kernel(const double* pool, const uint32_t* slot, uint64_t rows, uint64_t d, double* out) {
    const uint64_t i = blockIdx.x;
    if (i >= rows) return;
    const double* p = pool + (uint64_t)slot[i] * d;
    for (uint64_t j = threadIdx.x; j < d; j += blockDim.x) out[i * d + j] = p[j];
}

__global__ void scatter_rows_kernel(const double* in, const uint32_t* slot, uint64_t rows, uint64_t d, double* pool) {
    const uint64_t i = blockIdx.x;
    if (i >= rows) return;
    double* p = pool + (uint64_t)slot[i] * d;
    for (uint64_t j = threadIdx.x; j < d; j += blockDim.x) p[j] = in[i * d + j];
}

double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

Run::Run(const RunConfig& c) : cfg(c) {
    require(cfg.pop >= 2 && cfg.generations >= 1, "rvea_run: bad config");  // algorithms.hpp:229
    require(problem_known(cfg.problem), "make_problem: unknown problem");
    require(cfg.obj >= 2 && cfg.obj <= (uint64_t)kMaxObj, "rvea_run: objective count out of range");
    require(cfg.op >= kOpGa && cfg.op <= kOpRandom, "rvea_run: unknown operator");  // algorithms.hpp:270
    if (cfg.op == kOpDe) require(cfg.pop >= 4, "de_reproduce: needs at least four rows");
    preload_adapt_kernels();  // first used at the first adaptation: not in the middle of the loop
    n = cfg.pop;
    m = cfg.obj;
    if (cfg.problem == kToy2 || cfg.problem == kToy3) {  // problems.hpp:279-287: the environment fixes m and d
        m = cfg.problem == kToy2 ? 2 : 3;
        require(cfg.dim == 0 || cfg.dim == problem_default_dim(cfg.problem, m), "make_problem: toy env dimension is fixed");
    }
    d = cfg.dim ? cfg.dim : problem_default_dim(cfg.problem, m);
    require(d >= m, "make_problem: DTLZ needs d >= m");  // problems.hpp:269
    H = cfg.lattice_h ? cfg.lattice_h : lattice_density_for(m, n);  // algorithms.hpp:233-235
    r = lattice_count(m, H);
    require(r >= 2, "min_vector_angles: needs at least two vectors");
    const double ae = std::ceil(cfg.fr * (double)cfg.generations);  // algorithms.hpp:237-239
    adapt_every = ae < 1.0 ? 1 : (uint64_t)ae;
    rng = make_rng(cfg.seed, cfg.rng_mode);
    pcap = n > r ? n : r;
    cap = pcap + n;
    require(cap < 0xffffffffULL, "rvea_run: population too large for 32-bit slots");
    Context& cx = ctx();
    stream = cx.stream;

    pool = dev_alloc<double>(cap * d);
    for (int b = 0; b < 2; ++b) {
        fm[b] = dev_alloc<double>(cap * m);
        parent_slot[b] = dev_alloc<uint32_t>(pcap);
        free_slot[b] = dev_alloc<uint32_t>(n);
        TEMO_CUDA(cudaMallocHost(&h_perm[b], n * sizeof(uint32_t)));
    }
    src = dev_alloc<uint32_t>(n);
    perm_dev = dev_alloc<uint32_t>(n);
    if (cfg.op == kOpPso || cfg.op == kOpCso) {  // SwarmState + the scalarised fitness of the pool (algorithms.hpp:255-268)
        pool_idx_dev = dev_alloc<uint32_t>(n);
        pool_f = dev_alloc<double>(n * m);
        scores = dev_alloc<double>(n);
        sw_vel[0] = dev_alloc<double>(n * d);
        if (cfg.op == kOpPso) {
            sw_pbx = dev_alloc<double>(n * d);
            sw_pbs = dev_alloc<double>(n);
            sw_best = dev_alloc<uint32_t>(1);
        } else {
            sw_mean = dev_alloc<double>(d);
        }
    }
    used = dev_alloc<unsigned char>(cap);
    d_P = dev_alloc<uint32_t>(1);
    free_scratch = compact_state_alloc(cap);
    v0 = dev_alloc<double>(r * m);
    v = dev_alloc<double>(r * m);
    gamma = dev_alloc<double>(r);
    lower = dev_alloc<double>(d);
    upper = dev_alloc<double>(d);
    zmin = dev_alloc<double>(m);
    zmax = dev_alloc<double>(m);
    zscratch = col_minmax_scratch_alloc(m);
    skip_flag = dev_alloc<uint32_t>(1);
    TEMO_CUDA(cudaMallocHost(&h_status, 4 * sizeof(uint32_t)));
    ws.alloc(cap, r, m);
    for (int s2 = 0; s2 < 2; ++s2)
        for (int e = 0; e < kNumEvents; ++e) TEMO_CUDA(cudaEventCreate(&ev[s2][e]));

    // reference set (algorithms.hpp:236): lattice + unit vectors on the host (once), gamma on device
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
    TEMO_CUDA(cudaStreamSynchronize(stream));  // host vectors go out of scope

    // initial population (algorithms.hpp:241-242): slots 0..n-1, n*d draws
    iota_kernel<<<(unsigned)((pcap + 255) / 256), 256, 0, stream>>>(parent_slot[0], pcap, 0);
    iota_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(free_slot[0], n, (uint32_t)n);
    launch_random_reproduce(pool, nullptr, n, d, rng, 0, lower, upper, stream);
    counter = n * d;
    EvalArgs ea;
    ea.problem = cfg.problem;
    ea.x = pool;
    ea.n = n;
    ea.d = d;
    ea.m = m;
    ea.horizon = cfg.horizon;
    ea.f = fm[0];
    launch_evaluate(ea, stream);
    P = n;
    const uint32_t p32 = (uint32_t)P;
    TEMO_CUDA(cudaMemcpyAsync(d_P, &p32, sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
    check_status();
    t = 0;
    cur = 0;
    spec_valid = false;
}

Run::~Run() {
    cudaStreamSynchronize(stream);
    cudaFree(pool);
    for (int b = 0; b < 2; ++b) {
        cudaFree(fm[b]);
        cudaFree(parent_slot[b]);
        cudaFree(free_slot[b]);
        cudaFreeHost(h_perm[b]);
    }
    cudaFree(src); cudaFree(perm_dev); cudaFree(used); cudaFree(d_P); cudaFree(free_scratch);
    cudaFree(v0); cudaFree(v); cudaFree(gamma); cudaFree(lower); cudaFree(upper);
    cudaFree(zmin); cudaFree(zmax); cudaFree(zscratch); cudaFree(skip_flag); cudaFree(f_off_saved);
    cudaFree(mc_pf); cudaFree(mc_nearest); cudaFree(mc_hv_ref); cudaFree(mc_hits);
    cudaFree(pool_idx_dev); cudaFree(pool_f); cudaFree(scores); cudaFree(sw_vel[0]); cudaFree(sw_vel[1]);
    cudaFree(sw_pbx); cudaFree(sw_pbs); cudaFree(sw_mean); cudaFree(sw_best);
    cudaFree(arch_x[0]); cudaFree(arch_x[1]); cudaFree(arch_f[0]); cudaFree(arch_f[1]);
    cudaFree(arch_keep); cudaFree(arch_list); cudaFree(arch_scratch); cudaFree(arch_count);
    cudaFreeHost(h_status);
    ws.release();
    vindex.release();
    for (int s2 = 0; s2 < 2; ++s2)
        for (int e = 0; e < kNumEvents; ++e) cudaEventDestroy(ev[s2][e]);
}

// Reads n_elite / error flags back (one small D2H) and turns device-side contract violations
// into the reference's exceptions.
void Run::check_status() {
    TEMO_CUDA(cudaMemcpyAsync(h_status, ws.err_flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, stream));
    TEMO_CUDA(cudaMemcpyAsync(h_status + 1, d_P, sizeof(uint32_t), cudaMemcpyDeviceToHost, stream));
    TEMO_CUDA(cudaStreamSynchronize(stream));
    if (h_status[0] & 1u) fail(1, "min_vector_angles: duplicate reference vectors");  // refvec.hpp:97-98
    if (h_status[0] & 2u) fail(1, "normalize_to_unit: zero row");                      // refvec.hpp:72
}

// Draw-counter plan of one generation.
Run::Plan Run::plan_for(uint64_t P_now, uint64_t c) const {
    Plan p;
    p.c_pool = c;
    if (P_now != n) c += n;
    p.c_shuffle = c;
    if (uses_perm()) c += n - 1;  // ga: operators.hpp:155, cso: operators.hpp:254
    p.c_sbx = c;
    const uint64_t h = n / 2;
    switch (cfg.op) {
    case kOpGa:
        c += 3 * h * d + h;
        p.c_pm = c;
        c += 2 * n * d;
        break;
    case kOpDe: c += 4 * n + n * d; break;   // operators.hpp:170-172
    case kOpPso: c += 2 * n * d; break;      // operators.hpp:223-224
    case kOpCso: c += 3 * h * d; break;      // operators.hpp:256-258
    default: c += n * d; break;              // random_reproduce, operators.hpp:289
    }
    if (cfg.op != kOpGa) p.c_pm = c;
    p.c_end = c;
    return p;
}

void Run::ensure_permutation(const Plan& p) {
    if (!uses_perm()) return;
    if (spec_valid && spec_c_shuffle == p.c_shuffle) return;  // speculation hit
    uint64_t c = p.c_shuffle;
    shuffle_indices(cfg.seed, c, n, h_perm[hp]);
    spec_c_shuffle = p.c_shuffle;
    spec_valid = true;
}

void Run::launch_mating_table(const Plan& p) {
    const unsigned g = (unsigned)((n + 255) / 256);
    // ga mates rows in shuffled order; the other operators address the pool in its own order (cso applies its
    // permutation to pool rows itself)
    const uint32_t* perm = cfg.op == kOpGa ? perm_dev : nullptr;
    if (rng.mode == 0)
        build_src_kernel<0><<<g, 256, 0, stream>>>(perm, parent_slot[cur], n, P, rng, p.c_pool, src, pool_idx_dev);
    else
        build_src_kernel<1><<<g, 256, 0, stream>>>(perm, parent_slot[cur], n, P, rng, p.c_pool, src, pool_idx_dev);
}

// de / pso / cso / random in place of ga_reproduce (algorithms.hpp:253-268): operands are read through src[] (pool row
// i = storage row src[i]), children go to the free slots; pso and cso take apd_scores of the pool's objectives as
// fitness and carry the SwarmState, which is indexed by pool row like the reference's.
uint64_t Run::launch_other_operator(const Plan& p) {
    uint64_t launches = 0;
    if (cfg.op == kOpPso || cfg.op == kOpCso) {
        gather_f_kernel<<<(unsigned)((n * m + 255) / 256), 256, 0, stream>>>(fm[cur], pool_idx_dev, n, m, pool_f);  // :257,263
        const double penalty = apd_penalty(m, t, cfg.generations, cfg.alpha);
        launch_select(pool_f, n, nullptr, m, v, gamma, r, penalty, ws, stream, &vindex);  // apd_scores = rv_core's apd column
        TEMO_CUDA(cudaMemcpyAsync(scores, ws.apd, n * sizeof(double), cudaMemcpyDeviceToDevice, stream));
        launches += 1 + 9;
        if (!swarm_ready) {  // make_swarm_state (operators.hpp:58-60): zero velocities, personal bests = the pool
            TEMO_CUDA(cudaMemsetAsync(sw_vel[0], 0, n * d * sizeof(double), stream));
            if (cfg.op == kOpPso) {
                gather_rows_kernel<<<(unsigned)n, 256, 0, stream>>>(pool, src, n, d, sw_pbx);
                TEMO_CUDA(cudaMemcpyAsync(sw_pbs, scores, n * sizeof(double), cudaMemcpyDeviceToDevice, stream));
                ++launches;
            }
            sw_cur = 0;
            swarm_ready = true;
        }
    }
    switch (cfg.op) {
    case kOpDe:
        launch_de(pool, n, d, rng, p.c_sbx, cfg.de_f, cfg.de_cr, lower, upper, pool, stream, src, free_slot[cur]);
        launches += 1;
        break;
    case kOpPso:
        launch_pso(pool, scores, n, d, rng, p.c_sbx, cfg.pso_inertia, cfg.pso_c1, cfg.pso_c2, sw_vel[0], sw_pbx, sw_pbs, sw_best,
                   lower, upper, pool, stream, src, free_slot[cur]);
        launches += 3;
        break;
    case kOpCso:
        launch_cso(pool, scores, n, d, rng, p.c_sbx, cfg.cso_phi, perm_dev, sw_mean, sw_vel[0], sw_vel[0] /* in place: a row's velocity is touched by its own pair only */, lower,
                   upper, pool, stream, src, free_slot[cur]);
        launches += 2;
        break;
    default:  // random_reproduce (algorithms.hpp:266-267)
        launch_random_reproduce(pool, free_slot[cur], n, d, rng, p.c_sbx, lower, upper, stream);
        launches += 1;
        break;
    }
    return launches;
}

void Run::launch_reproduction(const Plan& p, bool fused) {
    ReproArgs ra;
    ra.pool = pool;
    ra.src = src;
    ra.out = pool;
    ra.dst = free_slot[cur];
    ra.n = n;
    ra.d = d;
    ra.rng = rng;
    ra.c_sbx = p.c_sbx;
    ra.c_pm = p.c_pm;
    ra.ga = cfg.ga;
    ra.lower = lower;
    ra.upper = upper;
    ra.seg = bound_seg;
    if (fused) {
        ra.eval_problem = cfg.problem;
        ra.m = m;
        ra.f_out = fm[cur];
        ra.f_row0 = P;
    }
    launch_reproduce(ra, stream);
}

void Run::launch_offspring_eval() {
    EvalArgs ea;
    ea.problem = cfg.problem;
    ea.x = pool;
    ea.rows = free_slot[cur];
    ea.n = n;
    ea.d = d;
    ea.m = m;
    ea.horizon = cfg.horizon;
    ea.f = fm[cur];
    ea.f_row0 = P;
    launch_evaluate(ea, stream);
}

bool Run::fusable() const { return cfg.op == kOpGa && cfg.fuse_eval && cfg.problem >= kDtlz1 && cfg.problem <= kDtlz4; }

uint64_t Run::step(double* survivors_f_host, const double* f_off_inject) {
    require(t < cfg.generations, "rvea_run: all generations already done");
    const double host0 = now_ms();
    P_before = P;
    const Plan p = plan_for(P, counter);
    ensure_permutation(p);
    const double host1 = now_ms();

    cudaEvent_t* const evs = ev[evp];
    TEMO_CUDA(cudaEventRecord(evs[0], stream));
    if (uses_perm())
        TEMO_CUDA(cudaMemcpyAsync(perm_dev, h_perm[hp], n * sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
    const bool fused = cfg.op == kOpGa && fuse_offspring_eval(cfg.fuse_eval, cfg.problem, d);
    launch_mating_table(p);
    TEMO_CUDA(cudaEventRecord(evs[1], stream));
    uint64_t launches = 1 + (fused ? 0 : 1) + 9 + 4;
    if (cfg.op == kOpGa) {
        launch_reproduction(p, fused);
        ++launches;
    } else {
        launches += launch_other_operator(p);
    }
    TEMO_CUDA(cudaEventRecord(evs[2], stream));
    if (!fused) launch_offspring_eval();
    TEMO_CUDA(cudaEventRecord(evs[3], stream));
    if (f_off_inject) {  // lock-step testing: keep the device's objectives aside, select on the given ones
        if (!f_off_saved) f_off_saved = dev_alloc<double>(n * m);
        TEMO_CUDA(cudaMemcpyAsync(f_off_saved, fm[cur] + P * m, n * m * sizeof(double), cudaMemcpyDeviceToDevice, stream));
        TEMO_CUDA(cudaMemcpyAsync(fm[cur] + P * m, f_off_inject, n * m * sizeof(double), cudaMemcpyHostToDevice, stream));
    }
    f_off_was_injected = f_off_inject != nullptr;

    // environmental selection over the merged population (algorithms.hpp:274-279)
    const double penalty = apd_penalty(m, t, cfg.generations, cfg.alpha);
    launch_select(fm[cur], P + n, nullptr, m, v, gamma, r, penalty, ws, stream, &vindex);
    TEMO_CUDA(cudaMemsetAsync(used, 0, cap, stream));
    const uint64_t kmax = r < P + n ? r : P + n;
    commit_survivors_kernel<<<(unsigned)((kmax + 255) / 256), 256, 0, stream>>>(
        ws.elite, ws.n_elite, P, m, parent_slot[cur], free_slot[cur], parent_slot[cur ^ 1], fm[cur], fm[cur ^ 1],
        used, d_P);
    launch_compact(cap, FreePred{used}, IdentityVal{}, free_scratch, n, free_slot[cur ^ 1], nullptr, stream);
    TEMO_CUDA(cudaEventRecord(evs[4], stream));

    // reference-vector adaptation (algorithms.hpp:281)
    if ((t + 1) % adapt_every == 0) {
        launch_col_minmax(fm[cur ^ 1], pcap, d_P, m, zmin, zmax, zscratch, stream);
        launch_adapt_vectors(v0, v, ws.vn, r, m, zmin, zmax, skip_flag, ws.err_flag, stream);
        if (!assoc_filter_preferred(m, r)) vindex.build(v, ws.vn, stream);  // m >= 5: the fp32-filtered scans need no index
        launch_gamma_auto(v, r, m, ws, &vindex, gamma, ws.err_flag, skip_flag, stream);
        launches += 6 + vindex.levels;
    }
    TEMO_CUDA(cudaEventRecord(evs[5], stream));
    // the survivors' objectives for the caller: at most kmax rows survive (one per reference vector), and they sit at the
    // head of the next generation's objective block; copied in the stream, so the step has ONE host round trip (the count
    // is only known afterwards: the caller's buffer holds r x m doubles by contract)
    if (survivors_f_host)
        TEMO_CUDA(cudaMemcpyAsync(survivors_f_host, fm[cur ^ 1], kmax * m * sizeof(double), cudaMemcpyDeviceToHost, stream));
    TEMO_CUDA(cudaMemcpyAsync(h_status, ws.err_flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, stream));
    TEMO_CUDA(cudaMemcpyAsync(h_status + 1, d_P, sizeof(uint32_t), cudaMemcpyDeviceToHost, stream));
    TEMO_CUDA(cudaGetLastError());

    // while the GPU works: speculative permutation of the next generation (|P'| != n assumed)
    const double host2 = now_ms();
    counter = p.c_end;
    hp ^= 1;
    spec_valid = false;
    if (t + 1 < cfg.generations) {
        const Plan next = plan_for(n + 1 /* any value != n */, counter);
        ensure_permutation(next);
    }
    const double host3 = now_ms();
    if (timings_pending) resolve_timings();  // the previous step's stage times, read while this one runs

    TEMO_CUDA(cudaStreamSynchronize(stream));
    if (h_status[0] & 1u) fail(1, "rv_select: gamma must be positive");
    if (h_status[0] & 2u) fail(1, "normalize_to_unit: zero row");
    P = h_status[1];
    cur ^= 1;
    ++t;
    if (track_archive) archive_insert();  // algorithms.hpp:282
    pending_host_ms = (host1 - host0) + (host3 - host2);
    pending_launches = (double)launches;
    timings_pending = true;
    evp ^= 1;
    return P;
}

void Run::resolve_timings() {
    if (!timings_pending) return;
    cudaEvent_t* const e = ev[evp ^ 1];  // the last finished step's set
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e[0], e[5]); timings[0] = ms;
    cudaEventElapsedTime(&ms, e[1], e[2]); timings[1] = ms;
    cudaEventElapsedTime(&ms, e[2], e[3]); timings[2] = ms;
    cudaEventElapsedTime(&ms, e[3], e[4]); timings[3] = ms;
    cudaEventElapsedTime(&ms, e[4], e[5]); timings[4] = ms;
    timings[5] = pending_host_ms;
    timings[6] = pending_launches;
    cudaEventElapsedTime(&ms, e[0], e[1]); timings[7] = ms;
    timings_pending = false;
    if (timing_log.empty()) timing_log.resize(kTimingLog * 8);
    std::memcpy(&timing_log[(timing_steps % kTimingLog) * 8], timings, 8 * sizeof(double));
    ++timing_steps;
}

uint64_t Run::timing_history(double* out, uint64_t max_steps, bool reset) {
    resolve_timings();
    const uint64_t have = std::min<uint64_t>(timing_steps, kTimingLog), count = std::min(have, max_steps);
    for (uint64_t i = 0; i < count; ++i)
        std::memcpy(out + i * 8, &timing_log[((timing_steps - count + i) % kTimingLog) * 8], 8 * sizeof(double));
    if (reset) timing_steps = 0;
    return count;
}

void Run::inject(uint64_t rows, const double* x, const double* f, const double* v_in, const double* gamma_in,
                 uint64_t counter_in, uint64_t t_in) {
    require(rows >= 1 && rows <= pcap, "inject: row count out of range");
    TEMO_CUDA(cudaStreamSynchronize(stream));
    if (x) {
        TEMO_CUDA(cudaMemcpy(pool, x, rows * d * sizeof(double), cudaMemcpyHostToDevice));
        iota_kernel<<<(unsigned)((pcap + 255) / 256), 256, 0, stream>>>(parent_slot[cur], pcap, 0);
        iota_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(free_slot[cur], n, (uint32_t)rows);
    } else {
        require(rows == P, "inject: row count must match when x is kept");
    }
    if (f) {
        TEMO_CUDA(cudaMemcpy(fm[cur], f, rows * m * sizeof(double), cudaMemcpyHostToDevice));
    } else if (x) {  // objectives of the injected rows come from the device evaluator
        EvalArgs ea;
        ea.problem = cfg.problem;
        ea.x = pool;
        ea.n = rows;
        ea.d = d;
        ea.m = m;
        ea.horizon = cfg.horizon;
    ea.horizon = cfg.horizon;
        ea.f = fm[cur];
        launch_evaluate(ea, stream);
    }
    if (v_in) {
        TEMO_CUDA(cudaMemcpy(v, v_in, r * m * sizeof(double), cudaMemcpyHostToDevice));
        launch_row_norms(v, r, m, ws.vn, stream);
        if (!assoc_filter_preferred(m, r)) vindex.build(v, ws.vn, stream);  // m >= 5: the fp32-filtered scans need no index
    }
    if (gamma_in) TEMO_CUDA(cudaMemcpy(gamma, gamma_in, r * sizeof(double), cudaMemcpyHostToDevice));
    P = rows;
    const uint32_t p32 = (uint32_t)P;
    TEMO_CUDA(cudaMemcpy(d_P, &p32, sizeof(uint32_t), cudaMemcpyHostToDevice));
    counter = counter_in;
    t = t_in;
    spec_valid = false;
    TEMO_CUDA(cudaStreamSynchronize(stream));
}

void Run::download(double* x, double* f, double* v_out, double* gamma_out) {
    TEMO_CUDA(cudaStreamSynchronize(stream));
    if (x) {
        double* tmp = dev_alloc<double>(P * d);
        gather_rows_kernel<<<(unsigned)P, 256, 0, stream>>>(pool, parent_slot[cur], P, d, tmp);
        const cudaError_t e = cudaMemcpyAsync(x, tmp, P * d * sizeof(double), cudaMemcpyDeviceToHost, stream);
        cudaStreamSynchronize(stream);
        cudaFree(tmp);
        TEMO_CUDA(e);
    }
    if (f) TEMO_CUDA(cudaMemcpy(f, fm[cur], P * m * sizeof(double), cudaMemcpyDeviceToHost));
    if (v_out) TEMO_CUDA(cudaMemcpy(v_out, v, r * m * sizeof(double), cudaMemcpyDeviceToHost));
    if (gamma_out) TEMO_CUDA(cudaMemcpy(gamma_out, gamma, r * sizeof(double), cudaMemcpyDeviceToHost));
}

// Offspring of the last generation still sit in the slots of the previous free list, their
// objectives in the previous merged matrix after the previous parents.
void Run::last_generation(double* offspring, double* f_off, uint64_t* elite_out) {
    require(t >= 1, "last_generation: no generation has run");
    TEMO_CUDA(cudaStreamSynchronize(stream));
    if (offspring) {
        double* tmp = dev_alloc<double>(n * d);
        gather_rows_kernel<<<(unsigned)n, 256, 0, stream>>>(pool, free_slot[cur ^ 1], n, d, tmp);
        const cudaError_t e = cudaMemcpyAsync(offspring, tmp, n * d * sizeof(double), cudaMemcpyDeviceToHost, stream);
        cudaStreamSynchronize(stream);
        cudaFree(tmp);
        TEMO_CUDA(e);
    }
    if (f_off)
        TEMO_CUDA(cudaMemcpy(f_off, f_off_was_injected ? f_off_saved : fm[cur ^ 1] + P_prev() * m,
                             n * m * sizeof(double), cudaMemcpyDeviceToHost));
    if (elite_out) {
        std::vector<uint32_t> tmp(P);
        TEMO_CUDA(cudaMemcpy(tmp.data(), ws.elite, P * sizeof(uint32_t), cudaMemcpyDeviceToHost));
        for (uint64_t k = 0; k < P; ++k) elite_out[k] = tmp[k];
    }
}

void Run::set_metrics(const double* pf_ref, uint64_t n_ref, const double* hv_ref, double hv_scale, uint64_t hv_samples,
                      uint64_t hv_seed, bool maximization) {
    TEMO_CUDA(cudaStreamSynchronize(stream));
    cudaFree(mc_pf); cudaFree(mc_nearest); cudaFree(mc_hv_ref); cudaFree(mc_hits);
    mc_pf = mc_nearest = mc_hv_ref = nullptr;
    mc_hits = nullptr;
    mc_n_ref = 0;
    mc_hv_ref_host.clear();
    if (pf_ref && n_ref) {
        mc_pf = dev_alloc<double>(n_ref * m);
        mc_nearest = dev_alloc<double>(n_ref);
        TEMO_CUDA(cudaMemcpy(mc_pf, pf_ref, n_ref * m * sizeof(double), cudaMemcpyHostToDevice));
        mc_n_ref = n_ref;
    }
    if (hv_ref) {
        require(hv_samples >= 1, "hv_mc: needs at least one sample");
        require(maximization || hv_scale > 0.0, "fill_metrics: hv_scale must be positive");
        mc_hv_ref_host.assign(hv_ref, hv_ref + m);
        if (maximization)  // algorithms.hpp:168-170: minimise f against -ref, unscaled
            for (double& x : mc_hv_ref_host) x = -x;
        mc_scale = maximization ? 1.0 : hv_scale;
        mc_samples = hv_samples;
        mc_seed = hv_seed;
        mc_hv_ref = dev_alloc<double>(m);
        mc_hits = dev_alloc<unsigned long long>(1);
        TEMO_CUDA(cudaMemcpy(mc_hv_ref, mc_hv_ref_host.data(), m * sizeof(double), cudaMemcpyHostToDevice));
    }
}

// fill_metrics (algorithms.hpp:161-180) of the population's objectives, or of the archive's when one is tracked (:288).
void Run::metrics(double* igd_out, double* hv_out) {
    const double nan = std::nan("");
    const double* fs = track_archive ? arch_f[acur] : fm[cur];
    const uint64_t rows = track_archive ? arch_rows : P;
    if (igd_out) *igd_out = mc_n_ref ? device_igd(fs, nullptr, rows, m, mc_pf, mc_n_ref, mc_nearest, stream) : nan;
    if (!hv_out) return;
    *hv_out = nan;
    if (mc_hv_ref_host.empty()) return;
    if (m == 2) {  // hv_exact_2d: a sort-based sweep, on a host copy of rows x 2 values
        std::vector<double> f(rows * 2);
        TEMO_CUDA(cudaMemcpyAsync(f.data(), fs, rows * 2 * sizeof(double), cudaMemcpyDeviceToHost, stream));
        TEMO_CUDA(cudaStreamSynchronize(stream));
        *hv_out = host_hv_exact_2d(f.data(), rows, mc_hv_ref_host.data(), mc_scale);
        return;
    }
    // hv_mc: the box's lower corner is col_min of the (scaled) objectives (metrics.hpp:121-124)
    launch_col_minmax(fs, rows, nullptr, m, zmin, zmax, zscratch, stream);
    double lo[kMaxObj];
    TEMO_CUDA(cudaMemcpyAsync(lo, zmin, m * sizeof(double), cudaMemcpyDeviceToHost, stream));
    TEMO_CUDA(cudaStreamSynchronize(stream));
    device_hv_mc_box(fs, nullptr, rows, m, zmin, lo, /*lo_scaled=*/true, mc_hv_ref, mc_hv_ref_host.data(), mc_scale, mc_samples,
                     mc_seed, mc_hits, hv_out, nullptr, stream);
}

// ---- Archive of the run (algorithms.hpp:68-142), resident in HBM -----------------------------------------------------
namespace {
struct KeepPred {
    const unsigned char* keep;
    __device__ bool operator()(uint64_t i) const { return keep[i] != 0; }
};
struct IndexVal {
    __device__ uint32_t operator()(uint64_t i) const { return (uint32_t)i; }
};
// out row k <- archive row list[k] (k < k_old) or survivor list[k] - n_old of the population (pool row through the slot table)
__global__ void archive_gather_kernel(const uint32_t* __restrict__ list, const uint32_t* __restrict__ counts, uint32_t n_old,
                                      const double* __restrict__ ax, const double* __restrict__ af, const double* __restrict__ pool,
                                      const uint32_t* __restrict__ slot, const double* __restrict__ pf, uint64_t d, uint64_t m,
                                      double* __restrict__ ox, double* __restrict__ of) {
    const uint32_t k = blockIdx.x;
    if (k >= counts[0]) return;
    const uint32_t e = list[k];
    const double* sx;
    const double* sf;
    if (e < n_old) {
        sx = ax + (uint64_t)e * d;
        sf = af + (uint64_t)e * m;
    } else {
        sx = pool + (uint64_t)slot[e - n_old] * d;
        sf = pf + (uint64_t)(e - n_old) * m;
    }
    for (uint64_t j = threadIdx.x; j < d; j += blockDim.x) ox[(uint64_t)k * d + j] = sx[j];
    for (uint64_t j = threadIdx.x; j < m; j += blockDim.x) of[(uint64_t)k * m + j] = sf[j];
}
// out row k <- archive row list[k]
__global__ void archive_take_kernel(const uint32_t* __restrict__ list, const double* __restrict__ ax, const double* __restrict__ af,
                                    uint64_t d, uint64_t m, double* __restrict__ ox, double* __restrict__ of) {
    const uint64_t k = blockIdx.x, e = list[k];
    for (uint64_t j = threadIdx.x; j < d; j += blockDim.x) ox[k * d + j] = ax[e * d + j];
    for (uint64_t j = threadIdx.x; j < m; j += blockDim.x) of[k * m + j] = af[e * m + j];
}
}  // namespace

void Run::archive_reserve(uint64_t rows) {
    if (rows <= arch_capacity) return;
    uint64_t want = arch_capacity ? arch_capacity : 2 * pcap;
    while (want < rows) want *= 2;
    TEMO_CUDA(cudaStreamSynchronize(stream));
    for (int b = 0; b < 2; ++b) {
        double* nx = dev_alloc<double>(want * d);
        double* nf = dev_alloc<double>(want * m);
        if (b == acur && arch_rows) {
            TEMO_CUDA(cudaMemcpy(nx, arch_x[b], arch_rows * d * sizeof(double), cudaMemcpyDeviceToDevice));
            TEMO_CUDA(cudaMemcpy(nf, arch_f[b], arch_rows * m * sizeof(double), cudaMemcpyDeviceToDevice));
        }
        cudaFree(arch_x[b]);
        cudaFree(arch_f[b]);
        arch_x[b] = nx;
        arch_f[b] = nf;
    }
    cudaFree(arch_keep); cudaFree(arch_list); cudaFree(arch_scratch);
    arch_keep = dev_alloc<unsigned char>(want);
    arch_list = dev_alloc<uint32_t>(want);
    arch_scratch = compact_state_alloc(want);
    if (!arch_count) arch_count = dev_alloc<uint32_t>(2);
    arch_capacity = want;
}

// Archive::insert(x, f, cap) with the current survivors (algorithms.hpp:72-122): the O(n^2 m) dominance / duplicate
// filter, the order-preserving compaction (kept archive rows first, then kept new rows) and the row gather run on the
// device; only the two row counts (and, beyond the cap, the objectives for the crowding sort) come back to the host.
void Run::archive_insert() {
    const uint64_t n_old = arch_rows, n_new = P;
    archive_reserve(n_old + n_new);
    unsigned char* keep_old = arch_keep;
    unsigned char* keep_new = arch_keep + n_old;
    launch_archive_filter(arch_f[acur], n_old, fm[cur], n_new, m, keep_old, keep_new, stream);
    // one compaction over the concatenated flags keeps "archive rows first, then new rows", each in its own order
    launch_compact(n_old + n_new, KeepPred{arch_keep}, IndexVal{}, arch_scratch, n_old + n_new, arch_list, arch_count, stream);
    uint32_t kept = 0;
    TEMO_CUDA(cudaMemcpyAsync(&kept, arch_count, sizeof(uint32_t), cudaMemcpyDeviceToHost, stream));
    TEMO_CUDA(cudaStreamSynchronize(stream));
    if (kept)
        archive_gather_kernel<<<kept, 256, 0, stream>>>(arch_list, arch_count, (uint32_t)n_old, arch_x[acur], arch_f[acur], pool,
                                                        parent_slot[cur], fm[cur], d, m, arch_x[acur ^ 1], arch_f[acur ^ 1]);
    TEMO_CUDA(cudaGetLastError());
    acur ^= 1;
    arch_rows = kept;
    if (archive_cap > 0 && arch_rows > archive_cap) {  // truncate_by_crowding (algorithms.hpp:124-143): two host sorts
        std::vector<double> f(arch_rows * m), crowd(arch_rows);
        TEMO_CUDA(cudaMemcpyAsync(f.data(), arch_f[acur], f.size() * sizeof(double), cudaMemcpyDeviceToHost, stream));
        TEMO_CUDA(cudaStreamSynchronize(stream));
        crowding_distance_host(f.data(), arch_rows, m, crowd.data());
        std::vector<uint32_t> order(arch_rows);
        for (uint64_t i = 0; i < arch_rows; ++i) order[i] = (uint32_t)i;
        std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
            if (crowd[a] != crowd[b]) return crowd[a] > crowd[b];
            return a < b;
        });
        order.resize(archive_cap);
        std::sort(order.begin(), order.end());  // keep insertion order
        TEMO_CUDA(cudaMemcpyAsync(arch_list, order.data(), archive_cap * sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
        archive_take_kernel<<<(unsigned)archive_cap, 256, 0, stream>>>(arch_list, arch_x[acur], arch_f[acur], d, m, arch_x[acur ^ 1],
                                                                       arch_f[acur ^ 1]);
        TEMO_CUDA(cudaGetLastError());
        TEMO_CUDA(cudaStreamSynchronize(stream));  // `order` goes away
        acur ^= 1;
        arch_rows = archive_cap;
    }
}

void Run::enable_archive(uint64_t cap_rows) {
    require(!track_archive, "track_archive: already enabled");
    track_archive = true;
    archive_cap = cap_rows;
    archive_insert();  // algorithms.hpp:243
}

void Run::archive_download(double* x, double* f) {
    require(track_archive, "archive: this run does not track one");
    TEMO_CUDA(cudaStreamSynchronize(stream));
    if (x && arch_rows) TEMO_CUDA(cudaMemcpy(x, arch_x[acur], arch_rows * d * sizeof(double), cudaMemcpyDeviceToHost));
    if (f && arch_rows) TEMO_CUDA(cudaMemcpy(f, arch_f[acur], arch_rows * m * sizeof(double), cudaMemcpyDeviceToHost));
}

double Run::time_stage(int stage, int reps) {
    require(reps >= 1, "time_stage: reps must be positive");
    require(cfg.op == kOpGa, "time_stage: the isolated stages are those of the ga loop");
    const Plan p = plan_for(P, counter);
    ensure_permutation(p);
    TEMO_CUDA(cudaMemcpyAsync(perm_dev, h_perm[hp], n * sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
    // make sure the offspring rows / merged objectives of this generation exist for stages 2 and 4
    launch_mating_table(p);
    launch_reproduction(p, false);
    launch_offspring_eval();
    const double penalty = apd_penalty(m, t < cfg.generations ? t : cfg.generations, cfg.generations, cfg.alpha);
    cudaEvent_t a, b;
    TEMO_CUDA(cudaEventCreate(&a));
    TEMO_CUDA(cudaEventCreate(&b));
    double total = 0.0;
    for (int it = 0; it < reps; ++it) {
        flush_l2();
        TEMO_CUDA(cudaEventRecord(a, stream));
        switch (stage) {
        case 1: launch_reproduction(p, false); break;
        case 2: launch_offspring_eval(); break;
        case 3:
            require(fusable(), "time_stage: the evaluation of this problem / shape cannot be fused");
            launch_reproduction(p, true);
            break;
        case 4: launch_select(fm[cur], P + n, nullptr, m, v, gamma, r, penalty, ws, stream, &vindex); break;
        case 5: launch_gamma_auto(v, r, m, ws, &vindex, gamma, ws.err_flag, nullptr, stream); break;
        case 6: launch_select(fm[cur], P + n, nullptr, m, v, gamma, r, penalty, ws, stream, nullptr); break;
        case 7: launch_gamma(v, ws.vn, r, m, gamma, ws.err_flag, nullptr, stream); break;
        default: fail(1, "time_stage: unknown stage");
        }
        TEMO_CUDA(cudaEventRecord(b, stream));
        TEMO_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        TEMO_CUDA(cudaEventElapsedTime(&ms, a, b));
        total += ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return total / reps;
}

void flush_l2() {
    Context& cx = ctx();
    const size_t bytes = 256u << 20;  // > 126 MB L2
    if (!cx.flush_buf) {
        cx.flush_buf = dev_alloc<unsigned char>(bytes);
        cx.flush_bytes = bytes;
    }
    TEMO_CUDA(cudaMemsetAsync(cx.flush_buf, 0x5a, cx.flush_bytes, cx.stream));
}

}  // namespace temo_b200
