// Device-resident RVEA run state (see run.cu). reference: rvea_run, algorithms.hpp:227-296.
#pragma once
#include <vector>

#include "internal.h"
#include "vecindex.h"

namespace temo_b200 {

// Offspring evaluation inside the reproduction kernel? DTLZ only; by shape (fuse_eval == 2): rows wider than 1024 genes -
// narrower ones are cheaper as single-warp reproduction plus the one-warp-per-row evaluator (config #4, d = 1000:
// 0.32 + 0.26 ms against 0.64 ms fused; d = 1536: 0.44 + 0.19 against 0.59).
inline bool fuse_offspring_eval(int fuse_eval, int problem, uint64_t d) {
    return fuse_eval != 0 && problem >= kDtlz1 && problem <= kDtlz4 && (fuse_eval == 1 || d > 1024);
}

struct RunConfig {  // reference: RunConfig, algorithms.hpp:21-41
    int problem = kDtlz2;
    int rng_mode = 0;
    uint64_t pop = 105, lattice_h = 0, generations = 100, seed = 42, dim = 0, obj = 3;
    double alpha = 2.0, fr = 0.1, time_budget_s = 0.0;
    GaParams ga;
    int fuse_eval = 2;  // 0 never, 1 whenever the problem has a fused evaluation, 2 by shape (fuse_offspring_eval)
    // reproduction operator (algorithms.hpp:250-268): 0 ga, 1 de, 2 pso, 3 cso, 4 random; the swarm operators take
    // apd_scores of the parent pool as fitness and carry a SwarmState across generations
    int op = 0;
    double de_f = 0.5, de_cr = 0.9;                          // DeParams, operators.hpp:28-31
    double pso_inertia = 0.4, pso_c1 = 1.5, pso_c2 = 1.5;    // PsoParams, operators.hpp:33-37
    double cso_phi = 0.1;                                    // CsoParams, operators.hpp:39-41
    uint64_t horizon = 100;                                  // toy environments: episode length (algorithms.hpp:35)
};
constexpr int kOpGa = 0, kOpDe = 1, kOpPso = 2, kOpCso = 3, kOpRandom = 4;  // TEMO_B200_OP_*

void flush_l2();

struct Run {
    static constexpr int kNumEvents = 6;
    struct Plan {
        uint64_t c_pool, c_shuffle, c_sbx, c_pm, c_end;  // c_sbx doubles as the first draw of de / pso / cso
    };

    explicit Run(const RunConfig& c);
    ~Run();
    Run(const Run&) = delete;
    Run& operator=(const Run&) = delete;

    uint64_t step(double* survivors_f_host, const double* f_off_inject = nullptr);
    void inject(uint64_t rows, const double* x, const double* f, const double* v_in, const double* gamma_in,
                uint64_t counter_in, uint64_t t_in);
    void download(double* x, double* f, double* v_out, double* gamma_out);
    void last_generation(double* offspring, double* f_off, uint64_t* elite_out);
    double time_stage(int stage, int reps);
    // MetricContext (algorithms.hpp:46-54) and fill_metrics (:161-180) on the current survivors' objectives, which stay
    // in HBM: IGD against pf_ref (n_ref x m, n_ref = 0: none), hypervolume against hv_ref (m values, nullptr: none).
    void set_metrics(const double* pf_ref, uint64_t n_ref, const double* hv_ref, double hv_scale, uint64_t hv_samples,
                     uint64_t hv_seed, bool maximization);
    void metrics(double* igd_out, double* hv_out);
    // Archive (algorithms.hpp:68-142) of a device-resident run, kept in HBM: enable_archive inserts the current
    // population (algorithms.hpp:243); every later step() inserts its survivors (:282). cap = RunConfig::archive_cap
    // (0: unbounded). With an archive the metrics are those of the archive's objectives (:288).
    void enable_archive(uint64_t archive_cap);
    void archive_download(double* x, double* f);

    RunConfig cfg;
    uint64_t n = 0, d = 0, m = 0, r = 0, H = 0, adapt_every = 1;
    uint64_t pcap = 0;  // max(n, r): most parents a generation can have
    uint64_t cap = 0;   // pool rows: pcap + n
    uint64_t P = 0;     // current survivor count (host copy)
    uint64_t P_before = 0;  // survivor count at the start of the last step
    uint64_t counter = 0, t = 0;
    Rng rng{};
    cudaStream_t stream = nullptr;

    double* pool = nullptr;          // cap x d
    double* fm[2] = {nullptr, nullptr};       // merged objectives, cap x m (double buffered)
    uint32_t* parent_slot[2] = {nullptr, nullptr};
    uint32_t* free_slot[2] = {nullptr, nullptr};
    int cur = 0;
    uint32_t* src = nullptr;
    uint32_t* perm_dev = nullptr;
    // pso / cso: survivor index of every pool row (its objective row), and the swarm state
    uint32_t* pool_idx_dev = nullptr;
    double *pool_f = nullptr, *scores = nullptr;                         // n x m, n
    double *sw_vel[2] = {nullptr, nullptr}, *sw_pbx = nullptr, *sw_pbs = nullptr;  // SwarmState (operators.hpp:46-56)
    double* sw_mean = nullptr;
    uint32_t* sw_best = nullptr;
    int sw_cur = 0;
    bool swarm_ready = false;
    unsigned char* used = nullptr;
    uint32_t* d_P = nullptr;
    uint32_t* free_scratch = nullptr;
    double *v0 = nullptr, *v = nullptr, *gamma = nullptr, *lower = nullptr, *upper = nullptr;
    BoundSegments bound_seg;  // the same bounds, piecewise constant (K1 keeps them in registers)
    double *zmin = nullptr, *zmax = nullptr;
    unsigned long long* zscratch = nullptr;
    uint32_t* skip_flag = nullptr;
    double* mc_pf = nullptr;       // IGD reference front on the device
    uint64_t mc_n_ref = 0;
    double* mc_nearest = nullptr;  // [n_ref]
    double* mc_hv_ref = nullptr;   // [m] (sign already applied)
    std::vector<double> mc_hv_ref_host;
    double mc_scale = 1.0;
    uint64_t mc_samples = 2048, mc_seed = 9001;
    unsigned long long* mc_hits = nullptr;
    bool track_archive = false;
    uint64_t archive_cap = 0, arch_rows = 0, arch_capacity = 0;
    double *arch_x[2] = {nullptr, nullptr}, *arch_f[2] = {nullptr, nullptr};  // double buffered: rows in insertion order
    int acur = 0;
    unsigned char* arch_keep = nullptr;   // [arch_capacity]: keep flags, archive rows first, then the inserted rows
    uint32_t* arch_list = nullptr;        // [arch_capacity]: kept archive rows, then kept inserted rows
    uint32_t* arch_scratch = nullptr;
    uint32_t* arch_count = nullptr;       // [2]
    double* f_off_saved = nullptr;  // device objectives of the last offspring when selection ran on injected ones
    bool f_off_was_injected = false;
    SelectWorkspace ws;
    VecIndex vindex;  // hierarchical direction index over v (rebuilt after every adaptation)

    uint32_t* h_perm[2] = {nullptr, nullptr};  // pinned
    int hp = 0;
    bool spec_valid = false;
    uint64_t spec_c_shuffle = 0;
    uint32_t* h_status = nullptr;  // pinned: [0] error flags, [1] survivor count
    // Stage events of a step, double-buffered: the elapsed times of step t are read while step t + 1 runs on the device
    // (or when somebody asks for them), not between the end of step t and the first launch of step t + 1.
    cudaEvent_t ev[2][kNumEvents]{};
    int evp = 0;                   // event set of the step being enqueued
    bool timings_pending = false;  // the last finished step's events (set evp ^ 1) have not been read yet
    double pending_host_ms = 0.0, pending_launches = 0.0;
    double timings[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    static constexpr uint64_t kTimingLog = 1024;  // steps kept
    std::vector<double> timing_log;               // 8 values per step, ring
    uint64_t timing_steps = 0;                    // steps logged since the last reset
    void resolve_timings();                       // reads the pending events into `timings` and the log
    uint64_t timing_history(double* out, uint64_t max_steps, bool reset);  // oldest first; returns the number of steps written

private:
    void check_status();
    Plan plan_for(uint64_t P_now, uint64_t c) const;
    void ensure_permutation(const Plan& p);
    void launch_mating_table(const Plan& p);
    void launch_reproduction(const Plan& p, bool fused);
    uint64_t launch_other_operator(const Plan& p);  // returns its launch count
    bool uses_perm() const { return cfg.op == kOpGa || cfg.op == kOpCso; }
    void launch_offspring_eval();
    bool fusable() const;
    void archive_reserve(uint64_t rows);
    void archive_insert();
    uint64_t P_prev() const { return P_before; }
};

}  // namespace temo_b200
