// Internal launch interface between the kernel translation units, the run driver and the
// C ABI (capi.cu). Everything lives in namespace temo_b200; nothing here is exported.
#pragma once

#include <cstdint>
#include <vector>

#include "common.cuh"

namespace temo_b200 {

// Problem ids (mirrors include/temo_b200.h).
constexpr int kDtlz1 = 1, kDtlz2 = 2, kDtlz3 = 3, kDtlz4 = 4, kLsmop1 = 101, kToy2 = 201, kToy3 = 202;
constexpr uint64_t kToyHidden = 16;  // make_problem's MlpArch{4, 16, 2} (problems.hpp:280)
constexpr int kMaxObj = 32;   // objectives supported by the on-device evaluators/selection
constexpr int kLsmopNk = 5;

// Canonical row mapping shared by the evaluation kernels (fused and standalone) so that
// their reductions associate identically: VEC genes per load, B threads per row.
inline int row_vec(uint64_t d) { return (d % 2 == 0) ? 2 : 1; }
inline int row_block(uint64_t d) {
    const uint64_t nvec = d / row_vec(d);
    uint64_t b = ((nvec + 31) / 32) * 32;
    if (b < 32) b = 32;
    if (b > 256) b = 256;
    return (int)b;
}

// LSMOP1 group layout (host-computed, passed by value to kernels).
struct LsmopLayout {
    uint32_t start[kMaxObj + 1];  // tail-relative first gene of each group
    uint32_t sublen[kMaxObj];
};
LsmopLayout lsmop1_layout(uint64_t d, uint64_t m);
const double* lsmop1_coef(uint64_t d, cudaStream_t s);  // device table 1 + (j + 1) / d, cached per d

struct GaParams {
    double pc = 1.0, eta = 20.0, pm = 1.0, xi = 20.0;  // operators.hpp:22-27
};

// Optional piecewise-constant description of the box bounds: genes [0, split) have (lo[0], hi[0]), genes
// [split, d) have (lo[1], hi[1]) (DTLZ: one segment; LSMOP: two). Lets K1 keep the bounds in registers instead
// of loading two arrays per gene; the arrays stay authoritative (valid == false: arrays only).
struct BoundSegments {
    bool valid = false;
    uint64_t split = 0;
    double lo[2] = {0.0, 0.0}, hi[2] = {0.0, 0.0};
};
BoundSegments find_bound_segments(const double* lower, const double* upper, uint64_t d);  // host arrays

// ---- K1: reproduction ---------------------------------------------------------------------
struct ReproArgs {
    const double* pool = nullptr;   // parent storage, row stride d
    const uint32_t* src = nullptr;  // [n] storage row of mating row i (nullptr: i)
    // optional (replaces pool / src): [n] address of the parent row of mating row i, each 16-byte aligned; rows may live in
    // other GPUs' pools mapped into this process (the sharded run: NVLink peer loads inside K1)
    const double* const* src_ptr = nullptr;
    double* out = nullptr;          // child storage, row stride d
    const uint32_t* dst = nullptr;  // [n] storage row of child i (nullptr: i)
    uint64_t n = 0, d = 0;
    Rng rng{};
    uint64_t c_sbx = 0;   // counter of the first SBX block (Mc); R1, R2, R3 follow (operators.hpp:70-73)
    uint64_t c_pm = 0;    // counter of the mask block R4; Mmut follows (operators.hpp:130-131)
    GaParams ga;
    const double* lower = nullptr;
    const double* upper = nullptr;
    BoundSegments seg;  // optional: same bounds as the arrays, piecewise constant
    bool do_sbx = true, do_pm = true;
    // fused evaluation of the children (0 = off): problem id, m, output rows f_out[(f_row0+i)*m..]
    int eval_problem = 0;
    uint64_t m = 0;
    double* f_out = nullptr;
    uint64_t f_row0 = 0;
    const uint32_t* f_row0_dev = nullptr;  // optional device-side row offset (survivor count)
    // sharded runs: this launch covers pairs [global_unit0, global_unit0 + n/2) of a global population of
    // global_n rows (0 = not sharded); draw counters are addressed globally, storage rows locally
    uint64_t global_n = 0, global_unit0 = 0;
    // optional: only the mating units [unit_begin, unit_begin + unit_count) of this launch's rows (0 = all); lets a
    // sharded run start on the pairs whose parents have already arrived
    uint64_t unit_begin = 0, unit_count = 0;
};
void launch_reproduce(const ReproArgs& a, cudaStream_t s);
// K1 path-selection knobs ("k1_generic", "k1_bound_arrays", "k1_cand_cap"); false for an unknown name.
bool set_k1_option(const char* name, long value);

// random_reproduce (operators.hpp:287-296) and uniform_tensor (rng.hpp:55-66).
void launch_random_reproduce(double* out, const uint32_t* dst, uint64_t n, uint64_t d, Rng rng,
                             uint64_t counter, const double* lower, const double* upper,
                             cudaStream_t s);
void launch_uniform_fill(double* out, uint64_t count, Rng rng, uint64_t counter, cudaStream_t s);
// pow with the host libm's bits (glibc_pow.cuh), elementwise; diagnostic/self-test entry.
void launch_pow_batch(const double* x, const double* y, uint64_t n, double* out, cudaStream_t s);

// ---- the other reproduction operators (swarm.cu) ------------------------------------
// de_reproduce (operators.hpp:166-200): draws consumed 4 n + n d.
// src / dst (optional, all three): operand row i is read from storage row src[i] of x, child i is written to storage row
// dst[i] of out (the device-resident run addresses its pool this way); nullptr = dense matrices.
void launch_de(const double* x, uint64_t n, uint64_t d, Rng rng, uint64_t counter, double f, double cr, const double* lower,
               const double* upper, double* out, cudaStream_t s, const uint32_t* src = nullptr, const uint32_t* dst = nullptr);
// pso_reproduce (operators.hpp:205-240): vel / pb_x / pb_score are the SwarmState, updated in place; draws 2 n d.
void launch_pso(const double* x, const double* scores, uint64_t n, uint64_t d, Rng rng, uint64_t counter, double inertia, double c1,
                double c2, double* vel, double* pb_x, double* pb_score, uint32_t* best_scratch, const double* lower,
                const double* upper, double* out, cudaStream_t s, const uint32_t* src = nullptr, const uint32_t* dst = nullptr);
// cso_reproduce (operators.hpp:246-284) after the caller's shuffle_indices (n - 1 draws): draws 3 (n / 2) d from `counter`.
// vel_out may be vel itself (in-place update: the winners' velocities are not rewritten).
void launch_cso(const double* x, const double* scores, uint64_t n, uint64_t d, Rng rng, uint64_t counter, double phi,
                const uint32_t* perm, double* mean_scratch, const double* vel, double* vel_out, const double* lower,
                const double* upper, double* out, cudaStream_t s, const uint32_t* src = nullptr, const uint32_t* dst = nullptr);

// ---- K2: evaluation -------------------------------------------------------------------------
struct EvalArgs {
    int problem = 0;
    const double* x = nullptr;      // storage base, row stride d
    const uint32_t* rows = nullptr; // [n] storage row of logical row i (nullptr: i)
    uint64_t n = 0, d = 0, m = 0;
    double* f = nullptr;            // f[(f_row0 + i) * m + j]
    uint64_t f_row0 = 0;
    const uint32_t* f_row0_dev = nullptr;
    bool allow_tma = true;
    uint64_t horizon = 100;         // toy2 / toy3: episode length (RunConfig::horizon, algorithms.hpp:35)
};
void launch_evaluate(const EvalArgs& a, cudaStream_t s);
// "eval_tma" (1 default; 0: the one-CTA-per-row kernels only); false for an unknown name
bool set_eval_option(const char* name, long value);
// second half of the streaming evaluators: rows holding {tail sum, position genes} -> objectives
void launch_dtlz_finish(int problem, double* f, uint64_t n, uint64_t m, uint64_t d, uint64_t f_row0, cudaStream_t s);

// ---- neuroevolution evaluator (toyenv.cu) ----------------------------------------------
uint64_t mlp_param_count(uint64_t hidden);
void launch_tanh_batch(const double* x, uint64_t n, double* out, cudaStream_t s);
void tanh_batch_host(const double* x, uint64_t n, double* out);
void launch_env_rollout(const double* params, const uint32_t* rows, uint64_t n, uint64_t d, uint64_t hidden, uint64_t horizon,
                        uint64_t m, bool negate, double* f, uint64_t f_row0, const uint32_t* f_row0_dev, cudaStream_t s);
void launch_mlp_forward(const double* params, uint64_t n, uint64_t d, uint64_t hidden, const double* obs, double* action,
                        cudaStream_t s);

// ---- K3: selection ----------------------------------------------------------------------------
struct SelectWorkspace {
    // sized for rows_cap merged rows and r vectors
    uint64_t rows_cap = 0, r = 0, m = 0;
    double* z = nullptr;              // [m] ideal point
    unsigned long long* zkey = nullptr;  // [m] ordered-int min keys
    double* vn = nullptr;             // [r] ||v_j||
    uint32_t* assoc = nullptr;        // [rows_cap]
    double* theta = nullptr;          // [rows_cap]
    double* apd = nullptr;            // [rows_cap]
    unsigned long long* best_key = nullptr;  // [r]
    uint32_t* best_row = nullptr;     // [r]
    uint32_t* first_row = nullptr;    // [r]
    uint32_t* elite = nullptr;        // [r] merged-row index per valid vector (compacted)
    unsigned char* valid = nullptr;   // [r]
    uint32_t* n_elite = nullptr;      // [1]
    uint32_t* err_flag = nullptr;     // [1] bit0: gamma <= 0
    uint32_t* tile_scratch = nullptr; // compaction tile counts
    float* v32 = nullptr;             // [r x (m+1)] fp32 copy of v and 1/|v| (filtered association, m >= 5)
    uint32_t* v32_flags = nullptr;    // [1] bit0: a vector component is negative / non-finite
    double* part_c = nullptr;         // [chunks x rows_cap] per-chunk winners of the filtered association (m >= 5 only)
    uint32_t* part_j = nullptr;
    uint32_t* row_flag = nullptr;       // [rows_cap] rows of the filtered scan that need the fallback (1 near-ties, 2 exact only)
    uint32_t* flag_list = nullptr;      // [rows_cap] those rows, compacted; flag_count [1]
    uint32_t* flag_count = nullptr;
    double* fb_c = nullptr;             // [rows_cap + kFallbackItems] partial winners of the fallback's (row, vector range) items
    uint32_t* fb_j = nullptr;
    float* seed32 = nullptr;            // [rows_cap] starting value of a row's running fp32 maximum (subsample scan)
    void alloc(uint64_t rows_cap_, uint64_t r_, uint64_t m_);
    void release();
};
// n_rows_dev (optional): device-side row count overriding n_rows (<= n_rows, which then only
// sizes the grid).
struct VecIndex;
// index (optional): hierarchical direction index over v (vecindex.h); nullptr = exhaustive scan.
void launch_select(const double* f, uint64_t n_rows, const uint32_t* n_rows_dev, uint64_t m,
                   const double* v, const double* gamma, uint64_t r, double penalty,
                   SelectWorkspace& ws, cudaStream_t s, VecIndex* index = nullptr);
void launch_row_norms(const double* v, uint64_t r, uint64_t m, double* vn, cudaStream_t s);
// Exact association + APD through a single-precision filter (many objectives, where the direction index prunes little);
// same outputs as the other association kernels. ws.vn must hold the norms of v.
bool assoc_filter_preferred(uint64_t m, uint64_t r);
void launch_assoc_filter(const double* f, uint64_t n_rows, uint64_t m, const double* v, const double* gamma, uint64_t r, double penalty,
                         SelectWorkspace& ws, uint32_t* assoc, double* theta, double* apd, cudaStream_t s, uint32_t row0);
// min_vector_angles through the same filtered scan (m >= 5); ws.vn must hold the norms of v. launch_gamma_auto picks the
// filtered scan or the direction index (index may be nullptr only when the filter is preferred).
void launch_gamma_filter(const double* v, uint64_t r, uint64_t m, SelectWorkspace& ws, double* gamma, uint32_t* err_flag,
                         const uint32_t* skip_flag, cudaStream_t s);
void launch_gamma_auto(const double* v, uint64_t r, uint64_t m, SelectWorkspace& ws, VecIndex* index, double* gamma,
                       uint32_t* err_flag, const uint32_t* skip_flag, cudaStream_t s);
// the stages of launch_select, separately (the sharded run puts collectives between them)
void launch_select_prepare(const double* f, uint64_t n_rows, uint64_t m, const double* gamma, uint64_t r,
                           SelectWorkspace& ws, cudaStream_t s);
void launch_elite_rows(uint64_t n_rows, const uint32_t* assoc, const double* apd, const unsigned long long* best_key,
                       uint32_t* best_row, uint32_t row0, cudaStream_t s);
void launch_select_finish(uint64_t r, SelectWorkspace& ws, bool nan_rule, cudaStream_t s);

// ---- K4: reference vectors ----------------------------------------------------------------------
// gamma_i = acos(max_{j != i} cos(v_i, v_j)) (refvec.hpp:81-100); err_flag bit0 set if any <= 0.
void launch_gamma(const double* v, const double* vn, uint64_t r, uint64_t m, double* gamma,
                  uint32_t* err_flag, const uint32_t* skip_flag, cudaStream_t s);
// zmin/zmax over rows [0, n_rows) of f (tensor.hpp:211-229).
void launch_col_minmax(const double* f, uint64_t n_rows, const uint32_t* n_rows_dev, uint64_t m,
                       double* zmin, double* zmax, unsigned long long* scratch2m /* col_minmax_scratch_alloc(m) */, cudaStream_t s);
unsigned long long* col_minmax_scratch_alloc(uint64_t m);
// adapt_vectors (refvec.hpp:119-131): v = unit(v0 * (zmax - zmin)); skip_flag[0] is set to 1
// (and v left untouched) unless every range is > 0; err bit1 on a zero row.
void preload_adapt_kernels();
void launch_adapt_vectors(const double* v0, double* v, double* vn, uint64_t r, uint64_t m,
                          const double* zmin, const double* zmax, uint32_t* skip_flag,
                          uint32_t* err_flag, cudaStream_t s);

// ---- quality indicators (metrics.cu) -----------------------------------------
// igd (metrics.hpp:21-44) of the n (or *n_dev) rows of f against f_ref; nearest_scratch holds n_ref doubles.
double device_igd(const double* f, const uint32_t* n_dev, uint64_t n, uint64_t m, const double* f_ref, uint64_t n_ref,
                  double* nearest_scratch, cudaStream_t s);
// hv_mc_box (metrics.hpp:76-117) of f / scale inside [lo, ref] (lo_scaled: the box corner is lo / scale, as when it is
// col_min of the unscaled objectives). lo / ref are given on both sides (device for the kernel, host for the volume).
void device_hv_mc_box(const double* f, const uint32_t* n_dev, uint64_t n, uint64_t m, const double* lo_dev, const double* lo_host,
                      bool lo_scaled, const double* ref_dev, const double* ref_host, double scale, uint64_t samples, uint64_t seed,
                      unsigned long long* hits_scratch, double* value, double* std_error, cudaStream_t s);
// Archive::insert's dominance filter (algorithms.hpp:76-100): keep flags of the archive rows and of the inserted rows.
void launch_archive_filter(const double* f_old, uint64_t n_old, const double* f_new, uint64_t n_new, uint64_t m, unsigned char* keep_old,
                           unsigned char* keep_new, cudaStream_t s);
// crowding_distance (selection.hpp:289-312), host: k x m front -> k distances.
void crowding_distance_host(const double* front, uint64_t k, uint64_t m, double* dist);
// hv_exact_2d (metrics.hpp:48-66) on a host copy of an n x 2 objective matrix divided by scale.
double host_hv_exact_2d(const double* f, uint64_t n, const double* ref, double scale);

// ---- host-side pieces (host_ops.cu) ---------------------------------------------------------------
uint64_t lattice_count(uint64_t m, uint64_t H);
uint64_t lattice_density_for(uint64_t m, uint64_t target);
std::vector<double> simplex_lattice(uint64_t m, uint64_t H);
std::vector<double> normalize_to_unit(const std::vector<double>& v, uint64_t r, uint64_t m);
void shuffle_indices(uint64_t seed, uint64_t& counter, uint64_t n, uint32_t* perm);
double apd_penalty(uint64_t m, uint64_t t, uint64_t t_max, double alpha);
void problem_bounds(int problem, uint64_t d, uint64_t m, double* lower, double* upper);
uint64_t problem_default_dim(int problem, uint64_t m);
bool problem_known(int problem);

// ---- device context -----------------------------------------------------------------------------------
struct Context {
    int device = -1;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;
    void* flush_buf = nullptr;
    size_t flush_bytes = 0;
};
void init_context(int device);
Context& ctx();  // initialises device 0 on first use; throws ENODEV without a GPU

template <class T>
T* dev_alloc(size_t count) {
    T* p = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) fail(4, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return p;
}

}  // namespace temo_b200
