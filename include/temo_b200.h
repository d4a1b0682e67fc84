/* temo_b200.h — C ABI of the B200-native TensorRVEA generation loop.
 *
 * Drop-in boundary for ONE path of the reference (arxiv 2404.01159 "temo" artifact):
 * the per-generation loop of rvea_run with the GA operator on DTLZ/LSMOP problems
 * (reference: proj/include/temo/algorithms.hpp:246-292). Every entry point below names
 * the reference interface it replaces. All matrices are dense row-major fp64 exactly
 * like temo::Tensor2D (tensor.hpp:22-59); index outputs are uint64 like std::size_t.
 *
 * Conventions
 *   - every function returns 0 on success; non-zero = failure, message via
 *     temo_b200_last_error(). TEMO_B200_EINVAL mirrors the reference's
 *     detail::require -> std::invalid_argument (tensor.hpp:63-65).
 *   - `counter` arguments are in/out and advance by exactly the reference's documented
 *     draw count (operators.hpp:3-13, rng.hpp:64), so a caller can interleave GPU and
 *     CPU operators on one RngStream.
 *   - host-pointer functions ("drop-ins") copy in, run the CUDA kernels, copy out.
 *     There is NO CPU fallback: without a CUDA device they fail with TEMO_B200_ENODEV.
 *   - the device-resident loop (temo_b200_run_*) keeps X, F, V, gamma in HBM for the
 *     whole run; per generation the host only ships the mating permutation (4 B/row)
 *     and reads back the survivor count.
 */
#ifndef TEMO_B200_H
#define TEMO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TEMO_B200_OK 0
#define TEMO_B200_EINVAL 1   /* contract violation (reference: std::invalid_argument) */
#define TEMO_B200_ECUDA 2    /* CUDA runtime error */
#define TEMO_B200_ENODEV 3   /* no usable CUDA device: the product has no CPU path */
#define TEMO_B200_ENOMEM 4
#define TEMO_B200_ERUNTIME 5 /* reference: std::runtime_error (algorithms.hpp:182-191) */

/* Problem ids (reference: make_problem, problems.hpp:261-296). LSMOP1 is an extension
 * required by BASELINE.json config #3; the reference has no LSMOP (parity unpinned). */
#define TEMO_B200_DTLZ1 1
#define TEMO_B200_DTLZ2 2
#define TEMO_B200_DTLZ3 3
#define TEMO_B200_DTLZ4 4
#define TEMO_B200_LSMOP1 101
#define TEMO_B200_TOY2 201   /* make_problem("toy2"): MLP 4-16-2 policy on the toy environment, 2 objectives (problems.hpp:279-294) */
#define TEMO_B200_TOY3 202   /* 3 objectives */

/* RNG policy. SPLITMIX64 reproduces RngStream::value_at bit for bit (rng.hpp:23-43) and is
 * the only mode with draw-for-draw parity; PHILOX is the north star's Philox4x32-10
 * throughput mode (not in the reference: parity unpinned, invariants only). */
#define TEMO_B200_RNG_SPLITMIX64 0
#define TEMO_B200_RNG_PHILOX 1

/* reference: GaParams, operators.hpp:22-27 */
typedef struct temo_b200_ga_params {
    double pc;  /* crossover probability per pair */
    double eta; /* SBX distribution index */
    double pm;  /* mutation numerator; per-gene rate pm/d */
    double xi;  /* mutation distribution index */
} temo_b200_ga_params;

/* reproduction operator of the run loop: RunConfig::op, algorithms.hpp:250-271 */
#define TEMO_B200_OP_GA 0
#define TEMO_B200_OP_DE 1
#define TEMO_B200_OP_PSO 2
#define TEMO_B200_OP_CSO 3
#define TEMO_B200_OP_RANDOM 4

/* reference: DeParams / PsoParams / CsoParams, operators.hpp:28-41 */
typedef struct temo_b200_op_params {
    double de_f, de_cr;
    double pso_inertia, pso_c1, pso_c2;
    double cso_phi;
} temo_b200_op_params;

/* reference: RunConfig, algorithms.hpp:21-41 (track_archive = false) */
typedef struct temo_b200_run_config {
    int32_t problem;      /* TEMO_B200_DTLZ1.. */
    int32_t rng_mode;     /* TEMO_B200_RNG_* */
    uint64_t pop;         /* n */
    uint64_t lattice_h;   /* 0 -> lattice_density_for(obj, pop) */
    uint64_t generations; /* t_max */
    uint64_t seed;
    uint64_t dim;         /* d (0 -> problem default: DTLZ1 7, DTLZ2-4 12, LSMOP1 100*obj) */
    uint64_t obj;         /* m */
    double alpha;         /* APD penalty exponent */
    double fr;            /* adaptation frequency: every ceil(fr * generations) generations */
    double time_budget_s; /* 0 -> run all generations */
    temo_b200_ga_params ga;
    int32_t fuse_eval;    /* evaluate offspring inside the reproduction kernel: 0 never, 1 whenever the problem allows, 2 by shape (default) */
    int32_t op;           /* TEMO_B200_OP_* (0 = ga); de / pso / cso / random: algorithms.hpp:253-268 */
    temo_b200_op_params opp;
    uint64_t horizon;     /* toy2 / toy3: episode length (RunConfig::horizon, algorithms.hpp:35; 0 -> 100) */
} temo_b200_run_config;

/* ---- library / device ------------------------------------------------------------- */
const char* temo_b200_last_error(void);
const char* temo_b200_version(void);
int temo_b200_device_count(void);
/* Selects the device for this process (one process per GPU) and creates the library's
 * stream. Implicitly called with device 0 by the first compute entry point. */
int temo_b200_init(int device);
void temo_b200_default_run_config(temo_b200_run_config* cfg);
void temo_b200_default_ga_params(temo_b200_ga_params* ga);

/* ---- rng.hpp ---------------------------------------------------------------------- */
/* uniform_tensor (rng.hpp:55-66): rows*cols draws, element e at counter+e. */
int temo_b200_uniform_tensor(uint64_t seed, uint64_t* counter, uint64_t rows, uint64_t cols,
                             int rng_mode, double* out);
/* shuffle_indices (rng.hpp:69-78): host-side Fisher-Yates, n-1 draws. */
int temo_b200_shuffle_indices(uint64_t seed, uint64_t* counter, uint64_t n, uint64_t* perm);
/* parent_pool_indices (algorithms.hpp:211-221). */
int temo_b200_parent_pool_indices(uint64_t current, uint64_t n, uint64_t seed, uint64_t* counter,
                                  uint64_t* idx);

/* ---- operators.hpp ---------------------------------------------------------------- */
/* sbx (operators.hpp:65-102): x n x d -> out n x d; 3*(n/2)*d + n/2 draws. */
int temo_b200_sbx(const double* x, uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter,
                  const temo_b200_ga_params* ga, const double* lower, const double* upper,
                  int rng_mode, double* out);
/* polynomial_mutation (operators.hpp:126-149): 2*n*d draws. */
int temo_b200_polynomial_mutation(const double* x, uint64_t n, uint64_t d, uint64_t seed,
                                  uint64_t* counter, const temo_b200_ga_params* ga,
                                  const double* lower, const double* upper, int rng_mode,
                                  double* out);
/* ga_reproduce (operators.hpp:153-161): shuffle + SBX + PM fused into one kernel pass. */
int temo_b200_ga_reproduce(const double* x, uint64_t n, uint64_t d, uint64_t seed,
                           uint64_t* counter, const temo_b200_ga_params* ga, const double* lower,
                           const double* upper, int rng_mode, double* out);
/* ---- the reference's other reproduction operators, host buffers, bit-identical to the
 * reference (no libm on these paths). `kernel_ms` (optional) receives the device time of the kernels of the call.
 * de_reproduce (operators.hpp:166-200): DE/rand/1/bin, needs n >= 4; advances *counter by 4 n + n d.
 * pso_reproduce (operators.hpp:205-240): velocities (n x d), pbest_x (n x d), pbest_score (n) are the SwarmState
 *   (operators.hpp:46-60), updated in place; `scores` are the caller's scalarised fitness (apd_scores); 2 n d draws.
 * cso_reproduce (operators.hpp:246-284): shuffle (n - 1 draws) + 3 (n / 2) d draws; velocities updated in place. */
int temo_b200_de_reproduce(const double* x, uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter, double f, double cr,
                           const double* lower, const double* upper, int rng_mode, double* out, double* kernel_ms);
int temo_b200_pso_reproduce(const double* x, const double* scores, uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter,
                            double inertia, double c1, double c2, double* velocities, double* pbest_x, double* pbest_score,
                            const double* lower, const double* upper, int rng_mode, double* out, double* kernel_ms);
int temo_b200_cso_reproduce(const double* x, const double* scores, uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter, double phi,
                            double* velocities, const double* lower, const double* upper, int rng_mode, double* out,
                            double* kernel_ms);
/* random_reproduce (operators.hpp:287-296): n*d draws. */
int temo_b200_random_reproduce(uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter,
                               const double* lower, const double* upper, int rng_mode, double* out);

/* ---- problems.hpp ----------------------------------------------------------------- */
/* dtlz_eval (problems.hpp:69-92) and ProblemInstance::evaluate (problems.hpp:252); also LSMOP1. */
int temo_b200_evaluate(int problem, const double* x, uint64_t n, uint64_t d, uint64_t m, double* f);
/* Neuroevolution evaluator, bit-identical to the reference on an FMA host (tanh follows the
 * C library's operation sequence, glibc_tanh.cuh).
 * env_rollout (problems.hpp:211-241): params n x d flat MLP parameters (d = 4h + h + 2h + 2, h = hidden <= 64) -> f n x num_obj
 *   cumulative returns of one episode of `horizon` steps, maximisation orientation; -1e9 for rows with non-finite parameters.
 * mlp_forward (problems.hpp:149-163), batched: obs n x 4 -> action n x 2.
 * temo_b200_evaluate_h: temo_b200_evaluate with the episode length make_problem(name, dim, m, horizon) takes (toy2 / toy3
 *   evaluate to the NEGATED returns, problems.hpp:288-292; temo_b200_evaluate uses horizon 100). */
int temo_b200_env_rollout(const double* params, uint64_t n, uint64_t d, uint64_t hidden, uint64_t horizon, uint64_t num_obj, double* f);
int temo_b200_mlp_forward(const double* params, uint64_t n, uint64_t d, uint64_t hidden, const double* obs, double* action);
int temo_b200_evaluate_h(int problem, const double* x, uint64_t n, uint64_t d, uint64_t m, uint64_t horizon, double* f);
/* make_problem bounds (problems.hpp:271-272): lower/upper 1 x d. */
int temo_b200_problem_bounds(int problem, uint64_t d, uint64_t m, double* lower, double* upper);
uint64_t temo_b200_problem_default_dim(int problem, uint64_t m);

/* ---- refvec.hpp ------------------------------------------------------------------- */
uint64_t temo_b200_lattice_count(uint64_t m, uint64_t H);            /* refvec.hpp:15-19 */
uint64_t temo_b200_lattice_density_for(uint64_t m, uint64_t target); /* refvec.hpp:22-35 */
int temo_b200_simplex_lattice(uint64_t m, uint64_t H, double* out);  /* refvec.hpp:40-62 */
/* make_ref_set (refvec.hpp:108-114): v0 (= v) r x m and gamma r. */
int temo_b200_make_ref_set(uint64_t m, uint64_t H, double* v0, double* gamma);
/* min_vector_angles (refvec.hpp:81-100), tiled on the device: no R x R matrix. */
int temo_b200_min_vector_angles(const double* v, uint64_t r, uint64_t m, double* gamma);
/* adapt (refvec.hpp:135-140): v, gamma in/out; untouched unless every range is > 0. */
int temo_b200_adapt(const double* v0, double* v, double* gamma, uint64_t r, uint64_t m,
                    const double* z_min, const double* z_max);

/* ---- selection.hpp ---------------------------------------------------------------- */
/* rv_select (selection.hpp:200-224, want_table = false) = rv_core (:148-192) + elites.
 * elite: capacity r; validity: r bytes. Optional per-row outputs (NULL to skip):
 * assoc[n], theta[n], apd[n] (RvCore, selection.hpp:139-143). */
int temo_b200_rv_select(const double* f, uint64_t n, uint64_t m, const double* v,
                        const double* gamma, uint64_t r, uint64_t t, uint64_t t_max, double alpha,
                        uint64_t* elite, uint64_t* n_elite, unsigned char* validity,
                        uint64_t* assoc, double* theta, double* apd);
/* detail::apd_penalty (selection.hpp:86-89), host scalar (glibc pow). */
double temo_b200_apd_penalty(uint64_t m, uint64_t t, uint64_t t_max, double alpha);

/* ---- algorithms.hpp: device-resident generation loop ------------------------------- */
typedef struct temo_b200_run temo_b200_run; /* opaque */

/* Initialisation of rvea_run (algorithms.hpp:229-243): reference set, initial population
 * (n*d draws), first evaluation. */
int temo_b200_run_create(const temo_b200_run_config* cfg, temo_b200_run** out);
/* One generation (algorithms.hpp:246-292). Returns the survivor count in *pop_size.
 * survivors_f (optional, capacity r*m doubles, host) receives the survivors' objectives
 * (the per-generation result the reference hands to fill_metrics, algorithms.hpp:287). */
int temo_b200_run_step(temo_b200_run* run, uint64_t* pop_size, double* survivors_f);
/* Lock-step testing hook: one generation whose environmental selection runs on the caller's
 * offspring objectives f_off (n x m, host) instead of the device-computed ones (those stay
 * readable through temo_b200_run_last_generation). With parents injected too, the selection
 * input is bit-identical to the CPU's, so the survivor set must be as well. */
int temo_b200_run_step_injected(temo_b200_run* run, const double* f_off, uint64_t* pop_size);
/* Lock-step testing hooks: overwrite / read the loop state with host data.
 * x: rows x d, f: rows x m, v: r x m, gamma: r (any may be NULL = keep; x without f
 * re-evaluates the injected rows on the device). */
int temo_b200_run_inject(temo_b200_run* run, uint64_t rows, const double* x, const double* f,
                         const double* v, const double* gamma, uint64_t counter, uint64_t t);
int temo_b200_run_state(temo_b200_run* run, uint64_t* rows, uint64_t* counter, uint64_t* t,
                        uint64_t* r, uint64_t* d, uint64_t* m);
/* Copies out x (rows x d), f (rows x m), v (r x m), gamma (r); any may be NULL. */
int temo_b200_run_download(temo_b200_run* run, double* x, double* f, double* v, double* gamma);
/* Last generation's offspring (n x d), their objectives (n x m) and the elite merged-row
 * indices (survivor k came from merged row elite[k]; parents first, algorithms.hpp:274-279). */
int temo_b200_run_last_generation(temo_b200_run* run, double* offspring, double* f_off,
                                  uint64_t* elite);
/* Device-side timings of the last step in ms (CUDA events on the library stream):
 * [0] whole generation, [1] reproduction kernel (+fused evaluation), [2] standalone evaluation,
 * [3] selection (+survivor commit), [4] adaptation, [5] host mating-permutation time (wall),
 * [6] number of kernels launched in the step, [7] permutation upload + mating table. */
int temo_b200_run_timings(temo_b200_run* run, double* ms8);
/* The same eight values for each of the last min(max_steps, 1024) steps since the last reset, oldest first (8 * steps
 * doubles); *steps_out = steps written. The library reads a step's events while the NEXT step runs on the device, so a
 * caller that wants per-step stage times of a timed loop asks once after the loop instead of once per step (no host
 * work between the end of a step and the first launch of the next). reset != 0 empties the log afterwards.
 * (Measurement support of the harness: no reference counterpart.) */
int temo_b200_run_timing_history(temo_b200_run* run, double* ms8_per_step, uint64_t max_steps, int reset, uint64_t* steps_out);
int temo_b200_run_destroy(temo_b200_run* run);

/* rvea_run (algorithms.hpp:227-296), whole run, RunRecord fields flattened:
 * final_x (cap x d, cap = max(pop, r)), final_f, rows per generation. */
int temo_b200_rvea_run(const temo_b200_run_config* cfg, double* final_x, double* final_f,
                       uint64_t* final_rows, uint64_t* rows_done, uint64_t* pop_size,
                       double* elapsed_ms);

/* ---- NSGA-II baseline ---------------------------------------- */
/* nondominated_sort (selection.hpp:251-283): front rank of each of the n rows of f (rank 0 = nondominated). */
int temo_b200_nondominated_sort(const double* f, uint64_t n, uint64_t m, uint64_t* rank);
/* nsga2_select (selection.hpp:316-346): `target` row indices, fronts in ascending rank, the last front split by
 * descending crowding distance (ties: lowest row). */
int temo_b200_nsga2_select(const double* f, uint64_t n, uint64_t m, uint64_t target, uint64_t* selected);
/* nsga2_run (algorithms.hpp:301-369, track_archive = false) as a device-resident session; cfg as for rvea_run
 * (lattice_h / alpha / fr / op are not used). */
typedef struct temo_b200_nsga2 temo_b200_nsga2; /* opaque */
int temo_b200_nsga2_create(const temo_b200_run_config* cfg, temo_b200_nsga2** out);
/* One generation. f_off (optional, n x m): selection runs on these offspring objectives instead of the device's
 * (lock-step testing). */
int temo_b200_nsga2_step(temo_b200_nsga2* run, const double* f_off);
int temo_b200_nsga2_inject(temo_b200_nsga2* run, const double* x, const double* f, uint64_t counter, uint64_t t);
int temo_b200_nsga2_state(temo_b200_nsga2* run, uint64_t* counter, uint64_t* t, uint64_t* d);
int temo_b200_nsga2_download(temo_b200_nsga2* run, double* x, double* f);
/* offspring (n x d), their device-evaluated objectives (n x m), the selected merged rows (n; parents first) and
 * the tournament winners (n) of the last generation; any may be NULL. */
int temo_b200_nsga2_last_generation(temo_b200_nsga2* run, double* offspring, double* f_off, uint64_t* selected,
                                    uint64_t* pool_idx);
int temo_b200_nsga2_destroy(temo_b200_nsga2* run);
/* whole run: final_x (pop x d), final_f (pop x m), cumulative elapsed ms per generation (may be NULL). */
int temo_b200_nsga2_run(const temo_b200_run_config* cfg, double* final_x, double* final_f, uint64_t* rows_done,
                        double* elapsed_ms);

/* ---- metrics.hpp (quality indicators) ----------------------- */
/* igd (metrics.hpp:21-44): mean distance from each row of f_ref (n_ref x m) to its nearest row of f (n x m). */
int temo_b200_igd(const double* f, uint64_t n, uint64_t m, const double* f_ref, uint64_t n_ref, double* out);
/* hv_mc_box (metrics.hpp:76-117): Monte-Carlo hypervolume of f inside the box [lo, ref] (m values each);
 * sample s uses draws s*m .. s*m+m-1 of RngStream{seed}. std_error may be NULL. */
int temo_b200_hv_mc_box(const double* f, uint64_t n, uint64_t m, const double* lo, const double* ref,
                        uint64_t samples, uint64_t seed, double* value, double* std_error);
/* hv_mc (metrics.hpp:121-124): the box is [col_min(f), ref]. */
int temo_b200_hv_mc(const double* f, uint64_t n, uint64_t m, const double* ref, uint64_t samples,
                    uint64_t seed, double* value, double* std_error);
/* Archive::insert (algorithms.hpp:72-122) on host buffers: the archive (x_old n_old x d, f_old n_old x m) receives the
 * rows (x_new, f_new); exact duplicates keep their earliest copy, dominated rows leave, kept archive rows come first and
 * insertion order is preserved; cap > 0 truncates by crowding distance (truncate_by_crowding, :124-143). The O(n^2)
 * dominance filter runs on the device, compaction and the crowding sort on the host. x_out / f_out hold up to
 * n_old + n_new rows and may not alias the inputs. */
int temo_b200_archive_insert(const double* x_old, const double* f_old, uint64_t n_old, const double* x_new,
                             const double* f_new, uint64_t n_new, uint64_t d, uint64_t m, uint64_t cap,
                             double* x_out, double* f_out, uint64_t* n_out);
/* crowding_distance (selection.hpp:289-312) of a k x m front (host code, no GPU needed). */
int temo_b200_crowding_distance(const double* front, uint64_t k, uint64_t m, double* dist);
/* MetricContext (algorithms.hpp:46-54) of a run: pf_ref (n_ref x m; n_ref = 0: no IGD), hv_ref (m values or
 * NULL: no HV), hv_scale, hv_samples, hv_seed, maximization. */
int temo_b200_run_set_metrics(temo_b200_run* run, const double* pf_ref, uint64_t n_ref, const double* hv_ref,
                              double hv_scale, uint64_t hv_samples, uint64_t hv_seed, int maximization);
/* Archive of a device-resident run (Archive, algorithms.hpp:68-142; RunConfig::track_archive / archive_cap, :31-33).
 * temo_b200_run_track_archive must follow temo_b200_run_create directly: it inserts the initial population
 * (algorithms.hpp:243); every later step inserts its survivors (:282) and temo_b200_run_metrics then reports the
 * archive's objectives (:288). archive_cap = 0: unbounded. The archive stays in HBM (dominance filter, compaction and
 * row gather on the device; crowding truncation beyond the cap on the host). temo_b200_run_archive copies out
 * x (rows x d) and f (rows x m) in insertion order; either may be NULL. */
int temo_b200_run_track_archive(temo_b200_run* run, uint64_t archive_cap);
int temo_b200_run_archive_rows(temo_b200_run* run, uint64_t* rows);
int temo_b200_run_archive(temo_b200_run* run, double* x, double* f);
/* fill_metrics (algorithms.hpp:161-180) on the current survivors' objectives without copying them to the host
 * (m = 2: hv_exact_2d on a host copy of rows x 2 values). NaN where the context has no reference. */
int temo_b200_run_metrics(temo_b200_run* run, double* igd, double* hv);

/* ---- device-pointer stage API (used by bench.py kernel timings and the multi-GPU host
 * orchestration in paper_2404_01159_b200/dist.py). Pointers are CUDA device pointers of
 * this process; all launches go to the library stream. ------------------------------ */
void* temo_b200_dev_alloc(size_t bytes);
int temo_b200_dev_free(void* p);
/* Page-locked host memory for buffers handed to the host-buffer entry points (e.g. the survivors_f of
 * temo_b200_run_step): copies to and from it run at full PCIe rate. Plain malloc'ed buffers work everywhere too. */
void* temo_b200_host_alloc(size_t bytes);
int temo_b200_host_free(void* p);
int temo_b200_dev_upload(void* dst, const void* src, size_t bytes);
int temo_b200_dev_download(void* dst, const void* src, size_t bytes);
int temo_b200_dev_sync(void);
/* Times `reps` back-to-back launches of a stage with CUDA events on the library stream,
 * returns the mean ms per launch. stage: 1 reproduction (ga, unfused), 2 evaluation,
 * 3 reproduction with fused evaluation, 4 selection, 5 gamma. Used for the roofline. */
int temo_b200_run_time_stage(temo_b200_run* run, int stage, int reps, double* mean_ms);
/* ---- sharded generation loop: stage-level entry points of ONE rank (one process per GPU). The host
 * orchestration (paper_2404_01159_b200/dist.py) only puts the small torch.distributed collectives between them:
 * all-gather of offspring objectives / free-slot lists, min-allreduces of the per-vector (APD key, row) minima
 * (SURVEY.md section 8e). Parents are NOT exchanged: every rank maps its peers' population pools (CUDA IPC) and the
 * reproduction kernel loads remote parent rows over NVLink itself; the survivor -> (owner, slot) tables and every
 * other piece of loop state live on the device. reference: rvea_run, algorithms.hpp:227-296. */
typedef struct temo_b200_shard temo_b200_shard; /* opaque */
const char* temo_b200_shard_last_error(void);
int temo_b200_shard_create(const temo_b200_run_config* cfg, int rank, int world, temo_b200_shard** out);
int temo_b200_shard_destroy(temo_b200_shard* s);
/* info8: n_loc, d, m, r, pcap, cap_loc, adapt_every, kernels + copies enqueued by this shard so far */
int temo_b200_shard_info(temo_b200_shard* s, uint64_t* info8);
/* state5: survivor count, draw counter, generations done, lo, hi (this rank's slice of the merged rows of the generation
 * begun last) */
int temo_b200_shard_state(temo_b200_shard* s, uint64_t* state5);
/* device buffers the collectives operate on: 0 f_off_loc (n_loc x m), 1 f_gather (world x n_loc x m), 2 best_key (int64
 * view, R), 3 first_row (int32 view, R), 4 best_row (int32 view, R), 5 free_slot (int32 view, n_loc), 6 free_all (int32
 * view, world x n_loc), 7 the population pool (cap_loc x d) */
void* temo_b200_shard_buffer(temo_b200_shard* s, int which);
/* The cudaStream_t all stages of this shard are enqueued on (collectives issued on it need no device-wide syncs). */
void* temo_b200_shard_stream(temo_b200_shard* s);
/* Peer pools: every rank exports the 64-byte CUDA IPC handle of its pool, the caller all-gathers the handles (world x 64
 * bytes) and every rank opens its peers' (world > 1; a world of 1 needs neither). set_peer_pointers is the same for
 * pools that are already addressable from this process (several shards of one process: tests). */
int temo_b200_shard_ipc_handle(temo_b200_shard* s, unsigned char* handle64);
int temo_b200_shard_open_peers(temo_b200_shard* s, const unsigned char* handles);
int temo_b200_shard_set_peer_pointers(temo_b200_shard* s, void* const* pools);
/* One generation = begin, reproduce, [all-gather f_off_loc -> f_gather, free_slot -> free_all], select_local,
 * [min-allreduce best_key, first_row], select_rows, [min-allreduce best_row], finish. Every call only enqueues work on
 * the shard's stream except finish, which reads the survivor count back (the one synchronisation of a generation).
 * place_initial_f follows the first all-gather of the initial population's objectives (algorithms.hpp:242). */
int temo_b200_shard_begin(temo_b200_shard* s);
int temo_b200_shard_reproduce(temo_b200_shard* s);
int temo_b200_shard_place_initial_f(temo_b200_shard* s);
int temo_b200_shard_select_local(temo_b200_shard* s);
int temo_b200_shard_select_rows(temo_b200_shard* s);
int temo_b200_shard_finish(temo_b200_shard* s, uint64_t* count);
/* Copies out the replicated state and this rank's rows: owner / slot tables (P entries each), x of the survivors this rank
 * owns (survivor order, own_rows x d; own_index receives their survivor indices), f (P x m), v, gamma. Any may be NULL. */
int temo_b200_shard_download(temo_b200_shard* s, uint32_t* owner, uint32_t* slot, uint64_t* own_rows, uint64_t* own_index, double* x,
                             double* f, double* v, double* gamma);

/* Self-test hook for the libm-exact pow used by SBX / polynomial mutation / DTLZ4
 * (reference call sites: operators.hpp:85-86,115-118; problems.hpp:79): out[e] = pow(x[e], y[e])
 * evaluated by the device kernel (on_device = 1) or by its host twin (on_device = 0, no GPU
 * needed). Must equal the host C library's pow bit for bit on the main path. */
int temo_b200_pow(const double* x, const double* y, uint64_t n, double* out, int on_device);
/* The same for tanh (glibc_tanh.cuh: the toy environment's policy network, problems.hpp:149-163). */
int temo_b200_tanh(const double* x, uint64_t n, double* out, int on_device);
/* Overwrites >= bytes of scratch HBM (L2 flush between timed iterations). */
int temo_b200_flush_l2(void);
/* Path-selection knobs for tests and A/B measurements (no reference counterpart; results are identical on every
 * path): "k1_generic" 0/1 routes reproduction through the generic kernel instead of the phased pair kernel;
 * "k1_bound_arrays" 0/1 makes the pair kernel read the bound arrays even when they are piecewise constant;
 * "k1_cand_cap" 0..8 sets its mutation-candidate slots per warp tile (0 forces the plain per-gene tile path);
 * "k1_dynamic_pairs" 1/0 hands the mating pairs to the persistent teams through a global counter (default) or
 * round-robin over the grid; "k1_single_warp" -1 gives a mating pair to one warp when the launch has a pair for every
 * resident warp and to a team of eight warps otherwise (default), 0 always teams, 1 always single warps;
 * "k1_nested_bounds" 1/0 sends two nested bound segments (LSMOP) through the one-segment kernel plus a fix-up of the row's
 * first genes (default) or selects the bounds per gene;
 * "eval_tma" 1/0 evaluates through the bulk-copy kernels (default) or the one-CTA-per-row kernels.
 * Returns TEMO_B200_EINVAL for an unknown name. */
int temo_b200_set_option(const char* name, long value);

#ifdef __cplusplus
}
#endif
#endif /* TEMO_B200_H */
