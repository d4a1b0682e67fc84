// TEST INFRASTRUCTURE — not product code.
//
// Thin extern "C" shim that compiles the UNMODIFIED reference headers where
// they lie (/root/reference/proj/include, passed with -I by oracle/Makefile)
// into oracle/_ref/libtemo_ref.so. Nothing from the reference is copied into
// this repository: this file only forwards flat C arrays to the reference's
// own inline functions and copies their results back out.
//
// Users: tests/ (validating the C restatement in temo_oracle.c and checking the
// CUDA path directly against the real reference), oracle/gen_golden.py (golden
// fixtures) and bench.py's cpu_baseline / --impl reference legs.
//
// Every entry point returns 0 on success, a negative value on a C++ exception
// (message retrievable with ref_last_error()).

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "temo/algorithms.hpp"
#include "temo/metrics.hpp"
#include "temo/operators.hpp"
#include "temo/oracle.hpp"
#include "temo/problems.hpp"
#include "temo/refvec.hpp"
#include "temo/rng.hpp"
#include "temo/selection.hpp"

namespace {

thread_local std::string g_err;

temo::Tensor2D wrap(const double* p, std::size_t r, std::size_t c) {
    temo::Tensor2D t(r, c);
    if (r * c) std::memcpy(t.data.data(), p, r * c * sizeof(double));
    return t;
}

void unwrap(const temo::Tensor2D& t, double* out) {
    if (t.size()) std::memcpy(out, t.data.data(), t.size() * sizeof(double));
}

temo::GaParams ga_of(const double* g) {
    temo::GaParams p;
    p.pc = g[0];
    p.eta = g[1];
    p.pm = g[2];
    p.xi = g[3];
    return p;
}

template <class F>
int guarded(F&& body) {
    try {
        body();
        return 0;
    } catch (const std::bad_alloc&) {
        g_err = "bad_alloc";
        return -2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

temo::RefVectorSet refs_of(const double* v, const double* gamma, std::size_t r, std::size_t m) {
    temo::RefVectorSet refs;
    refs.v0 = wrap(v, r, m);
    refs.v = refs.v0;
    refs.gamma = wrap(gamma, r, 1);
    return refs;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint64_t ref_num_threads() { return temo::num_threads(); }
void ref_set_num_threads(std::uint64_t n) { temo::set_num_threads(n); }

// ---- rng.hpp ---------------------------------------------------------------
double ref_value_at(std::uint64_t seed, std::uint64_t counter) {
    return temo::RngStream::value_at(seed, counter);
}

int ref_uniform_fill(std::uint64_t seed, std::uint64_t counter, double* out,
                     std::uint64_t rows, std::uint64_t cols) {
    return guarded([&] {
        temo::RngStream s{seed, counter};
        unwrap(temo::uniform_tensor(s, rows, cols), out);
    });
}

int ref_shuffle_indices(std::uint64_t seed, std::uint64_t* counter, std::uint64_t n,
                        std::uint64_t* out) {
    return guarded([&] {
        temo::RngStream s{seed, *counter};
        const auto perm = temo::shuffle_indices(s, n);
        for (std::size_t i = 0; i < n; ++i) out[i] = perm[i];
        *counter = s.counter;
    });
}

int ref_parent_pool_indices(std::uint64_t current, std::uint64_t n, std::uint64_t seed,
                            std::uint64_t* counter, std::uint64_t* out) {
    return guarded([&] {
        temo::RngStream s{seed, *counter};
        const auto idx = temo::parent_pool_indices(current, n, s);
        for (std::size_t i = 0; i < n; ++i) out[i] = idx[i];
        *counter = s.counter;
    });
}

// ---- operators.hpp ---------------------------------------------------------
// which: 0 sbx, 1 polynomial_mutation, 2 ga_reproduce, 3 oracle_sbx, 4 oracle_pm, 5 oracle_ga
int ref_operator(int which, const double* x, std::uint64_t n, std::uint64_t d,
                 std::uint64_t seed, std::uint64_t* counter, const double* ga,
                 const double* lower, const double* upper, double* out) {
    return guarded([&] {
        temo::RngStream s{seed, *counter};
        const temo::Tensor2D xt = wrap(x, n, d);
        const temo::Tensor2D lo = wrap(lower, 1, d), hi = wrap(upper, 1, d);
        const temo::GaParams p = ga_of(ga);
        temo::Tensor2D res;
        namespace orc = temo::oracle;
        switch (which) {
        case 0: res = temo::sbx(xt, s, p, lo, hi); break;
        case 1: res = temo::polynomial_mutation(xt, s, p, lo, hi); break;
        case 2: res = temo::ga_reproduce(xt, s, p, lo, hi); break;
        case 3: res = orc::to_tensor(orc::oracle_sbx(orc::to_matrix(xt), s, p, lo.data, hi.data)); break;
        case 4: res = orc::to_tensor(orc::oracle_pm(orc::to_matrix(xt), s, p, lo.data, hi.data)); break;
        case 5: res = orc::to_tensor(orc::oracle_ga(orc::to_matrix(xt), s, p, lo.data, hi.data)); break;
        default: throw std::invalid_argument("ref_operator: unknown operator id");
        }
        unwrap(res, out);
        *counter = s.counter;
    });
}

// DE / PSO / CSO (operators.hpp:166-284); batched (scalar == 0) or the reference's scalar oracle (oracle.hpp:206-295)
int ref_de_reproduce(int scalar, const double* x, std::uint64_t n, std::uint64_t d, std::uint64_t seed, std::uint64_t* counter,
                     const double* p, const double* lower, const double* upper, double* out) {
    return guarded([&] {
        temo::RngStream s{seed, *counter};
        const temo::Tensor2D xt = wrap(x, n, d), lo = wrap(lower, 1, d), hi = wrap(upper, 1, d);
        const temo::DeParams dp{p[0], p[1]};
        namespace orc = temo::oracle;
        unwrap(scalar ? orc::to_tensor(orc::oracle_de(orc::to_matrix(xt), s, dp, lo.data, hi.data)) : temo::de_reproduce(xt, s, dp, lo, hi), out);
        *counter = s.counter;
    });
}

int ref_pso_reproduce(int scalar, const double* x, const double* scores, std::uint64_t n, std::uint64_t d, std::uint64_t seed,
                      std::uint64_t* counter, const double* p, double* vel, double* pb_x, double* pb_score, const double* lower,
                      const double* upper, double* out) {
    return guarded([&] {
        temo::RngStream s{seed, *counter};
        const temo::Tensor2D xt = wrap(x, n, d), lo = wrap(lower, 1, d), hi = wrap(upper, 1, d), sc = wrap(scores, n, 1);
        temo::SwarmState st{wrap(vel, n, d), wrap(pb_x, n, d), wrap(pb_score, n, 1)};
        const temo::PsoParams pp{p[0], p[1], p[2]};
        namespace orc = temo::oracle;
        unwrap(scalar ? orc::to_tensor(orc::oracle_pso(orc::to_matrix(xt), st, sc.data, s, pp, lo.data, hi.data))
                      : temo::pso_reproduce(xt, st, sc, s, pp, lo, hi),
               out);
        unwrap(st.velocities, vel);
        unwrap(st.personal_best_x, pb_x);
        unwrap(st.personal_best_score, pb_score);
        *counter = s.counter;
    });
}

int ref_cso_reproduce(int scalar, const double* x, const double* scores, std::uint64_t n, std::uint64_t d, std::uint64_t seed,
                      std::uint64_t* counter, const double* p, double* vel, const double* lower, const double* upper, double* out) {
    return guarded([&] {
        temo::RngStream s{seed, *counter};
        const temo::Tensor2D xt = wrap(x, n, d), lo = wrap(lower, 1, d), hi = wrap(upper, 1, d), sc = wrap(scores, n, 1);
        temo::SwarmState st{wrap(vel, n, d), xt, sc};
        const temo::CsoParams cp{p[0]};
        namespace orc = temo::oracle;
        unwrap(scalar ? orc::to_tensor(orc::oracle_cso(orc::to_matrix(xt), sc.data, s, cp, lo.data, hi.data, st))
                      : temo::cso_reproduce(xt, sc, s, cp, lo, hi, st),
               out);
        unwrap(st.velocities, vel);
        *counter = s.counter;
    });
}

int ref_apd_scores(const double* f, std::uint64_t n, std::uint64_t m, const double* v, const double* gamma, std::uint64_t r,
                   std::uint64_t t, std::uint64_t t_max, double alpha, double* scores) {
    return guarded([&] {
        temo::RefVectorSet refs{wrap(v, r, m), wrap(v, r, m), wrap(gamma, r, 1)};
        unwrap(temo::apd_scores(wrap(f, n, m), refs, t, t_max, alpha), scores);
    });
}

int ref_random_reproduce(std::uint64_t n, std::uint64_t d, std::uint64_t seed,
                         std::uint64_t* counter, const double* lower, const double* upper,
                         double* out) {
    return guarded([&] {
        temo::RngStream s{seed, *counter};
        unwrap(temo::random_reproduce(n, d, s, wrap(lower, 1, d), wrap(upper, 1, d)), out);
        *counter = s.counter;
    });
}

double ref_polynomial_delta(double u, double x, double lo, double hi, double xi) {
    return temo::polynomial_delta(u, x, lo, hi, xi);
}

// ---- problems.hpp ----------------------------------------------------------
int ref_dtlz_eval(int id, const double* x, std::uint64_t n, std::uint64_t d, std::uint64_t m,
                  double* f) {
    return guarded([&] { unwrap(temo::dtlz_eval(id, wrap(x, n, d), m), f); });
}

// env_rollout / mlp_forward (problems.hpp:149-241) and make_problem("toy2"/"toy3").evaluate (:279-294)
int ref_env_rollout(const double* params, std::uint64_t n, std::uint64_t hidden, std::uint64_t horizon, std::uint64_t num_obj,
                    double* f) {
    return guarded([&] {
        const temo::MlpArch arch{temo::toy_obs_dim, hidden, temo::toy_act_dim};
        unwrap(temo::env_rollout(wrap(params, n, arch.param_count()), temo::ToyEnvSpec{horizon, num_obj}, arch), f);
    });
}

int ref_mlp_forward(const double* params, std::uint64_t hidden, const double* obs, double* action) {
    return guarded([&] {
        const temo::MlpArch arch{temo::toy_obs_dim, hidden, temo::toy_act_dim};
        const temo::MlpWeights w = temo::mlp_decode({params, arch.param_count()}, arch);
        temo::mlp_forward(w, {obs, temo::toy_obs_dim}, {action, temo::toy_act_dim});
    });
}

// any registered problem through make_problem(name, dim, m, horizon).evaluate; lower / upper may be NULL
int ref_problem_evaluate(const char* name, std::uint64_t dim, std::uint64_t m, std::uint64_t horizon, const double* x,
                         std::uint64_t n, double* f, double* lower, double* upper, std::uint64_t* dim_out, std::uint64_t* m_out) {
    return guarded([&] {
        const temo::ProblemInstance prob = temo::make_problem(name, dim, m, horizon);
        if (dim_out) *dim_out = prob.dim;
        if (m_out) *m_out = prob.num_obj;
        if (lower) unwrap(prob.lower, lower);
        if (upper) unwrap(prob.upper, upper);
        if (x && f && n) unwrap(prob.evaluate(wrap(x, n, prob.dim)), f);
    });
}

int ref_dtlz_pf_reference(int id, std::uint64_t m, std::uint64_t H, double* out) {
    return guarded([&] { unwrap(temo::dtlz_pf_reference(id, m, H), out); });
}

// ---- refvec.hpp ------------------------------------------------------------
std::uint64_t ref_lattice_count(std::uint64_t m, std::uint64_t H) {
    return temo::lattice_count(m, H);
}
std::uint64_t ref_lattice_density_for(std::uint64_t m, std::uint64_t target) {
    return temo::lattice_density_for(m, target);
}

int ref_simplex_lattice(std::uint64_t m, std::uint64_t H, double* out) {
    return guarded([&] { unwrap(temo::simplex_lattice(m, H), out); });
}

int ref_normalize_to_unit(const double* v, std::uint64_t r, std::uint64_t m, double* out) {
    return guarded([&] { unwrap(temo::normalize_to_unit(wrap(v, r, m)), out); });
}

int ref_make_ref_set(std::uint64_t m, std::uint64_t H, double* v0, double* gamma) {
    return guarded([&] {
        const temo::RefVectorSet refs = temo::make_ref_set(m, H);
        unwrap(refs.v0, v0);
        unwrap(refs.gamma, gamma);
    });
}

int ref_min_vector_angles(const double* v, std::uint64_t r, std::uint64_t m, double* gamma) {
    return guarded([&] { unwrap(temo::min_vector_angles(wrap(v, r, m)), gamma); });
}

// v and gamma are in/out (the reference mutates RefVectorSet in place).
int ref_adapt(const double* v0, double* v, double* gamma, std::uint64_t r, std::uint64_t m,
              const double* zmin, const double* zmax) {
    return guarded([&] {
        temo::RefVectorSet refs;
        refs.v0 = wrap(v0, r, m);
        refs.v = wrap(v, r, m);
        refs.gamma = wrap(gamma, r, 1);
        temo::adapt(refs, wrap(zmin, 1, m), wrap(zmax, 1, m));
        unwrap(refs.v, v);
        unwrap(refs.gamma, gamma);
    });
}

// ---- selection.hpp ---------------------------------------------------------
// which: 0 rv_select (production, rv_core), 1 oracle_rv_select (argmin-angle set form).
// Optional outputs (may be NULL): assoc[n], theta[n], apd[n] (rv_core only), table[n*r].
int ref_rv_select(int which, const double* f, std::uint64_t n, std::uint64_t m, const double* v,
                  const double* gamma, std::uint64_t r, std::uint64_t t, std::uint64_t t_max,
                  double alpha, std::uint64_t* elite, std::uint64_t* n_elite,
                  unsigned char* validity, std::uint64_t* assoc, double* theta, double* apd,
                  double* table) {
    return guarded([&] {
        const temo::Tensor2D ft = wrap(f, n, m);
        const temo::RefVectorSet refs = refs_of(v, gamma, r, m);
        const temo::SelectionOutcome out =
            which == 0 ? temo::rv_select(ft, refs, t, t_max, alpha, table != nullptr)
                       : temo::oracle::oracle_rv_select(ft, refs, t, t_max, alpha);
        *n_elite = out.elite_indices.size();
        for (std::size_t i = 0; i < out.elite_indices.size(); ++i) elite[i] = out.elite_indices[i];
        for (std::size_t j = 0; j < r; ++j) validity[j] = out.validity[j] ? 1 : 0;
        if (table && out.apd_table.size()) unwrap(out.apd_table, table);
        if (which == 0 && (assoc || theta || apd)) {
            const temo::detail::RvCore core = temo::detail::rv_core(ft, refs, t, t_max, alpha);
            for (std::size_t i = 0; i < n; ++i) {
                if (assoc) assoc[i] = core.assoc[i];
                if (theta) theta[i] = core.theta[i];
                if (apd) apd[i] = core.apd[i];
            }
        }
    });
}

double ref_apd_penalty(std::uint64_t m, std::uint64_t t, std::uint64_t t_max, double alpha) {
    return temo::detail::apd_penalty(m, t, t_max, alpha);
}

// ---- metrics.hpp -----------------------------------------------------------
int ref_igd(const double* f, std::uint64_t n, std::uint64_t m, const double* pf,
            std::uint64_t n_ref, double* out) {
    return guarded([&] { *out = temo::igd(wrap(f, n, m), wrap(pf, n_ref, m)); });
}

int ref_hv_mc(const double* f, std::uint64_t n, std::uint64_t m, const double* ref_point,
              std::uint64_t samples, std::uint64_t seed, double* out) {
    return guarded([&] {
        *out = temo::hv_mc(wrap(f, n, m), wrap(ref_point, 1, m), samples, seed).value;
    });
}

// ---- algorithms.hpp --------------------------------------------------------
// which: 0 rvea_run (batched, all lanes), 1 oracle_rvea_run (scalar loops).
// cfg_u: {pop, lattice_h, generations, seed, dim, obj}; cfg_d: {alpha, fr, time_budget_s};
// final_x/final_f must hold max(pop, R) rows. rows_* arrays hold `generations` entries.
// igd_H > 0 -> per-generation IGD against dtlz_pf_reference(id, m, igd_H) of the population.
int ref_rvea_run(int which, const char* problem, const std::uint64_t* cfg_u, const double* cfg_d,
                 const double* ga, std::uint64_t igd_H, double* final_x, double* final_f,
                 std::uint64_t* final_rows, std::uint64_t* rows_done, std::uint64_t* pop_size,
                 double* elapsed_ms, double* igd_out) {
    return guarded([&] {
        temo::RunConfig cfg;
        cfg.problem = problem;
        cfg.op = "ga";
        cfg.pop = cfg_u[0];
        cfg.lattice_h = cfg_u[1];
        cfg.generations = cfg_u[2];
        cfg.seed = cfg_u[3];
        cfg.dim = cfg_u[4];
        cfg.obj = cfg_u[5];
        cfg.alpha = cfg_d[0];
        cfg.fr = cfg_d[1];
        cfg.time_budget_s = cfg_d[2];
        cfg.track_archive = false;
        cfg.ga = ga_of(ga);
        const temo::ProblemInstance prob = temo::make_problem(cfg.problem, cfg.dim, cfg.obj);
        temo::MetricContext mc;
        if (igd_H > 0) mc.pf_ref = temo::dtlz_pf_reference(prob.dtlz_id, prob.num_obj, igd_H);
        const temo::RunRecord rec = which == 0 ? temo::rvea_run(prob, cfg, mc)
                                               : temo::oracle::oracle_rvea_run(prob, cfg, mc);
        *final_rows = rec.final_x.rows;
        if (final_x) unwrap(rec.final_x, final_x);
        if (final_f) unwrap(rec.final_f, final_f);
        *rows_done = rec.rows.size();
        for (std::size_t i = 0; i < rec.rows.size(); ++i) {
            if (pop_size) pop_size[i] = rec.rows[i].pop_size;
            if (elapsed_ms) elapsed_ms[i] = rec.rows[i].elapsed_ms;
            if (igd_out) igd_out[i] = rec.rows[i].igd_value;
        }
    });
}

// rvea_run with any operator of algorithms.hpp:250-271 (op = "ga" / "de" / "pso" / "cso" / "random");
// opp = {de.f, de.cr, pso.inertia, pso.c1, pso.c2, cso.phi}; cfg_u / cfg_d as in ref_rvea_run.
int ref_rvea_run_op(const char* problem, const char* op, const double* opp, const std::uint64_t* cfg_u, const double* cfg_d,
                    const double* ga, double* final_x, double* final_f, std::uint64_t* final_rows, std::uint64_t* rows_done,
                    std::uint64_t* pop_size) {
    return guarded([&] {
        temo::RunConfig cfg;
        cfg.problem = problem;
        cfg.op = op;
        cfg.pop = cfg_u[0];
        cfg.lattice_h = cfg_u[1];
        cfg.generations = cfg_u[2];
        cfg.seed = cfg_u[3];
        cfg.dim = cfg_u[4];
        cfg.obj = cfg_u[5];
        cfg.alpha = cfg_d[0];
        cfg.fr = cfg_d[1];
        cfg.time_budget_s = cfg_d[2];
        cfg.track_archive = false;
        cfg.ga = ga_of(ga);
        cfg.de.f = opp[0];
        cfg.de.cr = opp[1];
        cfg.pso.inertia = opp[2];
        cfg.pso.c1 = opp[3];
        cfg.pso.c2 = opp[4];
        cfg.cso.phi = opp[5];
        const temo::ProblemInstance prob = temo::make_problem(cfg.problem, cfg.dim, cfg.obj);
        const temo::RunRecord rec = temo::rvea_run(prob, cfg, temo::MetricContext{});
        *final_rows = rec.final_x.rows;
        if (final_x) unwrap(rec.final_x, final_x);
        if (final_f) unwrap(rec.final_f, final_f);
        *rows_done = rec.rows.size();
        for (std::size_t i = 0; i < rec.rows.size(); ++i)
            if (pop_size) pop_size[i] = rec.rows[i].pop_size;
    });
}

// rvea_run / oracle_rvea_run with track_archive = true (algorithms.hpp:243, 282-288): per-generation survivor count,
// archive size and IGD of the ARCHIVE against pf_ref; final archive in arch_x / arch_f (capacity arch_cap_rows rows).
int ref_rvea_run_archive(int which, const char* problem, const std::uint64_t* cfg_u, const double* cfg_d, std::uint64_t archive_cap,
                         const double* pf_ref, std::uint64_t n_ref, std::uint64_t* pop_size, std::uint64_t* arch_size,
                         double* igd_out, double* arch_x, double* arch_f, std::uint64_t arch_cap_rows, std::uint64_t* arch_rows) {
    return guarded([&] {
        temo::RunConfig cfg;
        cfg.problem = problem;
        cfg.op = "ga";
        cfg.pop = cfg_u[0];
        cfg.lattice_h = cfg_u[1];
        cfg.generations = cfg_u[2];
        cfg.seed = cfg_u[3];
        cfg.dim = cfg_u[4];
        cfg.obj = cfg_u[5];
        cfg.alpha = cfg_d[0];
        cfg.fr = cfg_d[1];
        cfg.track_archive = true;
        cfg.archive_history = true;
        cfg.archive_cap = archive_cap;
        const temo::ProblemInstance prob = temo::make_problem(cfg.problem, cfg.dim, cfg.obj);
        temo::MetricContext mc;
        if (pf_ref && n_ref) mc.pf_ref = wrap(pf_ref, n_ref, cfg.obj);
        const temo::RunRecord rec = which == 0 ? temo::rvea_run(prob, cfg, mc) : temo::oracle::oracle_rvea_run(prob, cfg, mc);
        for (std::size_t i = 0; i < rec.rows.size(); ++i) {
            pop_size[i] = rec.rows[i].pop_size;
            igd_out[i] = rec.rows[i].igd_value;
            arch_size[i] = i < rec.archive_f_history.size() ? rec.archive_f_history[i].rows : 0;
        }
        *arch_rows = rec.archive.f.rows;
        if (rec.archive.f.rows > arch_cap_rows) throw std::runtime_error("archive larger than the caller's buffers");
        if (arch_x) unwrap(rec.archive.x, arch_x);
        if (arch_f) unwrap(rec.archive.f, arch_f);
    });
}

// hv_mc_box / hv_mc with the standard error (metrics.hpp:76-124); lo == nullptr selects hv_mc. out = {value, std_error}.
int ref_hv_mc_box(const double* f, std::uint64_t n, std::uint64_t m, const double* lo, const double* ref_point,
                  std::uint64_t samples, std::uint64_t seed, double* out) {
    return guarded([&] {
        const temo::HvEstimate e = lo ? temo::hv_mc_box(wrap(f, n, m), wrap(lo, 1, m), wrap(ref_point, 1, m), samples, seed)
                                      : temo::hv_mc(wrap(f, n, m), wrap(ref_point, 1, m), samples, seed);
        out[0] = e.value;
        out[1] = e.std_error;
    });
}

// rvea_run with a MetricContext (algorithms.hpp:46-54, 161-180, 288): per-generation IGD / HV of the population.
// hv_ref may be nullptr; mcp = {hv_scale, hv_samples, hv_seed, maximization}.
int ref_rvea_run_metrics(const char* problem, const char* op, const std::uint64_t* cfg_u, const double* cfg_d, const double* pf_ref,
                         std::uint64_t n_ref, const double* hv_ref, const double* mcp, std::uint64_t* pop_size, double* igd_out,
                         double* hv_out) {
    return guarded([&] {
        temo::RunConfig cfg;
        cfg.problem = problem;
        cfg.op = op;
        cfg.pop = cfg_u[0];
        cfg.lattice_h = cfg_u[1];
        cfg.generations = cfg_u[2];
        cfg.seed = cfg_u[3];
        cfg.dim = cfg_u[4];
        cfg.obj = cfg_u[5];
        cfg.alpha = cfg_d[0];
        cfg.fr = cfg_d[1];
        cfg.track_archive = false;
        const temo::ProblemInstance prob = temo::make_problem(cfg.problem, cfg.dim, cfg.obj);
        temo::MetricContext mc;
        if (pf_ref && n_ref) mc.pf_ref = wrap(pf_ref, n_ref, cfg.obj);
        if (hv_ref) mc.hv_ref = wrap(hv_ref, 1, cfg.obj);
        mc.hv_scale = mcp[0];
        mc.hv_samples = static_cast<std::size_t>(mcp[1]);
        mc.hv_seed = static_cast<std::uint64_t>(mcp[2]);
        mc.maximization = mcp[3] != 0.0;
        const temo::RunRecord rec = temo::rvea_run(prob, cfg, mc);
        for (std::size_t i = 0; i < rec.rows.size(); ++i) {
            pop_size[i] = rec.rows[i].pop_size;
            igd_out[i] = rec.rows[i].igd_value;
            hv_out[i] = rec.rows[i].hv_value;
        }
    });
}

// Archive::insert (algorithms.hpp:72-144) on flat arrays; x_out / f_out hold n_old + n_new rows.
int ref_archive_insert(const double* x_old, const double* f_old, std::uint64_t n_old, const double* x_new, const double* f_new,
                       std::uint64_t n_new, std::uint64_t d, std::uint64_t m, std::uint64_t cap, double* x_out, double* f_out,
                       std::uint64_t* n_out) {
    return guarded([&] {
        temo::Archive a;
        if (n_old) {
            a.x = wrap(x_old, n_old, d);
            a.f = wrap(f_old, n_old, m);
        }
        a.insert(wrap(x_new, n_new, d), wrap(f_new, n_new, m), cap);
        *n_out = a.f.rows;
        unwrap(a.x, x_out);
        unwrap(a.f, f_out);
    });
}

int ref_crowding_distance(const double* front, std::uint64_t k, std::uint64_t m, double* dist) {
    return guarded([&] { unwrap(temo::crowding_distance(wrap(front, k, m)), dist); });
}

// ---- NSGA-II baseline (selection.hpp:251-346, algorithms.hpp:301-369) ----------------------------
int ref_nondominated_sort(const double* f, std::uint64_t n, std::uint64_t m, std::uint64_t* rank) {
    return guarded([&] {
        const std::vector<std::size_t> r = temo::nondominated_sort(wrap(f, n, m));
        for (std::size_t i = 0; i < r.size(); ++i) rank[i] = r[i];
    });
}

int ref_nsga2_select(const double* f, std::uint64_t n, std::uint64_t m, std::uint64_t target, std::uint64_t* selected) {
    return guarded([&] {
        const std::vector<std::size_t> s = temo::nsga2_select(wrap(f, n, m), target);
        for (std::size_t i = 0; i < s.size(); ++i) selected[i] = s[i];
    });
}

// cfg_u: {pop, generations, seed, dim, obj}
int ref_nsga2_run(const char* problem, const std::uint64_t* cfg_u, const double* ga, double* final_x, double* final_f) {
    return guarded([&] {
        temo::RunConfig cfg;
        cfg.problem = problem;
        cfg.pop = cfg_u[0];
        cfg.generations = cfg_u[1];
        cfg.seed = cfg_u[2];
        cfg.dim = cfg_u[3];
        cfg.obj = cfg_u[4];
        cfg.track_archive = false;
        cfg.ga = ga_of(ga);
        const temo::ProblemInstance prob = temo::make_problem(cfg.problem, cfg.dim, cfg.obj);
        const temo::RunRecord rec = temo::nsga2_run(prob, cfg, temo::MetricContext{});
        unwrap(rec.final_x, final_x);
        unwrap(rec.final_f, final_f);
    });
}

} // extern "C"
