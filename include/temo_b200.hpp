// temo_b200.hpp — reference-side binding: the reference's own signatures in namespace temo::b200,
// forwarding to the C ABI of libtemo_b200.so (temo_b200.h).
//
// A maintainer of the reference adds this header next to proj/include/temo/*.hpp, links
// libtemo_b200.so, and swaps one call: temo::sbx(...) -> temo::b200::sbx(...), temo::rv_select(...) ->
// temo::b200::rv_select(...), temo::rvea_run(...) -> temo::b200::rvea_run(...). Argument meaning, RngStream
// counter advance and exceptions are the reference's (std::invalid_argument for contract violations,
// std::runtime_error otherwise). Requires the reference headers on the include path.
//
// reference interfaces mirrored: rng.hpp:55-78, operators.hpp:65-161,287-296, problems.hpp:69-92,
// refvec.hpp:81-140, selection.hpp:131-135,200-346, algorithms.hpp:21-144,211-369, metrics.hpp:21-124.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "temo/algorithms.hpp"
#include "temo/metrics.hpp"
#include "temo/operators.hpp"
#include "temo/problems.hpp"
#include "temo/refvec.hpp"
#include "temo/rng.hpp"
#include "temo/selection.hpp"
#include "temo_b200.h"

namespace temo::b200 {

namespace detail {

inline void check(int rc) {
    if (rc == TEMO_B200_OK) return;
    const std::string msg = temo_b200_last_error();
    if (rc == TEMO_B200_EINVAL) throw std::invalid_argument(msg);
    if (rc == TEMO_B200_ENOMEM) throw std::bad_alloc();
    throw std::runtime_error(msg);
}

inline temo_b200_ga_params ga_of(const GaParams& p) { return {p.pc, p.eta, p.pm, p.xi}; }

inline int problem_id(const ProblemInstance& prob) {
    if (prob.dtlz_id >= 1 && prob.dtlz_id <= 4) return prob.dtlz_id;
    if (prob.name == "lsmop1") return TEMO_B200_LSMOP1;
    if (prob.name == "toy2") return TEMO_B200_TOY2;
    if (prob.name == "toy3") return TEMO_B200_TOY3;
    throw std::invalid_argument("temo::b200: problem '" + prob.name + "' has no device evaluator");
}

using OperatorFn = int (*)(const double*, uint64_t, uint64_t, uint64_t, uint64_t*, const temo_b200_ga_params*,
                           const double*, const double*, int, double*);

inline Tensor2D run_operator(OperatorFn fn, const Tensor2D& x, RngStream& stream, const GaParams& p,
                             const Tensor2D& lower, const Tensor2D& upper) {
    temo::detail::require(lower.size() == x.cols && upper.size() == x.cols, "operator: bounds shape mismatch");
    Tensor2D out(x.rows, x.cols);
    const temo_b200_ga_params ga = ga_of(p);
    uint64_t counter = stream.counter;
    check(fn(x.data.data(), x.rows, x.cols, stream.seed, &counter, &ga, lower.data.data(), upper.data.data(),
             TEMO_B200_RNG_SPLITMIX64, out.data.data()));
    stream.counter = counter;
    return out;
}

}  // namespace detail

// ---- rng.hpp ---------------------------------------------------------------------------------
inline Tensor2D uniform_tensor(RngStream& stream, std::size_t rows, std::size_t cols) {
    Tensor2D out(rows, cols);
    uint64_t counter = stream.counter;
    detail::check(temo_b200_uniform_tensor(stream.seed, &counter, rows, cols, TEMO_B200_RNG_SPLITMIX64, out.data.data()));
    stream.counter = counter;
    return out;
}

// ---- operators.hpp ---------------------------------------------------------------------------
inline Tensor2D sbx(const Tensor2D& x, RngStream& stream, const GaParams& p, const Tensor2D& lower,
                    const Tensor2D& upper) {
    return detail::run_operator(temo_b200_sbx, x, stream, p, lower, upper);
}

inline Tensor2D polynomial_mutation(const Tensor2D& x, RngStream& stream, const GaParams& p, const Tensor2D& lower,
                                    const Tensor2D& upper) {
    return detail::run_operator(temo_b200_polynomial_mutation, x, stream, p, lower, upper);
}

inline Tensor2D ga_reproduce(const Tensor2D& x, RngStream& stream, const GaParams& p, const Tensor2D& lower,
                             const Tensor2D& upper) {
    return detail::run_operator(temo_b200_ga_reproduce, x, stream, p, lower, upper);
}

inline Tensor2D random_reproduce(std::size_t n, std::size_t d, RngStream& stream, const Tensor2D& lower,
                                 const Tensor2D& upper) {
    Tensor2D out(n, d);
    uint64_t counter = stream.counter;
    detail::check(temo_b200_random_reproduce(n, d, stream.seed, &counter, lower.data.data(), upper.data.data(),
                                             TEMO_B200_RNG_SPLITMIX64, out.data.data()));
    stream.counter = counter;
    return out;
}

// DE / PSO / CSO (operators.hpp:166-284): same signatures, same in-place SwarmState updates, bit-identical results.
inline Tensor2D de_reproduce(const Tensor2D& x, RngStream& stream, const DeParams& p, const Tensor2D& lower,
                             const Tensor2D& upper) {
    temo::detail::require(lower.size() == x.cols && upper.size() == x.cols, "de_reproduce: bounds shape mismatch");
    Tensor2D out(x.rows, x.cols);
    uint64_t counter = stream.counter;
    detail::check(temo_b200_de_reproduce(x.data.data(), x.rows, x.cols, stream.seed, &counter, p.f, p.cr, lower.data.data(),
                                         upper.data.data(), TEMO_B200_RNG_SPLITMIX64, out.data.data(), nullptr));
    stream.counter = counter;
    return out;
}

inline Tensor2D pso_reproduce(const Tensor2D& x, SwarmState& state, const Tensor2D& scores, RngStream& stream,
                              const PsoParams& p, const Tensor2D& lower, const Tensor2D& upper) {
    const std::size_t n = x.rows, d = x.cols;
    temo::detail::require(state.velocities.rows == n && state.velocities.cols == d && state.personal_best_x.rows == n &&
                              scores.rows == n,
                          "pso_reproduce: state shape mismatch");  // operators.hpp:209-211
    Tensor2D out(n, d);
    uint64_t counter = stream.counter;
    detail::check(temo_b200_pso_reproduce(x.data.data(), scores.data.data(), n, d, stream.seed, &counter, p.inertia, p.c1, p.c2,
                                          state.velocities.data.data(), state.personal_best_x.data.data(),
                                          state.personal_best_score.data.data(), lower.data.data(), upper.data.data(),
                                          TEMO_B200_RNG_SPLITMIX64, out.data.data(), nullptr));
    stream.counter = counter;
    return out;
}

inline Tensor2D cso_reproduce(const Tensor2D& x, const Tensor2D& scores, RngStream& stream, const CsoParams& p,
                              const Tensor2D& lower, const Tensor2D& upper, SwarmState& state) {
    const std::size_t n = x.rows, d = x.cols;
    temo::detail::require(state.velocities.rows == n && state.velocities.cols == d && scores.rows == n,
                          "cso_reproduce: state shape mismatch");  // operators.hpp:251-253
    Tensor2D out(n, d);
    uint64_t counter = stream.counter;
    detail::check(temo_b200_cso_reproduce(x.data.data(), scores.data.data(), n, d, stream.seed, &counter, p.phi,
                                          state.velocities.data.data(), lower.data.data(), upper.data.data(),
                                          TEMO_B200_RNG_SPLITMIX64, out.data.data(), nullptr));
    stream.counter = counter;
    return out;
}

// ---- problems.hpp ----------------------------------------------------------------------------
inline Tensor2D dtlz_eval(int id, const Tensor2D& x, std::size_t m) {
    temo::detail::require(id >= 1 && id <= 4, "dtlz_eval: id must be in 1..4");
    Tensor2D f(x.rows, m);
    detail::check(temo_b200_evaluate(id, x.data.data(), x.rows, x.cols, m, f.data.data()));
    return f;
}

/// A ProblemInstance whose evaluate() runs on the device (drop-in for make_problem: dtlz1..dtlz4, toy2, toy3).
inline ProblemInstance make_problem(const std::string& name, std::size_t dim = 0, std::size_t m = 3, std::size_t toy_horizon = 100) {
    ProblemInstance p = temo::make_problem(name, dim, m, toy_horizon);
    const std::size_t mm = p.num_obj;
    if (p.dtlz_id != 0) {
        const int id = p.dtlz_id;
        p.evaluate = [id, mm](const Tensor2D& x) { return temo::b200::dtlz_eval(id, x, mm); };
    } else {  // toy2 / toy3: the negated returns of env_rollout (problems.hpp:288-292)
        const int id = name == "toy2" ? TEMO_B200_TOY2 : TEMO_B200_TOY3;
        p.evaluate = [id, mm, toy_horizon](const Tensor2D& x) {
            Tensor2D f(x.rows, mm);
            detail::check(temo_b200_evaluate_h(id, x.data.data(), x.rows, x.cols, mm, toy_horizon, f.data.data()));
            return f;
        };
    }
    return p;
}

// ---- refvec.hpp ------------------------------------------------------------------------------
inline Tensor2D min_vector_angles(const Tensor2D& v) {
    Tensor2D gamma(v.rows, 1);
    detail::check(temo_b200_min_vector_angles(v.data.data(), v.rows, v.cols, gamma.data.data()));
    return gamma;
}

inline RefVectorSet make_ref_set(std::size_t m, std::size_t H) {
    RefVectorSet refs;
    const std::size_t r = lattice_count(m, H);
    refs.v0 = Tensor2D(r, m);
    refs.gamma = Tensor2D(r, 1);
    detail::check(temo_b200_make_ref_set(m, H, refs.v0.data.data(), refs.gamma.data.data()));
    refs.v = refs.v0;
    return refs;
}

inline void adapt(RefVectorSet& refs, const Tensor2D& z_min, const Tensor2D& z_max) {
    temo::detail::require(z_min.size() == refs.v0.cols && z_max.size() == refs.v0.cols,
                          "adapt_vectors: range shape mismatch");
    detail::check(temo_b200_adapt(refs.v0.data.data(), refs.v.data.data(), refs.gamma.data.data(), refs.v0.rows,
                                  refs.v0.cols, z_min.data.data(), z_max.data.data()));
}

// ---- selection.hpp ---------------------------------------------------------------------------
inline SelectionOutcome rv_select(const Tensor2D& f, const RefVectorSet& refs, std::size_t t, std::size_t t_max,
                                  double alpha, bool want_table = true) {
    temo::detail::require(f.cols == refs.v.cols, "rv_select: objective count mismatch");
    const std::size_t n = f.rows, r = refs.v.rows;
    std::vector<uint64_t> elite(r ? r : 1), assoc(n);
    std::vector<unsigned char> valid(r);
    std::vector<double> apd(n);
    uint64_t count = 0;
    detail::check(temo_b200_rv_select(f.data.data(), n, f.cols, refs.v.data.data(), refs.gamma.data.data(), r, t, t_max,
                                      alpha, elite.data(), &count, valid.data(), assoc.data(), nullptr, apd.data()));
    SelectionOutcome out;
    out.elite_indices.assign(elite.begin(), elite.begin() + count);
    out.validity.assign(valid.begin(), valid.end());
    if (want_table) {  // selection.hpp:218-222
        out.apd_table = Tensor2D(n, r, inf);
        for (std::size_t i = 0; i < n; ++i) out.apd_table(i, assoc[i]) = apd[i];
    }
    return out;
}

/// apd_scores (selection.hpp:228-234): every row's APD against its associated vector, n x 1.
inline Tensor2D apd_scores(const Tensor2D& f, const RefVectorSet& refs, std::size_t t, std::size_t t_max, double alpha) {
    temo::detail::require(f.cols == refs.v.cols, "rv_select: objective count mismatch");
    const std::size_t n = f.rows, r = refs.v.rows;
    std::vector<uint64_t> elite(r ? r : 1);
    std::vector<unsigned char> valid(r);
    Tensor2D scores(n, 1);
    uint64_t count = 0;
    detail::check(temo_b200_rv_select(f.data.data(), n, f.cols, refs.v.data.data(), refs.gamma.data.data(), r, t, t_max, alpha,
                                      elite.data(), &count, valid.data(), nullptr, nullptr, scores.data.data()));
    return scores;
}

/// env_rollout (problems.hpp:211-241): n x d flat MLP parameters -> n x num_obj returns (maximisation orientation).
inline Tensor2D env_rollout(const Tensor2D& params, const ToyEnvSpec& spec, const MlpArch& arch) {
    temo::detail::require(params.cols == arch.param_count(), "env_rollout: parameter length mismatch");
    temo::detail::require(arch.obs_dim == toy_obs_dim && arch.act_dim == toy_act_dim, "env_rollout: arch does not match the environment");
    temo::detail::require(arch.hidden <= 64, "env_rollout: hidden layer too wide");
    Tensor2D f(params.rows, spec.num_obj);
    detail::check(temo_b200_env_rollout(params.data.data(), params.rows, params.cols, arch.hidden, spec.horizon, spec.num_obj,
                                        f.data.data()));
    return f;
}

/// mlp_forward (problems.hpp:149-163) for a batch: individual i (row i of params) acts on observation i.
inline Tensor2D mlp_forward(const Tensor2D& params, const MlpArch& arch, const Tensor2D& obs) {
    temo::detail::require(params.cols == arch.param_count(), "mlp_decode: length mismatch");
    temo::detail::require(obs.rows == params.rows && obs.cols == toy_obs_dim, "mlp_forward: observations must be n x 4");
    Tensor2D act(params.rows, toy_act_dim);
    detail::check(temo_b200_mlp_forward(params.data.data(), params.rows, params.cols, arch.hidden, obs.data.data(), act.data.data()));
    return act;
}

// ---- algorithms.hpp --------------------------------------------------------------------------
/// rvea_run (algorithms.hpp:227-296), device-resident for the whole run; cfg.op = ga / de / pso / cso / random
/// (algorithms.hpp:250-271). cfg.track_archive keeps the Archive in HBM (algorithms.hpp:243, 282) and fills
/// RunRecord.archive / archive_f_history; with a MetricContext every GenerationRow carries igd_value / hv_value of the
/// archive (of the population without one), algorithms.hpp:288. The expected-utility indicator is not on this path.
inline RunRecord rvea_run(const ProblemInstance& prob, const RunConfig& cfg, const MetricContext& mc = {}) {
    temo::detail::require(cfg.pop >= 2 && cfg.generations >= 1, "rvea_run: bad config");
    static const char* const kOps[] = {"ga", "de", "pso", "cso", "random"};
    int op = -1;
    for (int k = 0; k < 5; ++k)
        if (cfg.op == kOps[k]) op = k;
    if (op < 0) throw std::invalid_argument("rvea_run: unknown operator '" + cfg.op + "'");  // algorithms.hpp:270
    temo_b200_run_config c;
    temo_b200_default_run_config(&c);
    c.op = op;
    c.opp.de_f = cfg.de.f;
    c.opp.de_cr = cfg.de.cr;
    c.opp.pso_inertia = cfg.pso.inertia;
    c.opp.pso_c1 = cfg.pso.c1;
    c.opp.pso_c2 = cfg.pso.c2;
    c.opp.cso_phi = cfg.cso.phi;
    c.problem = detail::problem_id(prob);
    c.pop = cfg.pop;
    c.lattice_h = cfg.lattice_h;
    c.generations = cfg.generations;
    c.seed = cfg.seed;
    c.dim = prob.dim;
    c.obj = prob.num_obj;
    c.alpha = cfg.alpha;
    c.fr = cfg.fr;
    c.time_budget_s = cfg.time_budget_s;
    c.ga = detail::ga_of(cfg.ga);
    c.horizon = cfg.horizon;
    const std::size_t h = cfg.lattice_h ? cfg.lattice_h : lattice_density_for(prob.num_obj, cfg.pop);
    const std::size_t cap = std::max<std::size_t>(cfg.pop, lattice_count(prob.num_obj, h));
    Tensor2D x(cap, prob.dim), f(cap, prob.num_obj);
    RunRecord rec;
    uint64_t rows = 0;
    const bool with_metrics = mc.pf_ref.rows > 0 || mc.hv_ref.rows > 0;
    if (!cfg.track_archive && !with_metrics) {  // one call for the whole run
        std::vector<uint64_t> pops(cfg.generations);
        std::vector<double> ms(cfg.generations);
        uint64_t done = 0;
        detail::check(temo_b200_rvea_run(&c, x.data.data(), f.data.data(), &rows, &done, pops.data(), ms.data()));
        for (uint64_t t = 0; t < done; ++t) {
            GenerationRow row;
            row.t = t;
            row.elapsed_ms = ms[t];
            row.pop_size = pops[t];
            rec.rows.push_back(row);
        }
    } else {  // the session calls: one step per generation, archive and indicators stay on the device
        const temo::detail::GenerationTimer timer;
        temo_b200_run* run = nullptr;
        detail::check(temo_b200_run_create(&c, &run));
        struct Closer {
            temo_b200_run* r;
            ~Closer() { temo_b200_run_destroy(r); }
        } closer{run};
        auto fetch_archive = [&](Tensor2D* ax, Tensor2D& af) {
            uint64_t arows = 0;
            detail::check(temo_b200_run_archive_rows(run, &arows));
            if (ax) *ax = Tensor2D(arows, prob.dim);
            af = Tensor2D(arows, prob.num_obj);
            detail::check(temo_b200_run_archive(run, ax ? ax->data.data() : nullptr, af.data.data()));
        };
        if (cfg.track_archive) detail::check(temo_b200_run_track_archive(run, cfg.archive_cap));
        if (with_metrics)
            detail::check(temo_b200_run_set_metrics(run, mc.pf_ref.rows ? mc.pf_ref.data.data() : nullptr, mc.pf_ref.rows,
                                                    mc.hv_ref.rows ? mc.hv_ref.data.data() : nullptr, mc.hv_scale, mc.hv_samples,
                                                    mc.hv_seed, mc.maximization ? 1 : 0));
        for (std::size_t t = 0; t < cfg.generations; ++t) {
            uint64_t pop = 0;
            detail::check(temo_b200_run_step(run, &pop, nullptr));
            GenerationRow row;
            row.t = t;
            row.pop_size = pop;
            if (with_metrics) detail::check(temo_b200_run_metrics(run, &row.igd_value, &row.hv_value));
            if (cfg.track_archive && cfg.archive_history) {
                Tensor2D af;
                fetch_archive(nullptr, af);
                rec.archive_f_history.push_back(std::move(af));
            }
            row.elapsed_ms = timer.elapsed_ms();
            rec.rows.push_back(row);
            if (cfg.time_budget_s > 0.0 && row.elapsed_ms >= cfg.time_budget_s * 1e3) break;
        }
        uint64_t counter = 0, tt = 0, r = 0, d = 0, m = 0;
        detail::check(temo_b200_run_state(run, &rows, &counter, &tt, &r, &d, &m));
        detail::check(temo_b200_run_download(run, x.data.data(), f.data.data(), nullptr, nullptr));
        if (cfg.track_archive) fetch_archive(&rec.archive.x, rec.archive.f);
    }
    rec.final_x = Tensor2D(rows, prob.dim);
    rec.final_f = Tensor2D(rows, prob.num_obj);
    std::copy_n(x.data.begin(), rows * prob.dim, rec.final_x.data.begin());
    std::copy_n(f.data.begin(), rows * prob.num_obj, rec.final_f.data.begin());
    return rec;
}

// ---- metrics.hpp / Archive / NSGA-II baseline -----------------------------
/// igd (metrics.hpp:21-44).
inline double igd(const Tensor2D& f, const Tensor2D& f_ref) {
    temo::detail::require(f.rows >= 1 && f_ref.rows >= 1, "igd: empty set");
    temo::detail::require(f.cols == f_ref.cols, "igd: objective count mismatch");
    double out = 0.0;
    detail::check(temo_b200_igd(f.data.data(), f.rows, f.cols, f_ref.data.data(), f_ref.rows, &out));
    return out;
}

/// hv_mc_box (metrics.hpp:76-117).
inline HvEstimate hv_mc_box(const Tensor2D& f, const Tensor2D& lo, const Tensor2D& ref, std::size_t samples, std::uint64_t seed) {
    temo::detail::require(samples >= 1, "hv_mc: needs at least one sample");
    temo::detail::require(f.rows >= 1 && ref.rows == 1 && ref.cols == f.cols, "hv_mc: bad shapes");
    temo::detail::require(lo.rows == 1 && lo.cols == f.cols, "hv_mc: bad box");
    HvEstimate e;
    detail::check(temo_b200_hv_mc_box(f.data.data(), f.rows, f.cols, lo.data.data(), ref.data.data(), samples, seed, &e.value,
                                      &e.std_error));
    return e;
}

/// hv_mc (metrics.hpp:121-124).
inline HvEstimate hv_mc(const Tensor2D& f, const Tensor2D& ref, std::size_t samples, std::uint64_t seed) {
    temo::detail::require(samples >= 1, "hv_mc: needs at least one sample");
    temo::detail::require(f.rows >= 1 && ref.rows == 1 && ref.cols == f.cols, "hv_mc: bad shapes");
    HvEstimate e;
    detail::check(temo_b200_hv_mc(f.data.data(), f.rows, f.cols, ref.data.data(), samples, seed, &e.value, &e.std_error));
    return e;
}

/// Archive::insert (algorithms.hpp:72-122) as a free function on the reference's Archive.
inline void archive_insert(Archive& a, const Tensor2D& xn, const Tensor2D& fn, std::size_t cap = 0) {
    const std::size_t n_old = a.f.rows, n_new = fn.rows, total = n_old + n_new;
    Tensor2D nx(total, xn.cols), nf(total, fn.cols);
    uint64_t rows = 0;
    detail::check(temo_b200_archive_insert(a.x.data.data(), a.f.data.data(), n_old, xn.data.data(), fn.data.data(), n_new, xn.cols,
                                           fn.cols, cap, nx.data.data(), nf.data.data(), &rows));
    a.x = Tensor2D(rows, xn.cols);
    a.f = Tensor2D(rows, fn.cols);
    std::copy_n(nx.data.begin(), rows * xn.cols, a.x.data.begin());
    std::copy_n(nf.data.begin(), rows * fn.cols, a.f.data.begin());
}

/// nondominated_sort (selection.hpp:251-283).
inline std::vector<std::size_t> nondominated_sort(const Tensor2D& f) {
    std::vector<uint64_t> r(f.rows);
    detail::check(temo_b200_nondominated_sort(f.data.data(), f.rows, f.cols, r.data()));
    return std::vector<std::size_t>(r.begin(), r.end());
}

/// nsga2_select (selection.hpp:316-346).
inline std::vector<std::size_t> nsga2_select(const Tensor2D& f, std::size_t target) {
    temo::detail::require(target <= f.rows, "nsga2_select: target exceeds population");
    std::vector<uint64_t> s(target);
    detail::check(temo_b200_nsga2_select(f.data.data(), f.rows, f.cols, target, s.data()));
    return std::vector<std::size_t>(s.begin(), s.end());
}

/// nsga2_run (algorithms.hpp:301-369) with track_archive = false, device-resident for the whole run.
inline RunRecord nsga2_run(const ProblemInstance& prob, const RunConfig& cfg) {
    temo::detail::require(cfg.pop >= 2 && cfg.generations >= 1, "nsga2_run: bad config");
    temo_b200_run_config c;
    temo_b200_default_run_config(&c);
    c.problem = detail::problem_id(prob);
    c.pop = cfg.pop;
    c.generations = cfg.generations;
    c.seed = cfg.seed;
    c.dim = prob.dim;
    c.obj = prob.num_obj;
    c.time_budget_s = cfg.time_budget_s;
    c.ga = detail::ga_of(cfg.ga);
    RunRecord rec;
    rec.final_x = Tensor2D(cfg.pop, prob.dim);
    rec.final_f = Tensor2D(cfg.pop, prob.num_obj);
    std::vector<double> ms(cfg.generations);
    uint64_t done = 0;
    detail::check(temo_b200_nsga2_run(&c, rec.final_x.data.data(), rec.final_f.data.data(), &done, ms.data()));
    for (uint64_t t = 0; t < done; ++t) {
        GenerationRow row;
        row.t = t;
        row.elapsed_ms = ms[t];
        row.pop_size = cfg.pop;
        rec.rows.push_back(row);
    }
    return rec;
}

}  // namespace temo::b200
