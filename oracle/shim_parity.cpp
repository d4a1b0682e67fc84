// TEST INFRASTRUCTURE — the reference's own equivalence suites with the GPU path swapped in.
//
// Compiled (oracle/Makefile, only where /root/reference is mounted) against the UNMODIFIED reference
// headers and include/temo_b200.hpp into oracle/_ref/shim_parity; linked to libtemo_b200.so. Each suite
// re-hosts the instance generator of the reference's verify.hpp (same master seeds, same draw order) and
// replaces the batched CPU call by its temo::b200:: twin, comparing against the reference's scalar oracle
// (temo::oracle::*) exactly like the reference does:
//   rv_select_suite   verify.hpp:53-76   200 instances, seed 7001: elite indices + validity identical, APD 1e-9
//   operator_suite    verify.hpp:117-182 100 x {sbx, pm, de, pso, cso}, seed 7002 + op*1000003 + k: here bit-identical
//   ga pipeline       test_operators.cpp:104-114
//   whole run         test_algorithms.cpp:198-210 (seed 77) and BASELINE config #1
// Exit code = number of failed suites.
#include <cstdio>
#include <cstring>

#include "temo/verify.hpp"
#include "temo_b200.hpp"

using namespace temo;

static bool same_bits(const Tensor2D& a, const Tensor2D& b) {
    return a.same_shape(b) && std::memcmp(a.data.data(), b.data.data(), a.size() * sizeof(double)) == 0;
}

static int rv_select_suite_gpu() {
    int failed = 0;
    for (std::size_t k = 0; k < 200; ++k) {
        RngStream g{7001 + k, 0};
        const std::size_t n = verify::detail::pick(g, 1, 64);
        const std::size_t m = verify::detail::pick(g, 2, 3);
        const std::size_t h = m == 2 ? verify::detail::pick(g, 1, 14) : verify::detail::pick(g, 1, 4);
        const std::size_t t_max = verify::detail::pick(g, 1, 200);
        const std::size_t t = verify::detail::pick(g, 0, t_max);
        const RefVectorSet refs = make_ref_set(m, h);
        Tensor2D f = uniform_tensor(g, n, m);
        for (double& v : f.data) v *= 10.0;
        const SelectionOutcome a = b200::rv_select(f, refs, t, t_max, 2.0, true);
        const SelectionOutcome b = oracle::oracle_rv_select(f, refs, t, t_max, 2.0);
        bool ok = a.elite_indices == b.elite_indices && a.validity == b.validity;
        for (std::size_t i = 0; ok && i < a.apd_table.size(); ++i)
            ok = verify::detail::close(a.apd_table.data[i], b.apd_table.data[i], 1e-9);
        failed += !ok;
    }
    std::printf("rv_select_suite (gpu vs oracle_rv_select): %d/200 failed\n", failed);
    return failed;
}

static int operator_suite_gpu() {
    int failed = 0;
    for (std::size_t op = 0; op < 2; ++op) {
        for (std::size_t k = 0; k < 100; ++k) {
            const std::uint64_t seed = 7002 + op * 1000003 + k;
            RngStream g{seed, 0};
            auto inst = verify::detail::random_operator_instance(g, 2, 16, 8);
            RngStream sa{seed ^ 0x5eed, 0}, sb{seed ^ 0x5eed, 0};
            const GaParams p;
            Tensor2D got, exp;
            if (op == 0) {
                got = b200::sbx(inst.x, sa, p, inst.lower, inst.upper);
                exp = oracle::to_tensor(oracle::oracle_sbx(oracle::to_matrix(inst.x), sb, p, inst.lower.data, inst.upper.data));
            } else {
                got = b200::polynomial_mutation(inst.x, sa, p, inst.lower, inst.upper);
                exp = oracle::to_tensor(oracle::oracle_pm(oracle::to_matrix(inst.x), sb, p, inst.lower.data, inst.upper.data));
            }
            failed += !(same_bits(got, exp) && sa.counter == sb.counter);
        }
    }
    std::printf("operator_suite (gpu sbx/pm vs oracle, bit-exact): %d/200 failed\n", failed);
    return failed;
}

// verify.hpp:117-182, ops 2..4: DE / PSO / CSO through the shim against the reference's scalar oracles, bit-exact
static int swarm_suite_gpu() {
    int failed = 0;
    for (std::size_t op = 2; op < 5; ++op) {
        for (std::size_t k = 0; k < 100; ++k) {
            const std::uint64_t seed = 7002 + op * 1000003 + k;
            RngStream g{seed, 0};
            auto inst = verify::detail::random_operator_instance(g, op == 2 ? 4 : 2, 16, 8);
            const oracle::Matrix xm = oracle::to_matrix(inst.x);
            const oracle::Row lo = oracle::to_matrix(inst.lower)[0], hi = oracle::to_matrix(inst.upper)[0];
            RngStream sa{seed ^ 0xabcdef, 0}, sb{seed ^ 0xabcdef, 0};
            bool ok = true;
            if (op == 2) {
                const DeParams p;
                ok = same_bits(b200::de_reproduce(inst.x, sa, p, inst.lower, inst.upper), oracle::to_tensor(oracle::oracle_de(xm, sb, p, lo, hi)));
            } else if (op == 3) {
                const PsoParams p;
                SwarmState st_a = make_swarm_state(inst.x, inst.scores);
                for (double& v : st_a.personal_best_x.data) v *= 0.5;
                for (double& v : st_a.personal_best_score.data) v += 0.25;
                SwarmState st_b = st_a;
                const Tensor2D got = b200::pso_reproduce(inst.x, st_a, inst.scores, sa, p, inst.lower, inst.upper);
                const Tensor2D exp = oracle::to_tensor(oracle::oracle_pso(xm, st_b, inst.scores.data, sb, p, lo, hi));
                ok = same_bits(got, exp) && same_bits(st_a.velocities, st_b.velocities) && same_bits(st_a.personal_best_x, st_b.personal_best_x);
            } else {
                const CsoParams p;
                SwarmState st_a = make_swarm_state(inst.x, inst.scores), st_b = st_a;
                const Tensor2D got = b200::cso_reproduce(inst.x, inst.scores, sa, p, inst.lower, inst.upper, st_a);
                const Tensor2D exp = oracle::to_tensor(oracle::oracle_cso(xm, inst.scores.data, sb, p, lo, hi, st_b));
                ok = same_bits(got, exp) && same_bits(st_a.velocities, st_b.velocities);
            }
            failed += !(ok && sa.counter == sb.counter);
        }
    }
    std::printf("operator_suite (gpu de/pso/cso vs oracle, bit-exact): %d/300 failed\n", failed);
    return failed;
}

static int ga_pipeline_gpu() {
    int failed = 0;
    for (std::uint64_t seed = 43; seed < 63; ++seed) {
        RngStream g{seed, 0};
        auto inst = verify::detail::random_operator_instance(g, 2, 40, 30);
        RngStream sa{seed + 1, 7}, sb{seed + 1, 7};
        const GaParams p;
        const Tensor2D got = b200::ga_reproduce(inst.x, sa, p, inst.lower, inst.upper);
        const Tensor2D exp = ga_reproduce(inst.x, sb, p, inst.lower, inst.upper);
        failed += !(same_bits(got, exp) && sa.counter == sb.counter);
    }
    std::printf("ga_reproduce (gpu vs temo::ga_reproduce, bit-exact): %d/20 failed\n", failed);
    return failed;
}

static int whole_run_gpu() {
    int failed = 0;
    struct Case { const char* problem; std::size_t dim, obj, pop, h, gens; std::uint64_t seed; };
    const Case cases[] = {{"dtlz2", 8, 3, 12, 3, 10, 77}, {"dtlz1", 12, 3, 105, 13, 100, 42}};
    for (const Case& c : cases) {
        RunConfig cfg;
        cfg.problem = c.problem;
        cfg.pop = c.pop;
        cfg.lattice_h = c.h;
        cfg.generations = c.gens;
        cfg.seed = c.seed;
        cfg.track_archive = false;
        const ProblemInstance prob = make_problem(c.problem, c.dim, c.obj);
        const RunRecord a = b200::rvea_run(prob, cfg);
        const RunRecord b = oracle::oracle_rvea_run(prob, cfg);
        bool ok = a.rows.size() == b.rows.size();
        std::size_t same_pop = 0;
        for (std::size_t t = 0; ok && t < a.rows.size(); ++t) same_pop += a.rows[t].pop_size == b.rows[t].pop_size;
        const bool x_same = same_bits(a.final_x, b.final_x);
        std::size_t rows_same = 0;
        if (a.final_x.same_shape(b.final_x))
            for (std::size_t i = 0; i < a.final_x.rows; ++i)
                rows_same += std::memcmp(a.final_x.row(i).data(), b.final_x.row(i).data(), a.final_x.cols * sizeof(double)) == 0;
        bool f_close = a.final_f.same_shape(b.final_f);
        for (std::size_t i = 0; f_close && i < a.final_f.size(); ++i)
            f_close = verify::detail::close(a.final_f.data[i], b.final_f.data[i], 1e-9 * std::max(1.0, std::abs(b.final_f.data[i])));
        std::printf("rvea_run %s pop=%zu gens=%zu seed=%llu: survivor counts equal in %zu/%zu generations, final x %s "
                    "(%zu/%zu rows bit-identical), final f %s\n",
                    c.problem, c.pop, c.gens, (unsigned long long)c.seed, same_pop, a.rows.size(),
                    x_same ? "bit-identical" : "differs", rows_same, a.final_x.rows, f_close ? "within 1e-9" : "differs");
        // free-running: objectives carry the device evaluator's ulps, so an ulp-level copy of a parent may win or
        // lose its tie differently; the trajectory itself must still agree
        failed += !(ok && same_pop == a.rows.size() && f_close && rows_same * 2 >= a.final_x.rows);
    }
    return failed;
}

// metrics.hpp, Archive::insert and the NSGA-II selection pieces with the GPU path swapped in: all bit-identical
// (integer ranks / indices / hit counts; minima of exactly reproduced distances).
static int widened_suite_gpu() {
    int failed = 0;
    for (std::uint64_t k = 0; k < 40; ++k) {
        RngStream g{9000 + k, 0};
        const std::size_t n = verify::detail::pick(g, 1, 90), m = verify::detail::pick(g, 2, 6), n_ref = verify::detail::pick(g, 1, 40);
        const double q = static_cast<double>(verify::detail::pick(g, 2, 12));
        Tensor2D f = uniform_tensor(g, n, m), pf = uniform_tensor(g, n_ref, m), x = uniform_tensor(g, n, 3);
        for (double& v : f.data) v = std::floor(v * q) / q;  // coarse grid: duplicates and domination chains
        Tensor2D ref_pt(1, m, 1.25), lo(1, m, 0.0);
        bool ok = b200::igd(f, pf) == igd(f, pf);
        const HvEstimate a = b200::hv_mc(f, ref_pt, 700 + k, 5 + k), b = hv_mc(f, ref_pt, 700 + k, 5 + k);
        ok = ok && a.value == b.value && a.std_error == b.std_error;
        const HvEstimate c = b200::hv_mc_box(f, lo, ref_pt, 300, k), d = hv_mc_box(f, lo, ref_pt, 300, k);
        ok = ok && c.value == d.value && c.std_error == d.std_error;
        ok = ok && b200::nondominated_sort(f) == nondominated_sort(f);
        ok = ok && b200::nsga2_select(f, n / 2) == nsga2_select(f, n / 2);
        Archive ga, ca;
        const std::size_t half = n / 2;
        if (half) {
            Tensor2D x0(half, 3), f0(half, m);
            std::copy_n(x.data.begin(), half * 3, x0.data.begin());
            std::copy_n(f.data.begin(), half * m, f0.data.begin());
            b200::archive_insert(ga, x0, f0);
            ca.insert(x0, f0);
        }
        b200::archive_insert(ga, x, f, 7);
        ca.insert(x, f, 7);
        ok = ok && same_bits(ga.x, ca.x) && same_bits(ga.f, ca.f);
        failed += !ok;
    }
    std::printf("metrics / archive / nondominated_sort / nsga2_select (gpu vs reference, bit-exact): %d/40 failed\n", failed);
    return failed;
}

// rvea_run with RunConfig::op = de / pso / cso / random through the shim against the reference's own rvea_run
// (free-running: exact while the survivor counts agree).
static int operator_runs_gpu() {
    int failed = 0;
    for (const char* op : {"de", "pso", "cso", "random"}) {
        RunConfig cfg;
        cfg.problem = "dtlz2";
        cfg.op = op;
        cfg.pop = 40;
        cfg.generations = 12;
        cfg.seed = 3;
        cfg.track_archive = false;
        const ProblemInstance prob = make_problem("dtlz2", 9, 3);
        const RunRecord a = b200::rvea_run(prob, cfg), b = rvea_run(prob, cfg);
        std::size_t agree = 0;
        while (agree < a.rows.size() && agree < b.rows.size() && a.rows[agree].pop_size == b.rows[agree].pop_size) ++agree;
        const bool x_same = same_bits(a.final_x, b.final_x);
        std::printf("rvea_run op=%s: survivor counts equal in the first %zu/%zu generations, final x %s\n", op, agree, b.rows.size(),
                    x_same ? "bit-identical" : "differs");
        failed += !(a.rows.size() == b.rows.size() && agree >= 3);
    }
    bool threw = false;
    try {
        RunConfig cfg;
        cfg.op = "sa";
        (void)b200::rvea_run(make_problem("dtlz2", 9, 3), cfg);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    failed += !threw;
    return failed;
}

// The reference's convergence set-up (tests/acceptance.cpp:66-98) through the shim with the default track_archive = true:
// RunRecord.archive filled from the device-resident archive, archive IGD per generation, against the reference's own run.
static int archive_run_gpu() {
    RunConfig cfg;
    cfg.problem = "dtlz2";
    cfg.pop = 105;
    cfg.lattice_h = 13;
    cfg.generations = 200;
    cfg.seed = 4242;
    cfg.archive_history = true;
    const ProblemInstance prob = make_problem("dtlz2");
    MetricContext mc;
    std::size_t h = 1;
    while (lattice_count(prob.num_obj, h) < 300) ++h;
    mc.pf_ref = dtlz_pf_reference(prob.dtlz_id, prob.num_obj, h);
    const RunRecord a = b200::rvea_run(prob, cfg, mc);
    const RunRecord b = rvea_run(prob, cfg, mc);
    const double ia = a.rows.back().igd_value, ib = b.rows.back().igd_value;
    bool ok = a.rows.size() == b.rows.size() && a.archive.f.rows >= cfg.pop && a.archive.x.rows == a.archive.f.rows &&
              a.archive_f_history.size() == a.rows.size() && same_bits(a.archive_f_history.back(), a.archive.f);
    ok = ok && ia == igd(a.archive.f, mc.pf_ref);           // the device's IGD is the reference's arithmetic
    ok = ok && std::abs(ia - ib) <= 0.05 * ib && ia <= 1.1 * 0.037367406771666209;
    std::printf("rvea_run track_archive (dtlz2, 200 generations, seed 4242): archive %zu rows (reference %zu), final archive IGD %.17g "
                "(reference %.17g, pinned 0.037367406771666209)\n", a.archive.f.rows, b.archive.f.rows, ia, ib);
    return ok ? 0 : 1;
}

// MLP policy + toy environment through the shim: env_rollout, mlp_forward and make_problem("toy2" / "toy3").evaluate
// bit-identical to the reference's, a whole rvea_run on toy3 identical to the reference's run.
static int toyenv_gpu() {
    int failed = 0;
    RngStream g{9400, 0};
    const MlpArch arch{toy_obs_dim, 16, toy_act_dim};
    Tensor2D p = uniform_tensor(g, 300, arch.param_count());
    for (double& v : p.data) v = 2.0 * v - 1.0;
    p(5, 7) = std::numeric_limits<double>::quiet_NaN();
    for (const std::size_t m : {std::size_t{2}, std::size_t{3}}) {
        const ToyEnvSpec spec{m == 2 ? std::size_t{100} : std::size_t{41}, m};
        failed += !same_bits(b200::env_rollout(p, spec, arch), env_rollout(p, spec, arch));
    }
    Tensor2D obs = uniform_tensor(g, 300, toy_obs_dim), act(300, toy_act_dim);
    p(5, 7) = 0.25;
    for (std::size_t i = 0; i < 300; ++i) {
        const MlpWeights w = mlp_decode(p.row(i), arch);
        mlp_forward(w, obs.row(i), act.row(i));
    }
    failed += !same_bits(b200::mlp_forward(p, arch, obs), act);
    const ProblemInstance a = b200::make_problem("toy2", 0, 3, 60), b = make_problem("toy2", 0, 3, 60);
    failed += !same_bits(a.evaluate(p), b.evaluate(p));
    RunConfig cfg;
    cfg.problem = "toy3";
    cfg.pop = 66;
    cfg.generations = 10;
    cfg.seed = 8;
    cfg.track_archive = false;
    const ProblemInstance prob = make_problem("toy3");
    const RunRecord ra = b200::rvea_run(prob, cfg), rb = rvea_run(prob, cfg);
    failed += !(same_bits(ra.final_x, rb.final_x) && same_bits(ra.final_f, rb.final_f));
    std::printf("toy environment (env_rollout, mlp_forward, make_problem, rvea_run on toy3; bit-exact): %d/6 failed\n", failed);
    return failed;
}

int main() {
    if (temo_b200_device_count() < 1) {
        std::printf("no CUDA device\n");
        return 99;
    }
    int failed = 0;
    failed += rv_select_suite_gpu() != 0;
    failed += operator_suite_gpu() != 0;
    failed += swarm_suite_gpu() != 0;
    failed += ga_pipeline_gpu() != 0;
    failed += whole_run_gpu() != 0;
    failed += widened_suite_gpu() != 0;
    failed += operator_runs_gpu() != 0;
    failed += archive_run_gpu() != 0;
    failed += toyenv_gpu() != 0;
    std::printf("%s\n", failed ? "SHIM PARITY FAILED" : "SHIM PARITY OK");
    return failed;
}
