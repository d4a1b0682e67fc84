// C ABI of libtemo_b200.so — see include/temo_b200.h for the contract and the reference
// interface each entry point replaces. No torch types, no C++ types cross this boundary.
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "../../include/temo_b200.h"
#include "glibc_pow.cuh"
#include <algorithm>
#include "internal.h"
#include "nsga2.h"
#include "run.h"
#include "vecindex.h"

using namespace temo_b200;

namespace {

thread_local std::string g_error;

template <class F>
int guarded(F&& body) {
    try {
        body();
        return TEMO_B200_OK;
    } catch (const Error& e) {
        g_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_error = "host allocation failed";
        return TEMO_B200_ENOMEM;
    } catch (const std::exception& e) {
        g_error = e.what();
        return TEMO_B200_ERUNTIME;
    }
}

// RAII device buffer for the host-pointer drop-ins.
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t count = 0;
    explicit DevBuf(size_t n) : p(dev_alloc<T>(n)), count(n) {}
    DevBuf(const T* host, size_t n, cudaStream_t s) : DevBuf(n) {
        if (n) TEMO_CUDA(cudaMemcpyAsync(p, host, n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    ~DevBuf() { cudaFree(p); }
    void to_host(T* host, cudaStream_t s, size_t n = (size_t)-1) const {
        if (n == (size_t)-1) n = count;
        if (n) TEMO_CUDA(cudaMemcpyAsync(host, p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

GaParams ga_of(const temo_b200_ga_params* g) {
    GaParams p;
    if (g) {
        p.pc = g->pc;
        p.eta = g->eta;
        p.pm = g->pm;
        p.xi = g->xi;
    }
    return p;
}

RunConfig cfg_of(const temo_b200_run_config* c) {
    require(c != nullptr, "run config is null");
    RunConfig r;
    r.problem = c->problem;
    r.rng_mode = c->rng_mode;
    r.pop = c->pop;
    r.lattice_h = c->lattice_h;
    r.generations = c->generations;
    r.seed = c->seed;
    r.dim = c->dim;
    r.obj = c->obj;
    r.alpha = c->alpha;
    r.fr = c->fr;
    r.time_budget_s = c->time_budget_s;
    r.ga = ga_of(&c->ga);
    r.fuse_eval = c->fuse_eval;
    r.op = c->op;
    r.de_f = c->opp.de_f;
    r.de_cr = c->opp.de_cr;
    r.pso_inertia = c->opp.pso_inertia;
    r.pso_c1 = c->opp.pso_c1;
    r.pso_c2 = c->opp.pso_c2;
    r.cso_phi = c->opp.cso_phi;
    r.horizon = c->horizon ? c->horizon : 100;
    require(r.rng_mode == 0 || r.rng_mode == 1, "unknown rng mode");
    return r;
}

// below this many reference vectors the exhaustive scan is cheaper than building the index
constexpr uint64_t kIndexMinVectors = 1024;

void check_mode(int rng_mode) { require(rng_mode == 0 || rng_mode == 1, "unknown rng mode"); }

// Shared body of sbx / polynomial_mutation / ga_reproduce on host buffers.
void host_operator(bool do_shuffle, bool do_sbx, bool do_pm, const double* x, uint64_t n, uint64_t d,
                   uint64_t seed, uint64_t* counter, const temo_b200_ga_params* ga, const double* lower,
                   const double* upper, int rng_mode, double* out) {
    require(x && counter && lower && upper && out, "operator: null argument");
    require(n >= 1 && d >= 1, "operator: empty population");
    if (do_sbx) require(n >= 2, "sbx: needs at least two rows");
    check_mode(rng_mode);
    Context& cx = ctx();
    cudaStream_t s = cx.stream;
    DevBuf<double> dx(x, n * d, s), dlo(lower, d, s), dhi(upper, d, s), dout(n * d);
    uint64_t c = *counter;
    std::unique_ptr<DevBuf<uint32_t>> dperm;
    std::vector<uint32_t> perm;
    if (do_shuffle) {
        perm.resize(n);
        shuffle_indices(seed, c, n, perm.data());
        dperm.reset(new DevBuf<uint32_t>(perm.data(), n, s));
    }
    ReproArgs a;
    a.pool = dx.p;
    a.src = dperm ? dperm->p : nullptr;
    a.out = dout.p;
    a.n = n;
    a.d = d;
    a.rng = make_rng(seed, rng_mode);
    a.ga = ga_of(ga);
    a.lower = dlo.p;
    a.upper = dhi.p;
    a.seg = find_bound_segments(lower, upper, d);
    a.do_sbx = do_sbx;
    a.do_pm = do_pm;
    if (do_sbx) {
        a.c_sbx = c;
        c += 3 * (n / 2) * d + n / 2;
    }
    if (do_pm) {
        a.c_pm = c;
        c += 2 * n * d;
    }
    launch_reproduce(a, s);
    dout.to_host(out, s);
    TEMO_CUDA(cudaStreamSynchronize(s));
    *counter = c;
}

}  // namespace

extern "C" {

const char* temo_b200_last_error(void) { return g_error.c_str(); }
const char* temo_b200_version(void) { return "temo_b200 0.1 (sm_100a)"; }

int temo_b200_device_count(void) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return count;
}

int temo_b200_init(int device) {
    return guarded([&] { init_context(device); });
}

void temo_b200_default_ga_params(temo_b200_ga_params* ga) {
    if (!ga) return;
    ga->pc = 1.0;
    ga->eta = 20.0;
    ga->pm = 1.0;
    ga->xi = 20.0;
}

void temo_b200_default_run_config(temo_b200_run_config* cfg) {
    if (!cfg) return;
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->problem = TEMO_B200_DTLZ2;
    cfg->rng_mode = TEMO_B200_RNG_SPLITMIX64;
    cfg->pop = 105;
    cfg->lattice_h = 0;
    cfg->generations = 100;
    cfg->seed = 42;
    cfg->dim = 0;
    cfg->obj = 3;
    cfg->alpha = 2.0;
    cfg->fr = 0.1;
    cfg->time_budget_s = 0.0;
    temo_b200_default_ga_params(&cfg->ga);
    cfg->fuse_eval = 2;
    cfg->op = TEMO_B200_OP_GA;
    cfg->opp.de_f = 0.5;  // operators.hpp:28-41
    cfg->opp.de_cr = 0.9;
    cfg->opp.pso_inertia = 0.4;
    cfg->opp.pso_c1 = 1.5;
    cfg->opp.pso_c2 = 1.5;
    cfg->opp.cso_phi = 0.1;
    cfg->horizon = 100;  // algorithms.hpp:35
}

// ---- rng.hpp ------------------------------------------------------------------------------
int temo_b200_uniform_tensor(uint64_t seed, uint64_t* counter, uint64_t rows, uint64_t cols, int rng_mode,
                             double* out) {
    return guarded([&] {
        require(counter && out, "uniform_tensor: null argument");
        require(rows >= 1 && cols >= 1, "uniform_tensor: empty shape");  // rng.hpp:56
        check_mode(rng_mode);
        Context& cx = ctx();
        DevBuf<double> d(rows * cols);
        launch_uniform_fill(d.p, rows * cols, make_rng(seed, rng_mode), *counter, cx.stream);
        d.to_host(out, cx.stream);
        TEMO_CUDA(cudaStreamSynchronize(cx.stream));
        *counter += rows * cols;
    });
}

int temo_b200_shuffle_indices(uint64_t seed, uint64_t* counter, uint64_t n, uint64_t* perm) {
    return guarded([&] {
        require(counter && perm, "shuffle_indices: null argument");
        require(n >= 1 && n < 0xffffffffULL, "shuffle_indices: n must be positive");
        std::vector<uint32_t> p(n);
        shuffle_indices(seed, *counter, n, p.data());
        for (uint64_t i = 0; i < n; ++i) perm[i] = p[i];
    });
}

int temo_b200_parent_pool_indices(uint64_t current, uint64_t n, uint64_t seed, uint64_t* counter,
                                  uint64_t* idx) {
    return guarded([&] {
        require(counter && idx, "parent_pool_indices: null argument");
        if (current == n) {  // algorithms.hpp:214-217: no draws
            for (uint64_t i = 0; i < n; ++i) idx[i] = i;
            return;
        }
        const uint64_t base = mix64(seed);
        for (uint64_t i = 0; i < n; ++i) {
            const double u = (double)(mix64(base + (*counter + i) * kGolden) >> 11) * 0x1.0p-53;
            idx[i] = (uint64_t)(u * (double)current);
        }
        *counter += n;
    });
}

// ---- operators.hpp --------------------------------------------------------------------------
int temo_b200_sbx(const double* x, uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter,
                  const temo_b200_ga_params* ga, const double* lower, const double* upper, int rng_mode,
                  double* out) {
    return guarded([&] { host_operator(false, true, false, x, n, d, seed, counter, ga, lower, upper, rng_mode, out); });
}

int temo_b200_polynomial_mutation(const double* x, uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter,
                                  const temo_b200_ga_params* ga, const double* lower, const double* upper,
                                  int rng_mode, double* out) {
    return guarded([&] { host_operator(false, false, true, x, n, d, seed, counter, ga, lower, upper, rng_mode, out); });
}

int temo_b200_ga_reproduce(const double* x, uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter,
                           const temo_b200_ga_params* ga, const double* lower, const double* upper,
                           int rng_mode, double* out) {
    return guarded([&] { host_operator(true, true, true, x, n, d, seed, counter, ga, lower, upper, rng_mode, out); });
}

// ---- operators.hpp:166-284: DE / PSO / CSO on host buffers -----------------------
namespace {
struct KernelTimer {  // device time of the kernels of one call (CUDA events on the library stream)
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaStream_t s;
    double* out;
    KernelTimer(cudaStream_t st, double* o) : s(st), out(o) {
        if (out) {
            TEMO_CUDA(cudaEventCreate(&e0));
            TEMO_CUDA(cudaEventCreate(&e1));
            TEMO_CUDA(cudaEventRecord(e0, s));
        }
    }
    void stop() {
        if (out) TEMO_CUDA(cudaEventRecord(e1, s));
    }
    void read() {
        if (!out) return;
        float ms = 0.f;
        TEMO_CUDA(cudaEventSynchronize(e1));
        TEMO_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        *out = ms;
    }
    ~KernelTimer() {
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    }
};
}  // namespace

int temo_b200_de_reproduce(const double* x, uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter, double f, double cr,
                           const double* lower, const double* upper, int rng_mode, double* out, double* kernel_ms) {
    return guarded([&] {
        require(x && counter && lower && upper && out, "de_reproduce: null argument");
        require(n >= 4, "de_reproduce: needs at least four rows");  // operators.hpp:169
        require(d >= 1, "de_reproduce: empty rows");
        check_mode(rng_mode);
        cudaStream_t s = ctx().stream;
        DevBuf<double> dx(x, n * d, s), dlo(lower, d, s), dhi(upper, d, s), dout(n * d);
        KernelTimer tm(s, kernel_ms);
        launch_de(dx.p, n, d, make_rng(seed, rng_mode), *counter, f, cr, dlo.p, dhi.p, dout.p, s);
        tm.stop();
        dout.to_host(out, s);
        TEMO_CUDA(cudaStreamSynchronize(s));
        tm.read();
        *counter += 4 * n + n * d;  // r_sel n x 3, r_j n x 1, r_cr n x d
    });
}

int temo_b200_pso_reproduce(const double* x, const double* scores, uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter,
                            double inertia, double c1, double c2, double* velocities, double* pbest_x, double* pbest_score,
                            const double* lower, const double* upper, int rng_mode, double* out, double* kernel_ms) {
    return guarded([&] {
        require(x && scores && counter && velocities && pbest_x && pbest_score && lower && upper && out, "pso_reproduce: null argument");
        require(n >= 1 && d >= 1, "pso_reproduce: state shape mismatch");  // operators.hpp:209-211 (shapes are the caller's)
        check_mode(rng_mode);
        cudaStream_t s = ctx().stream;
        DevBuf<double> dx(x, n * d, s), dsc(scores, n, s), dv(velocities, n * d, s), dpx(pbest_x, n * d, s), dps(pbest_score, n, s),
            dlo(lower, d, s), dhi(upper, d, s), dout(n * d);
        DevBuf<uint32_t> best(1);
        KernelTimer tm(s, kernel_ms);
        launch_pso(dx.p, dsc.p, n, d, make_rng(seed, rng_mode), *counter, inertia, c1, c2, dv.p, dpx.p, dps.p, best.p, dlo.p, dhi.p,
                   dout.p, s);
        tm.stop();
        dout.to_host(out, s);
        dv.to_host(velocities, s);
        dpx.to_host(pbest_x, s);
        dps.to_host(pbest_score, s);
        TEMO_CUDA(cudaStreamSynchronize(s));
        tm.read();
        *counter += 2 * n * d;
    });
}

int temo_b200_cso_reproduce(const double* x, const double* scores, uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter, double phi,
                            double* velocities, const double* lower, const double* upper, int rng_mode, double* out,
                            double* kernel_ms) {
    return guarded([&] {
        require(x && scores && counter && velocities && lower && upper && out, "cso_reproduce: null argument");
        require(n >= 1 && n < 0xffffffffULL && d >= 1, "cso_reproduce: state shape mismatch");  // operators.hpp:251-253
        check_mode(rng_mode);
        cudaStream_t s = ctx().stream;
        uint64_t c = *counter;
        std::vector<uint32_t> perm(n);
        shuffle_indices(seed, c, n, perm.data());  // n - 1 draws (rng.hpp:69-78)
        DevBuf<double> dx(x, n * d, s), dsc(scores, n, s), dv(velocities, n * d, s), dlo(lower, d, s), dhi(upper, d, s), dout(n * d),
            dvo(n * d), dmean(d);
        DevBuf<uint32_t> dperm(perm.data(), n, s);
        KernelTimer tm(s, kernel_ms);
        launch_cso(dx.p, dsc.p, n, d, make_rng(seed, rng_mode), c, phi, dperm.p, dmean.p, dv.p, dvo.p, dlo.p, dhi.p, dout.p, s);
        tm.stop();
        dout.to_host(out, s);
        dvo.to_host(velocities, s);
        TEMO_CUDA(cudaStreamSynchronize(s));
        tm.read();
        *counter = c + 3 * (n / 2) * d;
    });
}

int temo_b200_random_reproduce(uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter, const double* lower,
                               const double* upper, int rng_mode, double* out) {
    return guarded([&] {
        require(counter && lower && upper && out, "random_reproduce: null argument");
        require(n >= 1 && d >= 1, "uniform_tensor: empty shape");
        check_mode(rng_mode);
        Context& cx = ctx();
        cudaStream_t s = cx.stream;
        DevBuf<double> dlo(lower, d, s), dhi(upper, d, s), dout(n * d);
        launch_random_reproduce(dout.p, nullptr, n, d, make_rng(seed, rng_mode), *counter, dlo.p, dhi.p, s);
        dout.to_host(out, s);
        TEMO_CUDA(cudaStreamSynchronize(s));
        *counter += n * d;
    });
}

// ---- problems.hpp -----------------------------------------------------------------------------
int temo_b200_evaluate(int problem, const double* x, uint64_t n, uint64_t d, uint64_t m, double* f) {
    return guarded([&] {
        require(x && f, "evaluate: null argument");
        Context& cx = ctx();
        cudaStream_t s = cx.stream;
        DevBuf<double> dx(x, n * d, s), df(n * m);
        EvalArgs a;
        a.problem = problem;
        a.x = dx.p;
        a.n = n;
        a.d = d;
        a.m = m;
        a.f = df.p;
        launch_evaluate(a, s);
        df.to_host(f, s);
        TEMO_CUDA(cudaStreamSynchronize(s));
    });
}

// env_rollout (problems.hpp:211-241): returns in maximisation orientation, -1e9 for non-finite parameter rows
int temo_b200_env_rollout(const double* params, uint64_t n, uint64_t d, uint64_t hidden, uint64_t horizon, uint64_t num_obj, double* f) {
    return guarded([&] {
        require(params && f, "env_rollout: null argument");
        cudaStream_t s = ctx().stream;
        DevBuf<double> dx(params, n * d, s), df(n * num_obj);
        launch_env_rollout(dx.p, nullptr, n, d, hidden, horizon, num_obj, /*negate=*/false, df.p, 0, nullptr, s);
        df.to_host(f, s);
        TEMO_CUDA(cudaStreamSynchronize(s));
    });
}

// mlp_forward (problems.hpp:149-163), batched: individual i acts on observation i (obs n x 4 -> action n x 2)
int temo_b200_mlp_forward(const double* params, uint64_t n, uint64_t d, uint64_t hidden, const double* obs, double* action) {
    return guarded([&] {
        require(params && obs && action, "mlp_forward: null argument");
        cudaStream_t s = ctx().stream;
        DevBuf<double> dx(params, n * d, s), dobs(obs, n * 4, s), dact(n * 2);
        launch_mlp_forward(dx.p, n, d, hidden, dobs.p, dact.p, s);
        dact.to_host(action, s);
        TEMO_CUDA(cudaStreamSynchronize(s));
    });
}

// problem evaluators with an episode length (toy2 / toy3; ignored by the others): make_problem(name, dim, m, horizon)
int temo_b200_evaluate_h(int problem, const double* x, uint64_t n, uint64_t d, uint64_t m, uint64_t horizon, double* f) {
    return guarded([&] {
        require(x && f, "evaluate: null argument");
        cudaStream_t s = ctx().stream;
        DevBuf<double> dx(x, n * d, s), df(n * m);
        EvalArgs a;
        a.problem = problem;
        a.x = dx.p;
        a.n = n;
        a.d = d;
        a.m = m;
        a.f = df.p;
        a.horizon = horizon;
        launch_evaluate(a, s);
        df.to_host(f, s);
        TEMO_CUDA(cudaStreamSynchronize(s));
    });
}

int temo_b200_problem_bounds(int problem, uint64_t d, uint64_t m, double* lower, double* upper) {
    return guarded([&] {
        require(lower && upper, "problem_bounds: null argument");
        problem_bounds(problem, d, m, lower, upper);
    });
}

uint64_t temo_b200_problem_default_dim(int problem, uint64_t m) { return problem_default_dim(problem, m); }

// ---- refvec.hpp ---------------------------------------------------------------------------------
uint64_t temo_b200_lattice_count(uint64_t m, uint64_t H) { return lattice_count(m, H); }
uint64_t temo_b200_lattice_density_for(uint64_t m, uint64_t target) { return lattice_density_for(m, target); }

int temo_b200_simplex_lattice(uint64_t m, uint64_t H, double* out) {
    return guarded([&] {
        require(out != nullptr, "simplex_lattice: null argument");
        const std::vector<double> lat = simplex_lattice(m, H);
        std::memcpy(out, lat.data(), lat.size() * sizeof(double));
    });
}

int temo_b200_min_vector_angles(const double* v, uint64_t r, uint64_t m, double* gamma) {
    return guarded([&] {
        require(v && gamma, "min_vector_angles: null argument");
        require(r >= 2, "min_vector_angles: needs at least two vectors");
        Context& cx = ctx();
        cudaStream_t s = cx.stream;
        DevBuf<double> dv(v, r * m, s), dvn(r), dg(r);
        DevBuf<uint32_t> err(1);
        TEMO_CUDA(cudaMemsetAsync(err.p, 0, sizeof(uint32_t), s));
        launch_row_norms(dv.p, r, m, dvn.p, s);
        if (assoc_filter_preferred(m, r)) {  // many objectives: the fp32-filtered exact scan (select.cu)
            SelectWorkspace ws;
            ws.alloc(r, r, m);
            struct Guard { SelectWorkspace& w; ~Guard() { w.release(); } } guard{ws};
            launch_row_norms(dv.p, r, m, ws.vn, s);
            launch_gamma_filter(dv.p, r, m, ws, dg.p, err.p, nullptr, s);
            TEMO_CUDA(cudaStreamSynchronize(s));
        } else if (r >= kIndexMinVectors) {
            VecIndex index;
            index.alloc(r, m);
            struct Guard { VecIndex& x; ~Guard() { x.release(); } } guard{index};
            index.set_order(v, s);
            index.build(dv.p, dvn.p, s);
            launch_gamma_indexed(dv.p, dvn.p, r, m, index, dg.p, err.p, nullptr, s);
            TEMO_CUDA(cudaStreamSynchronize(s));
        } else {
            launch_gamma(dv.p, dvn.p, r, m, dg.p, err.p, nullptr, s);
        }
        uint32_t flag = 0;
        err.to_host(&flag, s);
        dg.to_host(gamma, s);
        TEMO_CUDA(cudaStreamSynchronize(s));
        require(!(flag & 1u), "min_vector_angles: duplicate reference vectors");
    });
}

int temo_b200_make_ref_set(uint64_t m, uint64_t H, double* v0, double* gamma) {
    return guarded([&] {
        require(v0 && gamma, "make_ref_set: null argument");
        const uint64_t r = lattice_count(m, H);
        const std::vector<double> unit = normalize_to_unit(simplex_lattice(m, H), r, m);
        std::memcpy(v0, unit.data(), unit.size() * sizeof(double));
        const int rc = temo_b200_min_vector_angles(v0, r, m, gamma);
        if (rc) fail(rc, g_error);
    });
}

int temo_b200_adapt(const double* v0, double* v, double* gamma, uint64_t r, uint64_t m, const double* z_min,
                    const double* z_max) {
    return guarded([&] {
        require(v0 && v && gamma && z_min && z_max, "adapt: null argument");
        require(r >= 2, "min_vector_angles: needs at least two vectors");
        for (uint64_t k = 0; k < m; ++k)
            if (!(z_max[k] > z_min[k])) return;  // refvec.hpp:136-137: nothing changes
        Context& cx = ctx();
        cudaStream_t s = cx.stream;
        DevBuf<double> dv0(v0, r * m, s), dv(v, r * m, s), dvn(r), dg(r), dzmin(z_min, m, s), dzmax(z_max, m, s);
        DevBuf<uint32_t> flags(2);
        TEMO_CUDA(cudaMemsetAsync(flags.p, 0, 2 * sizeof(uint32_t), s));
        launch_adapt_vectors(dv0.p, dv.p, dvn.p, r, m, dzmin.p, dzmax.p, flags.p + 1, flags.p, s);
        if (assoc_filter_preferred(m, r)) {
            SelectWorkspace ws;
            ws.alloc(r, r, m);
            struct Guard { SelectWorkspace& w; ~Guard() { w.release(); } } guard{ws};
            TEMO_CUDA(cudaMemcpyAsync(ws.vn, dvn.p, r * sizeof(double), cudaMemcpyDeviceToDevice, s));
            launch_gamma_filter(dv.p, r, m, ws, dg.p, flags.p, flags.p + 1, s);
            TEMO_CUDA(cudaStreamSynchronize(s));
        } else if (r >= kIndexMinVectors) {
            VecIndex index;
            index.alloc(r, m);
            struct Guard { VecIndex& x; ~Guard() { x.release(); } } guard{index};
            index.set_order(v0, s);
            index.build(dv.p, dvn.p, s);
            launch_gamma_indexed(dv.p, dvn.p, r, m, index, dg.p, flags.p, flags.p + 1, s);
            TEMO_CUDA(cudaStreamSynchronize(s));
        } else {
            launch_gamma(dv.p, dvn.p, r, m, dg.p, flags.p, flags.p + 1, s);
        }
        uint32_t h[2] = {0, 0};
        flags.to_host(h, s);
        std::vector<double> nv(r * m), ng(r);
        dv.to_host(nv.data(), s);
        dg.to_host(ng.data(), s);
        TEMO_CUDA(cudaStreamSynchronize(s));
        require(!(h[0] & 2u), "normalize_to_unit: zero row");
        require(!(h[0] & 1u), "min_vector_angles: duplicate reference vectors");
        std::memcpy(v, nv.data(), nv.size() * sizeof(double));
        std::memcpy(gamma, ng.data(), ng.size() * sizeof(double));
    });
}

// ---- selection.hpp --------------------------------------------------------------------------------
double temo_b200_apd_penalty(uint64_t m, uint64_t t, uint64_t t_max, double alpha) {
    return apd_penalty(m, t, t_max, alpha);
}

int temo_b200_rv_select(const double* f, uint64_t n, uint64_t m, const double* v, const double* gamma, uint64_t r,
                        uint64_t t, uint64_t t_max, double alpha, uint64_t* elite, uint64_t* n_elite,
                        unsigned char* validity, uint64_t* assoc, double* theta, double* apd) {
    return guarded([&] {
        require(f && v && gamma && elite && n_elite && validity, "rv_select: null argument");
        require(t_max >= 1, "rv_select: t_max must be positive");  // selection.hpp:151
        require(n >= 1, "translate: empty objective tensor");
        require(r >= 1, "rv_select: no reference vectors");
        Context& cx = ctx();
        cudaStream_t s = cx.stream;
        DevBuf<double> df(f, n * m, s), dv(v, r * m, s), dg(gamma, r, s);
        SelectWorkspace ws;
        ws.alloc(n, r, m);
        struct Guard {
            SelectWorkspace& w;
            ~Guard() { w.release(); }
        } guard{ws};
        launch_row_norms(dv.p, r, m, ws.vn, s);
        VecIndex index;
        struct IndexGuard { VecIndex& x; ~IndexGuard() { x.release(); } } index_guard{index};
        const bool indexed = r >= kIndexMinVectors;
        if (indexed) {
            index.alloc(r, m);
            index.set_order(v, s);
            index.build(dv.p, ws.vn, s);
        }
        launch_select(df.p, n, nullptr, m, dv.p, dg.p, r, apd_penalty(m, t, t_max, alpha), ws, s, indexed ? &index : nullptr);
        uint32_t cnt = 0, flag = 0;
        std::vector<uint32_t> h_elite(r), h_assoc(assoc ? n : 0);
        TEMO_CUDA(cudaMemcpyAsync(&cnt, ws.n_elite, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        TEMO_CUDA(cudaMemcpyAsync(&flag, ws.err_flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        TEMO_CUDA(cudaMemcpyAsync(h_elite.data(), ws.elite, r * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        TEMO_CUDA(cudaMemcpyAsync(validity, ws.valid, r, cudaMemcpyDeviceToHost, s));
        if (assoc) TEMO_CUDA(cudaMemcpyAsync(h_assoc.data(), ws.assoc, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        if (theta) TEMO_CUDA(cudaMemcpyAsync(theta, ws.theta, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        if (apd) TEMO_CUDA(cudaMemcpyAsync(apd, ws.apd, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        TEMO_CUDA(cudaStreamSynchronize(s));
        require(!(flag & 1u), "rv_select: gamma must be positive");  // selection.hpp:152
        *n_elite = cnt;
        for (uint32_t k = 0; k < cnt; ++k) elite[k] = h_elite[k];
        if (assoc)
            for (uint64_t i = 0; i < n; ++i) assoc[i] = h_assoc[i];
    });
}

// ---- algorithms.hpp ----------------------------------------------------------------------------------
struct temo_b200_run {
    std::unique_ptr<Run> impl;
};

int temo_b200_run_create(const temo_b200_run_config* cfg, temo_b200_run** out) {
    return guarded([&] {
        require(out != nullptr, "run_create: null output");
        *out = nullptr;
        std::unique_ptr<temo_b200_run> h(new temo_b200_run);
        h->impl.reset(new Run(cfg_of(cfg)));
        *out = h.release();
    });
}

int temo_b200_run_step(temo_b200_run* run, uint64_t* pop_size, double* survivors_f) {
    return guarded([&] {
        require(run && run->impl, "run_step: null run");
        const uint64_t p = run->impl->step(survivors_f);
        if (pop_size) *pop_size = p;
    });
}

int temo_b200_run_step_injected(temo_b200_run* run, const double* f_off, uint64_t* pop_size) {
    return guarded([&] {
        require(run && run->impl && f_off, "run_step_injected: null argument");
        const uint64_t p = run->impl->step(nullptr, f_off);
        if (pop_size) *pop_size = p;
    });
}

int temo_b200_run_inject(temo_b200_run* run, uint64_t rows, const double* x, const double* f, const double* v,
                         const double* gamma, uint64_t counter, uint64_t t) {
    return guarded([&] {
        require(run && run->impl, "run_inject: null run");
        run->impl->inject(rows, x, f, v, gamma, counter, t);
    });
}

int temo_b200_run_state(temo_b200_run* run, uint64_t* rows, uint64_t* counter, uint64_t* t, uint64_t* r,
                        uint64_t* d, uint64_t* m) {
    return guarded([&] {
        require(run && run->impl, "run_state: null run");
        const Run& R = *run->impl;
        if (rows) *rows = R.P;
        if (counter) *counter = R.counter;
        if (t) *t = R.t;
        if (r) *r = R.r;
        if (d) *d = R.d;
        if (m) *m = R.m;
    });
}

int temo_b200_run_download(temo_b200_run* run, double* x, double* f, double* v, double* gamma) {
    return guarded([&] {
        require(run && run->impl, "run_download: null run");
        run->impl->download(x, f, v, gamma);
    });
}

int temo_b200_run_last_generation(temo_b200_run* run, double* offspring, double* f_off, uint64_t* elite) {
    return guarded([&] {
        require(run && run->impl, "run_last_generation: null run");
        run->impl->last_generation(offspring, f_off, elite);
    });
}

int temo_b200_run_timings(temo_b200_run* run, double* ms8) {
    return guarded([&] {
        require(run && run->impl && ms8, "run_timings: null argument");
        run->impl->resolve_timings();
        std::memcpy(ms8, run->impl->timings, 8 * sizeof(double));
    });
}

int temo_b200_run_timing_history(temo_b200_run* run, double* ms8_per_step, uint64_t max_steps, int reset, uint64_t* steps_out) {
    return guarded([&] {
        require(run && run->impl && steps_out && (ms8_per_step || max_steps == 0), "run_timing_history: null argument");
        *steps_out = run->impl->timing_history(ms8_per_step, max_steps, reset != 0);
    });
}

int temo_b200_run_time_stage(temo_b200_run* run, int stage, int reps, double* mean_ms) {
    return guarded([&] {
        require(run && run->impl && mean_ms, "run_time_stage: null argument");
        *mean_ms = run->impl->time_stage(stage, reps);
    });
}

int temo_b200_run_destroy(temo_b200_run* run) {
    return guarded([&] { delete run; });
}

int temo_b200_rvea_run(const temo_b200_run_config* cfg, double* final_x, double* final_f, uint64_t* final_rows,
                       uint64_t* rows_done, uint64_t* pop_size, double* elapsed_ms) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();  // GenerationTimer, algorithms.hpp:193-204
        Run run(cfg_of(cfg));
        uint64_t done = 0;
        for (uint64_t t = 0; t < run.cfg.generations; ++t) {
            const uint64_t p = run.step(nullptr);
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (pop_size) pop_size[t] = p;
            if (elapsed_ms) elapsed_ms[t] = ms;
            ++done;
            if (run.cfg.time_budget_s > 0.0 && ms >= run.cfg.time_budget_s * 1e3) break;  // algorithms.hpp:291
        }
        run.download(final_x, final_f, nullptr, nullptr);
        if (final_rows) *final_rows = run.P;
        if (rows_done) *rows_done = done;
    });
}

// ---- NSGA-II baseline ------------------------------------------------------------------------------------
int temo_b200_nondominated_sort(const double* f, uint64_t n, uint64_t m, uint64_t* rank) {
    return guarded([&] {
        require(n == 0 || (f && rank), "nondominated_sort: null argument");
        if (n == 0) return;
        cudaStream_t s = ctx().stream;
        DevBuf<double> df(f, n * m, s);
        SortScratch sc;
        struct Guard { SortScratch& x; ~Guard() { x.release(); } } guard{sc};
        sc.alloc(n);
        std::vector<uint32_t> r(n);
        device_nondominated_sort(df.p, n, m, sc, r.data(), s);
        for (uint64_t i = 0; i < n; ++i) rank[i] = r[i];
    });
}

int temo_b200_nsga2_select(const double* f, uint64_t n, uint64_t m, uint64_t target, uint64_t* selected) {
    return guarded([&] {
        require(target <= n, "nsga2_select: target exceeds population");  // selection.hpp:317
        if (target == 0) return;
        require(f && selected, "nsga2_select: null argument");
        cudaStream_t s = ctx().stream;
        DevBuf<double> df(f, n * m, s);
        SortScratch sc;
        struct Guard { SortScratch& x; ~Guard() { x.release(); } } guard{sc};
        sc.alloc(n);
        std::vector<uint32_t> r(n), sel(target);
        device_nondominated_sort(df.p, n, m, sc, r.data(), s);
        nsga2_select_host(f, r.data(), n, m, target, sel.data());
        for (uint64_t k = 0; k < target; ++k) selected[k] = sel[k];
    });
}

struct temo_b200_nsga2 {
    std::unique_ptr<Nsga2Run> impl;
};

int temo_b200_nsga2_create(const temo_b200_run_config* cfg, temo_b200_nsga2** out) {
    return guarded([&] {
        require(out != nullptr, "nsga2_create: null output");
        *out = nullptr;
        std::unique_ptr<temo_b200_nsga2> h(new temo_b200_nsga2);
        h->impl.reset(new Nsga2Run(cfg_of(cfg)));
        *out = h.release();
    });
}

int temo_b200_nsga2_step(temo_b200_nsga2* run, const double* f_off) {
    return guarded([&] {
        require(run && run->impl, "nsga2_step: null run");
        run->impl->step(f_off);
    });
}

int temo_b200_nsga2_inject(temo_b200_nsga2* run, const double* x, const double* f, uint64_t counter, uint64_t t) {
    return guarded([&] {
        require(run && run->impl, "nsga2_inject: null run");
        run->impl->inject(x, f, counter, t);
    });
}

int temo_b200_nsga2_state(temo_b200_nsga2* run, uint64_t* counter, uint64_t* t, uint64_t* d) {
    return guarded([&] {
        require(run && run->impl, "nsga2_state: null run");
        if (counter) *counter = run->impl->counter;
        if (t) *t = run->impl->t;
        if (d) *d = run->impl->d;
    });
}

int temo_b200_nsga2_download(temo_b200_nsga2* run, double* x, double* f) {
    return guarded([&] {
        require(run && run->impl, "nsga2_download: null run");
        run->impl->download(x, f);
    });
}

int temo_b200_nsga2_last_generation(temo_b200_nsga2* run, double* offspring, double* f_off, uint64_t* selected, uint64_t* pool_idx) {
    return guarded([&] {
        require(run && run->impl, "nsga2_last_generation: null run");
        run->impl->last_generation(offspring, f_off, selected, pool_idx);
    });
}

int temo_b200_nsga2_destroy(temo_b200_nsga2* run) {
    return guarded([&] { delete run; });
}

int temo_b200_nsga2_run(const temo_b200_run_config* cfg, double* final_x, double* final_f, uint64_t* rows_done, double* elapsed_ms) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        Nsga2Run run(cfg_of(cfg));
        uint64_t done = 0;
        for (uint64_t t = 0; t < run.cfg.generations; ++t) {
            run.step();
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (elapsed_ms) elapsed_ms[t] = ms;
            ++done;
            if (run.cfg.time_budget_s > 0.0 && ms >= run.cfg.time_budget_s * 1e3) break;  // algorithms.hpp:364
        }
        run.download(final_x, final_f);
        if (rows_done) *rows_done = done;
    });
}

// ---- metrics.hpp ------------------------------------------------------------------------------------------
int temo_b200_igd(const double* f, uint64_t n, uint64_t m, const double* f_ref, uint64_t n_ref, double* out) {
    return guarded([&] {
        require(f && f_ref && out, "igd: null argument");
        require(n >= 1 && n_ref >= 1, "igd: empty set");  // metrics.hpp:22
        cudaStream_t s = ctx().stream;
        DevBuf<double> df(f, n * m, s), dr(f_ref, n_ref * m, s), dn(n_ref);
        *out = device_igd(df.p, nullptr, n, m, dr.p, n_ref, dn.p, s);
    });
}

int temo_b200_hv_mc_box(const double* f, uint64_t n, uint64_t m, const double* lo, const double* ref, uint64_t samples,
                        uint64_t seed, double* value, double* std_error) {
    return guarded([&] {
        require(f && lo && ref && value, "hv_mc: null argument");
        require(samples >= 1, "hv_mc: needs at least one sample");  // metrics.hpp:78
        require(n >= 1, "hv_mc: bad shapes");
        cudaStream_t s = ctx().stream;
        DevBuf<double> df(f, n * m, s), dl(lo, m, s), dr(ref, m, s);
        DevBuf<unsigned long long> hits(1);
        device_hv_mc_box(df.p, nullptr, n, m, dl.p, lo, false, dr.p, ref, 1.0, samples, seed, hits.p, value, std_error, s);
    });
}

int temo_b200_hv_mc(const double* f, uint64_t n, uint64_t m, const double* ref, uint64_t samples, uint64_t seed,
                    double* value, double* std_error) {
    return guarded([&] {
        require(f && ref && value, "hv_mc: null argument");
        require(samples >= 1, "hv_mc: needs at least one sample");
        require(n >= 1, "col_min: empty tensor");  // tensor.hpp:212
        require(m >= 1 && m <= (uint64_t)kMaxObj, "hv_mc: unsupported objective count");
        cudaStream_t s = ctx().stream;
        DevBuf<double> df(f, n * m, s), dl(m), dr(ref, m, s);
        DevBuf<unsigned long long> hits(1);
        struct KeyScratch {
            unsigned long long* p;
            explicit KeyScratch(uint64_t mm) : p(col_minmax_scratch_alloc(mm)) {}
            ~KeyScratch() { cudaFree(p); }
        } scratch(m);
        launch_col_minmax(df.p, n, nullptr, m, dl.p, nullptr, scratch.p, s);
        double lo[kMaxObj];
        dl.to_host(lo, s);
        TEMO_CUDA(cudaStreamSynchronize(s));
        device_hv_mc_box(df.p, nullptr, n, m, dl.p, lo, false, dr.p, ref, 1.0, samples, seed, hits.p, value, std_error, s);
    });
}

int temo_b200_crowding_distance(const double* front, uint64_t k, uint64_t m, double* dist) {
    return guarded([&] {
        require(front && dist, "crowding_distance: null argument");
        crowding_distance_host(front, k, m, dist);
    });
}

int temo_b200_archive_insert(const double* x_old, const double* f_old, uint64_t n_old, const double* x_new, const double* f_new,
                             uint64_t n_new, uint64_t d, uint64_t m, uint64_t cap, double* x_out, double* f_out, uint64_t* n_out) {
    return guarded([&] {
        require(x_out && f_out && n_out, "Archive::insert: null output");
        require((n_old == 0 || (x_old && f_old)) && (n_new == 0 || (x_new && f_new)), "Archive::insert: null input");
        std::vector<unsigned char> keep_old(n_old), keep_new(n_new);
        if (n_old + n_new) {
            cudaStream_t s = ctx().stream;
            DevBuf<double> dfo(f_old, n_old * m, s), dfn(f_new, n_new * m, s);
            DevBuf<unsigned char> dko(n_old), dkn(n_new);
            launch_archive_filter(dfo.p, n_old, dfn.p, n_new, m, dko.p, dkn.p, s);
            dko.to_host(keep_old.data(), s, n_old);
            dkn.to_host(keep_new.data(), s, n_new);
            TEMO_CUDA(cudaStreamSynchronize(s));
        }
        // kept archive rows first, then kept new rows, both in their own order (algorithms.hpp:101-120)
        uint64_t row = 0;
        auto take = [&](const double* x, const double* f, uint64_t i) {
            std::memcpy(x_out + row * d, x + i * d, d * sizeof(double));
            std::memcpy(f_out + row * m, f + i * m, m * sizeof(double));
            ++row;
        };
        for (uint64_t j = 0; j < n_old; ++j)
            if (keep_old[j]) take(x_old, f_old, j);
        for (uint64_t i = 0; i < n_new; ++i)
            if (keep_new[i]) take(x_new, f_new, i);
        if (cap > 0 && row > cap) {  // truncate_by_crowding (algorithms.hpp:124-143)
            std::vector<double> crowd(row);
            crowding_distance_host(f_out, row, m, crowd.data());
            std::vector<uint64_t> order(row);
            for (uint64_t i = 0; i < row; ++i) order[i] = i;
            std::sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) {
                if (crowd[a] != crowd[b]) return crowd[a] > crowd[b];
                return a < b;
            });
            order.resize(cap);
            std::sort(order.begin(), order.end());  // keep insertion order
            for (uint64_t i = 0; i < cap; ++i) {    // order[i] >= i: an in-place forward compaction is safe
                if (order[i] == i) continue;
                std::memmove(x_out + i * d, x_out + order[i] * d, d * sizeof(double));
                std::memmove(f_out + i * m, f_out + order[i] * m, m * sizeof(double));
            }
            row = cap;
        }
        *n_out = row;
    });
}

int temo_b200_run_set_metrics(temo_b200_run* run, const double* pf_ref, uint64_t n_ref, const double* hv_ref, double hv_scale,
                              uint64_t hv_samples, uint64_t hv_seed, int maximization) {
    return guarded([&] {
        require(run && run->impl, "run_set_metrics: null run");
        run->impl->set_metrics(pf_ref, n_ref, hv_ref, hv_scale, hv_samples, hv_seed, maximization != 0);
    });
}

int temo_b200_run_track_archive(temo_b200_run* run, uint64_t archive_cap) {
    return guarded([&] {
        require(run && run->impl, "run_track_archive: null run");
        run->impl->enable_archive(archive_cap);
    });
}

int temo_b200_run_archive_rows(temo_b200_run* run, uint64_t* rows) {
    return guarded([&] {
        require(run && run->impl && rows, "run_archive_rows: null argument");
        require(run->impl->track_archive, "archive: this run does not track one");
        *rows = run->impl->arch_rows;
    });
}

int temo_b200_run_archive(temo_b200_run* run, double* x, double* f) {
    return guarded([&] {
        require(run && run->impl, "run_archive: null run");
        run->impl->archive_download(x, f);
    });
}

int temo_b200_run_metrics(temo_b200_run* run, double* igd, double* hv) {
    return guarded([&] {
        require(run && run->impl, "run_metrics: null run");
        run->impl->metrics(igd, hv);
    });
}

// ---- device-pointer helpers -------------------------------------------------------------------------------
void* temo_b200_dev_alloc(size_t bytes) {
    void* p = nullptr;
    const int rc = guarded([&] {
        ctx();
        p = dev_alloc<unsigned char>(bytes);
    });
    return rc ? nullptr : p;
}

void* temo_b200_host_alloc(size_t bytes) {
    void* p = nullptr;
    const int rc = guarded([&] {
        ctx();
        TEMO_CUDA(cudaMallocHost(&p, bytes ? bytes : 1));
    });
    return rc ? nullptr : p;
}

int temo_b200_host_free(void* p) {
    return guarded([&] { TEMO_CUDA(cudaFreeHost(p)); });
}

int temo_b200_dev_free(void* p) {
    return guarded([&] { TEMO_CUDA(cudaFree(p)); });
}

int temo_b200_dev_upload(void* dst, const void* src, size_t bytes) {
    return guarded([&] { TEMO_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice)); });
}

int temo_b200_dev_download(void* dst, const void* src, size_t bytes) {
    return guarded([&] { TEMO_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost)); });
}

int temo_b200_dev_sync(void) {
    return guarded([&] { TEMO_CUDA(cudaStreamSynchronize(ctx().stream)); });
}

int temo_b200_pow(const double* x, const double* y, uint64_t n, double* out, int on_device) {
    return guarded([&] {
        require(x && y && out, "pow: null argument");
        if (!on_device) {
            for (uint64_t e = 0; e < n; ++e) out[e] = glibc_pow_host(x[e], y[e]);
            return;
        }
        Context& cx = ctx();
        cudaStream_t s = cx.stream;
        DevBuf<double> dx(x, n, s), dy(y, n, s), dout(n);
        launch_pow_batch(dx.p, dy.p, n, dout.p, s);
        dout.to_host(out, s);
        TEMO_CUDA(cudaStreamSynchronize(s));
    });
}

int temo_b200_tanh(const double* x, uint64_t n, double* out, int on_device) {
    return guarded([&] {
        require(x && out, "tanh: null argument");
        if (!on_device) {
            tanh_batch_host(x, n, out);
            return;
        }
        cudaStream_t s = ctx().stream;
        DevBuf<double> dx(x, n, s), dout(n);
        launch_tanh_batch(dx.p, n, dout.p, s);
        dout.to_host(out, s);
        TEMO_CUDA(cudaStreamSynchronize(s));
    });
}

int temo_b200_set_option(const char* name, long value) {
    return guarded([&] { require(set_k1_option(name, value) || set_eval_option(name, value), "set_option: unknown option"); });
}

int temo_b200_flush_l2(void) {
    return guarded([&] { flush_l2(); });
}

}  // extern "C"
