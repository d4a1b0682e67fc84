/* TEST INFRASTRUCTURE — CPU restatement of the TensorRVEA generation loop.
 *
 * This file is the parity ORACLE for the CUDA path in paper_2404_01159_b200/csrc.
 * It is never linked into, imported by, or called from the product: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it. It restates, in plain C over flat row-major fp64 arrays, the arithmetic
 * of the reference (paths relative to /root/reference/proj/include/temo):
 *
 *   rng.hpp:23-78            SplitMix64 counter stream, uniform fill, Fisher-Yates
 *   operators.hpp:65-161     SBX, polynomial mutation, GA reproduction
 *   operators.hpp:287-296    random_reproduce (initial population)
 *   problems.hpp:24-92       DTLZ1-4
 *   refvec.hpp:15-140        lattice, unit vectors, gamma, adaptation
 *   selection.hpp:82-224     rv_core / rv_select (max-cosine association, APD, elites)
 *   algorithms.hpp:211-296   parent_pool_indices, rvea_run loop
 *
 * Pinning: tests/test_oracle_vs_ref.py checks every function here bit-for-bit
 * against oracle/_ref/libtemo_ref.so (the unmodified reference compiled by
 * oracle/Makefile) and tests/test_oracle_golden.py checks it against the committed
 * fixtures in tests/golden/ (generated from the reference by oracle/gen_golden.py)
 * and against the known answers in the reference's own tests.
 * LSMOP1 (to_lsmop1_*) has NO counterpart in the reference: parity unpinned.
 *
 * Bit-exactness rules followed throughout (reference: CMakeLists.txt:19-21
 * -ffp-contract=off; tensor.hpp:143-182 ascending-index accumulation from 0.0):
 * compile with -ffp-contract=off, accumulate in ascending index order, one
 * rounding per operation, libm pow/cos/sin/acos exactly where the reference calls them.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TO_PI 3.141592653589793238462643383279502884 /* std::numbers::pi rounds to the same double */

/* ------------------------------------------------------------------ rng.hpp */

/* rng.hpp:23-30 (Stafford variant 13 finalizer). */
static uint64_t to_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* rng.hpp:39-43: draw k of stream `seed`, top 53 bits scaled into [0,1). */
double to_value_at(uint64_t seed, uint64_t k) {
    const uint64_t word = to_mix64(to_mix64(seed) + k * 0x9e3779b97f4a7c15ULL);
    return (double)(word >> 11) * 0x1.0p-53;
}

/* rng.hpp:55-66: element e of a block starting at `counter` uses counter+e. */
void to_uniform_fill(uint64_t seed, uint64_t counter, double* out, uint64_t count) {
    for (uint64_t e = 0; e < count; ++e) out[e] = to_value_at(seed, counter + e);
}

/* rng.hpp:69-78: Fisher-Yates from the top index down, n-1 draws. */
void to_shuffle_indices(uint64_t seed, uint64_t* counter, uint64_t n, uint64_t* perm) {
    for (uint64_t i = 0; i < n; ++i) perm[i] = i;
    uint64_t c = *counter;
    for (uint64_t i = n; i-- > 1;) {
        const uint64_t j = (uint64_t)(to_value_at(seed, c++) * (double)(i + 1));
        const uint64_t tmp = perm[i];
        perm[i] = perm[j];
        perm[j] = tmp;
    }
    *counter = c;
}

/* algorithms.hpp:211-221: identity when the population already has n rows
 * (no draws), else n draws sampling with replacement. */
void to_parent_pool_indices(uint64_t current, uint64_t n, uint64_t seed, uint64_t* counter,
                            uint64_t* idx) {
    if (current == n) {
        for (uint64_t i = 0; i < n; ++i) idx[i] = i;
        return;
    }
    uint64_t c = *counter;
    for (uint64_t i = 0; i < n; ++i) idx[i] = (uint64_t)(to_value_at(seed, c++) * (double)current);
    *counter = c;
}

/* ------------------------------------------------------------- tensor.hpp */

static double to_step(double x) { return x >= 0.0 ? 1.0 : 0.0; }   /* tensor.hpp:76 */
static double to_sign(double x) { return x >= 0.0 ? 1.0 : -1.0; }  /* tensor.hpp:73 */
static double to_clip(double x, double lo, double hi) {            /* tensor.hpp:85-87 */
    return x < lo ? lo : (x > hi ? hi : x);
}
static double to_acos_clamped(double c) {                          /* tensor.hpp:79-83 */
    if (c > 1.0) c = 1.0;
    if (c < -1.0) c = -1.0;
    return acos(c);
}

/* ---------------------------------------------------------- operators.hpp */

/* ga = {pc, eta, pm, xi} (operators.hpp:22-27). */

/* operators.hpp:65-102. Draw blocks in order: Mc, R1, R2 (half x d each), R3 (half). */
void to_sbx(const double* x, uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter,
            const double* ga, const double* lower, const double* upper, double* out) {
    const uint64_t half = n / 2;
    const uint64_t c_mc = *counter, c_r1 = c_mc + half * d, c_r2 = c_r1 + half * d,
                   c_r3 = c_r2 + half * d;
    const double pc = ga[0], eta = ga[1];
    const double inv_exp = 1.0 / (eta + 1.0);
    for (uint64_t p = 0; p < half; ++p) {
        const double* pa = x + p * d;
        const double* pb = x + (half + p) * d;
        double* ca = out + p * d;
        double* cb = out + (half + p) * d;
        const double hc = to_step(to_value_at(seed, c_r3 + p) - pc);
        for (uint64_t j = 0; j < d; ++j) {
            const uint64_t e = p * d + j;
            const double mc = to_value_at(seed, c_mc + e);
            const double low = pow(2.0 * mc, inv_exp);
            const double high = pow(2.0 - 2.0 * mc, -inv_exp);
            const double hm = to_step(0.5 - mc);
            double beta = to_sign(to_value_at(seed, c_r1 + e) - 0.5) * (hm * low + (1.0 - hm) * high);
            const double hr = to_step(to_value_at(seed, c_r2 + e) - 0.5);
            beta = (1.0 - hc) * ((1.0 - hr) * beta + hr) + hc;
            ca[j] = to_clip(((1.0 + beta) * pa[j] + (1.0 - beta) * pb[j]) / 2.0, lower[j], upper[j]);
            cb[j] = to_clip(((1.0 - beta) * pa[j] + (1.0 + beta) * pb[j]) / 2.0, lower[j], upper[j]);
        }
    }
    if (n & 1) memcpy(out + (n - 1) * d, x + (n - 1) * d, d * sizeof(double)); /* :98-100 */
    *counter = c_r3 + half;
}

/* operators.hpp:106-121: both branches are always evaluated and blended by steps. */
double to_polynomial_delta(double u, double x, double lo, double hi, double xi) {
    const double range = hi - lo;
    const double e = xi + 1.0, inv_e = 1.0 / e;
    const double near_lo = 1.0 - (x - lo) / range;
    const double d_lo = range * (pow(2.0 * u + (1.0 - 2.0 * u) * pow(near_lo, e), inv_e) - 1.0);
    const double near_hi = 1.0 - (hi - x) / range;
    const double d_hi =
        range * (1.0 - pow(2.0 * (1.0 - u) + 2.0 * (u - 0.5) * pow(near_hi, e), inv_e));
    return d_lo * to_step(0.5 - u) + d_hi * to_step(u - 0.5);
}

/* operators.hpp:126-149. Draw blocks: R4 (mask), Mmut, n x d each. */
void to_polynomial_mutation(const double* x, uint64_t n, uint64_t d, uint64_t seed,
                            uint64_t* counter, const double* ga, const double* lower,
                            const double* upper, double* out) {
    const uint64_t c_mask = *counter, c_mut = c_mask + n * d;
    const double rate = ga[2] / (double)d, xi = ga[3];
    for (uint64_t e = 0; e < n * d; ++e) {
        const uint64_t j = e % d;
        const double xv = x[e];
        if (to_step(rate - to_value_at(seed, c_mask + e)) == 0.0 || upper[j] - lower[j] <= 0.0) {
            out[e] = xv;
            continue;
        }
        const double delta = to_polynomial_delta(to_value_at(seed, c_mut + e), xv, lower[j], upper[j], xi);
        out[e] = to_clip(xv + delta, lower[j], upper[j]);
    }
    *counter = c_mut + n * d;
}

/* operators.hpp:153-161: shuffle -> gather -> sbx -> pm. */
int to_ga_reproduce(const double* x, uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter,
                    const double* ga, const double* lower, const double* upper, double* out) {
    uint64_t* perm = (uint64_t*)malloc(n * sizeof(uint64_t));
    double* mates = (double*)malloc(n * d * sizeof(double));
    double* crossed = (double*)malloc(n * d * sizeof(double));
    if (!perm || !mates || !crossed) { free(perm); free(mates); free(crossed); return -2; }
    to_shuffle_indices(seed, counter, n, perm);
    for (uint64_t i = 0; i < n; ++i) memcpy(mates + i * d, x + perm[i] * d, d * sizeof(double));
    to_sbx(mates, n, d, seed, counter, ga, lower, upper, crossed);
    to_polynomial_mutation(crossed, n, d, seed, counter, ga, lower, upper, out);
    free(perm); free(mates); free(crossed);
    return 0;
}

/* Children of the mating pairs [unit0, unit0 + h_loc) of a GLOBAL shuffled population of n_g rows, the two
 * mates of every pair given explicitly (pa, pb: h_loc x d). Same arithmetic and the same draws as to_sbx followed by
 * to_polynomial_mutation for those rows (draw blocks addressed globally: SBX blocks are n_g/2 x d, PM blocks n_g x d),
 * i.e. what one shard of the multi-GPU run must produce. Used only by the sharded-orchestration tests. */
void to_reproduce_pairs(const double* pa, const double* pb, uint64_t h_loc, uint64_t d, uint64_t unit0, uint64_t n_g,
                        uint64_t seed, uint64_t c_sbx, uint64_t c_pm, const double* ga, const double* lower,
                        const double* upper, double* ca, double* cb) {
    const uint64_t half = n_g / 2;
    const uint64_t c_mc = c_sbx, c_r1 = c_mc + half * d, c_r2 = c_r1 + half * d, c_r3 = c_r2 + half * d;
    const uint64_t c_mask = c_pm, c_mut = c_pm + n_g * d;
    const double pc = ga[0], inv_exp = 1.0 / (ga[1] + 1.0), rate = ga[2] / (double)d, xi = ga[3];
    for (uint64_t p = 0; p < h_loc; ++p) {
        const uint64_t pg = unit0 + p;
        const double hc = to_step(to_value_at(seed, c_r3 + pg) - pc);
        for (uint64_t j = 0; j < d; ++j) {
            const uint64_t e = pg * d + j;
            const double mc = to_value_at(seed, c_mc + e);
            const double low = pow(2.0 * mc, inv_exp), high = pow(2.0 - 2.0 * mc, -inv_exp);
            const double hm = to_step(0.5 - mc);
            double beta = to_sign(to_value_at(seed, c_r1 + e) - 0.5) * (hm * low + (1.0 - hm) * high);
            const double hr = to_step(to_value_at(seed, c_r2 + e) - 0.5);
            beta = (1.0 - hc) * ((1.0 - hr) * beta + hr) + hc;
            const double xa = pa[p * d + j], xb = pb[p * d + j];
            double child[2];
            child[0] = to_clip(((1.0 + beta) * xa + (1.0 - beta) * xb) / 2.0, lower[j], upper[j]);
            child[1] = to_clip(((1.0 - beta) * xa + (1.0 + beta) * xb) / 2.0, lower[j], upper[j]);
            for (int w = 0; w < 2; ++w) {
                const uint64_t row = w == 0 ? pg : half + pg;
                const uint64_t em = row * d + j;
                double xv = child[w];
                if (!(to_step(rate - to_value_at(seed, c_mask + em)) == 0.0 || upper[j] - lower[j] <= 0.0)) {
                    const double delta = to_polynomial_delta(to_value_at(seed, c_mut + em), xv, lower[j], upper[j], xi);
                    xv = to_clip(xv + delta, lower[j], upper[j]);
                }
                (w == 0 ? ca : cb)[p * d + j] = xv;
            }
        }
    }
}

/* operators.hpp:287-296. */
void to_random_reproduce(uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter,
                         const double* lower, const double* upper, double* out) {
    const uint64_t c = *counter;
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = 0; j < d; ++j)
            out[i * d + j] = lower[j] + to_value_at(seed, c + i * d + j) * (upper[j] - lower[j]);
    *counter = c + n * d;
}

/* ------------------------------------------- operators.hpp: DE / PSO / CSO */

/* operators.hpp:166-200, DE/rand/1/bin. p = {f, cr}. Draw blocks: r_sel n x 3, r_j n x 1, r_cr n x d. */
int to_de_reproduce(const double* x, uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter, const double* p,
                    const double* lower, const double* upper, double* out) {
    if (n < 4) return 1;                                                 /* :169 */
    const uint64_t c_sel = *counter, c_j = c_sel + 3 * n, c_cr = c_j + n;
    const double nd = (double)n;
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t r1 = (i + 1 + (uint64_t)(to_value_at(seed, c_sel + i * 3 + 0) * (nd - 1.0))) % n;   /* :177-178 */
        const uint64_t excl_a = i < r1 ? i : r1, excl_b = i < r1 ? r1 : i;
        uint64_t r2 = (uint64_t)(to_value_at(seed, c_sel + i * 3 + 1) * (nd - 2.0));
        if (r2 >= excl_a) ++r2;
        if (r2 >= excl_b) ++r2;
        uint64_t e[3] = {i, r1, r2}, t;                                  /* sorted ascending, :183-184 */
        if (e[0] > e[1]) t = e[0], e[0] = e[1], e[1] = t;
        if (e[1] > e[2]) t = e[1], e[1] = e[2], e[2] = t;
        if (e[0] > e[1]) t = e[0], e[0] = e[1], e[1] = t;
        uint64_t r3 = (uint64_t)(to_value_at(seed, c_sel + i * 3 + 2) * (nd - 3.0));
        for (int k = 0; k < 3; ++k)
            if (r3 >= e[k]) ++r3;
        const uint64_t j_rand = (uint64_t)(to_value_at(seed, c_j + i) * (double)d);
        for (uint64_t j = 0; j < d; ++j) {
            if (to_value_at(seed, c_cr + i * d + j) < p[1] || j == j_rand) {
                const double trial = x[r1 * d + j] + p[0] * (x[r2 * d + j] - x[r3 * d + j]);        /* :191 */
                out[i * d + j] = to_clip(trial, lower[j], upper[j]);
            } else {
                out[i * d + j] = x[i * d + j];
            }
        }
    }
    *counter = c_cr + n * d;
    return 0;
}

/* operators.hpp:205-240. p = {inertia, c1, c2}; vel, pb_x (n x d) and pb_score (n) are the SwarmState, updated in place. */
int to_pso_reproduce(const double* x, const double* scores, uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter,
                     const double* p, double* vel, double* pb_x, double* pb_score, const double* lower, const double* upper,
                     double* out) {
    for (uint64_t i = 0; i < n; ++i)
        if (scores[i] < pb_score[i]) {                                   /* :213-219 */
            pb_score[i] = scores[i];
            memcpy(pb_x + i * d, x + i * d, d * sizeof(double));
        }
    uint64_t best = 0;
    for (uint64_t i = 1; i < n; ++i)
        if (pb_score[i] < pb_score[best]) best = i;                      /* :220-222 */
    const uint64_t c1 = *counter, c2 = c1 + n * d;
    const double* gbest = pb_x + best * d;
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = 0; j < d; ++j) {
            const double xv = x[i * d + j];
            const double v = p[0] * vel[i * d + j] + p[1] * to_value_at(seed, c1 + i * d + j) * (pb_x[i * d + j] - xv) +
                             p[2] * to_value_at(seed, c2 + i * d + j) * (gbest[j] - xv);            /* :230-232 */
            vel[i * d + j] = v;
            out[i * d + j] = to_clip(xv + v, lower[j], upper[j]);
        }
    *counter = c2 + n * d;
    return 0;
}

/* operators.hpp:246-284. p = {phi}; vel (n x d) updated in place. Shuffle (n - 1 draws), then r1, r2, r3 (pairs x d). */
int to_cso_reproduce(const double* x, const double* scores, uint64_t n, uint64_t d, uint64_t seed, uint64_t* counter,
                     const double* p, double* vel, const double* lower, const double* upper, double* out) {
    uint64_t* perm = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    double* mean = (double*)calloc(d ? d : 1, sizeof(double));
    double* nv = (double*)malloc((n * d ? n * d : 1) * sizeof(double));
    if (!perm || !mean || !nv) {
        free(perm); free(mean); free(nv);
        return 2;
    }
    to_shuffle_indices(seed, counter, n, perm);
    const uint64_t pairs = n / 2, c1 = *counter, c2 = c1 + pairs * d, c3 = c2 + pairs * d;
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = 0; j < d; ++j) mean[j] += x[i * d + j];        /* :257-259 */
    for (uint64_t j = 0; j < d; ++j) mean[j] /= (double)n;
    memcpy(out, x, n * d * sizeof(double));
    memcpy(nv, vel, n * d * sizeof(double));
    for (uint64_t q = 0; q < pairs; ++q) {
        const uint64_t a = perm[2 * q], b = perm[2 * q + 1];
        uint64_t win = a, lose = b;
        if (scores[b] < scores[a] || (scores[b] == scores[a] && b < a)) win = b, lose = a;          /* :267-271 */
        for (uint64_t j = 0; j < d; ++j) {
            const double xl = x[lose * d + j];
            const double v = to_value_at(seed, c1 + q * d + j) * vel[lose * d + j] +
                             to_value_at(seed, c2 + q * d + j) * (x[win * d + j] - xl) +
                             p[0] * to_value_at(seed, c3 + q * d + j) * (mean[j] - xl);             /* :273-275 */
            nv[lose * d + j] = v;
            out[lose * d + j] = to_clip(xl + v, lower[j], upper[j]);
        }
    }
    memcpy(vel, nv, n * d * sizeof(double));
    *counter = c3 + pairs * d;
    free(perm); free(mean); free(nv);
    return 0;
}

/* ----------------------------------------------------------- problems.hpp */

/* problems.hpp:69-92 with the g and shape helpers of :24-64 folded in. */
int to_dtlz_eval(int id, const double* x, uint64_t n, uint64_t d, uint64_t m, double* f) {
    if (id < 1 || id > 4 || m < 2 || d < m) return -1;
    const double half_pi = TO_PI / 2.0;
    double* pos = (double*)malloc((m - 1) * sizeof(double));
    if (!pos) return -2;
    for (uint64_t r = 0; r < n; ++r) {
        const double* row = x + r * d;
        double* fr = f + r * m;
        for (uint64_t j = 0; j + 1 < m; ++j) pos[j] = id == 4 ? pow(row[j], 100.0) : row[j];
        double g;
        if (id == 1 || id == 3) { /* :24-32 */
            g = (double)(d - m + 1);
            for (uint64_t i = m - 1; i < d; ++i) {
                const double t = row[i] - 0.5;
                g += t * t - cos(20.0 * TO_PI * t);
            }
            g = 100.0 * g;
        } else { /* :34-41 */
            g = 0.0;
            for (uint64_t i = m - 1; i < d; ++i) {
                const double t = row[i] - 0.5;
                g += t * t;
            }
        }
        for (uint64_t j = 0; j < m; ++j) {
            double v;
            if (id == 1) { /* :44-52 linear front */
                v = 0.5 * (1.0 + g);
                for (uint64_t i = 0; i + j + 1 < m; ++i) v *= pos[i];
                if (j > 0) v *= 1.0 - pos[m - 1 - j];
            } else { /* :55-64 spherical front */
                v = 1.0 + g;
                for (uint64_t i = 0; i + j + 1 < m; ++i) v *= cos(pos[i] * half_pi);
                if (j > 0) v *= sin(pos[m - 1 - j] * half_pi);
            }
            fr[j] = v;
        }
    }
    free(pos);
    return 0;
}

/* LSMOP1 — NOT in the reference: PARITY UNPINNED.
 * Definition restated from the LSMOP suite (Cheng, Jin, Olhofer, Sendhoff 2017,
 * "Test problems for large-scale multiobjective and many-objective optimization"),
 * as popularised by PlatEMO: nk = 5 sub-components per group; group sizes from the
 * logistic map c_1 = 3.8*0.1*0.9, c_i = 3.8 c_{i-1}(1-c_{i-1}); linear linkage
 * x'_j = (1 + j/d) x_j - 10 x_1 for the tail genes (1-based j = m..d); every group
 * uses the sphere basic function; linear front f_i = (1+g_i) prod x_k (1 - x_{m-i+1}).
 * Tail bounds are [0,10], position bounds [0,1]. */
void to_lsmop1_layout(uint64_t d, uint64_t m, uint64_t* sublen /* m */, uint64_t* start /* m+1 */) {
    double c[64];
    double sum = 0.0;
    c[0] = 3.8 * 0.1 * (1.0 - 0.1);
    for (uint64_t i = 1; i < m; ++i) c[i] = 3.8 * c[i - 1] * (1.0 - c[i - 1]);
    for (uint64_t i = 0; i < m; ++i) sum += c[i];
    start[0] = 0;
    for (uint64_t i = 0; i < m; ++i) {
        sublen[i] = (uint64_t)floor(c[i] / sum * (double)(d - m + 1) / 5.0);
        start[i + 1] = start[i] + sublen[i] * 5;
    }
}

void to_lsmop1_bounds(uint64_t d, uint64_t m, double* lower, double* upper) {
    for (uint64_t j = 0; j < d; ++j) {
        lower[j] = 0.0;
        upper[j] = j + 1 < m ? 1.0 : 10.0;
    }
}

int to_lsmop1_eval(const double* x, uint64_t n, uint64_t d, uint64_t m, double* f) {
    if (m < 2 || m > 64 || d < m) return -1;
    uint64_t sublen[64], start[65];
    to_lsmop1_layout(d, m, sublen, start);
    for (uint64_t r = 0; r < n; ++r) {
        const double* row = x + r * d;
        double* fr = f + r * m;
        for (uint64_t i = 0; i < m; ++i) {
            /* group i covers tail genes (0-based) m-1+start[i] .. m-1+start[i+1]-1; the nk
             * sub-blocks are contiguous so their spheres add up in ascending gene order. */
            double g = 0.0;
            for (uint64_t q = start[i]; q < start[i + 1]; ++q) {
                const uint64_t j = m - 1 + q; /* 0-based gene; 1-based index j+1 */
                const double y = (1.0 + (double)(j + 1) / (double)d) * row[j] - 10.0 * row[0];
                g += y * y;
            }
            g = sublen[i] ? g / (double)sublen[i] / 5.0 : 0.0;
            double v = 1.0 + g;
            for (uint64_t k = 0; k + i + 1 < m; ++k) v *= row[k];
            if (i > 0) v *= 1.0 - row[m - 1 - i];
            fr[i] = v;
        }
    }
    return 0;
}

/* MLP policy + toy control environment (problems.hpp:105-241). Parameters in the fixed order W1 (hidden x 4,
 * row-major), b1, W2 (2 x hidden, row-major), b2 (mlp_decode, problems.hpp:126-138). */
void to_mlp_forward(const double* p, uint64_t hidden, const double* obs, double* action) { /* problems.hpp:149-163 */
    const double *w1 = p, *b1 = p + 4 * hidden, *w2 = b1 + hidden, *b2 = w2 + 2 * hidden;
    double hid[64];
    for (uint64_t i = 0; i < hidden; ++i) {
        double s = b1[i];
        for (uint64_t j = 0; j < 4; ++j) s += w1[i * 4 + j] * obs[j];
        hid[i] = tanh(s);
    }
    for (uint64_t i = 0; i < 2; ++i) {
        double s = b2[i];
        for (uint64_t j = 0; j < hidden; ++j) s += w2[i * hidden + j] * hid[j];
        action[i] = tanh(s);
    }
}

/* env_rollout (problems.hpp:211-241) over toy_rollout (:176-206): n x d parameters -> n x num_obj returns
 * (maximisation orientation); a row with a non-finite parameter scores -1e9 everywhere. */
int to_env_rollout(const double* params, uint64_t n, uint64_t d, uint64_t hidden, uint64_t horizon, uint64_t num_obj, double* f) {
    if (hidden < 1 || hidden > 64 || d != 4 * hidden + hidden + 2 * hidden + 2 || (num_obj != 2 && num_obj != 3)) return -1;
    const double two_pi = 2.0 * 3.141592653589793238462643383279502884, h0 = 1.0;
    for (uint64_t r = 0; r < n; ++r) {
        const double* p = params + r * d;
        double* fr = f + r * num_obj;
        int finite = 1;
        for (uint64_t k = 0; k < d; ++k)
            if (!isfinite(p[k])) finite = 0;
        if (!finite) {
            for (uint64_t j = 0; j < num_obj; ++j) fr[j] = -1e9;
            continue;
        }
        double v = 0.0, h = h0, fwd = 0.0, ctrl = 0.0, height = 0.0, obs[4], act[2];
        for (uint64_t t = 0; t < horizon; ++t) {
            const double phase = two_pi * (double)t / (double)horizon;
            obs[0] = v;
            obs[1] = h;
            obs[2] = sin(phase);
            obs[3] = cos(phase);
            to_mlp_forward(p, hidden, obs, act);
            v = 0.9 * v + 0.1 * act[0];
            h = to_clip(0.95 * h + 0.1 * act[1], 0.0, 2.0);
            fwd += v;
            ctrl -= act[0] * act[0] + act[1] * act[1];
            height += 10.0 * (h - h0);
        }
        fr[0] = fwd;
        if (num_obj == 2) {
            fr[1] = ctrl;
        } else {
            fr[1] = height;
            fr[2] = ctrl;
        }
    }
    return 0;
}

/* make_problem("toy2" / "toy3").evaluate (problems.hpp:279-294): MlpArch{4, 16, 2}, the negated returns */
int to_toy_eval(int problem, const double* x, uint64_t n, uint64_t d, uint64_t m, uint64_t horizon, double* f) {
    if (m != (problem == 201 ? 2u : 3u)) return -1;
    const int rc = to_env_rollout(x, n, d, 16, horizon, m, f);
    if (rc) return rc;
    for (uint64_t e = 0; e < n * m; ++e) f[e] = -f[e];
    return 0;
}

/* ------------------------------------------------------------- refvec.hpp */

/* refvec.hpp:15-19: C(H+m-1, m-1) by the incremental product. */
uint64_t to_lattice_count(uint64_t m, uint64_t H) {
    uint64_t c = 1;
    for (uint64_t i = 1; i < m; ++i) c = c * (H + i) / i;
    return c;
}

/* refvec.hpp:22-35: closest lattice size, ties -> smaller H, stop once size >= target. */
uint64_t to_lattice_density_for(uint64_t m, uint64_t target) {
    uint64_t best_h = 1, best_gap = UINT64_MAX;
    for (uint64_t h = 1; h < 100000; ++h) {
        const uint64_t c = to_lattice_count(m, h);
        const uint64_t gap = c > target ? c - target : target - c;
        if (gap < best_gap) { best_gap = gap; best_h = h; }
        if (c >= target) break;
    }
    return best_h;
}

/* refvec.hpp:40-62: compositions of H into m parts, lexicographic with every
 * part descending from what is left; emitted iteratively instead of recursively. */
void to_simplex_lattice(uint64_t m, uint64_t H, double* out) {
    uint64_t* part = (uint64_t*)calloc(m, sizeof(uint64_t));
    part[0] = H; /* first row (H,0,...,0) */
    uint64_t row = 0;
    for (;;) {
        for (uint64_t j = 0; j < m; ++j) out[row * m + j] = (double)part[j] / (double)H;
        ++row;
        /* next composition: find the right-most position before the last that is
         * still positive, decrement it, and dump the remainder right after it. */
        uint64_t tail = part[m - 1];
        part[m - 1] = 0;
        uint64_t k = m - 1;
        while (k > 0 && part[k - 1] == 0) --k;
        if (k == 0) break;
        part[k - 1] -= 1;
        part[k] = tail + 1; /* the whole remainder goes to position k, later ones stay 0 */
    }
    free(part);
}

/* refvec.hpp:65-75. Returns -1 on a zero row. */
int to_normalize_to_unit(const double* v, uint64_t r, uint64_t m, double* out) {
    for (uint64_t i = 0; i < r; ++i) {
        double s = 0.0;
        for (uint64_t k = 0; k < m; ++k) s += v[i * m + k] * v[i * m + k];
        const double norm = sqrt(s);
        if (!(norm > 0.0)) return -1;
        for (uint64_t k = 0; k < m; ++k) out[i * m + k] = v[i * m + k] / norm;
    }
    return 0;
}

static void to_row_norms(const double* a, uint64_t r, uint64_t m, double* out) { /* tensor.hpp:171-182 */
    for (uint64_t i = 0; i < r; ++i) {
        double s = 0.0;
        for (uint64_t k = 0; k < m; ++k) s += a[i * m + k] * a[i * m + k];
        out[i] = sqrt(s);
    }
}

/* refvec.hpp:81-100, streamed: the reference materialises cos = V V^T (tensor.hpp:145-161,
 * ascending k from 0.0) and then scans it; scanning pair by pair performs the same
 * operations in the same order without the R x R matrix. Returns -1 if any gamma <= 0. */
int to_min_vector_angles(const double* v, uint64_t r, uint64_t m, double* gamma) {
    if (r < 2) return -3;
    double* norms = (double*)malloc(r * sizeof(double));
    if (!norms) return -2;
    to_row_norms(v, r, m, norms);
    int bad = 0;
    for (uint64_t i = 0; i < r; ++i) {
        double best = -INFINITY;
        for (uint64_t j = 0; j < r; ++j) {
            if (j == i) continue;
            double dot = 0.0;
            for (uint64_t k = 0; k < m; ++k) dot += v[i * m + k] * v[j * m + k];
            const double c = dot / (norms[i] * norms[j]);
            if (c > best) best = c;
        }
        gamma[i] = to_acos_clamped(best);
        if (!(gamma[i] > 0.0)) bad = 1;
    }
    free(norms);
    return bad ? -1 : 0;
}

/* refvec.hpp:81-100 for a SAMPLE of vectors: gamma[q] of vector rows[q] against the full set (every j != rows[q],
 * ascending j). The per-vector loop body is the one above; used where the full O(R^2) scan (or the reference's
 * R x R matrix, 137 GB at R = 130816) is out of reach: the BASELINE-size parity tests. */
int to_min_vector_angles_rows(const double* v, uint64_t r, uint64_t m, const uint64_t* rows, uint64_t n_rows,
                              double* gamma, double* best_cos) {
    if (r < 2) return -3;
    double* norms = (double*)malloc(r * sizeof(double));
    if (!norms) return -2;
    to_row_norms(v, r, m, norms);
    for (uint64_t q = 0; q < n_rows; ++q) {
        const uint64_t i = rows[q];
        if (i >= r) { free(norms); return -3; }
        double best = -INFINITY;
        for (uint64_t j = 0; j < r; ++j) {
            if (j == i) continue;
            double dot = 0.0;
            for (uint64_t k = 0; k < m; ++k) dot += v[i * m + k] * v[j * m + k];
            const double c = dot / (norms[i] * norms[j]);
            if (c > best) best = c;
        }
        gamma[q] = to_acos_clamped(best);
        if (best_cos) best_cos[q] = best;
    }
    free(norms);
    return 0;
}

/* refvec.hpp:119-131 (adapt_vectors alone, no gamma): v = unit(v0 (*) (zmax - zmin)); returns 1 when skipped. */
int to_adapt_vectors(const double* v0, double* v, uint64_t r, uint64_t m, const double* zmin, const double* zmax) {
    for (uint64_t k = 0; k < m; ++k)
        if (!(zmax[k] > zmin[k])) return 1;
    double* scaled = (double*)malloc(r * m * sizeof(double));
    if (!scaled) return -2;
    for (uint64_t i = 0; i < r; ++i)
        for (uint64_t k = 0; k < m; ++k) scaled[i * m + k] = v0[i * m + k] * (zmax[k] - zmin[k]);
    int rc = to_normalize_to_unit(scaled, r, m, v);
    free(scaled);
    return rc;
}

/* refvec.hpp:108-114. v0 and v start identical. */
int to_make_ref_set(uint64_t m, uint64_t H, double* v0, double* gamma) {
    const uint64_t r = to_lattice_count(m, H);
    double* lat = (double*)malloc(r * m * sizeof(double));
    if (!lat) return -2;
    to_simplex_lattice(m, H, lat);
    int rc = to_normalize_to_unit(lat, r, m, v0);
    free(lat);
    if (rc) return rc;
    return to_min_vector_angles(v0, r, m, gamma);
}

/* refvec.hpp:119-140: skipped (v, gamma untouched) unless every range is > 0. */
int to_adapt(const double* v0, double* v, double* gamma, uint64_t r, uint64_t m,
             const double* zmin, const double* zmax) {
    for (uint64_t k = 0; k < m; ++k)
        if (!(zmax[k] > zmin[k])) return 0;
    double* scaled = (double*)malloc(r * m * sizeof(double));
    if (!scaled) return -2;
    for (uint64_t i = 0; i < r; ++i)
        for (uint64_t k = 0; k < m; ++k) scaled[i * m + k] = v0[i * m + k] * (zmax[k] - zmin[k]);
    int rc = to_normalize_to_unit(scaled, r, m, v);
    free(scaled);
    if (rc) return rc;
    return to_min_vector_angles(v, r, m, gamma);
}

/* ---------------------------------------------------------- selection.hpp */

/* selection.hpp:86-89. */
double to_apd_penalty(uint64_t m, uint64_t t, uint64_t t_max, double alpha) {
    return (double)m * pow((double)t / (double)t_max, alpha);
}

/* selection.hpp:148-224 (rv_core + rv_select, want_table = false).
 * Outputs assoc/theta/apd are optional (NULL to skip). Returns -1 on a contract
 * violation (non-positive gamma, t_max == 0), like detail::require. */
int to_rv_select(const double* f, uint64_t n, uint64_t m, const double* v, const double* gamma,
                 uint64_t r, uint64_t t, uint64_t t_max, double alpha, uint64_t* elite,
                 uint64_t* n_elite, unsigned char* validity, uint64_t* assoc_out,
                 double* theta_out, double* apd_out) {
    if (t_max < 1 || n < 1) return -1;
    for (uint64_t j = 0; j < r; ++j)
        if (!(gamma[j] > 0.0)) return -1;
    double* z = (double*)malloc(m * sizeof(double));
    double* fp = (double*)malloc(m * sizeof(double));
    double* vn = (double*)malloc(r * sizeof(double));
    double* apd = (double*)malloc(n * sizeof(double));
    uint64_t* assoc = (uint64_t*)malloc(n * sizeof(uint64_t));
    uint64_t* best = (uint64_t*)calloc(r, sizeof(uint64_t));
    if (!z || !fp || !vn || !apd || !assoc || !best) return -2;
    /* ideal point: tensor.hpp:211-219 */
    for (uint64_t k = 0; k < m; ++k) z[k] = f[k];
    for (uint64_t i = 1; i < n; ++i)
        for (uint64_t k = 0; k < m; ++k)
            if (f[i * m + k] < z[k]) z[k] = f[i * m + k];
    to_row_norms(v, r, m, vn);
    const double penalty = to_apd_penalty(m, t, t_max, alpha);
    for (uint64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (uint64_t k = 0; k < m; ++k) {
            fp[k] = f[i * m + k] - z[k];
            s += fp[k] * fp[k];
        }
        const double nf = sqrt(s);
        uint64_t arg = 0;
        double theta = 0.0; /* a row at the ideal point: angle 0, vector 0 (:167-169) */
        if (nf != 0.0) {
            double top = -INFINITY;
            for (uint64_t j = 0; j < r; ++j) {
                double dot = 0.0;
                for (uint64_t k = 0; k < m; ++k) dot += fp[k] * v[j * m + k];
                const double c = dot / (nf * vn[j]);
                if (c > top) { top = c; arg = j; } /* first strict maximum wins */
            }
            theta = to_acos_clamped(top);
        }
        assoc[i] = arg;
        apd[i] = (1.0 + penalty * (theta / gamma[arg])) * nf; /* :82-84 */
        if (assoc_out) assoc_out[i] = arg;
        if (theta_out) theta_out[i] = theta;
        if (apd_out) apd_out[i] = apd[i];
    }
    /* :206-217: lowest row index among the minimal APD of each vector. */
    memset(validity, 0, r);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t j = assoc[i];
        if (!validity[j] || apd[i] < apd[best[j]]) { best[j] = i; validity[j] = 1; }
    }
    uint64_t cnt = 0;
    for (uint64_t j = 0; j < r; ++j)
        if (validity[j]) elite[cnt++] = best[j];
    *n_elite = cnt;
    free(z); free(fp); free(vn); free(apd); free(assoc); free(best);
    return 0;
}

/* --------------------------------------------------------- algorithms.hpp */

/* Problem ids: 1..4 DTLZ1-4 (problems.hpp:261-278), 101 LSMOP1 (unpinned). */
static int to_evaluate(int problem, const double* x, uint64_t n, uint64_t d, uint64_t m, double* f) {
    if (problem >= 1 && problem <= 4) return to_dtlz_eval(problem, x, n, d, m, f);
    if (problem == 101) return to_lsmop1_eval(x, n, d, m, f);
    if (problem == 201 || problem == 202) return to_toy_eval(problem, x, n, d, m, 100, f);  /* RunConfig::horizon default */
    return -1;
}

void to_problem_bounds(int problem, uint64_t d, uint64_t m, double* lower, double* upper) {
    if (problem == 101) { to_lsmop1_bounds(d, m, lower, upper); return; }
    if (problem == 201 || problem == 202) { /* problems.hpp:285-286 */
        for (uint64_t j = 0; j < d; ++j) { lower[j] = -1.0; upper[j] = 1.0; }
        return;
    }
    for (uint64_t j = 0; j < d; ++j) { lower[j] = 0.0; upper[j] = 1.0; }
}

/* One generation of algorithms.hpp:246-281 on explicit state, used by the lock-step
 * parity tests. In/out: x (rows_cap x d), f (rows_cap x m), *rows, v, gamma, *counter.
 * Optional outputs: offspring (n x d), f_off (n x m), elite (merged indices, <= r). */
int to_generation(int problem, uint64_t n, uint64_t d, uint64_t m, uint64_t seed, uint64_t* counter,
                  const double* ga, const double* lower, const double* upper, uint64_t t,
                  uint64_t t_max, double alpha, uint64_t adapt_every, const double* v0, double* v,
                  double* gamma, uint64_t r, double* x, double* f, uint64_t* rows,
                  double* offspring_out, double* f_off_out, uint64_t* elite_out,
                  uint64_t* n_elite_out) {
    const uint64_t P = *rows;
    uint64_t* pool_idx = (uint64_t*)malloc(n * sizeof(uint64_t));
    double* pool = (double*)malloc(n * d * sizeof(double));
    double* merged_x = (double*)malloc((P + n) * d * sizeof(double));
    double* merged_f = (double*)malloc((P + n) * m * sizeof(double));
    uint64_t* elite = (uint64_t*)malloc((r > P + n ? r : P + n) * sizeof(uint64_t));
    unsigned char* valid = (unsigned char*)malloc(r);
    if (!pool_idx || !pool || !merged_x || !merged_f || !elite || !valid) return -2;
    int rc = 0;
    to_parent_pool_indices(P, n, seed, counter, pool_idx);                       /* :247 */
    for (uint64_t i = 0; i < n; ++i) memcpy(pool + i * d, x + pool_idx[i] * d, d * sizeof(double)); /* :248 */
    memcpy(merged_x, x, P * d * sizeof(double));                                  /* :274 parents first */
    memcpy(merged_f, f, P * m * sizeof(double));
    double* off = merged_x + P * d;
    double* f_off = merged_f + P * m;
    rc = to_ga_reproduce(pool, n, d, seed, counter, ga, lower, upper, off);      /* :252 */
    if (!rc) rc = to_evaluate(problem, off, n, d, m, f_off);                      /* :273 */
    uint64_t cnt = 0;
    if (!rc) rc = to_rv_select(merged_f, P + n, m, v, gamma, r, t, t_max, alpha, elite, &cnt, valid,
                               NULL, NULL, NULL);                                 /* :276-277 */
    if (!rc) {
        if (offspring_out) memcpy(offspring_out, off, n * d * sizeof(double));
        if (f_off_out) memcpy(f_off_out, f_off, n * m * sizeof(double));
        for (uint64_t k = 0; k < cnt; ++k) {                                      /* :278-279 */
            memcpy(x + k * d, merged_x + elite[k] * d, d * sizeof(double));
            memcpy(f + k * m, merged_f + elite[k] * m, m * sizeof(double));
            if (elite_out) elite_out[k] = elite[k];
        }
        *rows = cnt;
        if (n_elite_out) *n_elite_out = cnt;
        if ((t + 1) % adapt_every == 0) {                                         /* :281 */
            double zmin[64], zmax[64];
            for (uint64_t k = 0; k < m; ++k) zmin[k] = zmax[k] = f[k];
            for (uint64_t i = 1; i < cnt; ++i)
                for (uint64_t k = 0; k < m; ++k) {
                    if (f[i * m + k] < zmin[k]) zmin[k] = f[i * m + k];
                    if (f[i * m + k] > zmax[k]) zmax[k] = f[i * m + k];
                }
            rc = to_adapt(v0, v, gamma, r, m, zmin, zmax);
        }
    }
    free(pool_idx); free(pool); free(merged_x); free(merged_f); free(elite); free(valid);
    return rc;
}

/* algorithms.hpp:227-296 with track_archive = false and the GA operator.
 * x_out/f_out need max(n, r) rows. pop_size[generations] receives the survivor counts. */
int to_rvea_run(int problem, uint64_t n, uint64_t d, uint64_t m, uint64_t lattice_h,
                uint64_t generations, double alpha, double fr, uint64_t seed, const double* ga,
                double* x_out, double* f_out, uint64_t* rows_out, uint64_t* pop_size,
                double* v_out, double* gamma_out, uint64_t* counter_out) {
    if (n < 2 || generations < 1 || m > 64) return -1;
    const uint64_t H = lattice_h ? lattice_h : to_lattice_density_for(m, n); /* :233-235 */
    const uint64_t r = to_lattice_count(m, H);
    const uint64_t cap = n > r ? n : r;
    double* v0 = (double*)malloc(r * m * sizeof(double));
    double* v = (double*)malloc(r * m * sizeof(double));
    double* gamma = (double*)malloc(r * sizeof(double));
    double* lower = (double*)malloc(d * sizeof(double));
    double* upper = (double*)malloc(d * sizeof(double));
    double* x = (double*)malloc(cap * d * sizeof(double));
    double* f = (double*)malloc(cap * m * sizeof(double));
    if (!v0 || !v || !gamma || !lower || !upper || !x || !f) return -2;
    int rc = to_make_ref_set(m, H, v0, gamma); /* :236 */
    memcpy(v, v0, r * m * sizeof(double));
    double ae = ceil(fr * (double)generations); /* :237-239 */
    uint64_t adapt_every = ae < 1.0 ? 1 : (uint64_t)ae;
    to_problem_bounds(problem, d, m, lower, upper);
    uint64_t counter = 0, rows = n;
    if (!rc) {
        to_random_reproduce(n, d, seed, &counter, lower, upper, x); /* :241 */
        rc = to_evaluate(problem, x, n, d, m, f);                   /* :242 */
    }
    for (uint64_t t = 0; !rc && t < generations; ++t) {
        rc = to_generation(problem, n, d, m, seed, &counter, ga, lower, upper, t, generations, alpha,
                           adapt_every, v0, v, gamma, r, x, f, &rows, NULL, NULL, NULL, NULL);
        if (pop_size) pop_size[t] = rows;
    }
    if (!rc) {
        memcpy(x_out, x, rows * d * sizeof(double));
        memcpy(f_out, f, rows * m * sizeof(double));
        *rows_out = rows;
        if (v_out) memcpy(v_out, v, r * m * sizeof(double));
        if (gamma_out) memcpy(gamma_out, gamma, r * sizeof(double));
        if (counter_out) *counter_out = counter;
    }
    free(v0); free(v); free(gamma); free(lower); free(upper); free(x); free(f);
    return rc;
}

/* algorithms.hpp:227-296 with track_archive = false and any operator of :250-271.
 * op: 0 ga, 1 de, 2 pso, 3 cso, 4 random. opp = {de.f, de.cr, pso.inertia, pso.c1, pso.c2, cso.phi}
 * (operators.hpp:28-41). pso / cso take apd_scores of the pool's objectives as fitness (:257-258, :263-264)
 * and carry a SwarmState created on first use (operators.hpp:58-60). */
int to_rvea_run_op(int problem, int op, const double* opp, uint64_t n, uint64_t d, uint64_t m, uint64_t lattice_h,
                   uint64_t generations, double alpha, double fr, uint64_t seed, const double* ga,
                   double* x_out, double* f_out, uint64_t* rows_out, uint64_t* pop_size, uint64_t* counter_out) {
    if (n < 2 || generations < 1 || m > 64 || op < 0 || op > 4) return -1;
    const uint64_t H = lattice_h ? lattice_h : to_lattice_density_for(m, n);
    const uint64_t r = to_lattice_count(m, H);
    const uint64_t cap = (n > r ? n : r) + n; /* merged rows */
    double* v0 = (double*)malloc(r * m * sizeof(double));
    double* v = (double*)malloc(r * m * sizeof(double));
    double* gamma = (double*)malloc(r * sizeof(double));
    double* lower = (double*)malloc(d * sizeof(double));
    double* upper = (double*)malloc(d * sizeof(double));
    double* x = (double*)malloc(cap * d * sizeof(double));
    double* f = (double*)malloc(cap * m * sizeof(double));
    double* nx = (double*)malloc(cap * d * sizeof(double));
    double* nf = (double*)malloc(cap * m * sizeof(double));
    double* pool = (double*)malloc(n * d * sizeof(double));
    double* pool_f = (double*)malloc(n * m * sizeof(double));
    double* scores = (double*)malloc(n * sizeof(double));
    double* vel = (double*)calloc(n * d, sizeof(double));
    double* pb_x = (double*)malloc(n * d * sizeof(double));
    double* pb_s = (double*)malloc(n * sizeof(double));
    uint64_t* pool_idx = (uint64_t*)malloc(n * sizeof(uint64_t));
    uint64_t* elite = (uint64_t*)malloc((r > cap ? r : cap) * sizeof(uint64_t));
    unsigned char* valid = (unsigned char*)malloc(r);
    if (!v0 || !v || !gamma || !lower || !upper || !x || !f || !nx || !nf || !pool || !pool_f || !scores || !vel || !pb_x ||
        !pb_s || !pool_idx || !elite || !valid)
        return -2;
    int rc = to_make_ref_set(m, H, v0, gamma);
    memcpy(v, v0, r * m * sizeof(double));
    const double ae = ceil(fr * (double)generations);
    const uint64_t adapt_every = ae < 1.0 ? 1 : (uint64_t)ae;
    to_problem_bounds(problem, d, m, lower, upper);
    uint64_t counter = 0, rows = n;
    int swarm_empty = 1;
    if (!rc) {
        to_random_reproduce(n, d, seed, &counter, lower, upper, x);
        rc = to_evaluate(problem, x, n, d, m, f);
    }
    for (uint64_t t = 0; !rc && t < generations; ++t) {
        const uint64_t P = rows;
        to_parent_pool_indices(P, n, seed, &counter, pool_idx);                                   /* :247 */
        for (uint64_t i = 0; i < n; ++i) memcpy(pool + i * d, x + pool_idx[i] * d, d * sizeof(double));
        double* off = x + P * d;   /* merged = parents first, then offspring (:274-275) */
        double* f_off = f + P * m;
        if (op == 2 || op == 3) {
            for (uint64_t i = 0; i < n; ++i) memcpy(pool_f + i * m, f + pool_idx[i] * m, m * sizeof(double));
            uint64_t cnt0 = 0;
            rc = to_rv_select(pool_f, n, m, v, gamma, r, t, generations, alpha, elite, &cnt0, valid, NULL, NULL, scores);
            if (rc) break;
            if (swarm_empty) { /* make_swarm_state */
                memset(vel, 0, n * d * sizeof(double));
                memcpy(pb_x, pool, n * d * sizeof(double));
                memcpy(pb_s, scores, n * sizeof(double));
                swarm_empty = 0;
            }
        }
        switch (op) {
        case 0: rc = to_ga_reproduce(pool, n, d, seed, &counter, ga, lower, upper, off); break;
        case 1: rc = to_de_reproduce(pool, n, d, seed, &counter, opp, lower, upper, off); break;
        case 2: rc = to_pso_reproduce(pool, scores, n, d, seed, &counter, opp + 2, vel, pb_x, pb_s, lower, upper, off); break;
        case 3: rc = to_cso_reproduce(pool, scores, n, d, seed, &counter, opp + 5, vel, lower, upper, off); break;
        default: to_random_reproduce(n, d, seed, &counter, lower, upper, off); break;
        }
        if (!rc) rc = to_evaluate(problem, off, n, d, m, f_off);
        uint64_t cnt = 0;
        if (!rc) rc = to_rv_select(f, P + n, m, v, gamma, r, t, generations, alpha, elite, &cnt, valid, NULL, NULL, NULL);
        if (rc) break;
        for (uint64_t k = 0; k < cnt; ++k) {
            memcpy(nx + k * d, x + elite[k] * d, d * sizeof(double));
            memcpy(nf + k * m, f + elite[k] * m, m * sizeof(double));
        }
        memcpy(x, nx, cnt * d * sizeof(double));
        memcpy(f, nf, cnt * m * sizeof(double));
        rows = cnt;
        if ((t + 1) % adapt_every == 0) {
            double zmin[64], zmax[64];
            for (uint64_t k = 0; k < m; ++k) zmin[k] = zmax[k] = f[k];
            for (uint64_t i = 1; i < cnt; ++i)
                for (uint64_t k = 0; k < m; ++k) {
                    if (f[i * m + k] < zmin[k]) zmin[k] = f[i * m + k];
                    if (f[i * m + k] > zmax[k]) zmax[k] = f[i * m + k];
                }
            rc = to_adapt(v0, v, gamma, r, m, zmin, zmax);
        }
        if (pop_size) pop_size[t] = rows;
    }
    if (!rc) {
        memcpy(x_out, x, rows * d * sizeof(double));
        memcpy(f_out, f, rows * m * sizeof(double));
        *rows_out = rows;
        if (counter_out) *counter_out = counter;
    }
    free(v0); free(v); free(gamma); free(lower); free(upper); free(x); free(f); free(nx); free(nf); free(pool);
    free(pool_f); free(scores); free(vel); free(pb_x); free(pb_s); free(pool_idx); free(elite); free(valid);
    return rc;
}

/* ------------------------------------------------------------------ metrics.hpp */

/* metrics.hpp:21-44 */
int to_igd(const double* f, uint64_t n, uint64_t m, const double* f_ref, uint64_t n_ref, double* out) {
    if (n < 1 || n_ref < 1) return 1;
    double sum = 0.0;
    for (uint64_t i = 0; i < n_ref; ++i) {
        double best = INFINITY;
        for (uint64_t j = 0; j < n; ++j) {
            double s = 0.0;
            for (uint64_t k = 0; k < m; ++k) {
                const double diff = f[j * m + k] - f_ref[i * m + k];
                s += diff * diff;
            }
            if (s < best) best = s;
        }
        sum += sqrt(best);
    }
    *out = sum / (double)n_ref;
    return 0;
}

/* metrics.hpp:76-117: sample s uses draws s*m .. s*m+m-1 of RngStream{seed}. out = {value, std_error}. */
int to_hv_mc_box(const double* f, uint64_t n, uint64_t m, const double* lo, const double* ref, uint64_t samples,
                 uint64_t seed, double* out) {
    if (samples < 1 || n < 1 || m > 64) return 1;
    double volume = 1.0;
    for (uint64_t k = 0; k < m; ++k) {
        const double side = ref[k] - lo[k];
        if (side <= 0.0) { out[0] = out[1] = 0.0; return 0; }
        volume *= side;
    }
    uint64_t hits = 0;
    double pt[64];
    for (uint64_t s = 0; s < samples; ++s) {
        for (uint64_t k = 0; k < m; ++k) pt[k] = lo[k] + to_value_at(seed, s * m + k) * (ref[k] - lo[k]);
        for (uint64_t i = 0; i < n; ++i) {
            int all_le = 1;
            for (uint64_t k = 0; k < m; ++k)
                if (f[i * m + k] > pt[k]) { all_le = 0; break; }
            if (all_le) { ++hits; break; }
        }
    }
    const double p = (double)hits / (double)samples;
    out[0] = volume * p;
    out[1] = volume * sqrt(p * (1.0 - p) / (double)samples);
    return 0;
}

/* metrics.hpp:121-124: the box is [col_min(f), ref]. */
int to_hv_mc(const double* f, uint64_t n, uint64_t m, const double* ref, uint64_t samples, uint64_t seed, double* out) {
    if (n < 1 || m > 64) return 1;
    double lo[64];
    for (uint64_t k = 0; k < m; ++k) lo[k] = f[k];
    for (uint64_t i = 1; i < n; ++i)
        for (uint64_t k = 0; k < m; ++k)
            if (f[i * m + k] < lo[k]) lo[k] = f[i * m + k];
    return to_hv_mc_box(f, n, m, lo, ref, samples, seed, out);
}

/* ------------------------------------------------ Archive::insert (algorithms.hpp:72-144), crowding_distance */

static int to_dominates(const double* a, const double* b, uint64_t m) { /* selection.hpp:240-247 */
    int strict = 0;
    for (uint64_t k = 0; k < m; ++k) {
        if (a[k] > b[k]) return 0;
        if (a[k] < b[k]) strict = 1;
    }
    return strict;
}
static int to_equal(const double* a, const double* b, uint64_t m) {
    for (uint64_t k = 0; k < m; ++k)
        if (!(a[k] == b[k])) return 0;
    return 1;
}

/* selection.hpp:289-312; ties in the per-objective order go to the lower row. */
static const double* g_sort_f;
static uint64_t g_sort_m, g_sort_obj;
static int to_cmp_obj(const void* pa, const void* pb) {
    const uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
    const double fa = g_sort_f[a * g_sort_m + g_sort_obj], fb = g_sort_f[b * g_sort_m + g_sort_obj];
    if (fa != fb) return fa < fb ? -1 : 1;
    return a < b ? -1 : (a > b ? 1 : 0);
}
int to_crowding_distance(const double* front, uint64_t k, uint64_t m, double* dist) {
    if (k < 1) return 1;
    for (uint64_t i = 0; i < k; ++i) dist[i] = k <= 2 ? INFINITY : 0.0;
    if (k <= 2) return 0;
    uint64_t* order = (uint64_t*)malloc(k * sizeof(uint64_t));
    if (!order) return 2;
    for (uint64_t obj = 0; obj < m; ++obj) {
        for (uint64_t i = 0; i < k; ++i) order[i] = i;
        g_sort_f = front; g_sort_m = m; g_sort_obj = obj;
        qsort(order, k, sizeof(uint64_t), to_cmp_obj); /* a total order: any sort gives the same permutation */
        const double range = front[order[k - 1] * m + obj] - front[order[0] * m + obj];
        if (range <= 0.0) continue;
        dist[order[0]] = INFINITY;
        dist[order[k - 1]] = INFINITY;
        for (uint64_t i = 1; i + 1 < k; ++i)
            dist[order[i]] += (front[order[i + 1] * m + obj] - front[order[i - 1] * m + obj]) / range;
    }
    free(order);
    return 0;
}

static const double* g_crowd;
static int to_cmp_crowd(const void* pa, const void* pb) {
    const uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
    if (g_crowd[a] != g_crowd[b]) return g_crowd[a] > g_crowd[b] ? -1 : 1;
    return a < b ? -1 : (a > b ? 1 : 0);
}
static int to_cmp_u64(const void* pa, const void* pb) {
    const uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* x_out / f_out hold n_old + n_new rows. */
int to_archive_insert(const double* x_old, const double* f_old, uint64_t n_old, const double* x_new, const double* f_new,
                      uint64_t n_new, uint64_t d, uint64_t m, uint64_t cap, double* x_out, double* f_out, uint64_t* n_out) {
    uint64_t row = 0;
    for (uint64_t j = 0; j < n_old; ++j) { /* :91-100 */
        int keep = 1;
        for (uint64_t i = 0; i < n_new && keep; ++i)
            if (to_dominates(f_new + i * m, f_old + j * m, m)) keep = 0;
        if (!keep) continue;
        memcpy(x_out + row * d, x_old + j * d, d * sizeof(double));
        memcpy(f_out + row * m, f_old + j * m, m * sizeof(double));
        ++row;
    }
    for (uint64_t i = 0; i < n_new; ++i) { /* :76-90 */
        const double* fi = f_new + i * m;
        int keep = 1;
        for (uint64_t j = 0; j < n_old && keep; ++j)
            if (to_equal(fi, f_old + j * m, m) || to_dominates(f_old + j * m, fi, m)) keep = 0;
        for (uint64_t k = 0; k < n_new && keep; ++k) {
            if (k == i) continue;
            if (to_dominates(f_new + k * m, fi, m) || (k < i && to_equal(fi, f_new + k * m, m))) keep = 0;
        }
        if (!keep) continue;
        memcpy(x_out + row * d, x_new + i * d, d * sizeof(double));
        memcpy(f_out + row * m, fi, m * sizeof(double));
        ++row;
    }
    if (cap > 0 && row > cap) { /* truncate_by_crowding, :124-143 */
        double* crowd = (double*)malloc(row * sizeof(double));
        uint64_t* order = (uint64_t*)malloc(row * sizeof(uint64_t));
        if (!crowd || !order) return 2;
        to_crowding_distance(f_out, row, m, crowd);
        for (uint64_t i = 0; i < row; ++i) order[i] = i;
        g_crowd = crowd;
        qsort(order, row, sizeof(uint64_t), to_cmp_crowd);
        qsort(order, cap, sizeof(uint64_t), to_cmp_u64);
        for (uint64_t i = 0; i < cap; ++i) {
            memmove(x_out + i * d, x_out + order[i] * d, d * sizeof(double));
            memmove(f_out + i * m, f_out + order[i] * m, m * sizeof(double));
        }
        row = cap;
        free(crowd); free(order);
    }
    *n_out = row;
    return 0;
}

/* ------------------------------------------- NSGA-II baseline */

/* selection.hpp:251-283. rank[i] = index of the front row i is peeled in = length of the longest chain of
 * dominators above it; computed here by peeling with dominator counts like the reference. */
int to_nondominated_sort(const double* f, uint64_t n, uint64_t m, uint64_t* rank) {
    uint32_t* cnt = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
    unsigned char* done = (unsigned char*)calloc(n ? n : 1, 1);
    uint64_t* cur = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    if (!cnt || !done || !cur) return 2;
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = 0; j < n; ++j)
            if (i != j && to_dominates(f + j * m, f + i * m, m)) ++cnt[i];
    uint64_t left = n, level = 0;
    while (left) {
        uint64_t k = 0;
        for (uint64_t i = 0; i < n; ++i)
            if (!done[i] && cnt[i] == 0) cur[k++] = i;
        if (!k) break; /* cannot happen for a strict partial order */
        for (uint64_t a = 0; a < k; ++a) {
            const uint64_t i = cur[a];
            rank[i] = level;
            done[i] = 1;
        }
        for (uint64_t a = 0; a < k; ++a)
            for (uint64_t j = 0; j < n; ++j)
                if (!done[j] && to_dominates(f + cur[a] * m, f + j * m, m)) --cnt[j];
        left -= k;
        ++level;
    }
    free(cnt); free(done); free(cur);
    return 0;
}

static const uint64_t* g_front_rows;
static int to_cmp_crowd_rows(const void* pa, const void* pb) { /* selection.hpp:336-339 */
    const uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
    if (g_crowd[a] != g_crowd[b]) return g_crowd[a] > g_crowd[b] ? -1 : 1;
    return g_front_rows[a] < g_front_rows[b] ? -1 : (g_front_rows[a] > g_front_rows[b] ? 1 : 0);
}

/* selection.hpp:316-346: fill by ascending rank, split the last front by descending crowding distance. */
int to_nsga2_select(const double* f, uint64_t n, uint64_t m, uint64_t target, uint64_t* selected) {
    if (target > n) return 1;
    uint64_t* rank = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    uint64_t* rows = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    uint64_t* by = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    double* front = (double*)malloc((n * m ? n * m : 1) * sizeof(double));
    double* crowd = (double*)malloc((n ? n : 1) * sizeof(double));
    if (!rank || !rows || !by || !front || !crowd) return 2;
    int rc = to_nondominated_sort(f, n, m, rank);
    uint64_t cnt = 0;
    for (uint64_t level = 0; !rc && cnt < target; ++level) {
        uint64_t k = 0;
        for (uint64_t i = 0; i < n; ++i)
            if (rank[i] == level) rows[k++] = i;
        if (cnt + k <= target) {
            for (uint64_t a = 0; a < k; ++a) selected[cnt++] = rows[a];
            continue;
        }
        for (uint64_t a = 0; a < k; ++a) memcpy(front + a * m, f + rows[a] * m, m * sizeof(double));
        to_crowding_distance(front, k, m, crowd);
        for (uint64_t a = 0; a < k; ++a) by[a] = a;
        g_crowd = crowd;
        g_front_rows = rows;
        qsort(by, k, sizeof(uint64_t), to_cmp_crowd_rows);
        for (uint64_t a = 0; cnt < target; ++a) selected[cnt++] = rows[by[a]];
    }
    free(rank); free(rows); free(by); free(front); free(crowd);
    return rc;
}

/* One generation of nsga2_run (algorithms.hpp:314-356) on explicit state: x (n x d), f (n x m) in/out, *counter in/out.
 * Optional outputs: offspring (n x d), f_off (n x m), sel (n merged-row indices), pool_idx (n). */
int to_nsga2_generation(int problem, uint64_t n, uint64_t d, uint64_t m, uint64_t seed, uint64_t* counter, const double* ga,
                        const double* lower, const double* upper, double* x, double* f, double* offspring_out, double* f_off_out,
                        uint64_t* sel_out, uint64_t* pool_idx_out) {
    uint64_t* rank = (uint64_t*)malloc(n * sizeof(uint64_t));
    uint64_t* members = (uint64_t*)malloc(n * sizeof(uint64_t));
    uint64_t* pool_idx = (uint64_t*)malloc(n * sizeof(uint64_t));
    uint64_t* sel = (uint64_t*)malloc(n * sizeof(uint64_t));
    double* crowd = (double*)calloc(n, sizeof(double));
    double* front = (double*)malloc(n * m * sizeof(double));
    double* cd = (double*)malloc(n * sizeof(double));
    double* pool = (double*)malloc(n * d * sizeof(double));
    double* crossed = (double*)malloc(n * d * sizeof(double));
    double* mx = (double*)malloc(2 * n * d * sizeof(double));
    double* mf = (double*)malloc(2 * n * m * sizeof(double));
    if (!rank || !members || !pool_idx || !sel || !crowd || !front || !cd || !pool || !crossed || !mx || !mf) return 2;
    int rc = to_nondominated_sort(f, n, m, rank);
    uint64_t levels = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (rank[i] + 1 > levels) levels = rank[i] + 1;
    for (uint64_t level = 0; level < levels; ++level) { /* :316-329 */
        uint64_t k = 0;
        for (uint64_t i = 0; i < n; ++i)
            if (rank[i] == level) members[k++] = i;
        if (!k) continue;
        for (uint64_t a = 0; a < k; ++a) memcpy(front + a * m, f + members[a] * m, m * sizeof(double));
        to_crowding_distance(front, k, m, cd);
        for (uint64_t a = 0; a < k; ++a) crowd[members[a]] = cd[a];
    }
    for (uint64_t i = 0; i < n; ++i) { /* binary tournament, :332-345 */
        const uint64_t a = (uint64_t)(to_value_at(seed, (*counter)++) * (double)n);
        const uint64_t b = (uint64_t)(to_value_at(seed, (*counter)++) * (double)n);
        int a_wins;
        if (rank[a] != rank[b]) a_wins = rank[a] < rank[b];
        else if (crowd[a] != crowd[b]) a_wins = crowd[a] > crowd[b];
        else a_wins = a <= b;
        pool_idx[i] = a_wins ? a : b;
    }
    for (uint64_t i = 0; i < n; ++i) memcpy(pool + i * d, x + pool_idx[i] * d, d * sizeof(double));
    to_sbx(pool, n, d, seed, counter, ga, lower, upper, crossed);               /* :347 */
    memcpy(mx, x, n * d * sizeof(double));
    memcpy(mf, f, n * m * sizeof(double));
    to_polynomial_mutation(crossed, n, d, seed, counter, ga, lower, upper, mx + n * d); /* :348-349 */
    if (!rc) rc = to_evaluate(problem, mx + n * d, n, d, m, mf + n * m);
    if (!rc) rc = to_nsga2_select(mf, 2 * n, m, n, sel);                         /* :353 */
    if (!rc) {
        if (offspring_out) memcpy(offspring_out, mx + n * d, n * d * sizeof(double));
        if (f_off_out) memcpy(f_off_out, mf + n * m, n * m * sizeof(double));
        for (uint64_t k = 0; k < n; ++k) {
            memcpy(x + k * d, mx + sel[k] * d, d * sizeof(double));
            memcpy(f + k * m, mf + sel[k] * m, m * sizeof(double));
            if (sel_out) sel_out[k] = sel[k];
            if (pool_idx_out) pool_idx_out[k] = pool_idx[k];
        }
    }
    free(rank); free(members); free(pool_idx); free(sel); free(crowd); free(front); free(cd); free(pool); free(crossed);
    free(mx); free(mf);
    return rc;
}

/* algorithms.hpp:301-369 with track_archive = false. */
int to_nsga2_run(int problem, uint64_t n, uint64_t d, uint64_t m, uint64_t generations, uint64_t seed, const double* ga,
                 double* x_out, double* f_out, uint64_t* counter_out) {
    if (n < 2 || generations < 1 || m > 64) return -1;
    double* lower = (double*)malloc(d * sizeof(double));
    double* upper = (double*)malloc(d * sizeof(double));
    if (!lower || !upper) return -2;
    to_problem_bounds(problem, d, m, lower, upper);
    uint64_t counter = 0;
    to_random_reproduce(n, d, seed, &counter, lower, upper, x_out);
    int rc = to_evaluate(problem, x_out, n, d, m, f_out);
    for (uint64_t t = 0; !rc && t < generations; ++t)
        rc = to_nsga2_generation(problem, n, d, m, seed, &counter, ga, lower, upper, x_out, f_out, NULL, NULL, NULL, NULL);
    if (counter_out) *counter_out = counter;
    free(lower); free(upper);
    return rc;
}
