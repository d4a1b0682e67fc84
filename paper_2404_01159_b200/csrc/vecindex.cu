// Exact nearest-reference-vector search without the O(rows x R) scan.
//
// reference: the association loop of detail::rv_core (selection.hpp:172-184: for every row the
// FIRST j with strictly greatest dot/(nf*vn[j])) and the max-cosine scan of min_vector_angles
// (refvec.hpp:89-94). At BASELINE config #3 those are 3.4e10 and 1.7e10 (row, vector) pairs —
// 50 ms and 30 ms per call on a B200 when done by brute force — although only the handful of
// vectors around a row's direction can win.
//
// Index: the R vectors are put in Hilbert-curve order of their simplex coordinates (host, once), so
// that every run of 32 consecutive positions ("group"), every run of 32 groups, ... is a
// compact patch of directions. Each node of that implicit 32-ary tree stores a member vector
// as its centre and the patch's angular radius rho as (cos rho, sin rho), rebuilt on the device
// whenever V changes. Search (one warp per row, depth-first, lanes = the 32 children of a node):
// a node can contain a vector with cosine >= L only if
//        cos(row, centre) >= cos(acos(L) + rho) = L cos(rho) - sqrt(1 - L^2) sin(rho),
// where L is the best cosine realised so far (a lower bound of the answer). Pruned nodes are
// provably worse than L by more than 1e-12 — three orders above fp64 rounding — so every vector
// whose COMPUTED cosine could equal or exceed the computed maximum is still visited, and the
// visited ones are scored with the reference's exact expression and reduced lexicographically
// (max cosine, then lowest original index) = the reference's first-strict-maximum rule.
// Requires V >= 0 and row >= 0 componentwise (always true for translated objectives and
// Das-Dennis sets); anything else takes the exhaustive warp scan, which is also the path for
// rows with non-finite norms (NaN handling identical to the reference's `c > best` loop).
#include <algorithm>
#include <numeric>

#include "internal.h"
#include "vecindex.h"

namespace temo_b200 {

namespace {

constexpr double kSlack = 1e-12;  // >> fp64 rounding of a cosine (~4e-16), << any decision it guards
// The search divides only where the reference's exact expression is needed. Everywhere else (the centres of the tree's
// nodes, and the leaf vectors that cannot reach the best cosine realised so far) a cosine is dot * rcp(nf * |v|) with the
// hardware's approximate fp64 reciprocal (rcp.approx.ftz.f64: relative error <= 1.0e-6 measured over 2.7e8 arguments on
// a B200, tools/rcp_check.cu; 2^-20 by the PTX manual). kApprox bounds the error of such a cosine (|cos| <= 1 up to
// rounding) with a factor of four in hand; every decision taken on an approximate cosine is widened by it.
constexpr double kApprox = 4e-6;
__device__ __forceinline__ double rcp_approx(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}

__device__ __forceinline__ unsigned long long order_key(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
constexpr unsigned long long kKeyMax = 0xffffffffffffffffULL;

// vp[p] = {v[orig[p]][0..m-1], vn[orig[p]]}
__global__ void gather_perm_kernel(const double* v, const double* vn, const uint32_t* orig, uint64_t r, uint64_t m,
                                   double* vp, uint32_t* flags) {
    const uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (p >= r) return;
    const uint64_t j = orig[p];
    bool neg = false;
    for (uint64_t k = 0; k < m; ++k) {
        const double x = v[j * m + k];
        vp[p * (m + 1) + k] = x;
        if (!(x >= 0.0)) neg = true;
    }
    vp[p * (m + 1) + m] = vn[j];
    if (neg) atomicOr(flags, 1u);
}

// One warp per node of level `lvl` (span = 32^lvl positions): centre = the member closest to the patch's
// mean direction, radius from the exact cosines to every member.
// Record: {centre[0..m-1], centre norm, cos rho, sin rho}.
__global__ void node_build_kernel(const double* vp, uint64_t r, uint64_t m, uint64_t span, uint64_t count,
                                  double* node, uint32_t* centre_pos) {
    const uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= count) return;
    const uint64_t a = i * span, b = (a + span < r) ? a + span : r;
    // mean direction of the members (vectors are unit up to rounding; any reasonable centre is valid —
    // the radius below is computed exactly for whichever member is chosen)
    double mean[kMaxObj];
    for (uint64_t k = 0; k < m; ++k) mean[k] = 0.0;
    for (uint64_t p = a + lane; p < b; p += 32)
        for (uint64_t k = 0; k < m; ++k) mean[k] += vp[p * (m + 1) + k] / vp[p * (m + 1) + m];
    for (uint64_t k = 0; k < m; ++k)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mean[k] += __shfl_xor_sync(0xffffffffu, mean[k], off);
    double best = -INFINITY;
    uint64_t best_p = a;
    for (uint64_t p = a + lane; p < b; p += 32) {
        double dot = 0.0;
        for (uint64_t k = 0; k < m; ++k) dot += mean[k] * vp[p * (m + 1) + k];
        dot /= vp[p * (m + 1) + m];
        if (dot > best) {
            best = dot;
            best_p = p;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, off);
        const uint64_t op = __shfl_xor_sync(0xffffffffu, best_p, off);
        if (ob > best || (ob == best && op < best_p)) {
            best = ob;
            best_p = op;
        }
    }
    const uint64_t c = best_p;
    const double* cv = vp + c * (m + 1);
    const double cn = cv[m];
    double lo = 2.0;
    for (uint64_t p = a + lane; p < b; p += 32) {
        const double* pv = vp + p * (m + 1);
        double dot = 0.0;
        for (uint64_t k = 0; k < m; ++k) dot += cv[k] * pv[k];
        const double cs = dot / (cn * pv[m]);
        lo = cs < lo ? cs : lo;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, lo, off);
        lo = o < lo ? o : lo;
    }
    if (lane == 0) {
        double cr = lo - kSlack;
        if (!(cr >= -1.0)) cr = -1.0;  // also catches NaN
        if (cr > 1.0) cr = 1.0;
        double* rec = node + i * (m + 3);
        for (uint64_t k = 0; k < m; ++k) rec[k] = cv[k];
        rec[m] = cn;
        rec[m + 1] = cr;
        rec[m + 2] = sqrt(fmax(0.0, 1.0 - cr * cr));
        centre_pos[i] = (uint32_t)c;
    }
}

// Same record for a node with many members (levels >= 2: spans of 1024 positions and more): one CTA per node instead
// of one warp, so that the few big nodes at the top of the tree do not serialise the rebuild after an adaptation.
// Identical arithmetic per member; the centre is again the member closest to the mean direction (ties -> lowest
// position) and the radius is exact for that centre, so any difference in the mean's summation order can only pick
// another valid centre.
__global__ void __launch_bounds__(256) node_build_block_kernel(const double* vp, uint64_t r, uint64_t m, uint64_t span, uint64_t count,
                                                                double* node, uint32_t* centre_pos) {
    __shared__ double s_mean[kMaxObj];
    __shared__ double s_val[8];
    __shared__ uint64_t s_pos[8];
    const uint64_t i = blockIdx.x;
    if (i >= count) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t a = i * span, b = (a + span < r) ? a + span : r;
    for (uint64_t k = 0; k < m; ++k) {  // mean direction, one component at a time (m <= 32)
        double acc = 0.0;
        for (uint64_t p = a + threadIdx.x; p < b; p += blockDim.x) acc += vp[p * (m + 1) + k] / vp[p * (m + 1) + m];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) s_val[warp] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < 8; ++w) t += s_val[w];
            s_mean[k] = t;
        }
        __syncthreads();
    }
    double best = -INFINITY;
    uint64_t best_p = a;
    for (uint64_t p = a + threadIdx.x; p < b; p += blockDim.x) {
        double dot = 0.0;
        for (uint64_t k = 0; k < m; ++k) dot += s_mean[k] * vp[p * (m + 1) + k];
        dot /= vp[p * (m + 1) + m];
        if (dot > best) {
            best = dot;
            best_p = p;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, off);
        const uint64_t op = __shfl_xor_sync(0xffffffffu, best_p, off);
        if (ob > best || (ob == best && op < best_p)) {
            best = ob;
            best_p = op;
        }
    }
    if (lane == 0) s_val[warp] = best, s_pos[warp] = best_p;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w)
            if (s_val[w] > s_val[0] || (s_val[w] == s_val[0] && s_pos[w] < s_pos[0])) s_val[0] = s_val[w], s_pos[0] = s_pos[w];
    }
    __syncthreads();
    const uint64_t c = s_pos[0];
    __syncthreads();
    const double* cv = vp + c * (m + 1);
    const double cn = cv[m];
    double lo = 2.0;
    for (uint64_t p = a + threadIdx.x; p < b; p += blockDim.x) {
        const double* pv = vp + p * (m + 1);
        double dot = 0.0;
        for (uint64_t k = 0; k < m; ++k) dot += cv[k] * pv[k];
        const double cs = dot / (cn * pv[m]);
        lo = cs < lo ? cs : lo;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, lo, off);
        lo = o < lo ? o : lo;
    }
    if (lane == 0) s_val[warp] = lo;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) lo = s_val[w] < lo ? s_val[w] : lo;
        double cr = lo - kSlack;
        if (!(cr >= -1.0)) cr = -1.0;  // also catches NaN
        if (cr > 1.0) cr = 1.0;
        double* rec = node + i * (m + 3);
        for (uint64_t k = 0; k < m; ++k) rec[k] = cv[k];
        rec[m] = cn;
        rec[m + 1] = cr;
        rec[m + 2] = sqrt(fmax(0.0, 1.0 - cr * cr));
        centre_pos[i] = (uint32_t)c;
    }
}

struct IndexView {
    const double* vp;
    const uint32_t* orig;
    uint64_t r;
    int levels;
    uint64_t count[VecIndex::kMaxLevels + 1];
    const double* node[VecIndex::kMaxLevels + 1];
    const uint32_t* centre[VecIndex::kMaxLevels + 1];
};

template <int M>
struct Row {
    double u[M > 0 ? M : kMaxObj];
    double nf;
    uint32_t self;  // original index to exclude (gamma) or 0xffffffff
};

// float lower bound of a non-negative cosine, warp-wide maximum (REDUX on the order-preserving bits)
__device__ __forceinline__ float warp_max_lower(double c, float cur) {
    float f = (c > 0.0) ? __double2float_rd(c) : 0.0f;
    if (!(f >= 0.0f)) f = 0.0f;  // NaN
    const unsigned bits = __reduce_max_sync(0xffffffffu, __float_as_uint(f));
    const float w = __uint_as_float(bits);
    return w > cur ? w : cur;
}

template <int M>
struct Searcher {
    static constexpr int MM = M > 0 ? M : kMaxObj;
    const IndexView& ix;
    const Row<M>& row;
    int m;
    int lane;
    double best_c;
    uint32_t best_j;
    float Lf;
    float Lf_seen;  // the L for which (Lb, Sb) below were computed
    double Lb, Sb;  // L - slack and sqrt(1 - Lb^2)
    bool exact_all;  // exhaustive scans (rows or vector sets with negative components): L says nothing about negative cosines

    __device__ __forceinline__ double dot_with(const double* rec) const {  // ascending k, multiply and add: the reference's dot
        double dot = 0.0;
#pragma unroll
        for (int k = 0; k < MM; ++k)
            if (k < m) dot += row.u[k] * rec[k];
        return dot;
    }
    __device__ __forceinline__ double cosine_approx(const double* rec) const {  // within kApprox of the exact expression
        return dot_with(rec) * rcp_approx(row.nf * rec[m]);
    }

    // q: approximate cosine to the node's centre
    __device__ __forceinline__ bool passes(double q, double cr, double sr) {
        if (Lf != Lf_seen) {  // warp-uniform: L is the same in every lane
            Lf_seen = Lf;
            Lb = (double)Lf - kSlack;
            Sb = sqrt(fmax(0.0, 1.0 - Lb * Lb));
        }
        return q + (kSlack + kApprox) >= Lb * cr - Sb * sr;
    }

    __device__ __forceinline__ void leaf(uint64_t group) {
        const uint64_t p = group * 32 + lane;
        double c = -1.0;
        if (p < ix.r) {
            const uint32_t j = ix.orig[p];
            if (j != row.self) {
                const double* rec = ix.vp + p * (m + 1);
                const double dot = dot_with(rec), den = row.nf * rec[m];
                // L is a lower bound of a cosine some vector has realised: a vector whose cosine cannot reach it is not
                // the maximum (nor a tie for it) and is not divided for
                if (exact_all || !(dot * rcp_approx(den) + kApprox < (double)Lf)) {
                    c = dot / den;  // selection.hpp:178 / refvec.hpp:92
                    if (c > best_c || (c == best_c && j < best_j)) {
                        best_c = c;
                        best_j = j;
                    }
                }
            }
        }
        Lf = warp_max_lower(c, Lf);
    }

    // Depth-first over the children [a, b) of a level-(lvl+1) node; lvl >= 1.
    template <int LVL>
    __device__ void descend(uint64_t a, uint64_t b) {
        for (uint64_t base = a; base < b; base += 32) {
            const uint64_t id = base + lane;
            const bool valid = id < b;
            double q = -1.0, cr = 1.0, sr = 0.0;
            if (valid) {
                const double* rec = ix.node[LVL] + id * (m + 3);
                q = cosine_approx(rec);
                cr = rec[m + 1];
                sr = rec[m + 2];
                if (!(q == q)) q = 2.0;  // a NaN cosine never prunes
            }
            // a centre is a realised cosine: it raises L (by its lower bound) unless it is the excluded vector itself
            const bool is_self = valid && row.self != 0xffffffffu && ix.orig[ix.centre[LVL][id]] == row.self;
            Lf = warp_max_lower((valid && !is_self && q <= 1.5) ? q - kApprox : -1.0, Lf);
            unsigned done = 0;
            // best-first: the passing child whose centre is closest to the row is opened first, which raises L to
            // (nearly) its final value at once and prunes most siblings; the order of visits does not change the
            // result (lexicographic reduction over everything visited, conservative pruning)
            const unsigned qkey = __float_as_uint(fminf(fmaxf(__double2float_rn(q), 0.0f), 4.0f));  // q in [0, 2]: bits are monotone
            for (;;) {
                const bool open = valid && !((done >> lane) & 1u) && passes(q, cr, sr);
                const unsigned mask = __ballot_sync(0xffffffffu, open);
                if (!mask) break;
                const unsigned top = __reduce_max_sync(0xffffffffu, open ? qkey : 0u);
                const unsigned pick = __ballot_sync(0xffffffffu, open && qkey == top);
                const int bsel = __ffs(pick ? pick : mask) - 1;
                done |= 1u << bsel;
                const uint64_t child = base + bsel;
                if (LVL == 1) {
                    leaf(child);
                } else {
                    const uint64_t ca = child * 32;
                    const uint64_t cb = ca + 32 < ix.count[LVL - 1] ? ca + 32 : ix.count[LVL - 1];
                    descend<(LVL > 1 ? LVL - 1 : 1)>(ca, cb);
                }
            }
        }
    }

    __device__ void exhaustive() {
        for (uint64_t g = 0; g * 32 < ix.r; ++g) leaf(g);
    }

    __device__ void finish() {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double oc = __shfl_xor_sync(0xffffffffu, best_c, off);
            const uint32_t oj = __shfl_xor_sync(0xffffffffu, best_j, off);
            if (oc > best_c || (oc == best_c && oj < best_j)) {
                best_c = oc;
                best_j = oj;
            }
        }
    }
};

template <int M>
__device__ __forceinline__ void search_row(const IndexView& ix, const Row<M>& row, int m, bool prunable,
                                           double* best_c, uint32_t* best_j) {
    Searcher<M> s{ix, row, m, (int)(threadIdx.x & 31), -INFINITY, 0xffffffffu, 0.0f, -1.0f, 0.0, 1.0, !prunable};
    if (!prunable) {
        s.exhaustive();
    } else {
        switch (ix.levels) {
        case 1: s.template descend<1>(0, ix.count[1]); break;
        case 2: s.template descend<2>(0, ix.count[2]); break;
        case 3: s.template descend<3>(0, ix.count[3]); break;
        default: s.template descend<4>(0, ix.count[4]); break;
        }
    }
    s.finish();
    *best_c = s.best_c;
    *best_j = s.best_j;
}

#ifndef TEMO_INDEX_WARPS
#define TEMO_INDEX_WARPS 4
#endif
constexpr int kWarpsPerCta = TEMO_INDEX_WARPS;
#ifndef TEMO_INDEX_MIN_CTAS
#define TEMO_INDEX_MIN_CTAS 8
#endif

// Association + APD for the merged objective rows (selection.hpp:148-192), one warp per row.
template <int M>
__global__ void __launch_bounds__(kWarpsPerCta * 32, TEMO_INDEX_MIN_CTAS) assoc_indexed_kernel(
    const double* __restrict__ f, uint64_t n_rows, const uint32_t* n_rows_dev, uint64_t m_rt,
    const double* __restrict__ z, const IndexView ix, const uint32_t* __restrict__ vflags, const double* __restrict__ gamma,
    double penalty, uint32_t* __restrict__ assoc, double* __restrict__ theta_out, double* __restrict__ apd_out,
    unsigned long long* __restrict__ best_key, uint32_t* __restrict__ first_row, uint32_t row0) {
    constexpr int MM = M > 0 ? M : kMaxObj;
    const int m = M > 0 ? M : (int)m_rt;
    const uint64_t n = n_rows_dev ? (uint64_t)*n_rows_dev : n_rows;
    const uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    if (i >= n) return;  // warp-uniform
    Row<M> row;
    row.self = 0xffffffffu;
    double s = 0.0;
    bool nonneg = true;
#pragma unroll
    for (int k = 0; k < MM; ++k) {
        if (k < m) {
            row.u[k] = f[i * m + k] - z[k];  // selection.hpp:155-157
            s += row.u[k] * row.u[k];
            if (!(row.u[k] >= 0.0)) nonneg = false;
        }
    }
    row.nf = sqrt(s);
    uint32_t arg = 0;
    double theta = 0.0;  // a row at the ideal point: angle 0 to vector 0 (selection.hpp:167-169)
    if (row.nf != 0.0) {
        const bool finite = row.nf < INFINITY;  // false for inf and NaN
        double best_c;
        uint32_t best_j;
        search_row<M>(ix, row, m, (*vflags & 1u) == 0 && nonneg && finite, &best_c, &best_j);
        if (best_j != 0xffffffffu) arg = best_j;  // no comparable cosine (NaN row): reference keeps arg = 0
        double c = best_j != 0xffffffffu ? best_c : -INFINITY;
        if (c > 1.0) c = 1.0;
        if (c < -1.0) c = -1.0;
        theta = acos(c);  // tensor.hpp:79-83
    }
    if ((threadIdx.x & 31) != 0) return;
    const double apd = (1.0 + penalty * (theta / gamma[arg])) * row.nf;  // selection.hpp:82-84
    assoc[i] = arg;
    theta_out[i] = theta;
    apd_out[i] = apd;
    const unsigned long long key = (apd != apd) ? kKeyMax : order_key(apd);
    atomicMin(&best_key[arg], key);
    atomicMin(&first_row[arg], row0 + (uint32_t)i);  // row0: merged-row number of this launch's first row
}

// gamma_i = acos(max_{j != i} cos(v_i, v_j)) (refvec.hpp:81-100), one warp per vector.
template <int M>
__global__ void __launch_bounds__(kWarpsPerCta * 32, TEMO_INDEX_MIN_CTAS) gamma_indexed_kernel(
    const double* __restrict__ v, const double* __restrict__ vn, uint64_t r, uint64_t m_rt, const IndexView ix,
    const uint32_t* __restrict__ vflags, double* __restrict__ gamma, uint32_t* err_flag, const uint32_t* skip_flag) {
    if (skip_flag && *skip_flag) return;
    constexpr int MM = M > 0 ? M : kMaxObj;
    const int m = M > 0 ? M : (int)m_rt;
    const uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    if (i >= r) return;
    Row<M> row;
    row.self = (uint32_t)i;
#pragma unroll
    for (int k = 0; k < MM; ++k)
        if (k < m) row.u[k] = v[i * m + k];
    row.nf = vn[i];
    double best_c;
    uint32_t best_j;
    search_row<M>(ix, row, m, (*vflags & 1u) == 0 && row.nf > 0.0 && row.nf < INFINITY, &best_c, &best_j);
    if ((threadIdx.x & 31) != 0) return;
    double c = best_j != 0xffffffffu ? best_c : -INFINITY;
    if (c > 1.0) c = 1.0;
    if (c < -1.0) c = -1.0;
    const double g = acos(c);
    gamma[i] = g;
    if (!(g > 0.0)) atomicOr(err_flag, 1u);  // refvec.hpp:97-98
}

IndexView view_of(const VecIndex& x) {
    IndexView v{};
    v.vp = x.vp;
    v.orig = x.orig;
    v.r = x.r;
    v.levels = x.levels;
    for (int l = 1; l <= x.levels; ++l) {
        v.count[l] = x.count[l];
        v.node[l] = x.node[l];
        v.centre[l] = x.centre[l];
    }
    return v;
}

}  // namespace

// Hilbert-curve order of the vectors' simplex coordinates v / sum(v) (first m-1 of them, quantised to
// B bits each). Consecutive cells of a Hilbert curve are always adjacent, so every run of 32^k consecutive
// positions is a connected, compact patch of directions (a Morton/Z-order run can straddle a long jump:
// measured on the m = 3, H = 510 lattice the worst 32-vector group spans 60 degrees in Z-order, 2.4 in
// Hilbert order, and the search visits 2.8x fewer nodes). Transform: J. Skilling, "Programming the Hilbert
// curve", AIP Conf. Proc. 707 (2004) — axes to transposed index, then bit interleave.
std::vector<uint32_t> morton_order(const double* v, uint64_t r, uint64_t m) {
    const int dims = (int)(m > 1 ? m - 1 : 1);
    int bits = 60 / dims;
    if (bits > 16) bits = 16;
    if (bits < 1) bits = 1;
    const double scale = (double)((1u << bits) - 1);
    std::vector<uint64_t> key(r);
    std::vector<uint32_t> x(dims);
    for (uint64_t j = 0; j < r; ++j) {
        double sum = 0.0;
        for (uint64_t k = 0; k < m; ++k) sum += std::fabs(v[j * m + k]);
        for (int k = 0; k < dims; ++k) {
            double a = sum > 0.0 ? std::fabs(v[j * m + k]) / sum : 0.0;
            if (!(a >= 0.0)) a = 0.0;
            if (a > 1.0) a = 1.0;
            x[k] = (uint32_t)(a * scale + 0.5);
        }
        if (bits > 1 && dims > 1) {
            const uint32_t top = 1u << (bits - 1);
            for (uint32_t q = top; q > 1; q >>= 1) {  // inverse undo of excess work
                const uint32_t pmask = q - 1;
                for (int i = 0; i < dims; ++i) {
                    if (x[i] & q) {
                        x[0] ^= pmask;
                    } else {
                        const uint32_t t = (x[0] ^ x[i]) & pmask;
                        x[0] ^= t;
                        x[i] ^= t;
                    }
                }
            }
            for (int i = 1; i < dims; ++i) x[i] ^= x[i - 1];  // Gray encode
            uint32_t t = 0;
            for (uint32_t q = top; q > 1; q >>= 1)
                if (x[dims - 1] & q) t ^= q - 1;
            for (int i = 0; i < dims; ++i) x[i] ^= t;
        }
        uint64_t code = 0;
        for (int b = bits - 1; b >= 0; --b)
            for (int k = 0; k < dims; ++k) code = (code << 1) | ((x[k] >> b) & 1u);
        key[j] = code;
    }
    std::vector<uint32_t> order(r);
    std::iota(order.begin(), order.end(), 0u);
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return key[a] < key[b]; });
    return order;
}

void VecIndex::alloc(uint64_t r_, uint64_t m_) {
    r = r_;
    m = m_;
    orig = dev_alloc<uint32_t>(r);
    vp = dev_alloc<double>(r * (m + 1));
    flags = dev_alloc<uint32_t>(1);
    levels = 0;
    uint64_t cnt = r;
    for (int l = 1; l <= kMaxLevels; ++l) {
        cnt = (cnt + 31) / 32;
        count[l] = cnt;
        node[l] = dev_alloc<double>(cnt * (m + 3));
        centre[l] = dev_alloc<uint32_t>(cnt);
        levels = l;
        if (cnt <= 32) break;
    }
    ordered = false;
    built = false;
}

void VecIndex::release() {
    cudaFree(orig);
    cudaFree(vp);
    cudaFree(flags);
    for (int l = 1; l <= kMaxLevels; ++l) {
        cudaFree(node[l]);
        cudaFree(centre[l]);
    }
    *this = VecIndex{};
}

void VecIndex::set_order(const double* v_host, cudaStream_t s) {
    const std::vector<uint32_t> order = morton_order(v_host, r, m);
    TEMO_CUDA(cudaMemcpyAsync(orig, order.data(), r * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    TEMO_CUDA(cudaStreamSynchronize(s));  // `order` goes out of scope
    ordered = true;
}

// (Re)builds the permuted copy and every node record from the current V; cheap (a few passes
// over R x m doubles), called at init and after each adaptation.
void VecIndex::build(const double* v, const double* vn, cudaStream_t s) {
    require(ordered, "VecIndex: order not set");
    TEMO_CUDA(cudaMemsetAsync(flags, 0, sizeof(uint32_t), s));
    gather_perm_kernel<<<(unsigned)((r + 255) / 256), 256, 0, s>>>(v, vn, orig, r, m, vp, flags);
    uint64_t span = 1;
    for (int l = 1; l <= levels; ++l) {
        span *= 32;
        if (l >= 2) {
            node_build_block_kernel<<<(unsigned)count[l], 256, 0, s>>>(vp, r, m, span, count[l], node[l], centre[l]);
        } else {
            const uint64_t threads = count[l] * 32;
            node_build_kernel<<<(unsigned)((threads + 127) / 128), 128, 0, s>>>(vp, r, m, span, count[l], node[l], centre[l]);
        }
    }
    TEMO_CUDA(cudaGetLastError());
    built = true;
}

#define TEMO_DISPATCH_M(m, CALL)        \
    switch (m) {                        \
    case 2: CALL(2); break;             \
    case 3: CALL(3); break;             \
    case 4: CALL(4); break;             \
    case 5: CALL(5); break;             \
    case 10: CALL(10); break;           \
    default: CALL(0); break;            \
    }

void launch_assoc_indexed(const double* f, uint64_t n_rows, const uint32_t* n_rows_dev, uint64_t m, const double* z,
                          VecIndex& index, const double* gamma, double penalty, uint32_t* assoc, double* theta,
                          double* apd, unsigned long long* best_key, uint32_t* first_row, cudaStream_t s, uint32_t row0) {
    require(index.built, "VecIndex: not built");
    const IndexView view = view_of(index);
    const unsigned grid = (unsigned)((n_rows + kWarpsPerCta - 1) / kWarpsPerCta);
#define CALL(MV) \
    assoc_indexed_kernel<MV><<<grid, kWarpsPerCta * 32, 0, s>>>(f, n_rows, n_rows_dev, m, z, view, index.flags, gamma, penalty, \
                                                               assoc, theta, apd, best_key, first_row, row0)
    TEMO_DISPATCH_M(m, CALL)
#undef CALL
    TEMO_CUDA(cudaGetLastError());
}

void launch_gamma_indexed(const double* v, const double* vn, uint64_t r, uint64_t m, VecIndex& index, double* gamma,
                          uint32_t* err_flag, const uint32_t* skip_flag, cudaStream_t s) {
    require(index.built, "VecIndex: not built");
    const IndexView view = view_of(index);
    const unsigned grid = (unsigned)((r + kWarpsPerCta - 1) / kWarpsPerCta);
#define CALL(MV) \
    gamma_indexed_kernel<MV><<<grid, kWarpsPerCta * 32, 0, s>>>(v, vn, r, m, view, index.flags, gamma, err_flag, skip_flag)
    TEMO_DISPATCH_M(m, CALL)
#undef CALL
    TEMO_CUDA(cudaGetLastError());
}

}  // namespace temo_b200
