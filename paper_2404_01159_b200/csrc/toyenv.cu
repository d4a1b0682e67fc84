// Neuroevolution evaluator: MLP policy + toy control environment.
//
// reference: MlpArch / mlp_decode / mlp_forward (problems.hpp:105-163), toy_rollout (:176-206), env_rollout (:211-241)
// and the toy2 / toy3 entries of make_problem (:279-294). One individual = the flat parameter vector of a
// 4 - hidden - 2 tanh network (W1 row-major, b1, W2 row-major, b2); an episode runs `horizon` steps of the point-mass
// dynamics with the network as policy and returns 2 or 3 cumulative rewards (maximisation orientation).
//
// Compute-bound and strictly sequential per individual (18 tanh per step, every step feeds the next): sixteen lanes
// share an individual (one hidden unit each, parameters in registers), two individuals per warp. Every operation is the
// reference's, in its order
// (--fmad=false keeps `s += w * x` a multiply and an add like -ffp-contract=off); tanh follows the host libm operation
// for operation (glibc_tanh.cuh) and sin / cos of the phase come from a table the host libm fills once per horizon, so
// the returns are bit-identical to env_rollout's.
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "glibc_tanh.cuh"
#include "internal.h"

namespace temo_b200 {

namespace {

constexpr int kToyObs = 4, kToyAct = 2, kToyMaxHidden = 64;  // problems.hpp:173-174, 217

struct ToyK {
    const double* params;   // storage base, row stride d
    const uint32_t* rows;   // optional storage row of individual i
    uint64_t n, d;
    uint32_t hidden, horizon, m;
    const double* phase;    // [2 * horizon]: sin, cos of 2 pi t / horizon
    double* f;
    uint64_t f_row0;
    const uint32_t* f_row0_dev;
    int negate;             // make_problem's evaluate returns the negated returns (minimisation)
    const double* obs;      // mlp_forward mode: n x 4 observations (nullptr: episodes)
};

// Sixteen lanes per individual (two individuals per warp): lane s owns the hidden units s, s + 16, ... (U = ceil(hidden / 16)
// of them, their W1 rows, biases and W2 columns in registers). One step of the episode:
//   hidden unit i:  s = b1[i]; s += W1(i, j) * obs[j] for j = 0..3; h_i = tanh(s)              (problems.hpp:151-156, all units at once)
//   output o:       p_i = W2(o, i) * h_i goes to shared memory; even lanes then add b2[0] + p_0 + p_1 + ... in ascending i (the
//                   reference's order, problems.hpp:157-162), odd lanes the same for output 1, and take its tanh
//   state update:   every lane keeps (v, h, returns) redundantly (problems.hpp:196-201)
// The thread-per-individual form of the first version is 4x leaner in instructions but cannot be kept busy: at the paper's
// population of 10^4 it gives 68 threads per SM and every instruction waits out its full FP64 latency (1.94 ms per
// evaluation; this form: see DESIGN.md section 3.9).
constexpr int kToyLanes = 16;

template <int U>
__global__ void __launch_bounds__(128) toy_rollout_kernel(const ToyK a) {
    __shared__ __align__(16) double s_p[4][2][kToyAct][kToyMaxHidden];  // [warp][group][output][hidden unit]
    const uint32_t lane = threadIdx.x & 31, sub = lane & (kToyLanes - 1), grp = lane >> 4, warp = threadIdx.x >> 5;
    const uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / kToyLanes;
    const bool live = i < a.n;
    const uint32_t H = a.hidden;
    const uint32_t o_b1 = H * kToyObs, o_w2 = o_b1 + H, o_b2 = o_w2 + kToyAct * H;
    const double* p = a.params + (live ? (a.rows ? (uint64_t)a.rows[i] : i) : 0) * a.d;
    double w1[U][kToyObs], b1[U], w2[U][kToyAct];
    bool finite = true;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint32_t unit = sub + kToyLanes * u;
        const bool has = unit < H;
#pragma unroll
        for (int j = 0; j < kToyObs; ++j) w1[u][j] = has ? p[unit * kToyObs + j] : 0.0;
        b1[u] = has ? p[o_b1 + unit] : 0.0;
#pragma unroll
        for (int o = 0; o < kToyAct; ++o) w2[u][o] = has ? p[o_w2 + o * H + unit] : 0.0;
#pragma unroll
        for (int j = 0; j < kToyObs; ++j) finite &= fabs(w1[u][j]) < INFINITY;
        finite &= fabs(b1[u]) < INFINITY && fabs(w2[u][0]) < INFINITY && fabs(w2[u][1]) < INFINITY;
    }
    const double b2_0 = p[o_b2], b2_1 = p[o_b2 + 1];
    finite &= fabs(b2_0) < INFINITY && fabs(b2_1) < INFINITY;
    const unsigned bad = __ballot_sync(0xffffffffu, !finite);
    finite = ((bad >> (grp * kToyLanes)) & 0xffffu) == 0;  // problems.hpp:224-226: any non-finite parameter of the individual
    double (*sp)[kToyMaxHidden] = s_p[warp][grp];

    // one policy evaluation: ob -> (act0, act1), the same bits in every lane of the group
    auto policy = [&](const double* ob, double& act0, double& act1) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t unit = sub + kToyLanes * u;
            double s = b1[u];
#pragma unroll
            for (int j = 0; j < kToyObs; ++j) s += w1[u][j] * ob[j];
            const double hid = glibc_tanh(s);
            if (unit < H) {
                sp[0][unit] = w2[u][0] * hid;
                sp[1][unit] = w2[u][1] * hid;
            }
        }
        __syncwarp();
        // even lanes add output 0, odd lanes output 1 (one add per hidden unit and warp instead of two)
        const double* mine = sp[sub & 1];
        double so = (sub & 1) ? b2_1 : b2_0;
        for (uint32_t k = 0; k + 1 < H; k += 2) {  // ascending hidden unit, two per 128-bit read
            const double2 q = *reinterpret_cast<const double2*>(&mine[k]);
            so += q.x;
            so += q.y;
        }
        if (H & 1) so += mine[H - 1];
        __syncwarp();
        const double act = glibc_tanh(so);  // lanes 0 / 1 of the group hold the two actions
        act0 = __shfl_sync(0xffffffffu, act, grp * kToyLanes);
        act1 = __shfl_sync(0xffffffffu, act, grp * kToyLanes + 1);
    };

    if (a.obs) {  // mlp_forward: a single evaluation per individual
        double ob[kToyObs], act0, act1;
#pragma unroll
        for (int j = 0; j < kToyObs; ++j) ob[j] = live ? a.obs[i * kToyObs + j] : 0.0;
        policy(ob, act0, act1);
        if (live && sub == 0) {
            a.f[i * kToyAct] = act0;
            a.f[i * kToyAct + 1] = act1;
        }
        return;
    }
    const double h0 = 1.0;
    double v = 0.0, h = h0, fwd = 0.0, ctrl = 0.0, height = 0.0;
    double ob[kToyObs];
    for (uint32_t t = 0; t < a.horizon; ++t) {  // problems.hpp:187-202
        ob[0] = v;
        ob[1] = h;
        ob[2] = a.phase[2 * t];
        ob[3] = a.phase[2 * t + 1];
        double act0, act1;
        policy(ob, act0, act1);
        v = 0.9 * v + 0.1 * act0;
        h = clampd(0.95 * h + 0.1 * act1, 0.0, 2.0);
        fwd += v;
        ctrl -= act0 * act0 + act1 * act1;
        height += 10.0 * (h - h0);
    }
    if (!live || sub != 0) return;
    const uint64_t f0 = a.f_row0 + (a.f_row0_dev ? (uint64_t)*a.f_row0_dev : 0);
    double* fr = a.f + (f0 + i) * a.m;
    if (!finite) {
        for (uint32_t j = 0; j < a.m; ++j) fr[j] = a.negate ? 1e9 : -1e9;  // problems.hpp:227-230
        return;
    }
    if (a.m == 2) {
        fr[0] = a.negate ? -fwd : fwd;
        fr[1] = a.negate ? -ctrl : ctrl;
    } else {
        fr[0] = a.negate ? -fwd : fwd;
        fr[1] = a.negate ? -height : height;
        fr[2] = a.negate ? -ctrl : ctrl;
    }
}

// sin / cos of 2 pi t / horizon for t < horizon, from the host libm (the bits the reference's std::sin / std::cos give
// on this machine), cached per horizon
const double* toy_phase_table(uint64_t horizon, cudaStream_t s) {
    static std::mutex mu;
    static std::map<uint64_t, double*> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(horizon);
    if (it != cache.end()) return it->second;
    std::vector<double> host(2 * horizon + 2);
    const double two_pi = 2.0 * kPi;
    for (uint64_t t = 0; t < horizon; ++t) {
        const double phase = two_pi * (double)t / (double)horizon;  // problems.hpp:188
        host[2 * t] = std::sin(phase);
        host[2 * t + 1] = std::cos(phase);
    }
    double* dev = dev_alloc<double>(host.size());
    TEMO_CUDA(cudaMemcpyAsync(dev, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    TEMO_CUDA(cudaStreamSynchronize(s));
    cache[horizon] = dev;
    return dev;
}

void launch_toy_kernel(const ToyK& k, cudaStream_t s) {
    const unsigned grid = (unsigned)((k.n * kToyLanes + 127) / 128);
    switch ((k.hidden + kToyLanes - 1) / kToyLanes) {  // hidden units per lane
    case 1: toy_rollout_kernel<1><<<grid, 128, 0, s>>>(k); break;
    case 2: toy_rollout_kernel<2><<<grid, 128, 0, s>>>(k); break;
    case 3: toy_rollout_kernel<3><<<grid, 128, 0, s>>>(k); break;
    default: toy_rollout_kernel<4><<<grid, 128, 0, s>>>(k); break;
    }
    TEMO_CUDA(cudaGetLastError());
}

}  // namespace

namespace {
__global__ void tanh_batch_kernel(const double* x, uint64_t n, double* out) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x) out[e] = glibc_tanh(x[e]);
}
}  // namespace

// tanh with the host libm's bits, elementwise (self-test entry); host = the same source compiled for the CPU
void launch_tanh_batch(const double* x, uint64_t n, double* out, cudaStream_t s) {
    if (n == 0) return;
    tanh_batch_kernel<<<(unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)kSMs * 8), 256, 0, s>>>(x, n, out);
    TEMO_CUDA(cudaGetLastError());
}
void tanh_batch_host(const double* x, uint64_t n, double* out) {
    for (uint64_t e = 0; e < n; ++e) out[e] = glibc_tanh(x[e]);
}

uint64_t mlp_param_count(uint64_t hidden) { return kToyObs * hidden + hidden + hidden * kToyAct + kToyAct; }  // problems.hpp:113-115

// env_rollout (problems.hpp:211-241): params n x d (device; optional row indirection) -> f[(f_row0 + i) * m ..]
void launch_env_rollout(const double* params, const uint32_t* rows, uint64_t n, uint64_t d, uint64_t hidden, uint64_t horizon,
                        uint64_t m, bool negate, double* f, uint64_t f_row0, const uint32_t* f_row0_dev, cudaStream_t s) {
    require(hidden >= 1 && hidden <= (uint64_t)kToyMaxHidden, "env_rollout: hidden layer too wide");        // problems.hpp:217
    require(d == mlp_param_count(hidden), "env_rollout: parameter length mismatch");                        // problems.hpp:213
    require(m == 2 || m == 3, "env_rollout: the toy environment has 2 or 3 objectives");
    require(horizon < 0x7fffffffULL, "env_rollout: horizon too long");
    if (n == 0) return;
    ToyK k{params, rows, n, d, (uint32_t)hidden, (uint32_t)horizon, (uint32_t)m, toy_phase_table(horizon, s), f, f_row0, f_row0_dev,
           negate ? 1 : 0, nullptr};
    launch_toy_kernel(k, s);
}

// mlp_forward (problems.hpp:149-163) for n individuals, each on its own observation: obs n x 4 -> action n x 2
void launch_mlp_forward(const double* params, uint64_t n, uint64_t d, uint64_t hidden, const double* obs, double* action,
                        cudaStream_t s) {
    require(hidden >= 1 && hidden <= (uint64_t)kToyMaxHidden, "mlp_forward: hidden layer too wide");
    require(d == mlp_param_count(hidden), "mlp_decode: length mismatch");  // problems.hpp:127
    if (n == 0) return;
    ToyK k{params, nullptr, n, d, (uint32_t)hidden, 0u, (uint32_t)kToyAct, nullptr, action, 0, nullptr, 0, obs};
    launch_toy_kernel(k, s);
}

}  // namespace temo_b200
