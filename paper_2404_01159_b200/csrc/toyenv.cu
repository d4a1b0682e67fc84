// Neuroevolution evaluator: MLP policy + toy control environment.
//
// reference: MlpArch / mlp_decode / mlp_forward (problems.hpp:105-163), toy_rollout (:176-206), env_rollout (:211-241)
// and the toy2 / toy3 entries of make_problem (:279-294). One individual = the flat parameter vector of a
// 4 - hidden - 2 tanh network (W1 row-major, b1, W2 row-major, b2); an episode runs `horizon` steps of the point-mass
// dynamics with the network as policy and returns 2 or 3 cumulative rewards (maximisation orientation).
//
// Compute-bound and strictly sequential per individual (18 tanh per step, every step feeds the next): one thread per
// individual walks the episode; the parameters of a CTA's individuals sit in shared memory, parameter-major, so a
// warp's reads of "parameter k of my individual" are conflict-free. Every operation is the reference's, in its order
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

// action = tanh(W2 tanh(W1 obs + b1) + b2) (problems.hpp:149-163); w(k) reads parameter k of this thread's individual
template <class W>
__device__ __forceinline__ void mlp_forward_dev(const W& w, uint32_t H, const double* obs, double* hid, double* act) {
    const uint32_t o_b1 = H * kToyObs, o_w2 = o_b1 + H, o_b2 = o_w2 + kToyAct * H;
    for (uint32_t i = 0; i < H; ++i) {
        double s = w(o_b1 + i);
        for (uint32_t j = 0; j < (uint32_t)kToyObs; ++j) s += w(i * kToyObs + j) * obs[j];
        hid[i] = glibc_tanh(s);
    }
    for (uint32_t i = 0; i < (uint32_t)kToyAct; ++i) {
        double s = w(o_b2 + i);
        for (uint32_t j = 0; j < H; ++j) s += w(o_w2 + i * H + j) * hid[j];
        act[i] = glibc_tanh(s);
    }
}

__global__ void toy_rollout_kernel(const ToyK a) {
    extern __shared__ double s_w[];  // d x blockDim: parameter k of thread t at s_w[k * blockDim + t]
    const uint32_t B = blockDim.x;
    const uint64_t row0 = blockIdx.x * (uint64_t)B;
    // cooperative, coalesced staging of the CTA's rows
    for (uint32_t t = 0; t < B; ++t) {
        const uint64_t i = row0 + t;
        if (i >= a.n) break;
        const double* p = a.params + (a.rows ? (uint64_t)a.rows[i] : i) * a.d;
        for (uint32_t k = threadIdx.x; k < a.d; k += B) s_w[k * B + t] = p[k];
    }
    __syncthreads();
    const uint64_t i = row0 + threadIdx.x;
    if (i >= a.n) return;
    const auto w = [&](uint32_t k) { return s_w[k * B + threadIdx.x]; };
    const uint64_t f0 = a.f_row0 + (a.f_row0_dev ? (uint64_t)*a.f_row0_dev : 0);
    double hid[kToyMaxHidden], act[kToyAct];
    if (a.obs) {  // a single forward pass per individual
        double ob[kToyObs];
        for (int j = 0; j < kToyObs; ++j) ob[j] = a.obs[i * kToyObs + j];
        mlp_forward_dev(w, a.hidden, ob, hid, act);
        a.f[i * kToyAct] = act[0];
        a.f[i * kToyAct + 1] = act[1];
        return;
    }
    double* fr = a.f + (f0 + i) * a.m;
    bool finite = true;
    for (uint32_t k = 0; k < a.d; ++k) {
        const double p = w(k);
        if (!(fabs(p) < INFINITY)) finite = false;  // problems.hpp:224-226
    }
    if (!finite) {
        for (uint32_t j = 0; j < a.m; ++j) fr[j] = a.negate ? 1e9 : -1e9;  // problems.hpp:227-230
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
        mlp_forward_dev(w, a.hidden, ob, hid, act);
        v = 0.9 * v + 0.1 * act[0];
        h = clampd(0.95 * h + 0.1 * act[1], 0.0, 2.0);
        fwd += v;
        ctrl -= act[0] * act[0] + act[1] * act[1];
        height += 10.0 * (h - h0);
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

void launch_toy_kernel(ToyK k, cudaStream_t s) {
    // threads per CTA: as many individuals as fit ~100 KB of parameters (two CTAs per SM), a multiple of 32, at most 128
    uint32_t B = (uint32_t)(100 * 1024 / (k.d * sizeof(double))) / 32 * 32;
    if (B < 32) B = 32;
    if (B > 128) B = 128;
    const size_t smem = (size_t)k.d * B * sizeof(double);
    static size_t configured = 0;
    if (smem > configured) {
        TEMO_CUDA(cudaFuncSetAttribute(toy_rollout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    toy_rollout_kernel<<<(unsigned)((k.n + B - 1) / B), B, smem, s>>>(k);
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
