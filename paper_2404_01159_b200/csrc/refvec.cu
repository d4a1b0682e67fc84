// K4 — reference-vector adaptation and the neighbour angles gamma.
//
// reference: adapt / adapt_vectors (refvec.hpp:119-140), normalize_to_unit (refvec.hpp:65-75)
// and min_vector_angles (refvec.hpp:81-100). The reference materialises the dense R x R cosine
// matrix (136.9 GB at R = 130816); here every thread owns one vector and streams all others
// through shared-memory tiles, keeping the exact per-pair arithmetic: ascending-k dot product,
// IEEE divide by (norm_i * norm_j), strict `>` max, one acos per vector.
#include "internal.h"

namespace temo_b200 {

namespace {

constexpr int kGammaThreads = 128;
constexpr int kGammaTile = 512;

template <int M>
__global__ void __launch_bounds__(kGammaThreads) gamma_kernel(const double* __restrict__ v,
                                                             const double* __restrict__ vn, uint64_t r,
                                                             uint64_t m_rt, double* __restrict__ gamma,
                                                             uint32_t* err_flag, const uint32_t* skip_flag) {
    if (skip_flag && *skip_flag) return;
    constexpr int MM = M > 0 ? M : kMaxObj;
    const int m = M > 0 ? M : (int)m_rt;
    extern __shared__ double s_tile[];
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const bool live = i < r;
    double vi[MM];
    double ni = 0.0;
    if (live) {
#pragma unroll
        for (int k = 0; k < MM; ++k)
            if (k < m) vi[k] = v[i * m + k];
        ni = vn[i];
    }
    double best = -INFINITY;
    const int stride = m + 1;
    for (uint64_t j0 = 0; j0 < r; j0 += kGammaTile) {
        const int tile = (int)((r - j0) < (uint64_t)kGammaTile ? (r - j0) : kGammaTile);
        __syncthreads();
        for (int e = threadIdx.x; e < tile * stride; e += blockDim.x) {
            const int jj = e / stride, k = e - jj * stride;
            s_tile[e] = k < m ? v[(j0 + jj) * m + k] : vn[j0 + jj];
        }
        __syncthreads();
        if (live) {
            for (int jj = 0; jj < tile; ++jj) {
                if (j0 + jj == i) continue;  // refvec.hpp:91
                const double* vr = s_tile + jj * stride;
                double dot = 0.0;
#pragma unroll
                for (int k = 0; k < MM; ++k)
                    if (k < m) dot += vi[k] * vr[k];
                const double c = dot / (ni * vr[m]);  // refvec.hpp:92
                if (c > best) best = c;
            }
        }
    }
    if (!live) return;
    double c = best;
    if (c > 1.0) c = 1.0;
    if (c < -1.0) c = -1.0;
    const double g = acos(c);
    gamma[i] = g;
    if (!(g > 0.0)) atomicOr(err_flag, 1u);  // refvec.hpp:97-98: duplicate reference vectors
}

__global__ void adapt_gate_kernel(const double* zmin, const double* zmax, uint64_t m, uint32_t* skip_flag) {
    uint32_t skip = 0;
    for (uint64_t k = 0; k < m; ++k)
        if (!(zmax[k] > zmin[k])) skip = 1;  // refvec.hpp:136-137
    *skip_flag = skip;
}

__global__ void adapt_vectors_kernel(const double* __restrict__ v0, double* __restrict__ v,
                                     double* __restrict__ vn, uint64_t r, uint64_t m,
                                     const double* __restrict__ zmin, const double* __restrict__ zmax,
                                     const uint32_t* skip_flag, uint32_t* err_flag) {
    if (*skip_flag) return;
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= r) return;
    double s = 0.0;
    for (uint64_t k = 0; k < m; ++k) {
        const double scaled = v0[i * m + k] * (zmax[k] - zmin[k]);  // refvec.hpp:126-129
        s += scaled * scaled;
    }
    const double norm = sqrt(s);  // refvec.hpp:69-71
    if (!(norm > 0.0)) {
        atomicOr(err_flag, 2u);
        return;
    }
    double s2 = 0.0;
    for (uint64_t k = 0; k < m; ++k) {
        const double scaled = v0[i * m + k] * (zmax[k] - zmin[k]);
        const double u = scaled / norm;
        v[i * m + k] = u;
        s2 += u * u;
    }
    vn[i] = sqrt(s2);  // row_norms of the new set (tensor.hpp:171-182), reused by selection
}

template <int M>
void launch_gamma_m(const double* v, const double* vn, uint64_t r, uint64_t m, double* gamma,
                    uint32_t* err_flag, const uint32_t* skip_flag, cudaStream_t s) {
    const size_t smem = (size_t)kGammaTile * (m + 1) * sizeof(double);
    if (smem > 48 * 1024) {
        static bool configured = false;
        if (!configured) {
            TEMO_CUDA(cudaFuncSetAttribute(gamma_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            configured = true;
        }
    }
    gamma_kernel<M><<<(unsigned)((r + kGammaThreads - 1) / kGammaThreads), kGammaThreads, smem, s>>>(
        v, vn, r, m, gamma, err_flag, skip_flag);
}

}  // namespace

void launch_gamma(const double* v, const double* vn, uint64_t r, uint64_t m, double* gamma,
                  uint32_t* err_flag, const uint32_t* skip_flag, cudaStream_t s) {
    require(r >= 2, "min_vector_angles: needs at least two vectors");  // refvec.hpp:82
    require(m >= 1 && m <= (uint64_t)kMaxObj, "min_vector_angles: unsupported objective count");
    switch (m) {
    case 2: launch_gamma_m<2>(v, vn, r, m, gamma, err_flag, skip_flag, s); break;
    case 3: launch_gamma_m<3>(v, vn, r, m, gamma, err_flag, skip_flag, s); break;
    case 4: launch_gamma_m<4>(v, vn, r, m, gamma, err_flag, skip_flag, s); break;
    case 5: launch_gamma_m<5>(v, vn, r, m, gamma, err_flag, skip_flag, s); break;
    case 10: launch_gamma_m<10>(v, vn, r, m, gamma, err_flag, skip_flag, s); break;
    default: launch_gamma_m<0>(v, vn, r, m, gamma, err_flag, skip_flag, s); break;
    }
    TEMO_CUDA(cudaGetLastError());
}

// Loads the kernels a run first needs at its first adaptation (lazy module loading would do it there, see init_context).
void preload_adapt_kernels() {
    cudaFuncAttributes attr;
    TEMO_CUDA(cudaFuncGetAttributes(&attr, adapt_gate_kernel));
    TEMO_CUDA(cudaFuncGetAttributes(&attr, adapt_vectors_kernel));
}

void launch_adapt_vectors(const double* v0, double* v, double* vn, uint64_t r, uint64_t m,
                          const double* zmin, const double* zmax, uint32_t* skip_flag,
                          uint32_t* err_flag, cudaStream_t s) {
    adapt_gate_kernel<<<1, 1, 0, s>>>(zmin, zmax, m, skip_flag);
    adapt_vectors_kernel<<<(unsigned)((r + 255) / 256), 256, 0, s>>>(v0, v, vn, r, m, zmin, zmax, skip_flag,
                                                                    err_flag);
    TEMO_CUDA(cudaGetLastError());
}

}  // namespace temo_b200
