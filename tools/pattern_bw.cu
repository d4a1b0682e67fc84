// Developer microbenchmark: HBM bandwidth of K1's access pattern without any compute.
// Each 8-warp team handles row pairs; warp w reads the 512-byte blocks w, w+8, ... of two random parent rows and writes
// the same blocks of two other rows. mode 0: warps free-running (as in K1), mode 1: plain streaming copy of the same bytes.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 3) pattern(const double2* pool, double2* out, const unsigned* src, const unsigned* dst, unsigned half,
                                                   unsigned nvec, int delay) {
    const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (unsigned unit = blockIdx.x; unit < half; unit += gridDim.x) {
        const double2* pa = pool + (size_t)src[unit] * nvec;
        const double2* pb = pool + (size_t)src[half + unit] * nvec;
        double2* oa = out + (size_t)dst[unit] * nvec;
        double2* ob = out + (size_t)dst[half + unit] * nvec;
        // emulate the compute passes between memory phases: spin `delay` clocks per warp tile before streaming
        if (delay) { long long t0 = clock64(); while (clock64() - t0 < delay * (long long)(1 + (w & 3))) {} }
        for (unsigned q = w * 32 + lane; q < nvec; q += 256) {
            const double2 a = __ldcs(pa + q), b = __ldcs(pb + q);
            __stcs(oa + q, make_double2(a.x + b.x, a.y));
            __stcs(ob + q, make_double2(b.x, a.y + b.y));
        }
    }
}
__global__ void stream_copy(const double2* in, double2* out, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) out[i] = in[i];
}
int main(int argc, char** argv) {
    const unsigned n = 1 << 17, d = 5000, nvec = d / 2, half = n / 2;
    const size_t rows = 2 * (size_t)n, bytes = rows * d * 8;
    double2 *pool; unsigned *src, *dst;
    cudaMalloc(&pool, bytes); cudaMemset(pool, 0, bytes);
    std::vector<unsigned> hs(n), hd(n);
    srand(1);
    std::vector<unsigned> perm(rows); for (size_t i = 0; i < rows; ++i) perm[i] = i;
    for (size_t i = rows - 1; i > 0; --i) { size_t j = ((size_t)rand() * RAND_MAX + rand()) % (i + 1); std::swap(perm[i], perm[j]); }
    for (unsigned i = 0; i < n; ++i) { hs[i] = perm[i]; hd[i] = perm[n + i]; }
    cudaMalloc(&src, n * 4); cudaMalloc(&dst, n * 4);
    cudaMemcpy(src, hs.data(), n * 4, cudaMemcpyHostToDevice); cudaMemcpy(dst, hd.data(), n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const double gb = 16.0 * n * d / 1e9;
    for (int delay : {0, 2000, 8000, 20000}) {
        for (int rep = 0; rep < 2; ++rep) pattern<<<148 * 3, 256>>>(pool, pool, src, dst, half, nvec, delay);
        cudaEventRecord(e0);
        for (int rep = 0; rep < 5; ++rep) pattern<<<148 * 3, 256>>>(pool, pool, src, dst, half, nvec, delay);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
        printf("pattern delay=%5d: %.3f ms  %.0f GB/s\n", delay, ms, gb / ms * 1e3 / 1e0 / 1e3 * 1e3);
    }
    cudaEventRecord(e0);
    for (int rep = 0; rep < 5; ++rep) stream_copy<<<148 * 8, 512>>>(pool, pool + (size_t)n * nvec, (size_t)n * nvec);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("stream copy: %.3f ms  %.0f GB/s\n", ms, gb / ms * 1e3);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
