// developer: maximum relative error of rcp.approx.ftz.f64 (the reciprocal behind the index search's approximate cosines)
#include <cstdio>
#include <cstdint>
__global__ void k(double* out) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    double worst = 0.0;
    for (uint64_t i = 0; i < 4096; ++i) {
        uint64_t z = (t * 4096 + i) * 0x9E3779B97F4A7C15ULL;
        z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL; z ^= z >> 27; z *= 0x94D049BB133111EBULL; z ^= z >> 31;
        const double m = 1.0 + (double)(z >> 11) * 0x1.0p-53;          // [1, 2)
        const double x = ldexp(m, (int)(z & 63) - 32);                 // 2^-32 .. 2^31
        double r;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
        const double e = fabs(r * x - 1.0);
        worst = e > worst ? e : worst;
    }
    out[t] = worst;
}
int main() {
    const int n = 1 << 16;
    double* d; cudaMalloc(&d, n * sizeof(double));
    k<<<n / 256, 256>>>(d);
    static double h[1 << 16];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double w = 0; for (int i = 0; i < n; ++i) w = h[i] > w ? h[i] : w;
    printf("rcp.approx.ftz.f64 max relative error over 2.7e8 arguments: %.3e (2^-20 = 9.54e-07)\n", w);
    return 0;
}
