// Micro-benchmark: time the phases of the in-register 32x32 warp Cholesky with clock64.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kCB = 32;
__device__ __forceinline__ void warp_chol32(double (&c)[kCB], double (&x)[kCB], int lane, long long* t) {
    long long t0 = clock64();
#pragma unroll
    for (int k = 0; k < kCB; ++k) {
        const double d = __shfl_sync(0xffffffffu, c[k], k);
        const double s = sqrt(d);
        const double inv = 1.0 / s;
        const double rkj = lane == k ? s : c[k] * inv;
        c[k] = rkj;
#pragma unroll
        for (int i = k + 1; i < kCB; ++i) {
            const double rki = __shfl_sync(0xffffffffu, rkj, i);
            c[i] = fma(-rki, rkj, c[i]);
        }
    }
    long long t1 = clock64();
#pragma unroll
    for (int j = 0; j < kCB; ++j) {
        double acc = lane == j ? 1.0 : 0.0;
#pragma unroll
        for (int p = 0; p < j; ++p) acc = fma(-x[p], __shfl_sync(0xffffffffu, c[p], j), acc);
        x[j] = acc / __shfl_sync(0xffffffffu, c[j], j);
    }
    long long t2 = clock64();
    if (lane == 0) { t[0] = t1 - t0; t[1] = t2 - t1; }
}
__global__ void k(const double* g, double* out, long long* t) {
    int lane = threadIdx.x;
    double c[kCB], x[kCB];
#pragma unroll
    for (int i = 0; i < kCB; ++i) { c[i] = g[i * 32 + lane]; x[i] = 0; }
    warp_chol32(c, x, lane, t);
#pragma unroll
    for (int i = 0; i < kCB; ++i) { out[i * 32 + lane] = c[i] + x[i]; }
}
int main() {
    double h[1024];
    for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) h[i * 32 + j] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + i + j);
    double *dg, *dout; long long* dt; long long ht[2];
    cudaMalloc(&dg, 8192); cudaMalloc(&dout, 8192); cudaMalloc(&dt, 16);
    cudaMemcpy(dg, h, 8192, cudaMemcpyHostToDevice);
    for (int r = 0; r < 3; ++r) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0); k<<<1, 32>>>(dg, dout, dt); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(ht, dt, 16, cudaMemcpyDeviceToHost);
        printf("chol %lld cycles, inverse %lld cycles, kernel %.1f us\n", ht[0], ht[1], ms * 1e3);
    }
    return 0;
}
