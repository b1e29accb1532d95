// Micro: FP64 dependent-chain latency and single-warp issue rate (clocks), unrolled.
#include <cstdio>
__global__ void lat(double* out, long long* t, double y) {
    double x = 1.0 + threadIdx.x * 1e-9;
    double a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = x + i;
    __syncthreads();
    long long c0; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c0));
#pragma unroll
    for (int i = 0; i < 256; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %0;" : "+d"(x) : "d"(y));
    long long c1; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c1));
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %0;" : "+d"(a[i]) : "d"(y));
    long long c2; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c2));
    float xf = (float)y;
#pragma unroll
    for (int i = 0; i < 256; ++i) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(xf));
    long long c3; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c3));
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    if (threadIdx.x % 32 == 0) { int w = threadIdx.x / 32; t[w * 4 + 0] = c1 - c0; t[w * 4 + 1] = c2 - c1; t[w * 4 + 2] = c3 - c2; }
    out[threadIdx.x] = x + xf + s;
}
int main() {
    double* o; long long* t; cudaMalloc(&o, 8 * 1024); cudaMalloc(&t, 8 * 4 * 32);
    for (int nt : {32, 128, 288, 512}) {
        for (int r = 0; r < 2; ++r) lat<<<1, nt>>>(o, t, 1.0000001);
        long long h[4 * 32]; cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
        printf("threads %3d (warp 0): DFMA chain %.1f clk/op, 256 indep DFMA %.2f clk/instr, FFMA chain %.1f clk/op\n", nt,
               h[0] / 256.0, h[1] / 256.0, h[2] / 256.0);
    }
}
