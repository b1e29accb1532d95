// Micro: FP64 CUDA-core throughput (DFMA) and libdevice log/sincos throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_k(double* out, int iters) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 0.999999, c = 1e-9;
    for (int i = 0; i < iters; ++i) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void ffma_k(float* out, int iters) {
    float a0 = threadIdx.x * 1e-3f, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const float b = 0.999999f, c = 1e-9f;
    for (int i = 0; i < iters; ++i) {
        a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
        a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void trans_k(double* out, int iters) {
    double x = 0.1 + threadIdx.x * 1e-4, acc = 0;
    for (int i = 0; i < iters; ++i) { double s, c; sincos(x, &s, &c); acc += log(x + 1.0) + s * c; x += 1e-7; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d; float* f; cudaMalloc(&d, 8 << 24); cudaMalloc(&f, 4 << 24);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
    int blocks = sms * 8, threads = 256, iters = 4096;
    dfma_k<<<blocks, threads>>>(d, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); dfma_k<<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA: %.2f TFLOP/s\n", 2.0 * 8 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12);
    ffma_k<<<blocks, threads>>>(f, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); ffma_k<<<blocks, threads>>>(f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA: %.2f TFLOP/s\n", 2.0 * 8 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12);
    trans_k<<<blocks, threads>>>(d, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); trans_k<<<blocks, threads>>>(d, 256); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("log+sincos: %.2f G/s (%.1f us)\n", 256.0 * blocks * threads / (ms * 1e-3) / 1e9, ms * 1e3);
    cudaEventRecord(e0); trans_k<<<1, 32>>>(d, 32); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("one warp, 32 x log+sincos latency: %.1f us\n", ms * 1e3);
    return 0;
}
