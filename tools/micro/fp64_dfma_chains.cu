// FP64 vector (non-tensor) DFMA throughput and latency on one SM and on the whole chip.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_rate fp64_rate.cu && ./fp64_rate
#include <cuda_runtime.h>
#include <cstdio>

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, long long* clk) {
    double a[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) a[c] = threadIdx.x * 1e-9 + c;
    const double x = 1.0000001, y = 1e-12;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) a[c] = fma(a[c], x, y);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int CHAINS>
void run(int blocks, int threads, int iters) {
    double* out;
    long long* clk;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaMalloc(&clk, sizeof(long long));
    dfma_kernel<CHAINS><<<blocks, threads>>>(out, iters, clk);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dfma_kernel<CHAINS><<<blocks, threads>>>(out, iters, clk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c = 0;
    cudaMemcpy(&c, clk, sizeof(long long), cudaMemcpyDeviceToHost);
    const double fmas = double(blocks) * threads * iters * CHAINS;
    std::printf("chains %2d, %4d blocks x %4d threads: %8.3f ms  %7.3f TFMA/s (%6.2f TFLOP/s)  clk/iter(thread0) %.1f\n",
                CHAINS, blocks, threads, ms, fmas / ms / 1e9, 2 * fmas / ms / 1e9, double(c) / iters);
    cudaFree(out);
    cudaFree(clk);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<1>(1, 32, 100000);       // latency: one warp, one chain
    run<8>(1, 32, 100000);       // one warp, 8 independent chains
    run<8>(1, 1024, 20000);      // one SM saturated
    run<8>(sms, 1024, 20000);    // whole chip
    run<1>(sms, 1024, 100000);   // whole chip, one chain per thread
    return 0;
}
