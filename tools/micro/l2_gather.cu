// Gather-bandwidth ceiling for the CSR passes: every warp repeatedly gathers one whole row of
// a row-major table X (w doubles per row, the rows a CSR nonzero pulls in), four rows in flight
// per warp step exactly like csr_spmm_kernel<4>, from random row indices (precomputed, read
// coalesced like a CSR column-index stream) and sums into registers (one FMA per element). Run
// with a table that fits in L2 (the L2 -> SM gather ceiling) and with one far larger than L2
// (the random-row HBM ceiling).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2_gather l2_gather.cu && ./l2_gather
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void __launch_bounds__(256) gather_kernel(const double* __restrict__ x, int w, const int* __restrict__ idx,
                                                     long long nidx, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * 256LL + threadIdx.x) >> 5, nw = (gridDim.x * 256LL) >> 5;
    double acc[4] = {0, 0, 0, 0};
    for (long long e0 = warp * 32; e0 < nidx; e0 += nw * 32) {
        const int my = idx[e0 + lane];
        for (int j = 0; j < 32; j += 4) {
            const double* r0 = x + static_cast<long long>(__shfl_sync(~0u, my, j)) * w;
            const double* r1 = x + static_cast<long long>(__shfl_sync(~0u, my, j + 1)) * w;
            const double* r2 = x + static_cast<long long>(__shfl_sync(~0u, my, j + 2)) * w;
            const double* r3 = x + static_cast<long long>(__shfl_sync(~0u, my, j + 3)) * w;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int c = lane + 32 * q;
                if (c < w) {
                    acc[q] = fma(__ldg(r0 + c), 1.0, acc[q]);
                    acc[q] = fma(__ldg(r1 + c), 1.0, acc[q]);
                    acc[q] = fma(__ldg(r2 + c), 1.0, acc[q]);
                    acc[q] = fma(__ldg(r3 + c), 1.0, acc[q]);
                }
            }
        }
    }
    out[blockIdx.x * 256 + threadIdx.x] = acc[0] + acc[1] + acc[2] + acc[3];
}

int main(int argc, char** argv) {
    const int w = argc > 1 ? std::atoi(argv[1]) : 100;
    const long long nidx = 1LL << 26;  // 67M gathers per launch
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    std::vector<int> hidx(nidx);
    int* didx;
    double *dout, *dx;
    cudaMalloc(&didx, nidx * sizeof(int));
    cudaMalloc(&dout, 16LL * sms * 256 * sizeof(double));
    for (long long rows : {50000LL, 80000LL, 150000LL, 500000LL, 5000000LL}) {
        std::uint64_t s = 88172645463325252ULL;
        for (long long i = 0; i < nidx; ++i) {
            s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            hidx[i] = static_cast<int>(s % static_cast<std::uint64_t>(rows));
        }
        cudaMemcpy(didx, hidx.data(), nidx * sizeof(int), cudaMemcpyHostToDevice);
        cudaMalloc(&dx, rows * w * sizeof(double));
        cudaMemset(dx, 0, rows * w * sizeof(double));
        for (int blocks_per_sm : {2, 4, 8, 16}) {
            const int grid = blocks_per_sm * sms;
            gather_kernel<<<grid, 256>>>(dx, w, didx, nidx, dout);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            for (int r = 0; r < 3; ++r) gather_kernel<<<grid, 256>>>(dx, w, didx, nidx, dout);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            ms /= 3;
            const double bytes = static_cast<double>(nidx) * w * 8;
            std::printf("table %8lld rows (%7.1f MB), grid %2d x SMs: %7.3f ms  %6.2f TB/s gathered\n", rows,
                        rows * w * 8 / 1e6, blocks_per_sm, ms, bytes / ms / 1e9);
        }
        cudaFree(dx);
    }
    std::printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
