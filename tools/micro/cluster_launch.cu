// Launch overhead of a thread-block cluster kernel vs cluster size and dynamic shared memory:
// an (almost) empty kernel, timed with CUDA events over back-to-back launches and by ncu.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_launch cluster_launch.cu && ./cluster_launch
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(256, 1) k_cluster(double* out, int do_sync) {
    extern __shared__ double sm[];
    cg::cluster_group cluster = cg::this_cluster();
    sm[threadIdx.x] = threadIdx.x;
    if (do_sync) cluster.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = sm[0] + cluster.num_blocks();
}
__global__ void __launch_bounds__(256, 1) k_plain(double* out) {
    extern __shared__ double sm[];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = sm[0];
}

int main() {
    double* d;
    cudaMalloc(&d, 64);
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int smem_kb : {8, 100, 200}) {
        const int smem = smem_kb * 1024;
        cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(k_plain, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int cs : {0, 1, 2, 4, 8, 16}) {
            const int grid = cs == 0 ? 8 : (cs < 8 ? 8 : cs);
            auto launch = [&]() {
                if (cs == 0) {
                    k_plain<<<grid, 256, smem, st>>>(d);
                } else {
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(grid);
                    cfg.blockDim = dim3(256);
                    cfg.dynamicSmemBytes = smem;
                    cfg.stream = st;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeClusterDimension;
                    at[0].val.clusterDim.x = cs;
                    at[0].val.clusterDim.y = 1;
                    at[0].val.clusterDim.z = 1;
                    cfg.attrs = at;
                    cfg.numAttrs = 1;
                    cudaLaunchKernelEx(&cfg, k_cluster, d, 1);
                }
            };
            for (int i = 0; i < 10; ++i) launch();
            cudaStreamSynchronize(st);
            cudaEventRecord(e0, st);
            for (int i = 0; i < 200; ++i) launch();
            cudaEventRecord(e1, st);
            cudaStreamSynchronize(st);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("smem %3d KB  cluster %2d (grid %2d): %.2f us per launch (back-to-back)  err=%s\n", smem_kb, cs, grid,
                   ms * 1e3 / 200, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
