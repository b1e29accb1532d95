// Micro: phase timing of chol_small (small.cu compiled in with QB_CHOL_TIMING).
#define QB_CHOL_TIMING 1
#include "../../paper_1606_09402_b200/csrc/small.cu"
namespace qbgpu { std::atomic<long long> g_kernel_launches{0}; int gemm_num_sms() { return 148; } }
#include <cstdio>
#include <vector>
int main() {
    using namespace qbgpu;
    for (int b : {20, 50, 112}) {
        std::vector<double> g(b * b);
        for (int i = 0; i < b; ++i) for (int j = 0; j < b; ++j) g[i + j * b] = (i == j ? 3.0 * b : 0.0) + 1.0 / (1 + i + j);
        double *dg, *dr, *dri; SmallStatus* ds;
        cudaMalloc(&dg, 8 * b * b); cudaMalloc(&dr, 8 * b * b); cudaMalloc(&dri, 8 * b * b); cudaMalloc(&ds, 64);
        cudaMemcpy(dg, g.data(), 8 * b * b, cudaMemcpyHostToDevice);
        for (int rep = 0; rep < 3; ++rep) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            chol_small(0, dg, b, b, dr, dri, b, ds);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            long long t[4]; cudaMemcpyFromSymbol(t, g_chol_t, sizeof(t));
            printf("b=%d: load %lld, warpchol %lld, total-to-output %lld cycles; event %.1f us (%s)\n", b, t[0], t[1], t[2], ms * 1e3,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
}
