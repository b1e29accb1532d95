// Probe: TMA tile::gather4 of FP64 rows (cp.async.bulk.tensor.2d ... tile::gather4) on sm_100a.
// Builds a 2-D tensor map over X (n x w row-major) with box {w, B1} for B1 in {1, 4}, gathers 4
// arbitrary rows into shared memory and compares with a plain copy.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void k(const __grid_constant__ CUtensorMap map, int w, int r0, int r1, int r2, int r3, double* out) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bar;
    const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar));
    for (int i = threadIdx.x; i < 4 * w; i += blockDim.x) sm[i] = -1.0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(4 * w * 8) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(sm))),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b)
            : "memory");
    }
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(b) : "memory");
    for (int i = threadIdx.x; i < 4 * w; i += blockDim.x) out[i] = sm[i];
}

int main() {
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    const int n = 1000;
    for (int w : {50, 100, 128}) {
        for (int ld : {w, w + 4}) {
            std::vector<double> hx(static_cast<size_t>(n) * ld);
            for (size_t i = 0; i < hx.size(); ++i) hx[i] = static_cast<double>(i);
            double *dx, *dout;
            cudaMalloc(&dx, hx.size() * 8);
            cudaMalloc(&dout, 4 * w * 8);
            cudaMemcpy(dx, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice);
            for (int b1 : {1, 4}) {
                CUtensorMap map;
                const cuuint64_t dims[2] = {static_cast<cuuint64_t>(w), static_cast<cuuint64_t>(n)};
                const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
                const cuuint32_t box[2] = {static_cast<cuuint32_t>(w), static_cast<cuuint32_t>(b1)};
                const cuuint32_t es[2] = {1, 1};
                CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dx, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                if (r != CUDA_SUCCESS) { printf("w=%d ld=%d box1=%d: encode failed %d\n", w, ld, b1, (int)r); continue; }
                const int rows[4] = {7, 999, 3, 500};
                cudaMemset(dout, 0, 4 * w * 8);
                k<<<1, 128, 4 * w * 8>>>(map, w, rows[0], rows[1], rows[2], rows[3], dout);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("w=%d ld=%d box1=%d: kernel error %s\n", w, ld, b1, cudaGetErrorString(e)); return 1; }
                std::vector<double> ho(4 * w);
                cudaMemcpy(ho.data(), dout, 4 * w * 8, cudaMemcpyDeviceToHost);
                int bad = 0;
                for (int rr = 0; rr < 4; ++rr)
                    for (int c = 0; c < w; ++c)
                        if (ho[rr * w + c] != hx[static_cast<size_t>(rows[rr]) * ld + c]) ++bad;
                printf("w=%d ld=%d box1=%d: %s (%d mismatches; first %.0f expect %.0f)\n", w, ld, b1, bad ? "WRONG" : "ok", bad,
                       ho[0], hx[static_cast<size_t>(rows[0]) * ld]);
            }
            cudaFree(dx);
            cudaFree(dout);
        }
    }
    return 0;
}
