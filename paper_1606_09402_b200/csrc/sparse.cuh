// CSR passes (see sparse.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace qbgpu {

struct CsrView {
    std::int64_t rows = 0, cols = 0, nnz = 0;
    const std::int64_t* rp = nullptr;
    const std::int32_t* ci = nullptr;
    const double* v = nullptr;
};

// Y(rows x w, row-major ldy) = alpha * A X + beta * Y, X (cols x w, row-major ldx).
void csr_spmm(cudaStream_t st, const CsrView& a, const double* x, std::int64_t ldx, double* y, std::int64_t ldy,
              int w, double alpha, double beta, int sms);

// Returns validation flags (0 = valid, bit 0 = structure, bit 1 = non-finite value).
int csr_validate(cudaStream_t st, std::int64_t m, std::int64_t n, std::int64_t nnz, const std::int64_t* rp,
                 const std::int32_t* ci, const double* v, int sms);

// Builds the CSR of A^T (n x m) with row-ascending entries per column.
void csr_transpose(cudaStream_t st, std::int64_t m, std::int64_t n, std::int64_t nnz, const std::int64_t* rp,
                   const std::int32_t* ci, const double* v, std::int64_t* ct_rp, std::int32_t* ct_ci,
                   double* ct_v, int sms);

}  // namespace qbgpu
