// CSR passes (see sparse.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace qbgpu {

// Rows longer than kHeavyRow nonzeros (Zipf-like dense rows, popular columns in the
// transposed CSR) are cut into segments of at most kHeavyRow entries that separate
// warps process; their partial rows are then summed in segment order.
constexpr std::int64_t kHeavyRow = 4096;

struct HeavyPlan {
    std::int64_t nseg = 0, nrows = 0;
    std::int64_t* seg = nullptr;      // device: 3 x nseg (row, lo, hi), segments of a row contiguous
    std::int64_t* rows = nullptr;     // device: 3 x nrows (row, first segment, segment count)
};

struct CsrView {
    std::int64_t rows = 0, cols = 0, nnz = 0;
    const std::int64_t* rp = nullptr;
    const std::int32_t* ci = nullptr;
    const double* v = nullptr;
    HeavyPlan heavy;
};

// Build the heavy-row plan from a host copy of row_ptr (device arrays allocated here).
HeavyPlan make_heavy_plan(const std::int64_t* rp_host, std::int64_t rows, cudaStream_t st);
void free_heavy_plan(HeavyPlan& p);

// Y(rows x w, row-major ldy) = alpha * A X + beta * Y, X (cols x w, row-major ldx).
void csr_spmm(cudaStream_t st, const CsrView& a, const double* x, std::int64_t ldx, double* y, std::int64_t ldy,
              int w, double alpha, double beta, int sms, double* partial = nullptr);
// Scratch (doubles) csr_spmm needs for the heavy rows at width w.
inline std::size_t csr_spmm_scratch(const CsrView& a, int w) { return static_cast<std::size_t>(a.heavy.nseg) * w; }

// Returns validation flags (0 = valid, bit 0 = structure, bit 1 = non-finite value).
int csr_validate(cudaStream_t st, std::int64_t m, std::int64_t n, std::int64_t nnz, const std::int64_t* rp,
                 const std::int32_t* ci, const double* v, int sms);

// Builds the CSR of A^T (n x m) with row-ascending entries per column.
void csr_transpose(cudaStream_t st, std::int64_t m, std::int64_t n, std::int64_t nnz, const std::int64_t* rp,
                   const std::int32_t* ci, const double* v, std::int64_t* ct_rp, std::int32_t* ct_ci,
                   double* ct_v, int sms);

}  // namespace qbgpu
