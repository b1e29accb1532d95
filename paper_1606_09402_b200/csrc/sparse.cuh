// CSR passes (see sparse.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace qbgpu {

// Rows longer than kHeavyRow nonzeros (Zipf-like dense rows, popular columns in the
// transposed CSR) are cut into segments of at most kHeavyRow entries that separate
// warps process; their partial rows are then summed in segment order. A warp walks its row
// 4 gathers per step, so one long row on one warp is a serial tail: config 5's passes went
// 15.7 / 15.1 ms -> 12.2 / 11.9 ms when the threshold dropped from 4096 to 256
// (tools/spmm_bench.py sweep 4096/1024/512/256/128/64; 128 was 2 % faster on config 5 but
// segmented config 3's ~100-entry transposed columns, +10 %).
constexpr std::int64_t kHeavyRow = 256;

struct HeavyPlan {
    std::int64_t nseg = 0, nrows = 0;
    std::int64_t thr = kHeavyRow;     // rows longer than thr are segmented (segments of thr entries)
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
// Segment length / heavy-row threshold (QBFAC_HEAVY_ROW overrides kHeavyRow).
std::int64_t heavy_row_threshold();
void free_heavy_plan(HeavyPlan& p);

// Y(rows x w, row-major ldy) = alpha * A X + beta * Y, X (cols x w, row-major ldx).
void csr_spmm(cudaStream_t st, const CsrView& a, const double* x, std::int64_t ldx, double* y, std::int64_t ldy,
              int w, double alpha, double beta, int sms, double* partial = nullptr);
// Scratch (doubles) csr_spmm needs for the heavy rows at width w.
inline std::size_t csr_spmm_scratch(const CsrView& a, int w) { return static_cast<std::size_t>(a.heavy.nseg) * w; }

// Returns validation flags (0 = valid, bit 0 = structure, bit 1 = non-finite value).
int csr_validate(cudaStream_t st, std::int64_t m, std::int64_t n, std::int64_t nnz, const std::int64_t* rp,
                 const std::int32_t* ci, const double* v, int sms);

// Hybrid split of a power-law CSR (A = S + P_R^T D_r + D_c P_C^T): rows flagged in rowflag
// (entire rows) go to the dense row block D_r (dr x n, row-major), entries of the columns with
// colmap[c] = j >= 0 (outside flagged rows) to the dense column block D_c (m x dc, column-major,
// ld m); everything else stays in S (same order). d_r / d_c must be zeroed; s_rp has m+1 slots.
// Returns nnz(S).
std::int64_t csr_split_dense(cudaStream_t st, std::int64_t m, std::int64_t n, const std::int64_t* rp,
                             const std::int32_t* ci, const double* v, const std::int32_t* rowmap,
                             const std::int32_t* colmap, std::int64_t* s_rp, std::int32_t** s_ci, double** s_v,
                             double* d_r, double* d_c, int sms);
// dst(k x w, row-major ld w) = src rows idx[0..k) (row-major ld lds)
void gather_rows(cudaStream_t st, const double* src, std::int64_t lds, const std::int64_t* idx, std::int64_t k, int w,
                 double* dst);
// dst rows idx[i] += alpha * src row i (rows distinct: no races)
void scatter_add_rows(cudaStream_t st, const double* src, const std::int64_t* idx, std::int64_t k, int w, double alpha,
                      double* dst, std::int64_t ldd);

// Builds the CSR of A^T (n x m) with row-ascending entries per column.
void csr_transpose(cudaStream_t st, std::int64_t m, std::int64_t n, std::int64_t nnz, const std::int64_t* rp,
                   const std::int32_t* ci, const double* v, std::int64_t* ct_rp, std::int32_t* ct_ci,
                   double* ct_v, int sms);

}  // namespace qbgpu
