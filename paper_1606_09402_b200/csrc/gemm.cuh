// Device-side building blocks of the qbfac B200 path: FP64 DMMA GEMM, small
// dense kernels (CholQR pieces, indicator), reductions. See gemm.cu / small.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "common.cuh"

namespace qbgpu {

// Growable device scratch buffer (never shrinks; freed with its owner).
struct Workspace {
    double* ptr = nullptr;
    std::size_t cap = 0;  // doubles
    double* get(std::size_t n) {
        if (n > cap) {
            if (ptr) QB_CUDA(cudaFree(ptr));
            ptr = nullptr;
            cap = 0;
            std::size_t want = n + n / 4 + 1024;
            QB_CUDA(cudaMalloc(&ptr, want * sizeof(double)));
            cap = want;
        }
        return ptr;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
    }
    ~Workspace() { release(); }
};

int gemm_num_sms();
// 2-D tensor map over a row-major rows x w FP64 matrix (leading dimension ld), box = one row
// (for TMA tile::gather4); `map` points to a 64-byte aligned CUtensorMap.
void make_tensor_map_rows(void* map, const double* base, std::int64_t rows, int w, std::int64_t ld);
// 2-D tensor map over a row-major outer x inner FP64 matrix (row stride ld), box box0 x box1 elements;
// elements outside the matrix are zero-filled by the TMA unit.
void make_tensor_map_2d(void* map, const double* base, std::int64_t inner, std::int64_t outer, std::int64_t ld,
                        int box0, int box1);

// C = alpha * A * B + beta * C, all FP64 views in device memory (any layouts).
// beta == 0 never reads C. Deterministic (fixed split-K reduction order).
// flags: kGemmTriB   - B is upper triangular (K range of an output tile limited);
//        kGemmUpperC - only tiles touching the upper triangle of C are computed
//                      (symmetric results such as Grams; the strict lower part is untouched).
constexpr int kGemmTriB = 1;
constexpr int kGemmUpperC = 2;
void gemm(cudaStream_t st, Workspace& ws, double alpha, const MatView& a, const MatView& b,
          double beta, const MatView& c, int flags = 0);

// ---- small.cu -------------------------------------------------------------------
void scale_matrix(cudaStream_t st, const MatView& c, double beta);
void copy_matrix(cudaStream_t st, const MatView& src, const MatView& dst);  // dst = src (any layouts)
void set_identity(cudaStream_t st, const MatView& c);
void add_matrix(cudaStream_t st, const MatView& src, const MatView& dst, double alpha);  // dst += alpha*src

// out[0] = sum of squares of all entries of v (deterministic two-stage tree).
void sum_squares(cudaStream_t st, Workspace& ws, const MatView& v, double* out);
void sum_squares_vec(cudaStream_t st, Workspace& ws, const double* x, std::int64_t n, double* out);
// out[j] = sum_i v(i,j)^2 for j < v.cols (deterministic).
void column_sumsq(cudaStream_t st, Workspace& ws, const MatView& v, double* out);

// Small dense factorization status written by chol_small / cholqr checks.
struct SmallStatus {
    int breakdown;        // 1 if Cholesky met a non-positive pivot
    int bad_index;        // first failing pivot index
    double diag_min;      // min_j R(j,j)
    double diag_max;      // max_j R(j,j)
    double gram_dev;      // max |G(i,j) - delta_ij| of the input Gram (orthogonality of input)
};

// b x b Gram G (col-major, ld) -> R = chol(G) upper (col-major ldr), Rinv = R^{-1}
// (upper, col-major). One CTA. b <= kSmallMax.
constexpr int kPanelTraceSlots = 12;
constexpr int kSmallMax = 112;  // chol_small keeps [G | I] (b x 2b) in shared memory
void chol_small(cudaStream_t st, const double* g, std::int64_t ldg, int b, double* r,
                double* rinv, std::int64_t ldr, SmallStatus* status);
// Blocked Cholesky W = R^T R (upper triangle of the l x l col-major W, overwritten) and
// R^{-1}, one cooperative launch; r and rinv (ld ldr) must be zero on entry; one status
// per 64-column diagonal block.
void chol_wide(cudaStream_t st, double* w, std::int64_t ldw, int l, double* r, double* rinv, std::int64_t ldr,
               SmallStatus* stats);
// One-sided Jacobi SVD of the r x r column-major N in place (N W = U Sigma, W must hold I on
// entry): one cooperative launch, returns the number of sweeps.
int jacobi_svd(cudaStream_t st, double* nmat, double* w, int r, unsigned* gbar, int max_sweeps = 40);

// Fused CholQR2 of a tall row-major panel Y (rows x b, b <= 112) in one cooperative launch:
// g <- Y^T Y, (ra, rainv) <- chol, t1 <- Y ra^{-1}, g <- t1^T t1, (rb, rbinv) <- chol,
// q <- t1 rb^{-1}; statuses of both Choleskies in st0 / st1. q may alias y. Small
// matrices are column-major with ld kSmallMax. gbar: two zero-initialised words per
// context (grid barrier).
void panel_trace(unsigned long long* out);
void chol_wide_trace(unsigned long long* out);  // 64 x 4 step stamps of the last chol_wide launch  // phase timestamps of the last panel launch
void cholqr2_panel(cudaStream_t st, Workspace& ws, const double* y, std::int64_t rows, int b, std::int64_t ldy,
                   double* t1, double* q, std::int64_t ldq, double* g, double* ra, double* rainv, double* rb,
                   double* rbinv, SmallStatus* st0, SmallStatus* st1, unsigned* gbar, bool span_only = false);
// C = A * B for upper-triangular b x b (col-major, ld); C must not alias.
void trmm_upper_small(cudaStream_t st, const double* a, const double* b, double* c, int n,
                      std::int64_t ld);
// c0 = a0*b0 and (if c1) c1 = a1*b1 for upper-triangular n x n, one launch.
void trmm_upper_pair(cudaStream_t st, const double* a0, const double* b0, double* c0, const double* a1,
                     const double* b1, double* c1, int n, std::int64_t ld);
// Rinv = R^{-1} for upper-triangular R (one CTA).
void tri_inverse_small(cudaStream_t st, const double* r, double* rinv, int n, std::int64_t ld);

// Error-indicator step: for j < b: E -= norms[j]; if check and
// E < eps2 stop after row j. Writes the new E and the kept row count.
struct IndicatorOut {
    double e;
    int keep;
    int met;
};
void indicator_step(cudaStream_t st, double* e_dev, const double* norms, int b, double eps2,
                    int check, IndicatorOut* out);

// Householder economic QR of a column-major m x b panel (b <= kSmallMax), diag(R) >= 0:
// the exact-semantics fallback when CholQR is unreliable. y is overwritten by Q.
// Cooperative grid; deterministic reductions.
void householder_panel(cudaStream_t st, Workspace& ws, double* y, std::int64_t m, int b,
                       std::int64_t ld, double* r, std::int64_t ldr);

}  // namespace qbgpu
