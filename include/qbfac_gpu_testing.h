/*
 * qbfac_gpu_testing.h — kernel-level hooks of libqbfac_gpu.so for the parity tests.
 * Not part of the drop-in boundary (include/qbfac_gpu.h); device pointers only,
 * every call synchronizes the context stream before returning.
 *
 *   qbfac_gpu_test_gemm      the DMMA GEMM behind every dense product
 *                            (replaces kernels::gemm_nn / gemm_tn, kernels_drivers.cpp:21-65)
 *   qbfac_gpu_test_chol      the in-CTA Cholesky + inverse used by CholQR
 *   qbfac_gpu_test_cholqr2   the fused one-launch CholQR2 of a tall panel
 *   qbfac_gpu_test_chol_wide the blocked (cooperative) Cholesky + inverse of the wide CholQR
 *   qbfac_gpu_test_householder  the Householder panel QR (orth_qr, qr.hpp:15-18)
 *   qbfac_gpu_test_orth_wide the power step's orth() of a wide sketch (CholQR2 or BCGS2)
 *   qbfac_gpu_test_colsumsq  per-column sums of squares (the indicator's row norms)
 *   qbfac_gpu_test_create_local_group  in-process rank group on one GPU (sharded-engine tests)
 *   qbfac_gpu_test_allreduce the context's allreduce (NCCL, or the local group) on a device buffer
 *   qbfac_gpu_test_collective its reduce-scatter / all-gather (the column-sharded n-side of EI)
 *   qbfac_gpu_test_chol_wide_trace  per-step stamps of the wide Cholesky
 *   qbfac_gpu_test_panel_trace  per-phase %globaltimer stamps (ns) of the last CholQR2 panel launch
 *   qbfac_gpu_test_csr_spmm  CSR pass Y = alpha A X + beta Y on device arrays
 *                            (replaces csr_gemm_n, kernels_drivers.cpp:67-79)
 */
#ifndef QBFAC_GPU_TESTING_H
#define QBFAC_GPU_TESTING_H

#include <stdint.h>

#include "qbfac_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* C(M x N) = alpha * A(M x K) * B(K x N) + beta * C; *_row selects row-major storage. */
int qbfac_gpu_test_gemm(qbfac_gpu_ctx* ctx, double alpha, const double* a, int64_t m, int64_t k, int64_t lda,
                        int a_row, const double* b, int64_t n, int64_t ldb, int b_row, double beta, double* c,
                        int64_t ldc, int c_row);
/* b x b Gram (col-major, ld b) -> R, R^{-1} (col-major, ld b); returns breakdown flag in *status. */
int qbfac_gpu_test_chol(qbfac_gpu_ctx* ctx, const double* g, int b, double* r, double* rinv, int* status);
/* blocked Cholesky + inverse of an l x l Gram (col-major, upper triangle read and overwritten), one cooperative launch */
/* fused CholQR2 of a row-major panel (rows x b, b <= 112): q (may alias y), R and R^{-1} (ld 112, column-major) */
int qbfac_gpu_test_cholqr2(qbfac_gpu_ctx* ctx, const double* y, int64_t rows, int b, int64_t ldy, double* q,
                           int64_t ldq, double* r, double* rinv, int* status);
/* 12 stamps: 0 start, 1 Gram A done, 2 partials written, 3 Gram reduced, 4/5 chol A done / published,
   6 phase B done, 7 Gram B reduced, 8/9 chol B done / published, 10 end (two-pass), 11 end (one pass);
   then 32 clock64 stamps of the last in-CTA Cholesky (out must hold 44 values) */
int qbfac_gpu_test_panel_trace(qbfac_gpu_ctx* ctx, unsigned long long* out);
/* `world` contexts on ONE device forming an in-process rank group: the row-sharded engine's
   allreduces meet at a host barrier and rank 0 sums the buffers in rank order. Each rank must be
   driven by its own host thread (qbfac_gpu_run blocks in the collectives). Test harness for the
   NCCL path's arithmetic on a single GPU; outs[world] receives the contexts. */
int qbfac_gpu_test_create_local_group(int device, int world, qbfac_gpu_ctx** outs);
/* In-place sum over the context's ranks of count doubles at dev (ncclAllReduce for an NCCL
   context, including a one-rank communicator made with qbfac_gpu_create_dist(dev, 0, 1, id)). */
int qbfac_gpu_test_allreduce(qbfac_gpu_ctx* ctx, double* dev, int64_t count);
/* op 1: recv (count) = this rank's block of the sum over ranks of send (world * count), ncclReduceScatter;
   op 2: recv (world * count) = every rank's send (count) in rank order, ncclAllGather. */
int qbfac_gpu_test_collective(qbfac_gpu_ctx* ctx, int op, const double* send, double* recv, int64_t count);
/* 64 x 4 %globaltimer stamps (ns) per step k of the last chol_wide launch (CTA 0): step start, phase 2
   done, phase 3 done (incl. the next diagonal Cholesky on CTA 0), step end */
int qbfac_gpu_test_chol_wide_trace(qbfac_gpu_ctx* ctx, unsigned long long* out);
int qbfac_gpu_test_chol_wide(qbfac_gpu_ctx* ctx, double* g, int l, double* r, double* rinv, int* breakdown);
/* Householder QR of a column-major m x b panel in place (Q overwrites y); R col-major ld b. */
int qbfac_gpu_test_householder(qbfac_gpu_ctx* ctx, double* y, int64_t m, int b, int64_t ld, double* r);
/* Orthonormalise a wide row-major rows x l panel in place (CholQR2 / BCGS2, the power step's orth). */
int qbfac_gpu_test_orth_wide(qbfac_gpu_ctx* ctx, double* x, int64_t rows, int64_t l, int force_bcgs2);
int qbfac_gpu_test_colsumsq(qbfac_gpu_ctx* ctx, const double* x, int64_t rows, int64_t cols, int64_t ld, int row,
                            double* out);
int qbfac_gpu_test_csr_spmm(qbfac_gpu_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz, const int64_t* rp,
                            const int32_t* ci, const double* v, const double* x, int64_t ldx, double* y,
                            int64_t ldy, int w, double alpha, double beta);

#ifdef __cplusplus
}
#endif

#endif /* QBFAC_GPU_TESTING_H */
