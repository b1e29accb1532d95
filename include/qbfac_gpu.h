/*
 * qbfac_gpu.h — C-ABI of the B200-native randQB_EI / randQB_FP hot path.
 *
 * Drop-in boundary for the reference's algorithm entry points, whose C++
 * signatures survive in /root/reference/SPEC.md (the header qb.hpp and the
 * implementation src/qb.cpp are missing from the snapshot,
 * /root/reference/proj/CMakeLists.txt:26):
 *
 *   qbfac_gpu_run(.. alg = QBFAC_ALG_EI ..)        replaces rand_qb_ei
 *   qbfac_gpu_run(.. alg = QBFAC_ALG_FP ..)        replaces rand_qb_fp
 *   qbfac_gpu_run(.. alg = QBFAC_ALG_FP_FIXED_RANK) replaces rand_qb_fp_fixed_rank SPEC.md:282-290
 *   qbfac_gpu_run(.. alg = QBFAC_ALG_SINGLE_PASS ..) replaces single_pass_fp
 *
 * and for the operator layer the algorithms call
 * (/root/reference/proj/include/qbfac/matrix_handle.hpp:41-86):
 *
 *   qbfac_gpu_matrix_dense / _csr   replace MatrixHandle(DenseMatrix) / (SparseCsrMatrix)
 *                                   matrix_handle.hpp:43-44, validation as
 *                                   SparseCsrMatrix::from_parts sparse_csr.cpp:10-40
 *   qbfac_gpu_frob_norm_sq          replaces MatrixHandle::frob_norm_sq  matrix_handle.cpp:104-110
 *   qbfac_gpu_multiply              replaces MatrixHandle::multiply      matrix_handle.cpp:112-116
 *   qbfac_gpu_gaussian              replaces gaussian(rows, cols, rng)   rng.cpp:72-79
 *
 * Conventions: plain pointers and sizes, no exceptions cross this boundary,
 * every entry point returns a status (enum qbfac_status) that mirrors the
 * reference exception hierarchy (/root/reference/proj/include/qbfac/types.hpp:16-66);
 * qbfac_gpu_last_error() returns the message of the last failure on a context.
 * Host matrices are column-major double (the reference DenseMatrix layout,
 * dense_matrix.hpp:11-26); CSR arrays follow sparse_csr.hpp:46-48 (int64 row_ptr,
 * int32 col_idx, double values). Inputs are borrowed and copied during the call;
 * outputs go to caller-allocated buffers (two-phase: run -> info.rank -> copy).
 * There is no CPU fallback: every call needs a CUDA device (sm_100a).
 */
#ifndef QBFAC_GPU_H
#define QBFAC_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum qbfac_status {
    QBFAC_OK = 0,
    QBFAC_DIMENSION_ERROR = 1,       /* DimensionError         types.hpp:21-24 */
    QBFAC_SINGULARITY_ERROR = 2,     /* SingularityError       types.hpp:26-34 */
    QBFAC_TOLERANCE_FLOOR_ERROR = 3, /* ToleranceFloorError    types.hpp:38-46 */
    QBFAC_FORMAT_ERROR = 4,          /* FormatError            types.hpp:53-56 */
    QBFAC_RESOURCE_ERROR = 5,        /* ResourceError (OOM)    types.hpp:63-66 */
    QBFAC_ERROR = 6,                 /* Error (CUDA/NCCL, non-finite, ...) types.hpp:16-19 */
    QBFAC_INTERNAL = 7
};

/* QBFactorization::terminated_by */
enum qbfac_termination {
    QBFAC_RANK_REACHED = 0,
    QBFAC_TOLERANCE_MET = 1,
    QBFAC_SKETCH_EXHAUSTED = 2,
    QBFAC_RANK_COLLAPSE = 3
};

enum qbfac_alg {
    QBFAC_ALG_EI = 0,
    QBFAC_ALG_FP = 1,
    QBFAC_ALG_FP_FIXED_RANK = 2,
    QBFAC_ALG_SINGLE_PASS = 3,
    /* baselines: randQB (l = k + s, power), randQB_b (stop rule, b; dense A),
     * adaptive range finder (eps_abs = spectral tolerance, b = r window, max_rank) */
    QBFAC_ALG_QB = 4,
    QBFAC_ALG_QB_B = 5,
    QBFAC_ALG_RANGE_FINDER = 6
};

/* StopRule plus the algorithm parameters of SPEC.md:273-308. */
typedef struct qbfac_params {
    int32_t alg;          /* enum qbfac_alg */
    int32_t mode;         /* 0 = StopRule::fixed_rank(k, s), 1 = fixed_precision(eps_abs) */
    int64_t b;            /* block size */
    int64_t power;        /* power-iteration count P */
    int64_t k, s;         /* fixed rank / oversampling (mode 0; FP fixed rank; single pass l = k+s) */
    int64_t max_rank;     /* rank cap (0 = min(m, n)) */
    int64_t l_budget;     /* randQB_FP sketch width l~ */
    int64_t max_restarts; /* randQB_FP restart cap (default 8) */
    double eps_abs;       /* absolute Frobenius tolerance */
    uint64_t seed;        /* RngStream(seed, stream) rng.hpp:23 */
    uint64_t stream;
    int32_t reorth;       /* FP fixed rank: apply steps 9a-9c */
    int32_t flags;        /* reserved, 0 */
} qbfac_params;

/* Everything QBFactorization carries besides Q and B,
 * plus diagnostics. */
typedef struct qbfac_info {
    int64_t rank;              /* Q.cols() == B.rows() */
    double error_indicator;    /* E = ||A||_F^2 - ||B||_F^2 */
    double norm_a_sq;          /* ||A||_F^2 */
    int64_t passes;            /* PassCounter delta */
    int32_t terminated_by;     /* enum qbfac_termination */
    int32_t status;            /* enum qbfac_status of the run */
    int64_t diag_index;        /* SingularityError::diag_index */
    double floor;              /* ToleranceFloorError::floor_value */
    int64_t m, n;
    int64_t blocks;            /* blocks processed */
    int64_t gaussians_used;    /* next_gaussian() draws consumed from (seed, stream) */
    int64_t restarts;          /* randQB_FP sketch regenerations */
    int64_t householder_fallbacks; /* CholQR -> Householder panel fallbacks */
    double device_ms;          /* CUDA-event time of the run on the device */
} qbfac_info;

typedef struct qbfac_gpu_ctx qbfac_gpu_ctx;
typedef struct qbfac_gpu_matrix qbfac_gpu_matrix;
typedef struct qbfac_gpu_result qbfac_gpu_result;

/* ---- context -------------------------------------------------------------------- */
int qbfac_gpu_create(int device, qbfac_gpu_ctx** out);
/* Row-sharded context: this process is `rank` of `world`, one GPU each; the
 * 128-byte NCCL unique id comes from qbfac_gpu_nccl_unique_id() on rank 0. world == 1
 * with a non-NULL id builds a one-rank NCCL communicator (same results as
 * qbfac_gpu_create). */
int qbfac_gpu_create_dist(int device, int rank, int world, const void* nccl_id, qbfac_gpu_ctx** out);
int qbfac_gpu_nccl_unique_id(void* out128);
void qbfac_gpu_destroy(qbfac_gpu_ctx* ctx);
const char* qbfac_gpu_last_error(const qbfac_gpu_ctx* ctx);
int qbfac_gpu_synchronize(qbfac_gpu_ctx* ctx);
/* The CUDA stream (cudaStream_t) every call of this context is ordered on. */
void* qbfac_gpu_stream(qbfac_gpu_ctx* ctx);
/* Number of kernels this context launched so far (counted per context; NULL = the
 * process-wide total). */
int64_t qbfac_gpu_kernel_launches(const qbfac_gpu_ctx* ctx);

/* ---- the matrix A (MatrixHandle) ----------------------------------------------- */
/* Dense m x n column-major host matrix (lda >= m). With world > 1 pass this rank's
 * row block: m = local rows, row0 = its first global row, m_global = total rows. */
int qbfac_gpu_matrix_dense(qbfac_gpu_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda,
                           qbfac_gpu_matrix** out);
int qbfac_gpu_matrix_dense_device(qbfac_gpu_ctx* ctx, int64_t m, int64_t n, const double* dev_a,
                                  int64_t lda, qbfac_gpu_matrix** out);
int qbfac_gpu_matrix_dense_shard(qbfac_gpu_ctx* ctx, int64_t m_global, int64_t row0, int64_t m_local,
                                 int64_t n, const double* a, int64_t lda, qbfac_gpu_matrix** out);
/* CSR host arrays (validated as SparseCsrMatrix::from_parts). The transposed CSR
 * used for A^T products is built on the device. */
/* Asynchronous dense upload: the copy is cut into row chunks (chunk_rows, 0 = ~9 chunks of
 * whole 128-row tiles) issued on the context's copy stream, and the first A*X pass of the
 * next run consumes each chunk as soon as it lands (H2D overlapped with the first pass;
 * pinned host memory gives a true overlap; when that pass feeds the wide CholQR of
 * randQB_FP's power scheme, the sketch's Gram is accumulated per chunk behind it). `a` must stay valid and unchanged until a run
 * has consumed the matrix, qbfac_gpu_synchronize(), or qbfac_gpu_matrix_free(). The
 * DenseMatrix::from_data finiteness check (dense_matrix.cpp:17-18) happens at the first
 * norm computation instead of at upload. */
int qbfac_gpu_matrix_dense_async(qbfac_gpu_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda,
                                 int64_t chunk_rows, qbfac_gpu_matrix** out);
/* Host-streamed dense matrix — the RowStream of single_pass_fp (matrix_handle.hpp:30-37,
 * SPEC.md:300-308): A stays in host memory (column-major, lda; borrowed, must outlive the
 * run) and QBFAC_ALG_SINGLE_PASS streams row chunks (chunk_rows, 0 = ~128 MB) through a
 * 3-deep device ring, overlapping each chunk's copy with G_c = A_c Omega, H += A_c^T G_c and
 * ||A_c||^2 of the previous ones. Pinned host memory gives full-rate DMA. Any other use of
 * the handle returns QBFAC_ERROR. */
int qbfac_gpu_matrix_dense_stream(qbfac_gpu_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda,
                                  int64_t chunk_rows, qbfac_gpu_matrix** out);
int qbfac_gpu_matrix_csr(qbfac_gpu_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr,
                         const int32_t* col_idx, const double* values, qbfac_gpu_matrix** out);
/* Host-streamed CSR — the CsrRowStream of single_pass_fp (matrix_handle.cpp:60-73,
 * SPEC.md:300-308): the arrays stay in host memory (borrowed, must outlive the run) and
 * QBFAC_ALG_SINGLE_PASS uploads row chunks of about chunk_nnz entries (0 = 16 Mi) one at a
 * time, validating each as SparseCsrMatrix::from_parts (FormatError / Error) before
 * G_c = A_c Omega, H += A_c^T G_c and ||A_c||^2. row_ptr is checked whole at creation.
 * Any other use of the handle returns QBFAC_ERROR; world must be 1. */
int qbfac_gpu_matrix_csr_stream(qbfac_gpu_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr,
                                const int32_t* col_idx, const double* values, int64_t chunk_nnz,
                                qbfac_gpu_matrix** out);
int qbfac_gpu_matrix_csr_shard(qbfac_gpu_ctx* ctx, int64_t m_global, int64_t row0, int64_t m_local,
                               int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                               const double* values, qbfac_gpu_matrix** out);
/* ---- Matrix Market ingest / export (CSR built as
 * SparseCsrMatrix::from_triplets, sparse_csr.cpp:42-64). Host-only helpers (no
 * device needed): coordinate or array, real/integer, general; any other banner ->
 * QBFAC_FORMAT_ERROR; duplicate or out-of-range coordinates -> QBFAC_FORMAT_ERROR;
 * non-finite values -> QBFAC_ERROR. Two-phase: info, then read into caller buffers
 * (row_ptr m+1, col_idx/values nnz; dense: column-major with lda >= m). Writers emit
 * shortest round-trip decimal, so write -> read reproduces every double exactly.
 * Messages of these context-free calls: qbfac_mtx_last_error(). */
const char* qbfac_mtx_last_error(void);
int qbfac_mtx_info(const char* path, int* coordinate, int64_t* m, int64_t* n, int64_t* nnz);
int qbfac_mtx_read_csr(const char* path, int64_t* row_ptr, int32_t* col_idx, double* values);
int qbfac_mtx_read_dense(const char* path, double* a, int64_t lda);
int qbfac_mtx_write_csr(const char* path, int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr,
                        const int32_t* col_idx, const double* values);
int qbfac_mtx_write_dense(const char* path, int64_t m, int64_t n, const double* a, int64_t lda);
/* read_matrix_market(path) -> MatrixHandle on the device (coordinate -> CSR plus its
 * device-built transpose, array -> dense). */
int qbfac_gpu_matrix_mtx(qbfac_gpu_ctx* ctx, const char* path, qbfac_gpu_matrix** out);
/* shape of a handle and copies of its device arrays back to the host (the reference's
 * MatrixHandle::matrix() accessors, matrix_handle.hpp:58-74) */
int qbfac_gpu_matrix_shape(const qbfac_gpu_matrix* mat, int* sparse, int64_t* m, int64_t* n, int64_t* nnz);
int qbfac_gpu_matrix_export_csr(qbfac_gpu_ctx* ctx, const qbfac_gpu_matrix* mat, int64_t* row_ptr, int32_t* col_idx,
                                double* values);
int qbfac_gpu_matrix_export_dense(qbfac_gpu_ctx* ctx, const qbfac_gpu_matrix* mat, double* a, int64_t lda);

void qbfac_gpu_matrix_free(qbfac_gpu_matrix* mat);
/* Passes counted on this handle so far (PassCounter, matrix_handle.hpp:20-27). */
int64_t qbfac_gpu_matrix_passes(const qbfac_gpu_matrix* mat);

/* ||A||_F^2 (one pass). */
int qbfac_gpu_frob_norm_sq(qbfac_gpu_ctx* ctx, qbfac_gpu_matrix* mat, double* out);
/* Y = A X (trans = 0) or A^T X (trans = 1), host column-major buffers; one pass. */
int qbfac_gpu_multiply(qbfac_gpu_ctx* ctx, qbfac_gpu_matrix* mat, const double* x, int64_t w, int trans,
                       double* y);
/* Same product on device buffers: X (w columns) and Y row-major with leading dimensions
 * ldx, ldy (the layout of the engine's block vectors); ordered on qbfac_gpu_stream(). */
int qbfac_gpu_multiply_device(qbfac_gpu_ctx* ctx, qbfac_gpu_matrix* mat, const double* x, int64_t ldx, int64_t w,
                              int trans, double* y, int64_t ldy);
/* gaussian(rows, cols, rng) after `skip` earlier draws, into a host column-major buffer. */
int qbfac_gpu_gaussian(qbfac_gpu_ctx* ctx, uint64_t seed, uint64_t stream, uint64_t skip, int64_t rows,
                       int64_t cols, double* out);
/* Same, into device memory (column-major, leading dimension ld). */
int qbfac_gpu_gaussian_device(qbfac_gpu_ctx* ctx, uint64_t seed, uint64_t stream, uint64_t skip,
                              int64_t rows, int64_t cols, double* dev_out, int64_t ld);

/* ---- the algorithms ------------------------------------------------------------ */
int qbfac_gpu_run(qbfac_gpu_ctx* ctx, qbfac_gpu_matrix* mat, const qbfac_params* params,
                  qbfac_gpu_result** out, qbfac_info* info);
/* Q: this rank's m x rank rows, column-major, leading dimension ldq >= m. */
int qbfac_gpu_result_copy_q(qbfac_gpu_result* res, double* q, int64_t ldq);
/* B: rank x n, column-major, leading dimension ldb >= rank. */
int qbfac_gpu_result_copy_b(qbfac_gpu_result* res, double* b, int64_t ldb);
/* E after every block boundary (Theorem 2 checks); returns the count written. */
int64_t qbfac_gpu_result_copy_trace(qbfac_gpu_result* res, double* out, int64_t cap);
/* qb_to_svd(f, k) (PAPER Eq. 1.3): truncated SVD of Q*B computed on the
 * device — Q_b = orth(B^T) (wide CholQR2 / BCGS2), N = B Q_b, one-sided Jacobi N W = U_r S,
 * U = Q U_r(:, 1..k), V = Q_b W(:, 1..k). Outputs: u (m x k, ldu >= m), s (k, non-increasing),
 * v (n x k, ldv >= n), column-major host buffers; k > rank -> QBFAC_DIMENSION_ERROR.
 * `sweeps` (optional) receives the Jacobi sweep count. */
int qbfac_gpu_result_svd(qbfac_gpu_result* res, int64_t k, double* u, int64_t ldu, double* s, double* v,
                         int64_t ldv, int* sweeps);
void qbfac_gpu_result_free(qbfac_gpu_result* res);

/* Theorem 3 validity: returns 1 iff eps > sqrt(4 u / delta) ||A||_F. */
int qbfac_gpu_validate_epsilon(double eps, double frob_a, double delta, double* floor_out);

#ifdef __cplusplus
}
#endif

#endif /* QBFAC_GPU_H */
