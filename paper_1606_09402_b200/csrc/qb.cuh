// Host-side engine of the B200 randQB path: context, device matrix handle,
// result, and the algorithm drivers (qb.cu). The C-ABI (capi.cu) is a thin
// exception-to-status layer over these.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "comm.cuh"
#include "common.cuh"
#include "gemm.cuh"
#include "rng.cuh"
#include "sparse.cuh"

namespace qbgpu {

// Stream-ordered device allocation (cudaMallocAsync pool).
struct DBuf {
    double* p = nullptr;
    std::size_t n = 0;
    cudaStream_t st = nullptr;
    DBuf() = default;
    DBuf(std::size_t count, cudaStream_t s) : n(count), st(s) {
        if (count) QB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(double), s));
    }
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), st(o.st) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { reset(); p = o.p; n = o.n; st = o.st; o.p = nullptr; o.n = 0; }
        return *this;
    }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    void reset() {
        if (p) cudaFreeAsync(p, st);
        p = nullptr;
        n = 0;
    }
    ~DBuf() { reset(); }
};

struct Context {
    int device = 0;
    cudaStream_t st = nullptr;
    cudaStream_t st_copy = nullptr;  // host->device uploads overlapped with compute
    int sms = 148;
    Workspace ws_gemm, ws_red, ws_hh, ws_sp, ws_panel;
    RngTables rng;
    std::unique_ptr<Comm> comm;
    int rank = 0, world = 1;
    std::string last_error;
    // small device scratch: b x b matrices (ld kSmallMax) and scalars
    double* d_small = nullptr;
    SmallStatus* d_status = nullptr;
    unsigned* d_gbar = nullptr;  // grid-barrier words of the cooperative kernels (zeroed once)
    IndicatorOut* d_ind = nullptr;
    static constexpr int kLazyCap = 256;    // optimistic CholQR statuses per block
    SmallStatus* d_lazy = nullptr;
    SmallStatus* h_lazy = nullptr;
    // pinned host mirrors
    SmallStatus* h_status = nullptr;
    IndicatorOut* h_ind = nullptr;
    double* h_scalar = nullptr;

    explicit Context(int dev, int rank_ = 0, int world_ = 1, const void* nccl_id = nullptr,
                     std::shared_ptr<LocalGroup> local = nullptr);
    ~Context();
    void allreduce(double* p, std::size_t count) {
        if (comm) comm->allreduce_sum(p, count, st);
    }
    void reduce_scatter(const double* send, double* recv, std::size_t recvcount) {
        if (comm) comm->reduce_scatter_sum(send, recv, recvcount, st);
        else if (recvcount && recv != send)
            QB_CUDA(cudaMemcpyAsync(recv, send, recvcount * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    void all_gather(const double* send, double* recv, std::size_t sendcount) {
        if (comm) comm->all_gather(send, recv, sendcount, st);
        else if (sendcount && recv != send)
            QB_CUDA(cudaMemcpyAsync(recv, send, sendcount * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
};

struct Matrix {
    Context* ctx = nullptr;
    bool sparse = false;
    std::int64_t m = 0, n = 0;          // local rows, columns
    std::int64_t m_global = 0, row0 = 0;
    std::int64_t passes = 0;            // PassCounter (matrix_handle.hpp:20-27)
    // dense, column-major
    double* a = nullptr;
    std::int64_t lda = 0;
    bool owns_a = true;
    bool pooled_a = false;  // `a` from the stream-ordered pool (freed with cudaFreeAsync on ctx->st)
    // CSR + device-built transposed CSR
    std::int64_t nnz = 0;
    std::int64_t* rp = nullptr;
    std::int32_t* ci = nullptr;
    double* v = nullptr;
    std::int64_t* ct_rp = nullptr;
    std::int32_t* ct_ci = nullptr;
    double* ct_v = nullptr;
    HeavyPlan heavy, heavy_t;  // heavy-row segment plans of the CSR and its transpose
    // Hybrid split of power-law matrices (make_csr): the SpMM runs on the remainder S
    // (s_* arrays, transposed into ct_*), dense rows / dense columns go to DMMA GEMMs.
    std::int64_t s_nnz = 0;
    std::int64_t* s_rp = nullptr;
    std::int32_t* s_ci = nullptr;
    double* s_v = nullptr;
    std::int64_t dr = 0, dc = 0;
    std::int64_t* d_rows = nullptr;  // dr row indices (local)
    std::int64_t* d_cols = nullptr;  // dc column indices
    double* d_r = nullptr;           // dr x n, row-major
    double* d_c = nullptr;           // m x dc, column-major (ld m)
    bool hybrid() const { return d_r || d_c; }
    // Asynchronous dense upload (qbfac_gpu_matrix_dense_async): row chunks [row_end of the
    // previous, row_end) become resident when their event completes on ctx->st_copy. The
    // first A*X pass consumes them chunk by chunk; every other use waits for all of them.
    struct Chunk {
        std::int64_t row_end;
        cudaEvent_t ready;
    };
    std::vector<Chunk> pending;
    bool check_finite = false;  // validate ||A||^2 at the first norm (from_data, dense_matrix.cpp:17-18)
    // Host-streamed dense rows (qbfac_gpu_matrix_dense_stream, the RowStream of
    // matrix_handle.hpp:30-37): A stays in host memory and single_pass_fp streams row chunks.
    bool host_stream = false;
    const double* host_a = nullptr;
    std::int64_t host_lda = 0, chunk_rows = 0;
    // Host-streamed CSR (qbfac_gpu_matrix_csr_stream, CsrRowStream of matrix_handle.cpp:60-73):
    // row chunks of about chunk_nnz entries are uploaded, validated and multiplied one at a time.
    const std::int64_t* host_rp = nullptr;
    const std::int32_t* host_ci = nullptr;
    const double* host_v = nullptr;
    std::int64_t chunk_nnz = 0;
    void wait_resident(cudaStream_t s);

    ~Matrix();
    MatView dense_view() const { return MatView{a, m, n, lda, false}; }
    CsrView csr() const {
        return hybrid() ? CsrView{m, n, s_nnz, s_rp, s_ci, s_v, heavy} : CsrView{m, n, nnz, rp, ci, v, heavy};
    }
    CsrView csr_t() const { return CsrView{n, m, hybrid() ? s_nnz : nnz, ct_rp, ct_ci, ct_v, heavy_t}; }
};

std::unique_ptr<Matrix> make_dense(Context& c, std::int64_t m_global, std::int64_t row0, std::int64_t m,
                                   std::int64_t n, const double* a, std::int64_t lda, bool device_src);
// Chunked asynchronous upload of a host dense matrix (pinned memory gives a true overlap;
// the host buffer must stay unchanged until the matrix has been consumed or synchronized).
std::unique_ptr<Matrix> make_dense_async(Context& c, std::int64_t m, std::int64_t n, const double* a,
                                         std::int64_t lda, std::int64_t chunk_rows);
// Host-streamed dense matrix (borrowed host pointer, column-major, lda): consumed only by
// single_pass_fp, which streams row chunks through a device ring.
std::unique_ptr<Matrix> make_dense_stream(Context& c, std::int64_t m, std::int64_t n, const double* a,
                                          std::int64_t lda, std::int64_t chunk_rows);
std::unique_ptr<Matrix> make_csr(Context& c, std::int64_t m_global, std::int64_t row0, std::int64_t m,
                                 std::int64_t n, std::int64_t nnz, const std::int64_t* rp,
                                 const std::int32_t* ci, const double* v, bool allow_hybrid = true);
// Host-streamed CSR (borrowed host arrays): consumed only by single_pass_fp, chunk by chunk.
std::unique_ptr<Matrix> make_csr_stream(Context& c, std::int64_t m, std::int64_t n, std::int64_t nnz,
                                        const std::int64_t* rp, const std::int32_t* ci, const double* v,
                                        std::int64_t chunk_nnz);

struct Params {
    int alg = 0;          // 0 EI, 1 FP, 2 FP fixed rank, 3 single pass
    int mode = 1;         // 0 fixed rank, 1 fixed precision
    std::int64_t b = 10, power = 0, k = 0, s = 0, max_rank = 0, l_budget = 0, max_restarts = 8;
    double eps_abs = 0.0;
    std::uint64_t seed = 0, stream = 0;
    bool reorth = true;
};

struct Result {
    Context* ctx = nullptr;
    std::int64_t m = 0, n = 0, rank = 0;
    DBuf q, bt;            // Q: m x cap row-major (ld), B^T: n x cap row-major (ld)
    std::int64_t ld = 0;
    double e = -1.0, norm_a_sq = 0.0;
    std::int64_t passes = 0;
    int terminated_by = 0;
    std::int64_t blocks = 0, gaussians_used = 0, restarts = 0, hh_fallbacks = 0;
    double device_ms = 0.0;
    std::vector<double> trace;

    MatView q_view() const { return MatView{q.p, m, rank, ld, true}; }
    MatView bt_view() const { return MatView{bt.p, n, rank, ld, true}; }
};

std::unique_ptr<Result> run(Context& c, Matrix& a, const Params& p);

// qb_to_svd: top-k U (m x k), S, V (n x k) of Q B into host buffers
// (column-major, ldu >= m, ldv >= n); returns the Jacobi sweep count.
int qb_to_svd(Context& c, Result& r, std::int64_t k, double* u, std::int64_t ldu, double* s, double* v,
              std::int64_t ldv);

// Kernel-level hook (include/qbfac_gpu_testing.h): orthonormalise a wide row-major panel.
void test_orth_wide(Context& c, const MatView& x, bool force_bcgs2);

// Operator layer (MatrixHandle::frob_norm_sq / multiply) on device buffers.
double frob_norm_sq(Context& c, Matrix& a);
// Y (rows x w, row-major) = op(A) X (row-major), one pass; A^T results are allreduced.
void multiply(Context& c, Matrix& a, const MatView& x, const MatView& y, bool trans);

}  // namespace qbgpu
