// extern "C" boundary (include/qbfac_gpu.h): exception -> status translation over
// the engine in qb.cu. No C++ exception crosses this layer.

#include <cmath>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "../../include/qbfac_gpu.h"
#include "mtx.cuh"
#include "qb.cuh"

struct qbfac_gpu_ctx {
    std::unique_ptr<qbgpu::Context> c;
    std::string last_error;
    long long launches = 0;  // kernels launched by this context's C-ABI calls
};
struct qbfac_gpu_matrix {
    qbfac_gpu_ctx* ctx = nullptr;
    std::unique_ptr<qbgpu::Matrix> m;
};
struct qbfac_gpu_result {
    qbfac_gpu_ctx* ctx = nullptr;
    std::unique_ptr<qbgpu::Result> r;
};

namespace {

thread_local std::string g_create_error;

template <class Fn>
int guard(qbfac_gpu_ctx* ctx, Fn&& fn, qbfac_info* info = nullptr) {
    auto fail = [&](int st, const std::string& msg) {
        if (ctx) ctx->last_error = msg;
        else g_create_error = msg;
        if (info) info->status = st;
        return st;
    };
    // launches made while this call runs are this context's (QB_LAUNCH_CHECK)
    struct CounterScope {
        long long* prev;
        explicit CounterScope(long long* c) : prev(qbgpu::t_launch_counter) { qbgpu::t_launch_counter = c; }
        ~CounterScope() { qbgpu::t_launch_counter = prev; }
    } scope(ctx ? &ctx->launches : qbgpu::t_launch_counter);
    try {
        if (ctx && ctx->c) {
            cudaError_t e = cudaSetDevice(ctx->c->device);
            if (e != cudaSuccess) return fail(QBFAC_ERROR, cudaGetErrorString(e));
        }
        fn();
        if (info) info->status = QBFAC_OK;
        return QBFAC_OK;
    } catch (const qbgpu::QbError& e) {
        if (info) {
            info->diag_index = e.diag_index;
            info->floor = e.floor;
        }
        return fail(e.status, e.what());
    } catch (const std::bad_alloc&) {
        return fail(QBFAC_RESOURCE_ERROR, "host out of memory");
    } catch (const std::exception& e) {
        return fail(QBFAC_INTERNAL, e.what());
    }
}

}  // namespace

extern "C" {

int qbfac_gpu_create(int device, qbfac_gpu_ctx** out) { return qbfac_gpu_create_dist(device, 0, 1, nullptr, out); }

int qbfac_gpu_create_dist(int device, int rank, int world, const void* nccl_id, qbfac_gpu_ctx** out) {
    if (!out) return QBFAC_ERROR;
    *out = nullptr;
    auto h = std::make_unique<qbfac_gpu_ctx>();
    int st = guard(nullptr, [&] {
        if (world > 1 && !nccl_id) throw qbgpu::QbError(qbgpu::kError, "world > 1 needs an NCCL unique id");
        if (world < 1 || rank < 0 || rank >= world) throw qbgpu::QbError(qbgpu::kDimensionError, "bad rank/world");
        h->c = std::make_unique<qbgpu::Context>(device, rank, world, nccl_id);
    });
    if (st == QBFAC_OK) *out = h.release();
    return st;
}

int qbfac_gpu_nccl_unique_id(void* out128) {
    return guard(nullptr, [&] { qbgpu::Comm::unique_id(out128); });
}

void qbfac_gpu_destroy(qbfac_gpu_ctx* ctx) { delete ctx; }

const char* qbfac_gpu_last_error(const qbfac_gpu_ctx* ctx) {
    return ctx ? ctx->last_error.c_str() : g_create_error.c_str();
}

int qbfac_gpu_synchronize(qbfac_gpu_ctx* ctx) {
    return guard(ctx, [&] {
        QB_CUDA(cudaStreamSynchronize(ctx->c->st_copy));
        QB_CUDA(cudaStreamSynchronize(ctx->c->st));
    });
}

void* qbfac_gpu_stream(qbfac_gpu_ctx* ctx) { return ctx ? static_cast<void*>(ctx->c->st) : nullptr; }

int64_t qbfac_gpu_kernel_launches(const qbfac_gpu_ctx* ctx) {
    return ctx ? ctx->launches : qbgpu::g_kernel_launches.load();
}

// ---- matrices ---------------------------------------------------------------------
int qbfac_gpu_matrix_dense(qbfac_gpu_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda,
                           qbfac_gpu_matrix** out) {
    return qbfac_gpu_matrix_dense_shard(ctx, m, 0, m, n, a, lda, out);
}

int qbfac_gpu_matrix_dense_shard(qbfac_gpu_ctx* ctx, int64_t m_global, int64_t row0, int64_t m_local, int64_t n,
                                 const double* a, int64_t lda, qbfac_gpu_matrix** out) {
    if (!ctx || !out) return QBFAC_ERROR;
    *out = nullptr;
    return guard(ctx, [&] {
        auto h = std::make_unique<qbfac_gpu_matrix>();
        h->ctx = ctx;
        h->m = qbgpu::make_dense(*ctx->c, m_global, row0, m_local, n, a, lda, false);
        *out = h.release();
    });
}

int qbfac_gpu_matrix_dense_device(qbfac_gpu_ctx* ctx, int64_t m, int64_t n, const double* dev_a, int64_t lda,
                                  qbfac_gpu_matrix** out) {
    if (!ctx || !out) return QBFAC_ERROR;
    *out = nullptr;
    return guard(ctx, [&] {
        auto h = std::make_unique<qbfac_gpu_matrix>();
        h->ctx = ctx;
        h->m = qbgpu::make_dense(*ctx->c, m, 0, m, n, dev_a, lda, true);
        *out = h.release();
    });
}

int qbfac_gpu_matrix_dense_async(qbfac_gpu_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda,
                                 int64_t chunk_rows, qbfac_gpu_matrix** out) {
    if (!ctx || !out) return QBFAC_ERROR;
    *out = nullptr;
    return guard(ctx, [&] {
        auto h = std::make_unique<qbfac_gpu_matrix>();
        h->ctx = ctx;
        h->m = qbgpu::make_dense_async(*ctx->c, m, n, a, lda, chunk_rows);
        *out = h.release();
    });
}

int qbfac_gpu_matrix_dense_stream(qbfac_gpu_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda,
                                  int64_t chunk_rows, qbfac_gpu_matrix** out) {
    if (!ctx || !out) return QBFAC_ERROR;
    *out = nullptr;
    return guard(ctx, [&] {
        auto h = std::make_unique<qbfac_gpu_matrix>();
        h->ctx = ctx;
        h->m = qbgpu::make_dense_stream(*ctx->c, m, n, a, lda, chunk_rows);
        *out = h.release();
    });
}

int qbfac_gpu_matrix_csr(qbfac_gpu_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr,
                         const int32_t* col_idx, const double* values, qbfac_gpu_matrix** out) {
    return qbfac_gpu_matrix_csr_shard(ctx, m, 0, m, n, nnz, row_ptr, col_idx, values, out);
}

int qbfac_gpu_matrix_csr_stream(qbfac_gpu_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr,
                                const int32_t* col_idx, const double* values, int64_t chunk_nnz,
                                qbfac_gpu_matrix** out) {
    if (!ctx || !out) return QBFAC_ERROR;
    *out = nullptr;
    return guard(ctx, [&] {
        auto h = std::make_unique<qbfac_gpu_matrix>();
        h->ctx = ctx;
        h->m = qbgpu::make_csr_stream(*ctx->c, m, n, nnz, row_ptr, col_idx, values, chunk_nnz);
        *out = h.release();
    });
}

int qbfac_gpu_matrix_csr_shard(qbfac_gpu_ctx* ctx, int64_t m_global, int64_t row0, int64_t m_local, int64_t n,
                               int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx, const double* values,
                               qbfac_gpu_matrix** out) {
    if (!ctx || !out) return QBFAC_ERROR;
    *out = nullptr;
    return guard(ctx, [&] {
        auto h = std::make_unique<qbfac_gpu_matrix>();
        h->ctx = ctx;
        h->m = qbgpu::make_csr(*ctx->c, m_global, row0, m_local, n, nnz, row_ptr, col_idx, values);
        *out = h.release();
    });
}

// ---- Matrix Market and matrix export ------------------------------------
const char* qbfac_mtx_last_error(void) { return g_create_error.c_str(); }

int qbfac_mtx_info(const char* path, int* coordinate, int64_t* m, int64_t* n, int64_t* nnz) {
    return guard(nullptr, [&] {
        const auto i = qbgpu::mtx_info(path);
        *coordinate = i.coordinate ? 1 : 0;
        *m = i.m;
        *n = i.n;
        *nnz = i.nnz;
    });
}

int qbfac_mtx_read_csr(const char* path, int64_t* row_ptr, int32_t* col_idx, double* values) {
    return guard(nullptr, [&] {
        qbgpu::MtxInfo i{};
        std::vector<int64_t> rp;
        std::vector<int32_t> ci;
        std::vector<double> v;
        qbgpu::mtx_read_csr(path, i, rp, ci, v);
        std::memcpy(row_ptr, rp.data(), sizeof(int64_t) * rp.size());
        if (!v.empty()) {
            std::memcpy(col_idx, ci.data(), sizeof(int32_t) * ci.size());
            std::memcpy(values, v.data(), sizeof(double) * v.size());
        }
    });
}

int qbfac_mtx_read_dense(const char* path, double* a, int64_t lda) {
    return guard(nullptr, [&] {
        qbgpu::MtxInfo i{};
        std::vector<double> v;
        qbgpu::mtx_read_dense(path, i, v);
        for (int64_t j = 0; j < i.n; ++j)
            for (int64_t r = 0; r < i.m; ++r) a[r + j * lda] = v[static_cast<size_t>(r + j * i.m)];
    });
}

int qbfac_mtx_write_csr(const char* path, int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr,
                        const int32_t* col_idx, const double* values) {
    return guard(nullptr, [&] { qbgpu::mtx_write_csr(path, m, n, nnz, row_ptr, col_idx, values); });
}

int qbfac_mtx_write_dense(const char* path, int64_t m, int64_t n, const double* a, int64_t lda) {
    return guard(nullptr, [&] { qbgpu::mtx_write_dense(path, m, n, a, lda); });
}

int qbfac_gpu_matrix_mtx(qbfac_gpu_ctx* ctx, const char* path, qbfac_gpu_matrix** out) {
    if (!ctx || !out) return QBFAC_ERROR;
    *out = nullptr;
    return guard(ctx, [&] {
        auto h = std::make_unique<qbfac_gpu_matrix>();
        h->ctx = ctx;
        qbgpu::MtxInfo i{};
        const auto head = qbgpu::mtx_info(path);
        if (head.coordinate) {
            std::vector<int64_t> rp;
            std::vector<int32_t> ci;
            std::vector<double> v;
            qbgpu::mtx_read_csr(path, i, rp, ci, v);
            h->m = qbgpu::make_csr(*ctx->c, i.m, 0, i.m, i.n, i.nnz, rp.data(), ci.data(), v.data());
        } else {
            std::vector<double> a;
            qbgpu::mtx_read_dense(path, i, a);
            h->m = qbgpu::make_dense(*ctx->c, i.m, 0, i.m, i.n, a.data(), std::max<int64_t>(i.m, 1), false);
        }
        *out = h.release();
    });
}

int qbfac_gpu_matrix_shape(const qbfac_gpu_matrix* mat, int* sparse, int64_t* m, int64_t* n, int64_t* nnz) {
    if (!mat || !mat->m) return QBFAC_ERROR;
    *sparse = mat->m->sparse ? 1 : 0;
    *m = mat->m->m;
    *n = mat->m->n;
    *nnz = mat->m->sparse ? mat->m->nnz : mat->m->m * mat->m->n;
    return QBFAC_OK;
}

int qbfac_gpu_matrix_export_csr(qbfac_gpu_ctx* ctx, const qbfac_gpu_matrix* mat, int64_t* row_ptr, int32_t* col_idx,
                                double* values) {
    return guard(ctx, [&] {
        const auto& a = *mat->m;
        if (!a.sparse) throw qbgpu::QbError(qbgpu::kDimensionError, "export_csr: dense matrix");
        QB_CUDA(cudaMemcpyAsync(row_ptr, a.rp, sizeof(int64_t) * (a.m + 1), cudaMemcpyDeviceToHost, ctx->c->st));
        if (a.nnz > 0) {
            QB_CUDA(cudaMemcpyAsync(col_idx, a.ci, sizeof(int32_t) * a.nnz, cudaMemcpyDeviceToHost, ctx->c->st));
            QB_CUDA(cudaMemcpyAsync(values, a.v, sizeof(double) * a.nnz, cudaMemcpyDeviceToHost, ctx->c->st));
        }
        QB_CUDA(cudaStreamSynchronize(ctx->c->st));
    });
}

int qbfac_gpu_matrix_export_dense(qbfac_gpu_ctx* ctx, const qbfac_gpu_matrix* mat, double* a, int64_t lda) {
    return guard(ctx, [&] {
        const auto& x = *mat->m;
        if (x.sparse) throw qbgpu::QbError(qbgpu::kDimensionError, "export_dense: sparse matrix");
        if (x.m > 0 && x.n > 0)
            QB_CUDA(cudaMemcpy2DAsync(a, sizeof(double) * lda, x.a, sizeof(double) * x.lda, sizeof(double) * x.m, x.n,
                                      cudaMemcpyDeviceToHost, ctx->c->st));
        QB_CUDA(cudaStreamSynchronize(ctx->c->st));
    });
}

void qbfac_gpu_matrix_free(qbfac_gpu_matrix* mat) {
    if (!mat) return;
    if (mat->ctx && mat->ctx->c) cudaSetDevice(mat->ctx->c->device);
    delete mat;
}

int64_t qbfac_gpu_matrix_passes(const qbfac_gpu_matrix* mat) { return mat ? mat->m->passes : 0; }

int qbfac_gpu_frob_norm_sq(qbfac_gpu_ctx* ctx, qbfac_gpu_matrix* mat, double* out) {
    return guard(ctx, [&] { *out = qbgpu::frob_norm_sq(*ctx->c, *mat->m); });
}

int qbfac_gpu_multiply(qbfac_gpu_ctx* ctx, qbfac_gpu_matrix* mat, const double* x, int64_t w, int trans, double* y) {
    return guard(ctx, [&] {
        auto& c = *ctx->c;
        auto& a = *mat->m;
        const int64_t xr = trans ? a.m : a.n;
        const int64_t yr = trans ? a.n : a.m;
        qbgpu::DBuf xc(static_cast<size_t>(xr * w), c.st), xrm(static_cast<size_t>(xr * w), c.st);
        qbgpu::DBuf yrm(static_cast<size_t>(yr * w), c.st), yc(static_cast<size_t>(yr * w), c.st);
        if (xr * w > 0) QB_CUDA(cudaMemcpyAsync(xc.p, x, sizeof(double) * xr * w, cudaMemcpyHostToDevice, c.st));
        qbgpu::MatView xcv{xc.p, xr, w, std::max<int64_t>(xr, 1), false};
        qbgpu::MatView xrv{xrm.p, xr, w, std::max<int64_t>(w, 1), true};
        qbgpu::MatView yrv{yrm.p, yr, w, std::max<int64_t>(w, 1), true};
        qbgpu::MatView ycv{yc.p, yr, w, std::max<int64_t>(yr, 1), false};
        qbgpu::copy_matrix(c.st, xcv, xrv);
        qbgpu::multiply(c, a, xrv, yrv, trans != 0);
        qbgpu::copy_matrix(c.st, yrv, ycv);
        if (yr * w > 0) QB_CUDA(cudaMemcpyAsync(y, yc.p, sizeof(double) * yr * w, cudaMemcpyDeviceToHost, c.st));
        QB_CUDA(cudaStreamSynchronize(c.st));
    });
}

int qbfac_gpu_multiply_device(qbfac_gpu_ctx* ctx, qbfac_gpu_matrix* mat, const double* x, int64_t ldx, int64_t w,
                              int trans, double* y, int64_t ldy) {
    return guard(ctx, [&] {
        auto& a = *mat->m;
        const int64_t xr = trans ? a.m : a.n;
        const int64_t yr = trans ? a.n : a.m;
        qbgpu::MatView xv{const_cast<double*>(x), xr, w, ldx, true};
        qbgpu::MatView yv{y, yr, w, ldy, true};
        qbgpu::multiply(*ctx->c, a, xv, yv, trans != 0);
    });
}

int qbfac_gpu_gaussian(qbfac_gpu_ctx* ctx, uint64_t seed, uint64_t stream, uint64_t skip, int64_t rows, int64_t cols,
                       double* out) {
    return guard(ctx, [&] {
        if (rows < 1 || cols < 1) throw qbgpu::QbError(qbgpu::kDimensionError, "gaussian: dimensions must be at least 1");
        auto& c = *ctx->c;
        qbgpu::DBuf d(static_cast<size_t>(rows * cols), c.st);
        qbgpu::gaussian_fill(c.st, c.rng, seed, stream, skip, qbgpu::MatView{d.p, rows, cols, rows, false});
        QB_CUDA(cudaMemcpyAsync(out, d.p, sizeof(double) * rows * cols, cudaMemcpyDeviceToHost, c.st));
        QB_CUDA(cudaStreamSynchronize(c.st));
    });
}

int qbfac_gpu_gaussian_device(qbfac_gpu_ctx* ctx, uint64_t seed, uint64_t stream, uint64_t skip, int64_t rows,
                              int64_t cols, double* dev_out, int64_t ld) {
    return guard(ctx, [&] {
        if (rows < 1 || cols < 1) throw qbgpu::QbError(qbgpu::kDimensionError, "gaussian: dimensions must be at least 1");
        auto& c = *ctx->c;
        qbgpu::gaussian_fill(c.st, c.rng, seed, stream, skip, qbgpu::MatView{dev_out, rows, cols, ld, false});
    });
}

// ---- algorithms ---------------------------------------------------------------------
int qbfac_gpu_run(qbfac_gpu_ctx* ctx, qbfac_gpu_matrix* mat, const qbfac_params* params, qbfac_gpu_result** out,
                  qbfac_info* info) {
    if (!ctx || !mat || !params || !out) return QBFAC_ERROR;
    *out = nullptr;
    qbfac_info local{};
    qbfac_info* inf = info ? info : &local;
    std::memset(inf, 0, sizeof(*inf));
    return guard(
        ctx,
        [&] {
            qbgpu::Params p;
            p.alg = params->alg;
            p.mode = params->mode;
            p.b = params->b;
            p.power = params->power;
            p.k = params->k;
            p.s = params->s;
            p.max_rank = params->max_rank;
            p.l_budget = params->l_budget;
            p.max_restarts = params->max_restarts;
            p.eps_abs = params->eps_abs;
            p.seed = params->seed;
            p.stream = params->stream;
            p.reorth = params->reorth != 0;
            if (p.power < 0) throw qbgpu::QbError(qbgpu::kDimensionError, "power must be >= 0");
            auto h = std::make_unique<qbfac_gpu_result>();
            h->ctx = ctx;
            h->r = qbgpu::run(*ctx->c, *mat->m, p);
            const auto& r = *h->r;
            inf->rank = r.rank;
            inf->error_indicator = r.e;
            inf->norm_a_sq = r.norm_a_sq;
            inf->passes = r.passes;
            inf->terminated_by = r.terminated_by;
            inf->m = r.m;
            inf->n = r.n;
            inf->blocks = r.blocks;
            inf->gaussians_used = r.gaussians_used;
            inf->restarts = r.restarts;
            inf->householder_fallbacks = r.hh_fallbacks;
            inf->device_ms = r.device_ms;
            *out = h.release();
        },
        inf);
}

int qbfac_gpu_result_copy_q(qbfac_gpu_result* res, double* q, int64_t ldq) {
    if (!res) return QBFAC_ERROR;
    return guard(res->ctx, [&] {
        auto& r = *res->r;
        auto& c = *res->ctx->c;
        if (r.rank == 0 || r.m == 0) return;
        if (ldq < r.m) throw qbgpu::QbError(qbgpu::kDimensionError, "copy_q: ldq < m");
        qbgpu::DBuf t(static_cast<size_t>(r.m * r.rank), c.st);
        qbgpu::MatView tv{t.p, r.m, r.rank, r.m, false};
        qbgpu::copy_matrix(c.st, r.q_view(), tv);
        QB_CUDA(cudaMemcpy2DAsync(q, ldq * sizeof(double), t.p, r.m * sizeof(double), r.m * sizeof(double), r.rank,
                                  cudaMemcpyDeviceToHost, c.st));
        QB_CUDA(cudaStreamSynchronize(c.st));
    });
}

int qbfac_gpu_result_copy_b(qbfac_gpu_result* res, double* b, int64_t ldb) {
    if (!res) return QBFAC_ERROR;
    return guard(res->ctx, [&] {
        auto& r = *res->r;
        auto& c = *res->ctx->c;
        if (r.rank == 0 || r.n == 0) return;
        if (ldb < r.rank) throw qbgpu::QbError(qbgpu::kDimensionError, "copy_b: ldb < rank");
        // B(i, j) = B^T(j, i): column j of B is row j of the row-major B^T.
        QB_CUDA(cudaMemcpy2DAsync(b, ldb * sizeof(double), r.bt.p, r.ld * sizeof(double), r.rank * sizeof(double), r.n,
                                  cudaMemcpyDeviceToHost, c.st));
        QB_CUDA(cudaStreamSynchronize(c.st));
    });
}

int64_t qbfac_gpu_result_copy_trace(qbfac_gpu_result* res, double* out, int64_t cap) {
    if (!res) return 0;
    const auto& tr = res->r->trace;
    const int64_t n = std::min<int64_t>(cap, static_cast<int64_t>(tr.size()));
    if (out && n > 0) std::memcpy(out, tr.data(), sizeof(double) * n);
    return static_cast<int64_t>(tr.size());
}

int qbfac_gpu_result_svd(qbfac_gpu_result* res, int64_t k, double* u, int64_t ldu, double* s, double* v,
                         int64_t ldv, int* sweeps) {
    if (!res) return QBFAC_ERROR;
    return guard(res->ctx, [&] {
        const int sw = qbgpu::qb_to_svd(*res->ctx->c, *res->r, k, u, ldu, s, v, ldv);
        if (sweeps) *sweeps = sw;
    });
}

void qbfac_gpu_result_free(qbfac_gpu_result* res) {
    if (!res) return;
    if (res->ctx && res->ctx->c) cudaSetDevice(res->ctx->c->device);
    delete res;
}

int qbfac_gpu_validate_epsilon(double eps, double frob_a, double delta, double* floor_out) {
    const double floor = std::sqrt(4.0 * 1.1102230246251565e-16 / delta) * frob_a;
    if (floor_out) *floor_out = floor;
    return eps > floor ? 1 : 0;
}

}  // extern "C"

// ---- kernel-level test hooks (include/qbfac_gpu_testing.h) ------------------------------
#include "../../include/qbfac_gpu_testing.h"

extern "C" {

int qbfac_gpu_test_gemm(qbfac_gpu_ctx* ctx, double alpha, const double* a, int64_t m, int64_t k, int64_t lda,
                        int a_row, const double* b, int64_t n, int64_t ldb, int b_row, double beta, double* c,
                        int64_t ldc, int c_row) {
    return guard(ctx, [&] {
        auto& cx = *ctx->c;
        qbgpu::MatView av{const_cast<double*>(a), m, k, lda, a_row != 0};
        qbgpu::MatView bv{const_cast<double*>(b), k, n, ldb, b_row != 0};
        qbgpu::MatView cv{c, m, n, ldc, c_row != 0};
        qbgpu::gemm(cx.st, cx.ws_gemm, alpha, av, bv, beta, cv);
        QB_CUDA(cudaStreamSynchronize(cx.st));
    });
}

int qbfac_gpu_test_chol(qbfac_gpu_ctx* ctx, const double* g, int b, double* r, double* rinv, int* status) {
    return guard(ctx, [&] {
        auto& cx = *ctx->c;
        qbgpu::chol_small(cx.st, g, b, b, r, rinv, b, cx.d_status);
        QB_CUDA(cudaMemcpyAsync(cx.h_status, cx.d_status, sizeof(qbgpu::SmallStatus), cudaMemcpyDeviceToHost, cx.st));
        QB_CUDA(cudaStreamSynchronize(cx.st));
        *status = cx.h_status->breakdown;
    });
}

int qbfac_gpu_test_chol_wide(qbfac_gpu_ctx* ctx, double* g, int l, double* r, double* rinv, int* breakdown) {
    return guard(ctx, [&] {
        auto& cx = *ctx->c;
        const int nt = (l + 63) / 64;
        qbgpu::DBuf st(static_cast<std::size_t>(nt) * 4, cx.st);
        QB_CUDA(cudaMemsetAsync(r, 0, sizeof(double) * l * l, cx.st));
        QB_CUDA(cudaMemsetAsync(rinv, 0, sizeof(double) * l * l, cx.st));
        auto* stats = reinterpret_cast<qbgpu::SmallStatus*>(st.p);
        qbgpu::chol_wide(cx.st, g, l, l, r, rinv, l, stats);
        std::vector<qbgpu::SmallStatus> hs(static_cast<std::size_t>(nt));
        QB_CUDA(cudaMemcpyAsync(hs.data(), stats, sizeof(qbgpu::SmallStatus) * nt, cudaMemcpyDeviceToHost, cx.st));
        QB_CUDA(cudaStreamSynchronize(cx.st));
        *breakdown = 0;
        for (const auto& s : hs) *breakdown |= s.breakdown;
    });
}

int qbfac_gpu_test_cholqr2(qbfac_gpu_ctx* ctx, const double* y, int64_t rows, int b, int64_t ldy, double* q,
                           int64_t ldq, double* r, double* rinv, int* status) {
    return guard(ctx, [&] {
        auto& cx = *ctx->c;
        constexpr int S = qbgpu::kSmallMax * qbgpu::kSmallMax;
        qbgpu::DBuf small(static_cast<std::size_t>(S) * 5, cx.st);
        qbgpu::DBuf t1(static_cast<std::size_t>(std::max<int64_t>(rows, 1)) * b, cx.st);
        qbgpu::DBuf st(8, cx.st);
        auto* sts = reinterpret_cast<qbgpu::SmallStatus*>(st.p);
        double* sl = small.p;
        qbgpu::cholqr2_panel(cx.st, cx.ws_panel, y, rows, b, ldy, t1.p, q, ldq, sl, sl + S, sl + 2 * S, sl + 3 * S,
                             sl + 4 * S, sts, sts + 1, cx.d_gbar);
        qbgpu::trmm_upper_pair(cx.st, sl + 3 * S, sl + S, r, sl + 2 * S, sl + 4 * S, rinv, b, qbgpu::kSmallMax);
        qbgpu::SmallStatus h[2];
        QB_CUDA(cudaMemcpyAsync(h, sts, sizeof(h), cudaMemcpyDeviceToHost, cx.st));
        QB_CUDA(cudaStreamSynchronize(cx.st));
        *status = h[0].breakdown | (h[1].breakdown << 1);
    });
}

int qbfac_gpu_test_create_local_group(int device, int world, qbfac_gpu_ctx** outs) {
    if (!outs || world < 2) return QBFAC_ERROR;
    for (int r = 0; r < world; ++r) outs[r] = nullptr;
    std::vector<std::unique_ptr<qbfac_gpu_ctx>> hs;
    int st = guard(nullptr, [&] {
        auto g = std::make_shared<qbgpu::LocalGroup>(world);
        for (int r = 0; r < world; ++r) {
            hs.push_back(std::make_unique<qbfac_gpu_ctx>());
            hs.back()->c = std::make_unique<qbgpu::Context>(device, r, world, nullptr, g);
        }
    });
    if (st == QBFAC_OK)
        for (int r = 0; r < world; ++r) outs[r] = hs[static_cast<std::size_t>(r)].release();
    return st;
}

int qbfac_gpu_test_allreduce(qbfac_gpu_ctx* ctx, double* dev, int64_t count) {
    if (!ctx) return QBFAC_ERROR;
    return guard(ctx, [&] {
        if (!ctx->c->comm) throw qbgpu::QbError(qbgpu::kError, "context has no communicator");
        ctx->c->allreduce(dev, static_cast<std::size_t>(count));
        QB_CUDA(cudaStreamSynchronize(ctx->c->st));
    });
}

int qbfac_gpu_test_collective(qbfac_gpu_ctx* ctx, int op, const double* send, double* recv, int64_t count) {
    if (!ctx) return QBFAC_ERROR;
    return guard(ctx, [&] {
        if (!ctx->c->comm) throw qbgpu::QbError(qbgpu::kError, "context has no communicator");
        if (op == 1) ctx->c->reduce_scatter(send, recv, static_cast<std::size_t>(count));
        else if (op == 2) ctx->c->all_gather(send, recv, static_cast<std::size_t>(count));
        else throw qbgpu::QbError(qbgpu::kDimensionError, "collective: op must be 1 (reduce-scatter) or 2 (all-gather)");
        QB_CUDA(cudaStreamSynchronize(ctx->c->st));
    });
}

int qbfac_gpu_test_chol_wide_trace(qbfac_gpu_ctx* ctx, unsigned long long* out) {
    return guard(ctx, [&] {
        QB_CUDA(cudaStreamSynchronize(ctx->c->st));
        qbgpu::chol_wide_trace(out);
    });
}

int qbfac_gpu_test_panel_trace(qbfac_gpu_ctx* ctx, unsigned long long* out) {
    return guard(ctx, [&] {
        QB_CUDA(cudaStreamSynchronize(ctx->c->st));
        qbgpu::panel_trace(out);
    });
}

int qbfac_gpu_test_householder(qbfac_gpu_ctx* ctx, double* y, int64_t m, int b, int64_t ld, double* r) {
    return guard(ctx, [&] {
        auto& cx = *ctx->c;
        qbgpu::householder_panel(cx.st, cx.ws_hh, y, m, b, ld, r, b);
        QB_CUDA(cudaStreamSynchronize(cx.st));
    });
}

int qbfac_gpu_test_orth_wide(qbfac_gpu_ctx* ctx, double* x, int64_t rows, int64_t l, int force_bcgs2) {
    return guard(ctx, [&] {
        qbgpu::test_orth_wide(*ctx->c, qbgpu::MatView{x, rows, l, l, true}, force_bcgs2 != 0);
    });
}

int qbfac_gpu_test_colsumsq(qbfac_gpu_ctx* ctx, const double* x, int64_t rows, int64_t cols, int64_t ld, int row,
                            double* out) {
    return guard(ctx, [&] {
        auto& cx = *ctx->c;
        qbgpu::column_sumsq(cx.st, cx.ws_red, qbgpu::MatView{const_cast<double*>(x), rows, cols, ld, row != 0}, out);
        QB_CUDA(cudaStreamSynchronize(cx.st));
    });
}

int qbfac_gpu_test_csr_spmm(qbfac_gpu_ctx* ctx, int64_t rows, int64_t cols, int64_t nnz, const int64_t* rp,
                            const int32_t* ci, const double* v, const double* x, int64_t ldx, double* y, int64_t ldy,
                            int w, double alpha, double beta) {
    return guard(ctx, [&] {
        auto& cx = *ctx->c;
        qbgpu::CsrView a{rows, cols, nnz, rp, ci, v, {}};
        std::vector<int64_t> rph(static_cast<size_t>(rows + 1));
        QB_CUDA(cudaMemcpy(rph.data(), rp, sizeof(int64_t) * (rows + 1), cudaMemcpyDeviceToHost));
        a.heavy = qbgpu::make_heavy_plan(rph.data(), rows, cx.st);
        double* part = a.heavy.nseg ? cx.ws_sp.get(qbgpu::csr_spmm_scratch(a, std::min(w, 256))) : nullptr;
        qbgpu::csr_spmm(cx.st, a, x, ldx, y, ldy, w, alpha, beta, cx.sms, part);
        QB_CUDA(cudaStreamSynchronize(cx.st));
        qbgpu::free_heavy_plan(a.heavy);
        QB_CUDA(cudaStreamSynchronize(cx.st));
    });
}

}  // extern "C"
