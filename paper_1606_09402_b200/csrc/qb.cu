// Device drivers of randQB_EI / randQB_FP / single pass on B200.
//
// Reference semantics (the reference's src/qb.cpp is missing; restated from
// /root/reference/SPEC.md:204-363 and PAPER.md, identically to oracle/qb_restated.cpp):
//   randQB_EI  Alg. 2, with per-block power iteration
//   randQB_FP  Alg. 4, steps 9a-9c PAPER.md:441-447, restarts SPEC.md:347
//   Alg. 3     PAPER.md:352-376 (fixed rank), single pass Remark 4.2 PAPER.md:466-467
//   row-by-row error indicator PAPER.md:206-220, validate_epsilon SPEC.md:327-335
//
// Everything between the upload of A and the copy-out of Q/B runs on the GPU:
// Omega is generated on the device from the reference's stream, the passes over
// A are DMMA GEMMs (dense) or CSR SpMM (sparse), orth() is CholQR2 with a
// Householder-panel fallback (same Q, R as the reference's Householder QR with
// diag(R) >= 0 up to rounding; rank-collapse decisions are taken on the
// Householder R), and the indicator E -= ||B_i(j,:)||^2 with the row truncation
// runs in a device kernel. The host only reads a few status words per block.
//
// Layouts: A dense column-major (lda padded to a multiple of 8); every block vector
// (Omega_i, Y_i, Q_i, B_i^T, G, H) and the accumulated Q (m x cap) and B^T (n x cap)
// are row-major, so CSR passes gather contiguous rows and appending a block is a
// write into a column slot.

#include "qb.cuh"

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <tuple>

namespace qbgpu {

std::atomic<long long> g_kernel_launches{0};
thread_local long long* t_launch_counter = nullptr;

namespace {

constexpr double kRankTol = 1e-12;
constexpr double kEpsMach = 1.1102230246251565e-16;  // types.hpp:14
constexpr double kCholRatioMin = 1e-7;      // below: CholQR R not trusted -> Householder
constexpr double kCholGramDevMax = 0.5;     // second CholQR pass must see a near-identity Gram
constexpr int kSlot = kSmallMax * kSmallMax;
enum SmallSlot { kG = 0, kRa, kRainv, kRb, kRbinv, kR1, kR1inv, kR2, kR2inv, kR, kRinv, kTmp, kNorms, kNumSlots };

}  // namespace

// ---------------------------------------------------------------------------------
Context::Context(int dev, int rank_, int world_, const void* nccl_id, std::shared_ptr<LocalGroup> local)
    : device(dev), rank(rank_), world(world_) {
    QB_CUDA(cudaSetDevice(dev));
    cudaDeviceProp prop{};
    QB_CUDA(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10)
        throw QbError(kError, std::string("qbfac_gpu needs an sm_100 (B200) device, found ") + prop.name);
    sms = prop.multiProcessorCount;
    QB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    QB_CUDA(cudaStreamCreateWithFlags(&st_copy, cudaStreamNonBlocking));
    QB_CUDA(cudaMalloc(&d_small, sizeof(double) * kSlot * kNumSlots + 64 * sizeof(double)));
    QB_CUDA(cudaMalloc(&d_status, sizeof(SmallStatus) * 4));
    QB_CUDA(cudaMalloc(&d_gbar, 64 * sizeof(unsigned)));
    QB_CUDA(cudaMemset(d_gbar, 0, 64 * sizeof(unsigned)));
    QB_CUDA(cudaMalloc(&d_lazy, sizeof(SmallStatus) * kLazyCap));
    QB_CUDA(cudaMallocHost(&h_lazy, sizeof(SmallStatus) * kLazyCap));
    QB_CUDA(cudaMalloc(&d_ind, sizeof(IndicatorOut)));
    QB_CUDA(cudaMallocHost(&h_status, sizeof(SmallStatus) * 4));
    QB_CUDA(cudaMallocHost(&h_ind, sizeof(IndicatorOut)));
    QB_CUDA(cudaMallocHost(&h_scalar, sizeof(double) * 8));
    // Grow the stream-ordered pool's retention so per-run buffers are reused.
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        std::uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    rng.device();
    // world == 1 with an NCCL id: a one-rank communicator (exercises the NCCL path on one GPU)
    if (world > 1 || nccl_id)
        comm = local ? std::make_unique<Comm>(rank, world, std::move(local)) : std::make_unique<Comm>(rank, world, nccl_id);
}

Context::~Context() {
    cudaSetDevice(device);
    if (st) cudaStreamSynchronize(st);
    comm.reset();
    ws_gemm.release();
    ws_red.release();
    ws_hh.release();
    ws_sp.release();
    ws_panel.release();
    if (st_copy) cudaStreamDestroy(st_copy);
    if (d_small) cudaFree(d_small);
    if (d_status) cudaFree(d_status);
    if (d_gbar) cudaFree(d_gbar);
    if (d_lazy) cudaFree(d_lazy);
    if (h_lazy) cudaFreeHost(h_lazy);
    if (d_ind) cudaFree(d_ind);
    if (h_status) cudaFreeHost(h_status);
    if (h_ind) cudaFreeHost(h_ind);
    if (h_scalar) cudaFreeHost(h_scalar);
    if (st) cudaStreamDestroy(st);
}

Matrix::~Matrix() {
    for (auto& ch : pending) {
        cudaEventSynchronize(ch.ready);
        cudaEventDestroy(ch.ready);
    }
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (a && owns_a) {
        if (pooled_a) cudaFreeAsync(a, ctx->st);
        else cudaFree(a);
    }
    if (rp) cudaFree(rp);
    if (ci) cudaFree(ci);
    if (v) cudaFree(v);
    if (ct_rp) cudaFree(ct_rp);
    if (ct_ci) cudaFree(ct_ci);
    if (ct_v) cudaFree(ct_v);
    free_heavy_plan(heavy);
    free_heavy_plan(heavy_t);
    for (void* p : {static_cast<void*>(s_rp), static_cast<void*>(s_ci), static_cast<void*>(s_v),
                    static_cast<void*>(d_rows), static_cast<void*>(d_cols), static_cast<void*>(d_r),
                    static_cast<void*>(d_c)})
        if (p) cudaFree(p);
}

std::unique_ptr<Matrix> make_dense(Context& c, std::int64_t m_global, std::int64_t row0, std::int64_t m,
                                   std::int64_t n, const double* a, std::int64_t lda, bool device_src) {
    if (m < 0 || n < 0 || lda < std::max<std::int64_t>(1, m))
        throw QbError(kDimensionError, "matrix_dense: bad dimensions");
    auto mat = std::make_unique<Matrix>();
    mat->ctx = &c;
    mat->m = m;
    mat->n = n;
    mat->m_global = m_global;
    mat->row0 = row0;
    mat->lda = std::max<std::int64_t>(8, round_up(m, 8));
    // stream-ordered pool (retained across calls): no cudaMalloc/cudaFree of the whole matrix per upload
    QB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&mat->a), sizeof(double) * mat->lda * std::max<std::int64_t>(n, 1), c.st));
    mat->pooled_a = true;
    if (mat->lda != m) QB_CUDA(cudaMemsetAsync(mat->a, 0, sizeof(double) * mat->lda * std::max<std::int64_t>(n, 1), c.st));
    if (m > 0 && n > 0)
        QB_CUDA(cudaMemcpy2DAsync(mat->a, mat->lda * sizeof(double), a, lda * sizeof(double), m * sizeof(double), n,
                                  device_src ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.st));
    // DenseMatrix::from_data rejects non-finite entries (dense_matrix.cpp:17-18).
    if (m > 0 && n > 0) {
        sum_squares(c.st, c.ws_red, mat->dense_view(), c.d_small + kSlot * kNumSlots);
        QB_CUDA(cudaMemcpyAsync(c.h_scalar, c.d_small + kSlot * kNumSlots, sizeof(double), cudaMemcpyDeviceToHost, c.st));
    }
    QB_CUDA(cudaStreamSynchronize(c.st));
    if (m > 0 && n > 0 && !std::isfinite(c.h_scalar[0])) throw QbError(kError, "from_data: non-finite entry");
    return mat;
}

std::unique_ptr<Matrix> make_dense_async(Context& c, std::int64_t m, std::int64_t n, const double* a,
                                         std::int64_t lda, std::int64_t chunk_rows) {
    if (m < 0 || n < 0 || lda < std::max<std::int64_t>(1, m))
        throw QbError(kDimensionError, "matrix_dense: bad dimensions");
    auto mat = std::make_unique<Matrix>();
    mat->ctx = &c;
    mat->m = m;
    mat->n = n;
    mat->m_global = m;
    mat->lda = std::max<std::int64_t>(8, round_up(m, 8));
    QB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&mat->a), sizeof(double) * mat->lda * std::max<std::int64_t>(n, 1),
                            c.st_copy));
    mat->pooled_a = true;
    if (mat->lda != m) {
        QB_CUDA(cudaMemsetAsync(mat->a, 0, sizeof(double) * mat->lda * std::max<std::int64_t>(n, 1), c.st_copy));
    }
    if (m == 0 || n == 0) return mat;
    // ~9 row chunks of whole 128-row GEMM tiles (896 rows at m = 8000: measured best for the config-2
    // first pass with the per-chunk Gram behind it, tools/e2e_chunk_sweep.py)
    if (chunk_rows <= 0) chunk_rows = std::max<std::int64_t>(896, round_up(ceil_div(m, 9), 128));
    for (std::int64_t r0 = 0; r0 < m; r0 += chunk_rows) {
        const std::int64_t rows = std::min(chunk_rows, m - r0);
        QB_CUDA(cudaMemcpy2DAsync(mat->a + r0, mat->lda * sizeof(double), a + r0, lda * sizeof(double),
                                  rows * sizeof(double), n, cudaMemcpyHostToDevice, c.st_copy));
        cudaEvent_t ev;
        QB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        QB_CUDA(cudaEventRecord(ev, c.st_copy));
        mat->pending.push_back(Matrix::Chunk{r0 + rows, ev});
    }
    mat->check_finite = true;
    return mat;
}

std::unique_ptr<Matrix> make_dense_stream(Context& c, std::int64_t m, std::int64_t n, const double* a,
                                          std::int64_t lda, std::int64_t chunk_rows) {
    if (m < 0 || n < 0 || lda < std::max<std::int64_t>(1, m) || (m > 0 && n > 0 && !a))
        throw QbError(kDimensionError, "matrix_dense_stream: bad dimensions");
    // the streamed single pass forms H and ||A||^2 of the local rows only: no row-sharded RowStream
    if (c.world > 1) throw QbError(kError, "matrix_dense_stream: a host RowStream is single-GPU (world == 1)");
    auto mat = std::make_unique<Matrix>();
    mat->ctx = &c;
    mat->m = m;
    mat->n = n;
    mat->m_global = m;
    mat->host_stream = true;
    mat->host_a = a;
    mat->host_lda = lda;
    // ~128 MB per chunk, whole 128-row GEMM tiles
    if (chunk_rows <= 0)
        chunk_rows = std::max<std::int64_t>(128, round_up((std::int64_t{128} << 20) / (8 * std::max<std::int64_t>(n, 1)), 128));
    mat->chunk_rows = chunk_rows;
    return mat;
}

void Matrix::wait_resident(cudaStream_t s) {
    for (auto& ch : pending) {
        QB_CUDA(cudaStreamWaitEvent(s, ch.ready, 0));
        cudaEventDestroy(ch.ready);
    }
    pending.clear();
}

std::unique_ptr<Matrix> make_csr_stream(Context& c, std::int64_t m, std::int64_t n, std::int64_t nnz,
                                        const std::int64_t* rp, const std::int32_t* ci, const double* v,
                                        std::int64_t chunk_nnz) {
    if (n > static_cast<std::int64_t>(INT32_MAX))
        throw QbError(kDimensionError, "csr: column count exceeds 32-bit index range");
    if (m < 0 || n < 0 || nnz < 0 || !rp || (nnz > 0 && (!ci || !v)))
        throw QbError(kFormatError, "csr: inconsistent structure arrays");
    if (c.world > 1) throw QbError(kError, "matrix_csr_stream: a host RowStream is single-GPU (world == 1)");
    // row_ptr must be a valid partition before it is used to cut chunks (sparse_csr.cpp:16-20);
    // column indices and values are validated per chunk on the device as each one is uploaded
    if (rp[0] != 0 || rp[m] != nnz) throw QbError(kFormatError, "csr: row_ptr does not span the entries");
    for (std::int64_t i = 0; i < m; ++i)
        if (rp[i + 1] < rp[i]) throw QbError(kFormatError, "csr: row_ptr not non-decreasing");
    auto mat = std::make_unique<Matrix>();
    mat->ctx = &c;
    mat->sparse = true;
    mat->m = m;
    mat->n = n;
    mat->m_global = m;
    mat->nnz = nnz;
    mat->host_stream = true;
    mat->host_rp = rp;
    mat->host_ci = ci;
    mat->host_v = v;
    mat->chunk_nnz = chunk_nnz > 0 ? chunk_nnz : (std::int64_t{16} << 20);  // ~200 MB of entries
    return mat;
}

std::unique_ptr<Matrix> make_csr(Context& c, std::int64_t m_global, std::int64_t row0, std::int64_t m,
                                 std::int64_t n, std::int64_t nnz, const std::int64_t* rp, const std::int32_t* ci,
                                 const double* v, bool allow_hybrid) {
    if (n > static_cast<std::int64_t>(INT32_MAX))
        throw QbError(kDimensionError, "csr: column count exceeds 32-bit index range");
    if (m < 0 || n < 0 || nnz < 0) throw QbError(kFormatError, "csr: inconsistent structure arrays");
    auto mat = std::make_unique<Matrix>();
    mat->ctx = &c;
    mat->sparse = true;
    mat->m = m;
    mat->n = n;
    mat->m_global = m_global;
    mat->row0 = row0;
    mat->nnz = nnz;
    QB_CUDA(cudaMalloc(&mat->rp, sizeof(std::int64_t) * (m + 1)));
    QB_CUDA(cudaMalloc(&mat->ci, sizeof(std::int32_t) * std::max<std::int64_t>(nnz, 1)));
    QB_CUDA(cudaMalloc(&mat->v, sizeof(double) * std::max<std::int64_t>(nnz, 1)));
    QB_CUDA(cudaMalloc(&mat->ct_rp, sizeof(std::int64_t) * (n + 1)));
    QB_CUDA(cudaMalloc(&mat->ct_ci, sizeof(std::int32_t) * std::max<std::int64_t>(nnz, 1)));
    QB_CUDA(cudaMalloc(&mat->ct_v, sizeof(double) * std::max<std::int64_t>(nnz, 1)));
    QB_CUDA(cudaMemcpyAsync(mat->rp, rp, sizeof(std::int64_t) * (m + 1), cudaMemcpyHostToDevice, c.st));
    if (nnz > 0) {
        QB_CUDA(cudaMemcpyAsync(mat->ci, ci, sizeof(std::int32_t) * nnz, cudaMemcpyHostToDevice, c.st));
        QB_CUDA(cudaMemcpyAsync(mat->v, v, sizeof(double) * nnz, cudaMemcpyHostToDevice, c.st));
    }
    const int flags = csr_validate(c.st, m, n, nnz, mat->rp, mat->ci, mat->v, c.sms);
    if (flags & 1) throw QbError(kFormatError, "csr: invalid structure (row_ptr / column indices)");
    if (flags & 2) throw QbError(kError, "csr: non-finite value");
    // Power-law matrices: rows with >= max(1024, n/16) entries and (outside those rows) columns
    // with >= max(4096, m/16) entries are stored dense and multiplied on the FP64 tensor cores;
    // a dense block costs 2w flops per stored element on DMMA, a CSR entry an 8w-byte L2/HBM
    // gather, which DMMA beats above ~6 % density (config 5 measured best at 1/16 among 1/8,
    // 1/16, 1/32; QBFAC_DENSE_DIVR / _DIVC override, QBFAC_CSR_DENSE=0 disables). Blocks are
    // capped at 4 GB each.
    const char* hyb_env = std::getenv("QBFAC_CSR_DENSE");
    const bool hyb_ok = allow_hybrid && !(hyb_env && hyb_env[0] == '0') && m > 0 && n > 0 && nnz > 0;
    std::vector<std::int32_t> rowmap, colmap;
    std::vector<std::int64_t> drows, dcols;
    std::int64_t extracted = 0;
    if (hyb_ok) {
        const int div_r = std::getenv("QBFAC_DENSE_DIVR") ? std::atoi(std::getenv("QBFAC_DENSE_DIVR")) : 16;
        const int div_c = std::getenv("QBFAC_DENSE_DIVC") ? std::atoi(std::getenv("QBFAC_DENSE_DIVC")) : 16;
        const std::int64_t row_thr = std::max<std::int64_t>(1024, n / div_r), col_thr = std::max<std::int64_t>(4096, m / div_c);
        const std::int64_t cap_rows = (std::int64_t{4} << 30) / (8 * n), cap_cols = (std::int64_t{4} << 30) / (8 * m);
        rowmap.assign(static_cast<std::size_t>(m), -1);
        std::vector<std::pair<std::int64_t, std::int64_t>> rl;
        for (std::int64_t i = 0; i < m; ++i)
            if (rp[i + 1] - rp[i] >= row_thr) rl.push_back({rp[i + 1] - rp[i], i});
        std::stable_sort(rl.begin(), rl.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
        if (static_cast<std::int64_t>(rl.size()) > cap_rows) rl.resize(static_cast<std::size_t>(cap_rows));
        for (const auto& x : rl) drows.push_back(x.second);
        std::sort(drows.begin(), drows.end());
        for (std::size_t r = 0; r < drows.size(); ++r) {
            rowmap[static_cast<std::size_t>(drows[r])] = static_cast<std::int32_t>(r);
            extracted += rp[drows[r] + 1] - rp[drows[r]];
        }
        std::vector<std::int64_t> cc(static_cast<std::size_t>(n), 0);
        for (std::int64_t i = 0; i < m; ++i)
            if (rowmap[i] < 0)
                for (std::int64_t e = rp[i]; e < rp[i + 1]; ++e) ++cc[ci[e]];
        std::vector<std::pair<std::int64_t, std::int64_t>> cl;
        for (std::int64_t j = 0; j < n; ++j)
            if (cc[j] >= col_thr) cl.push_back({cc[j], j});
        std::stable_sort(cl.begin(), cl.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
        if (static_cast<std::int64_t>(cl.size()) > cap_cols) cl.resize(static_cast<std::size_t>(cap_cols));
        colmap.assign(static_cast<std::size_t>(n), -1);
        for (const auto& x : cl) dcols.push_back(x.second);
        std::sort(dcols.begin(), dcols.end());
        for (std::size_t j = 0; j < dcols.size(); ++j) {
            colmap[static_cast<std::size_t>(dcols[j])] = static_cast<std::int32_t>(j);
            extracted += cc[dcols[j]];
        }
    }
    if (hyb_ok && 20 * extracted >= nnz) {  // worth it when >= 5 % of the entries move to DMMA
        mat->dr = static_cast<std::int64_t>(drows.size());
        mat->dc = static_cast<std::int64_t>(dcols.size());
        std::int32_t *d_rowmap = nullptr, *d_colmap = nullptr;
        QB_CUDA(cudaMalloc(&d_rowmap, sizeof(std::int32_t) * m));
        QB_CUDA(cudaMalloc(&d_colmap, sizeof(std::int32_t) * n));
        QB_CUDA(cudaMemcpyAsync(d_rowmap, rowmap.data(), sizeof(std::int32_t) * m, cudaMemcpyHostToDevice, c.st));
        QB_CUDA(cudaMemcpyAsync(d_colmap, colmap.data(), sizeof(std::int32_t) * n, cudaMemcpyHostToDevice, c.st));
        if (mat->dr) {
            QB_CUDA(cudaMalloc(&mat->d_rows, sizeof(std::int64_t) * mat->dr));
            QB_CUDA(cudaMemcpyAsync(mat->d_rows, drows.data(), sizeof(std::int64_t) * mat->dr, cudaMemcpyHostToDevice, c.st));
            QB_CUDA(cudaMalloc(&mat->d_r, sizeof(double) * mat->dr * n));
            QB_CUDA(cudaMemsetAsync(mat->d_r, 0, sizeof(double) * mat->dr * n, c.st));
        }
        if (mat->dc) {
            QB_CUDA(cudaMalloc(&mat->d_cols, sizeof(std::int64_t) * mat->dc));
            QB_CUDA(cudaMemcpyAsync(mat->d_cols, dcols.data(), sizeof(std::int64_t) * mat->dc, cudaMemcpyHostToDevice, c.st));
            QB_CUDA(cudaMalloc(&mat->d_c, sizeof(double) * mat->dc * m));
            QB_CUDA(cudaMemsetAsync(mat->d_c, 0, sizeof(double) * mat->dc * m, c.st));
        }
        QB_CUDA(cudaMalloc(&mat->s_rp, sizeof(std::int64_t) * (m + 1)));
        mat->s_nnz = csr_split_dense(c.st, m, n, mat->rp, mat->ci, mat->v, d_rowmap, d_colmap, mat->s_rp, &mat->s_ci,
                                     &mat->s_v, mat->d_r, mat->d_c, c.sms);
        QB_CUDA(cudaStreamSynchronize(c.st));
        cudaFree(d_rowmap);
        cudaFree(d_colmap);
        csr_transpose(c.st, m, n, mat->s_nnz, mat->s_rp, mat->s_ci, mat->s_v, mat->ct_rp, mat->ct_ci, mat->ct_v, c.sms);
        std::vector<std::int64_t> s_rp_host(static_cast<std::size_t>(m + 1));
        QB_CUDA(cudaMemcpyAsync(s_rp_host.data(), mat->s_rp, sizeof(std::int64_t) * (m + 1), cudaMemcpyDeviceToHost, c.st));
        QB_CUDA(cudaStreamSynchronize(c.st));
        mat->heavy = make_heavy_plan(s_rp_host.data(), m, c.st);
    } else {
        csr_transpose(c.st, m, n, nnz, mat->rp, mat->ci, mat->v, mat->ct_rp, mat->ct_ci, mat->ct_v, c.sms);
        mat->heavy = make_heavy_plan(rp, m, c.st);
    }
    std::vector<std::int64_t> ct_rp_host(static_cast<std::size_t>(n + 1));
    QB_CUDA(cudaMemcpyAsync(ct_rp_host.data(), mat->ct_rp, sizeof(std::int64_t) * (n + 1), cudaMemcpyDeviceToHost, c.st));
    QB_CUDA(cudaStreamSynchronize(c.st));
    mat->heavy_t = make_heavy_plan(ct_rp_host.data(), n, c.st);
    return mat;
}

// ---------------------------------------------------------------------------------
namespace {

class Engine {
public:
    Engine(Context& c, Matrix& a) : c_(c), a_(a), st_(c.st) {}

    double* slot(int s) const { return c_.d_small + static_cast<std::size_t>(s) * kSlot; }
    MatView small(int s, std::int64_t r, std::int64_t cc) const { return MatView{slot(s), r, cc, kSmallMax, false}; }

    void gemm(double alpha, const MatView& a, const MatView& b, double beta, const MatView& c) {
        qbgpu::gemm(st_, c_.ws_gemm, alpha, a, b, beta, c);
    }

    // Y (m x w) = A X (X: n x w). Dense: DMMA GEMM; sparse: CSR SpMM.
    void apply(const MatView& x, const MatView& y, double alpha = 1.0, double beta = 0.0) {
        const bool want_pregram = want_pregram_;
        want_pregram_ = false;
        if (a_.host_stream) throw QbError(kError, "host-streamed matrix: only single_pass_fp consumes a RowStream");
        if (a_.sparse) {
            if (!x.rowmajor || !y.rowmajor) throw QbError(kInternal, "sparse pass needs row-major blocks");
            const CsrView av = a_.csr();
            double* part = av.heavy.nseg ? c_.ws_sp.get(csr_spmm_scratch(av, std::min<int>(static_cast<int>(x.cols), 256))) : nullptr;
            csr_spmm(st_, av, x.p, x.ld, y.p, y.ld, static_cast<int>(x.cols), alpha, beta, c_.sms, part);
            if (a_.hybrid()) {
                const int w = static_cast<int>(x.cols);
                if (a_.dr) {  // y[R] += alpha D_r X
                    DBuf t(static_cast<std::size_t>(a_.dr) * w, st_);
                    gemm(1.0, MatView{a_.d_r, a_.dr, a_.n, a_.n, true}, x, 0.0, MatView{t.p, a_.dr, w, w, true});
                    scatter_add_rows(st_, t.p, a_.d_rows, a_.dr, w, alpha, y.p, y.ld);
                }
                if (a_.dc) {  // y += alpha D_c X[C]
                    DBuf xc(static_cast<std::size_t>(a_.dc) * w, st_);
                    gather_rows(st_, x.p, x.ld, a_.d_cols, a_.dc, w, xc.p);
                    gemm(alpha, MatView{a_.d_c, a_.m, a_.dc, std::max<std::int64_t>(a_.m, 1), false},
                         MatView{xc.p, a_.dc, w, w, true}, 1.0, y);
                }
            }
        } else if (!a_.pending.empty()) {
            // first pass over an asynchronously uploaded A: one GEMM per row chunk as it lands.
            // When the caller orthonormalises Y next by the wide CholQR (request_pregram), the
            // chunk's share of the Gram Y^T Y is accumulated behind its GEMM, in the gaps the copy
            // leaves on the compute stream, and orth_wide_cholqr2 starts from that Gram.
            const std::int64_t l = y.cols;
            const bool pregram = want_pregram && pregram_enabled() && alpha == 1.0 && beta == 0.0 && y.rowmajor &&
                                 y.ld == l && l > kSmallMax && c_.world == 1 && a_.pending.size() > 1;
            const std::size_t ll = static_cast<std::size_t>(l) * l;
            if (pregram && wide_.n < 3 * ll) wide_ = DBuf(3 * ll, st_);
            std::int64_t r0 = 0;
            for (auto& ch : a_.pending) {
                QB_CUDA(cudaStreamWaitEvent(st_, ch.ready, 0));
                const std::int64_t rows = ch.row_end - r0;
                MatView ab{a_.a + r0, rows, a_.n, a_.lda, false};
                MatView yb = y.rowmajor ? MatView{y.p + r0 * y.ld, rows, y.cols, y.ld, true}
                                        : MatView{y.p + r0, rows, y.cols, y.ld, false};
                gemm(alpha, ab, x, beta, yb);
                if (pregram)
                    qbgpu::gemm(st_, c_.ws_gemm, 1.0, yb.t(), yb, r0 == 0 ? 0.0 : 1.0, MatView{wide_.p, l, l, l, false},
                                kGemmUpperC);
                r0 = ch.row_end;
            }
            if (pregram) pregram_for_ = y.p;
            a_.wait_resident(st_);
        } else {
            gemm(alpha, a_.dense_view(), x, beta, y);
        }
    }
    // One pass over a host-streamed A (single_pass_fp): row chunks are copied
    // on the copy stream into a 3-deep device ring while the compute stream forms, per chunk,
    // G_c = A_c Omega, H += A_c^T G_c and ||A_c||^2 (summed in chunk order). Returns ||A||^2.
    double stream_single_pass(const MatView& om, const MatView& g, const MatView& h) {
        if (!a_.host_stream) throw QbError(kInternal, "stream_single_pass on a resident matrix");
        if (a_.sparse) return stream_single_pass_csr(om, g, h);
        const std::int64_t m = a_.m, n = a_.n, cr = a_.chunk_rows;
        const std::int64_t nchunk = ceil_div(m, cr);
        constexpr int kRing = 3;
        const std::int64_t ld = round_up(cr, 8);
        DBuf ring(static_cast<std::size_t>(kRing) * ld * std::max<std::int64_t>(n, 1), st_);
        DBuf norms(static_cast<std::size_t>(std::max<std::int64_t>(nchunk, 1)), st_);
        cudaEvent_t landed[kRing], freed[kRing];
        for (int i = 0; i < kRing; ++i) {
            QB_CUDA(cudaEventCreateWithFlags(&landed[i], cudaEventDisableTiming));
            QB_CUDA(cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming));
        }
        // the ring is allocated on the compute stream: make the copy stream wait for it
        cudaEvent_t ready;
        QB_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
        QB_CUDA(cudaEventRecord(ready, st_));
        QB_CUDA(cudaStreamWaitEvent(c_.st_copy, ready, 0));
        for (std::int64_t ci = 0; ci < nchunk; ++ci) {
            const int slot = static_cast<int>(ci % kRing);
            const std::int64_t r0 = ci * cr, rows = std::min(cr, m - r0);
            double* buf = ring.p + static_cast<std::size_t>(slot) * ld * n;
            if (ci >= kRing) QB_CUDA(cudaStreamWaitEvent(c_.st_copy, freed[slot], 0));
            QB_CUDA(cudaMemcpy2DAsync(buf, ld * sizeof(double), a_.host_a + r0, a_.host_lda * sizeof(double),
                                      rows * sizeof(double), n, cudaMemcpyHostToDevice, c_.st_copy));
            QB_CUDA(cudaEventRecord(landed[slot], c_.st_copy));
            QB_CUDA(cudaStreamWaitEvent(st_, landed[slot], 0));
            MatView ac{buf, rows, n, ld, false};
            MatView gc = g.rowmajor ? MatView{g.p + r0 * g.ld, rows, g.cols, g.ld, true}
                                    : MatView{g.p + r0, rows, g.cols, g.ld, false};
            gemm(1.0, ac, om, 0.0, gc);
            sum_squares(st_, c_.ws_red, ac, norms.p + ci);
            gemm(1.0, ac.t(), gc, ci == 0 ? 0.0 : 1.0, h);
            QB_CUDA(cudaEventRecord(freed[slot], st_));
        }
        std::vector<double> hn(static_cast<std::size_t>(nchunk));
        if (nchunk) QB_CUDA(cudaMemcpyAsync(hn.data(), norms.p, sizeof(double) * nchunk, cudaMemcpyDeviceToHost, st_));
        QB_CUDA(cudaStreamSynchronize(st_));
        for (int i = 0; i < kRing; ++i) {
            cudaEventDestroy(landed[i]);
            cudaEventDestroy(freed[i]);
        }
        cudaEventDestroy(ready);
        double nrm = 0.0;
        for (double x : hn) nrm += x;
        if (!std::isfinite(nrm)) throw QbError(kError, "from_data: non-finite entry");  // dense_matrix.cpp:17-18
        return nrm;
    }

    // CsrRowStream (matrix_handle.cpp:60-73) over host CSR arrays: row chunks of about
    // chunk_nnz entries are uploaded and validated as SparseCsrMatrix::from_parts would
    // (make_csr on the chunk: FormatError / Error), then G_c = A_c Omega (CSR SpMM),
    // H += A_c^T G_c (CSR SpMM over the chunk's device-built transpose) and ||A_c||^2 over
    // its values, in chunk order. Only one chunk of A is ever resident.
    double stream_single_pass_csr(const MatView& om, const MatView& g, const MatView& h) {
        const std::int64_t m = a_.m, n = a_.n, w = om.cols;
        const std::int64_t* rp = a_.host_rp;
        std::vector<std::int64_t> cuts{0};  // chunk row boundaries
        while (cuts.back() < m) {
            const std::int64_t r0 = cuts.back();
            std::int64_t r1 = static_cast<std::int64_t>(std::upper_bound(rp + r0 + 1, rp + m + 1, rp[r0] + a_.chunk_nnz) - rp) - 1;
            cuts.push_back(std::max(r1, r0 + 1));
        }
        const std::size_t nchunk = cuts.size() - 1;
        if (nchunk == 0) {  // no rows: G is empty and H = A^T G = 0
            if (h.rows * h.cols) QB_CUDA(cudaMemsetAsync(h.p, 0, sizeof(double) * h.rows * h.ld, st_));
            return 0.0;
        }
        DBuf ht(nchunk > 1 ? static_cast<std::size_t>(n) * std::max<std::int64_t>(w, 1) : 0, st_);
        MatView htv{ht.p, n, w, w, true};
        DBuf dn(nchunk, st_);
        for (std::size_t k = 0; k < nchunk; ++k) {
            const std::int64_t r0 = cuts[k], r1 = cuts[k + 1], e0 = rp[r0], nnz_c = rp[r1] - e0;
            std::vector<std::int64_t> lrp(static_cast<std::size_t>(r1 - r0 + 1));
            for (std::int64_t i = r0; i <= r1; ++i) lrp[static_cast<std::size_t>(i - r0)] = rp[i] - e0;
            auto chunk = make_csr(c_, m, r0, r1 - r0, n, nnz_c, lrp.data(), a_.host_ci + e0, a_.host_v + e0, false);
            Engine ec(c_, *chunk);
            MatView gc = g.rowmajor ? MatView{g.p + r0 * g.ld, r1 - r0, g.cols, g.ld, true}
                                    : MatView{g.p + r0, r1 - r0, g.cols, g.ld, false};
            ec.apply(om, gc);
            if (k == 0) {
                ec.apply_t(gc, h);
            } else {
                ec.apply_t(gc, htv);
                add_matrix(st_, htv, h, 1.0);
            }
            sum_squares_vec(st_, c_.ws_red, chunk->v, nnz_c, dn.p + k);
            QB_CUDA(cudaStreamSynchronize(st_));  // the chunk's device arrays are released next
        }
        std::vector<double> norms(nchunk);
        QB_CUDA(cudaMemcpyAsync(norms.data(), dn.p, sizeof(double) * nchunk, cudaMemcpyDeviceToHost, st_));
        QB_CUDA(cudaStreamSynchronize(st_));
        double nrm = 0.0;
        for (double x : norms) nrm += x;
        return nrm;
    }

    // Y (n x w) = A^T X (X: m x w), summed over ranks.
    void apply_t(const MatView& x, const MatView& y, bool reduce = true) {
        if (a_.host_stream) throw QbError(kError, "host-streamed matrix: only single_pass_fp consumes a RowStream");
        a_.wait_resident(st_);
        const bool contiguous = (y.rowmajor && y.ld == y.cols) || (!y.rowmajor && y.ld == y.rows);
        if (reduce && c_.world > 1 && !contiguous) {
            // allreduce needs a packed buffer: compute there, reduce, scatter into y
            if (scratch_t_.n < static_cast<std::size_t>(y.rows * y.cols))
                scratch_t_ = DBuf(static_cast<std::size_t>(y.rows * y.cols), st_);
            MatView t{scratch_t_.p, y.rows, y.cols, y.cols, true};
            apply_t(x, t);
            copy_matrix(st_, t, y);
            return;
        }
        if (a_.sparse) {
            if (!x.rowmajor || !y.rowmajor) throw QbError(kInternal, "sparse pass needs row-major blocks");
            const CsrView av = a_.csr_t();
            double* part = av.heavy.nseg ? c_.ws_sp.get(csr_spmm_scratch(av, std::min<int>(static_cast<int>(x.cols), 256))) : nullptr;
            csr_spmm(st_, av, x.p, x.ld, y.p, y.ld, static_cast<int>(x.cols), 1.0, 0.0, c_.sms, part);
            if (a_.hybrid()) {
                const int w = static_cast<int>(x.cols);
                if (a_.dr) {  // z += D_r^T X[R]
                    DBuf xr(static_cast<std::size_t>(a_.dr) * w, st_);
                    gather_rows(st_, x.p, x.ld, a_.d_rows, a_.dr, w, xr.p);
                    gemm(1.0, MatView{a_.d_r, a_.dr, a_.n, a_.n, true}.t(), MatView{xr.p, a_.dr, w, w, true}, 1.0, y);
                }
                if (a_.dc) {  // z[C] += D_c^T X
                    DBuf t(static_cast<std::size_t>(a_.dc) * w, st_);
                    gemm(1.0, MatView{a_.d_c, a_.m, a_.dc, std::max<std::int64_t>(a_.m, 1), false}.t(), x, 0.0,
                         MatView{t.p, a_.dc, w, w, true});
                    scatter_add_rows(st_, t.p, a_.d_cols, a_.dc, w, 1.0, y.p, y.ld);
                }
            }
        } else {
            gemm(1.0, a_.dense_view().t(), x, 0.0, y);
        }
        if (reduce) allreduce_view(y);
    }
    // Column-sharded n-side (randQB_EI at world > 1): yl (blk x w, rows [rank blk, rank blk + blk) of
    // the n rows padded to n_pad = world blk) = this rank's block of A^T X summed over ranks — one
    // reduce-scatter instead of an allreduce of the whole n x w. Rows past n are zero.
    void apply_t_rs(const MatView& x, const MatView& yl, std::int64_t n_pad, std::int64_t blk) {
        const std::int64_t w = x.cols;
        if (rs_full_.n < static_cast<std::size_t>(n_pad * w)) rs_full_ = DBuf(static_cast<std::size_t>(n_pad * w), st_);
        if (n_pad > a_.n)
            QB_CUDA(cudaMemsetAsync(rs_full_.p + a_.n * w, 0, sizeof(double) * (n_pad - a_.n) * w, st_));
        apply_t(x, MatView{rs_full_.p, a_.n, w, w, true}, false);
        if (yl.rowmajor && yl.ld == w && yl.rows == blk) {
            c_.reduce_scatter(rs_full_.p, yl.p, static_cast<std::size_t>(blk * w));
            return;
        }
        if (rs_loc_.n < static_cast<std::size_t>(blk * w)) rs_loc_ = DBuf(static_cast<std::size_t>(blk * w), st_);
        c_.reduce_scatter(rs_full_.p, rs_loc_.p, static_cast<std::size_t>(blk * w));
        if (yl.rows) copy_matrix(st_, MatView{rs_loc_.p, yl.rows, w, w, true}, yl);
    }
    void allreduce_view(const MatView& y) {
        if (c_.world == 1) return;
        if (!(y.rowmajor && y.ld == y.cols) && !(!y.rowmajor && y.ld == y.rows))
            throw QbError(kInternal, "allreduce needs a contiguous view");
        c_.allreduce(y.p, static_cast<std::size_t>(y.rows * y.cols));
    }

    double frob_device(double* out) {  // ||A||_F^2 into device scalar `out` (+ allreduce)
        if (a_.host_stream) throw QbError(kError, "host-streamed matrix: only single_pass_fp consumes a RowStream");
        a_.wait_resident(st_);
        if (a_.sparse) sum_squares_vec(st_, c_.ws_red, a_.v, a_.nnz, out);
        else sum_squares(st_, c_.ws_red, a_.dense_view(), out);
        c_.allreduce(out, 1);
        QB_CUDA(cudaMemcpyAsync(c_.h_scalar, out, sizeof(double), cudaMemcpyDeviceToHost, st_));
        QB_CUDA(cudaStreamSynchronize(st_));
        if (a_.check_finite) {  // deferred DenseMatrix::from_data check of an async upload
            if (!std::isfinite(c_.h_scalar[0])) throw QbError(kError, "from_data: non-finite entry");
            a_.check_finite = false;
        }
        return c_.h_scalar[0];
    }

    // orth(Y): Q (rows x b, may alias Y) and upper R (slot r_slot) with inverse
    // (slot rinv_slot), such that Y = Q R, diag(R) > 0. `sharded`: rows are split over
    // ranks (Grams are allreduced). Returns the leading rank d (first index with
    // R_jj <= 1e-12 max R_jj, qr.hpp:20-21), b when full rank.
    // Optimistic CholQR (per block): Cholesky statuses are written to a device array and
    // checked once, together with the indicator read, at the end of the block. If any
    // pass needed the fallback the caller re-runs the whole block with force_hh.
    bool optimistic = false, force_hh = false;
    int lazy_n = 0;
    void begin_block(bool opt, bool force) {
        optimistic = opt;
        force_hh = force;
        lazy_n = 0;
    }
    void fetch_lazy() {
        if (lazy_n)
            QB_CUDA(cudaMemcpyAsync(c_.h_lazy, c_.d_lazy, sizeof(SmallStatus) * 2 * lazy_n, cudaMemcpyDeviceToHost, st_));
    }
    bool lazy_ok() const {  // after the stream sync that follows fetch_lazy()
        for (int i = 0; i < lazy_n; ++i)
            if (!cholqr_ok(c_.h_lazy[2 * i], c_.h_lazy[2 * i + 1])) return false;
        return true;
    }
    static bool cholqr_ok(const SmallStatus& s0, const SmallStatus& s1) {
        return !s0.breakdown && !s1.breakdown && s0.diag_max > 0.0 && s0.diag_min >= kCholRatioMin * s0.diag_max &&
               s1.gram_dev <= kCholGramDevMax && std::isfinite(s0.diag_max) && std::isfinite(s1.diag_max);
    }

    // span_only: the caller uses span(Y) only (a sketch inside the power iteration); the fused panel
    // then stops after one CholQR pass when that pass is orthonormal to 1e-6 (cholqr2_panel).
    int orth_block(const MatView& y, const MatView& qout, int r_slot, int rinv_slot, bool sharded, DBuf& tmp,
                   bool need_r = true, bool span_only = false) {
        const int b = static_cast<int>(y.cols);
        const std::int64_t rows = y.rows;
        if (b == 0) return 0;
        if (b > kSmallMax || wide_mode) return orth_block_wide(y, qout, r_slot, rinv_slot, sharded, tmp, need_r);
        MatView t1{tmp.p, rows, b, b, true};
        last_wide = false;
        if (!force_hh) {
            const bool lazy = optimistic && lazy_n < Context::kLazyCap / 2;
            SmallStatus* st0 = lazy ? c_.d_lazy + 2 * lazy_n : c_.d_status + 0;
            SmallStatus* st1 = st0 + 1;
            // Unsharded panels: the whole CholQR2 in one cooperative launch (q may alias y
            // only when the statuses are checked lazily: the Householder redo restarts the block).
            if (!sharded && rows > 0 && y.rowmajor && qout.rowmajor && (lazy || qout.p != y.p)) {
                cholqr2_panel(st_, c_.ws_panel, y.p, rows, b, y.ld, t1.p, qout.p, qout.ld, slot(kG), slot(kRa),
                              slot(kRainv), slot(kRb), slot(kRbinv), st0, st1, c_.d_gbar, span_only);
                bool ok = true;
                if (lazy) {
                    ++lazy_n;
                } else {
                    QB_CUDA(cudaMemcpyAsync(c_.h_status, st0, sizeof(SmallStatus) * 2, cudaMemcpyDeviceToHost, st_));
                    QB_CUDA(cudaStreamSynchronize(st_));
                    ok = cholqr_ok(c_.h_status[0], c_.h_status[1]);
                }
                if (ok) {
                    if (need_r)
                        trmm_upper_pair(st_, slot(kRb), slot(kRa), slot(r_slot), slot(kRainv), slot(kRbinv),
                                        slot(rinv_slot), b, kSmallMax);
                    return b;
                }
            } else {
            // pass 1
            gemm(1.0, y.t(), y, 0.0, small(kG, b, b));
            if (sharded) c_.allreduce(slot(kG), kSlot);
            chol_small(st_, slot(kG), kSmallMax, b, slot(kRa), slot(kRainv), kSmallMax, st0);
            gemm(1.0, y, small(kRainv, b, b), 0.0, t1);
            // pass 2
            gemm(1.0, t1.t(), t1, 0.0, small(kG, b, b));
            if (sharded) c_.allreduce(slot(kG), kSlot);
            chol_small(st_, slot(kG), kSmallMax, b, slot(kRb), slot(kRbinv), kSmallMax, st1);
            bool ok = true;
            if (lazy) {
                ++lazy_n;
            } else {
                QB_CUDA(cudaMemcpyAsync(c_.h_status, st0, sizeof(SmallStatus) * 2, cudaMemcpyDeviceToHost, st_));
                QB_CUDA(cudaStreamSynchronize(st_));
                ok = cholqr_ok(c_.h_status[0], c_.h_status[1]);
            }
            if (ok) {
                gemm(1.0, t1, small(kRbinv, b, b), 0.0, qout);
                if (need_r)
                    trmm_upper_pair(st_, slot(kRb), slot(kRa), slot(r_slot), slot(kRainv), slot(kRbinv),
                                    slot(rinv_slot), b, kSmallMax);
                return b;
            }
            }
        }
        // Householder fallback: exact deficiency decisions (qr.hpp:15-21).
        ++hh_fallbacks;
        if (sharded && c_.world > 1) {
            // Row-sharded panel: assemble the whole m x b panel on every rank (each rank writes its
            // rows into a zeroed buffer; the sum over ranks adds only zeros to them, so it is exact),
            // factor it redundantly (identical inputs, identical R and deficiency decision on every
            // rank) and keep this rank's rows of Q.
            const std::int64_t mg = geo_rows >= 0 ? geo_rows : a_.m_global, r0 = geo_rows >= 0 ? geo_row0 : a_.row0;
            DBuf full(static_cast<std::size_t>(std::max<std::int64_t>(mg, 1)) * b, st_);
            QB_CUDA(cudaMemsetAsync(full.p, 0, sizeof(double) * full.n, st_));
            MatView fv{full.p, mg, b, std::max<std::int64_t>(mg, 1), false};
            if (rows) copy_matrix(st_, y, fv.rows_range(r0, rows));
            c_.allreduce(full.p, full.n);
            householder_panel(st_, c_.ws_hh, fv.p, mg, b, fv.ld, slot(r_slot), kSmallMax);
            const int d = householder_rank(r_slot, b);
            if (rows) copy_matrix(st_, fv.rows_range(r0, rows), qout);
            if (d > 0) tri_inverse_small(st_, slot(r_slot), slot(rinv_slot), d, kSmallMax);
            return d;
        }
        MatView ycol{t1.p, rows, b, std::max<std::int64_t>(rows, 1), false};
        copy_matrix(st_, y, ycol);
        householder_panel(st_, c_.ws_hh, ycol.p, rows, b, ycol.ld, slot(r_slot), kSmallMax);
        const int d = householder_rank(r_slot, b);
        copy_matrix(st_, ycol, qout);
        if (d > 0) tri_inverse_small(st_, slot(r_slot), slot(rinv_slot), d, kSmallMax);
        return d;
    }
    // ---- blocks wider than the in-CTA panel kernels (b > kSmallMax = 112) ----------------
    // orth(Y) for a wide block: block Gram-Schmidt with re-orthogonalisation (BCGS2) over
    // panels of <= 112 columns, each orthonormalised by the narrow orth_block (fused CholQR2,
    // Householder on failure — the same deficiency machinery). R is assembled block by block:
    //   R[j, j] = R2_j R1_j,   R[<j, j] = S1_j + S2_j R1_j      (S1, S2: the two projections)
    //   R^{-1}[j, j] = R1_j^{-1} R2_j^{-1},
    //   R^{-1}[<j, j] = -R^{-1}[<j, <j] R[<j, j] R^{-1}[j, j],
    // in wide slots (b x b, column-major) read through rmat(). diag(R) = diag(R2_j) diag(R1_j)
    // gives the reference's deficiency decision over the whole block: the first j with
    // R_jj <= 1e-12 max R_jj (qr.hpp:20-21; R of a QR with diag > 0 is unique, so the panel
    // diagonals are the Householder R's up to rounding).
    // wide_mode (set per randQB_FP block of width > 112) keeps every orth of that block on this
    // path, so R_i = R~_i R_i and the B_i update read one storage.
    bool wide_mode = false;
    bool last_wide = false;
    double* wslot(int s, std::int64_t b) {
        const std::size_t need = static_cast<std::size_t>(b) * b;
        if (wslot_[s].n < need) wslot_[s] = DBuf(need, st_);
        return wslot_[s].p;
    }
    MatView rmat(int s, std::int64_t d) const {
        return last_wide ? MatView{wslot_[s].p, d, d, wld_, false} : small(s, d, d);
    }
    // R = R2 R1 and R^{-1} = R1^{-1} R2^{-1} (d x d upper) for the narrow slots or the wide ones.
    void tri_pair(int s2, int s1, int sr, int s1inv, int s2inv, int srinv, int d) {
        if (!last_wide) {
            trmm_upper_pair(st_, slot(s2), slot(s1), slot(sr), slot(s1inv), slot(s2inv), slot(srinv), d, kSmallMax);
            return;
        }
        wslot(sr, wld_);
        wslot(srinv, wld_);
        gemm(1.0, rmat(s2, d), rmat(s1, d), 0.0, rmat(sr, d));
        gemm(1.0, rmat(s1inv, d), rmat(s2inv, d), 0.0, rmat(srinv, d));
    }
    int orth_block_wide(const MatView& y, const MatView& qout, int r_slot, int rinv_slot, bool sharded, DBuf& tmp,
                        bool need_r) {
        const std::int64_t b = y.cols;
        if (qout.p != y.p) copy_matrix(st_, y, qout);
        const std::int64_t np = ceil_div(b, kSmallMax);
        const std::int64_t pw = ceil_div(b, np);
        if (wld_ < b) {  // wide slots share one leading dimension (the widest block so far)
            for (auto& w : wslot_) w = DBuf();
            wld_ = b;
        }
        double* wr = wslot(r_slot, wld_);
        double* wri = wslot(rinv_slot, wld_);
        QB_CUDA(cudaMemsetAsync(wr, 0, sizeof(double) * wld_ * wld_, st_));
        QB_CUDA(cudaMemsetAsync(wri, 0, sizeof(double) * wld_ * wld_, st_));
        MatView R{wr, b, b, wld_, false}, Ri{wri, b, b, wld_, false};
        const std::size_t sneed = static_cast<std::size_t>(b) * pw;
        if (wide_s_.n < 3 * sneed) wide_s_ = DBuf(3 * sneed, st_);
        if (wide_diag_.n < static_cast<std::size_t>(b)) wide_diag_ = DBuf(static_cast<std::size_t>(b), st_);
        const bool saved = wide_mode;
        wide_mode = false;  // the panels themselves take the narrow path
        for (std::int64_t j0 = 0; j0 < b; j0 += pw) {
            const int bj = static_cast<int>(std::min(pw, b - j0));
            MatView xj = qout.cols_range(j0, bj);
            MatView prev = qout.cols_range(0, j0);
            MatView s1{wide_s_.p, j0, bj, bj, true}, s2{wide_s_.p + sneed, j0, bj, bj, true};
            if (j0 > 0) {
                gemm(1.0, prev.t(), xj, 0.0, s1);
                if (sharded) allreduce_view(s1);
                gemm(-1.0, prev, s1, 1.0, xj);
            }
            orth_block(xj, xj, kR1, kR1inv, sharded, tmp, true);
            if (j0 > 0) {
                gemm(1.0, prev.t(), xj, 0.0, s2);
                if (sharded) allreduce_view(s2);
                gemm(-1.0, prev, s2, 1.0, xj);
                orth_block(xj, xj, kR2, kR2inv, sharded, tmp, true);
                trmm_upper_pair(st_, slot(kR2), slot(kR1), slot(kR), slot(kR1inv), slot(kR2inv), slot(kRinv), bj,
                                kSmallMax);
            } else {
                copy_matrix(st_, small(kR1, bj, bj), small(kR, bj, bj));
                copy_matrix(st_, small(kR1inv, bj, bj), small(kRinv, bj, bj));
            }
            // diag(R_jj): the stride-(ld+1) view of the slot
            copy_matrix(st_, MatView{slot(kR), bj, 1, kSmallMax + 1, true}, MatView{wide_diag_.p + j0, bj, 1, 1, true});
            if (need_r) {
                copy_matrix(st_, small(kR, bj, bj), R.block(j0, j0, bj, bj));
                copy_matrix(st_, small(kRinv, bj, bj), Ri.block(j0, j0, bj, bj));
                if (j0 > 0) {
                    copy_matrix(st_, s1, R.block(0, j0, j0, bj));
                    gemm(1.0, s2, small(kR1, bj, bj), 1.0, R.block(0, j0, j0, bj));
                    MatView t{wide_s_.p + 2 * sneed, j0, bj, bj, true};
                    gemm(1.0, Ri.block(0, 0, j0, j0), R.block(0, j0, j0, bj), 0.0, t);
                    gemm(-1.0, t, small(kRinv, bj, bj), 0.0, Ri.block(0, j0, j0, bj));
                }
            }
        }
        wide_mode = saved;
        last_wide = true;
        std::vector<double> dg(static_cast<std::size_t>(b));
        QB_CUDA(cudaMemcpyAsync(dg.data(), wide_diag_.p, sizeof(double) * b, cudaMemcpyDeviceToHost, st_));
        QB_CUDA(cudaStreamSynchronize(st_));
        double mx = 0.0;
        for (double x : dg) mx = std::max(mx, std::fabs(x));
        for (std::int64_t j = 0; j < b; ++j)
            if (!(std::fabs(dg[static_cast<std::size_t>(j)]) > kRankTol * mx)) return static_cast<int>(j);
        return static_cast<int>(b);
    }

    // Leading rank of the Householder R in `r_slot`: the first j with |R_jj| <= 1e-12 max |R_jj|
    // (rank_deficiency_report, qr.hpp:20-21); b when none.
    int householder_rank(int r_slot, int b) {
        std::vector<double> rh(static_cast<std::size_t>(kSlot));
        QB_CUDA(cudaMemcpyAsync(rh.data(), slot(r_slot), sizeof(double) * kSlot, cudaMemcpyDeviceToHost, st_));
        QB_CUDA(cudaStreamSynchronize(st_));
        double mx = 0.0;
        for (int j = 0; j < b; ++j) mx = std::max(mx, std::fabs(rh[j + j * kSmallMax]));
        for (int j = 0; j < b; ++j)
            if (std::fabs(rh[j + j * kSmallMax]) <= kRankTol * mx) return j;
        return b;
    }

    // Blocked right-looking Cholesky of the l x l SPD matrix W (column-major, upper
    // triangle read, overwritten) into R (upper) and R^{-1}, both column-major (ld l).
    // One cooperative launch (chol_wide, small.cu): right-looking over 64-column tiles,
    // diagonal blocks by chol_small's register-tiled elimination of [W_kk | I], row panels
    // R_kk^{-T} W_kj and trailing updates as DMMA tile products; R^{-1} is accumulated
    // alongside (the transposed right half of the elimination of [W | I]).
    // Returns false on breakdown or when min diag(R) < kCholRatioMin * max diag(R).
    bool chol_blocked(double* w, int l, double* r, double* rinv, double max_gram_dev, double* ratio = nullptr) {
        const int nb = 64;
        const int nt = static_cast<int>(ceil_div(l, nb));
        QB_CUDA(cudaMemsetAsync(r, 0, sizeof(double) * l * l, st_));
        QB_CUDA(cudaMemsetAsync(rinv, 0, sizeof(double) * l * l, st_));
        if (stat_.n < static_cast<std::size_t>(nt) * 4) stat_ = DBuf(static_cast<std::size_t>(nt) * 4, st_);
        auto* stats = reinterpret_cast<SmallStatus*>(stat_.p);
        static_assert(sizeof(SmallStatus) <= 4 * sizeof(double), "status size");
        chol_wide(st_, w, l, l, r, rinv, l, stats);
        std::vector<SmallStatus> hs(static_cast<std::size_t>(nt));
        QB_CUDA(cudaMemcpyAsync(hs.data(), stats, sizeof(SmallStatus) * nt, cudaMemcpyDeviceToHost, st_));
        QB_CUDA(cudaStreamSynchronize(st_));
        double dmin = INFINITY, dmax = 0.0, dev = 0.0;
        for (const auto& s : hs) {
            if (s.breakdown || !std::isfinite(s.diag_max)) return false;
            dmin = std::min(dmin, s.diag_min);
            dmax = std::max(dmax, s.diag_max);
            dev = std::max(dev, s.gram_dev);
        }
        if (ratio) *ratio = dmax > 0.0 ? dmin / dmax : 0.0;
        return dmax > 0.0 && dmin >= kCholRatioMin * dmax && dev <= max_gram_dev;
    }

    // CholQR of a wide panel X (rows x l, row-major) in place: one l x l Gram (DMMA SYRK),
    // blocked Cholesky, X R^{-1} as a triangular-B GEMM. The second pass of CholQR2 is
    // run only when the first leaves a loss of orthogonality u*kappa^2 (kappa estimated
    // by the diagonal ratio of R) above 1e-6: the power step needs a basis with the
    // reference's leading-column spans, which any upper-triangular R preserves.
    // Returns false (X unchanged, or holding the one-pass basis) when the Gram is too
    // ill-conditioned for Cholesky; orth_wide then falls back to BCGS2.
    bool orth_wide_cholqr2(const MatView& x, bool sharded) {
        const int l = static_cast<int>(x.cols);
        const std::size_t ll = static_cast<std::size_t>(l) * l;
        if (wide_.n < 3 * ll) wide_ = DBuf(3 * ll, st_);
        if (wide_y_.n < static_cast<std::size_t>(x.rows) * l) wide_y_ = DBuf(static_cast<std::size_t>(x.rows) * l, st_);
        double* g = wide_.p;
        double* r = wide_.p + ll;
        double* rinv = wide_.p + 2 * ll;
        MatView y{wide_y_.p, x.rows, l, l, true};
        MatView gv{g, l, l, l, false};
        MatView rinv_v{rinv, l, l, l, false};
        for (int pass = 0; pass < 2; ++pass) {
            const MatView& src = pass == 0 ? x : y;
            const MatView& dst = pass == 0 ? y : x;
            if (pass == 0 && !sharded && pregram_for_ == x.p) {
                // the Gram of X was accumulated chunk by chunk behind the upload's first pass
            } else {
                qbgpu::gemm(st_, c_.ws_gemm, 1.0, src.t(), src, 0.0, gv, kGemmUpperC);
            }
            pregram_for_ = nullptr;
            if (sharded) c_.allreduce(g, ll);
            double ratio = 0.0;
            if (!chol_blocked(g, l, r, rinv, pass == 0 ? INFINITY : kCholGramDevMax, &ratio)) {
                if (pass == 1) copy_matrix(st_, y, x);
                return false;
            }
            qbgpu::gemm(st_, c_.ws_gemm, 1.0, src, rinv_v, 0.0, dst, kGemmTriB);
            ++wide_passes;
            if (pass == 0 && kEpsMach / (ratio * ratio) <= 1e-6) {
                copy_matrix(st_, y, x);
                return true;
            }
        }
        return true;
    }

    // Orthonormal basis of the leading-column spans of X (rows x l) in place:
    // CholQR2 with one wide Gram when well conditioned, else block Gram-Schmidt with
    // re-orthogonalisation (BCGS2) over CholQR2 panels.
    void orth_wide(const MatView& x, bool sharded, DBuf& tmp, DBuf& sbuf) {
        if (x.cols > kSmallMax && x.rowmajor && x.ld == x.cols && orth_wide_cholqr2(x, sharded)) return;
        orth_wide_bcgs2(x, sharded, tmp, sbuf);
    }

    void orth_wide_bcgs2(const MatView& x, bool sharded, DBuf& tmp, DBuf& sbuf) {
        const std::int64_t l = x.cols;
        const std::int64_t bw = 64;
        for (std::int64_t j0 = 0; j0 < l; j0 += bw) {
            const std::int64_t bj = std::min(bw, l - j0);
            MatView xj = x.cols_range(j0, bj);
            for (int rep = 0; rep < 2; ++rep) {
                if (j0 > 0) {
                    MatView prev = x.cols_range(0, j0);
                    MatView s{sbuf.p, j0, bj, bj, true};
                    gemm(1.0, prev.t(), xj, 0.0, s);
                    if (sharded) allreduce_view(s);
                    gemm(-1.0, prev, s, 1.0, xj);
                }
                orth_block(xj, xj, kR2, kR2inv, sharded, tmp);
            }
        }
    }

    // The next apply() feeds orth_wide: over a chunked asynchronous upload it may accumulate the
    // wide Gram per chunk (QBFAC_PREGRAM=0 switches this off).
    void request_pregram() { want_pregram_ = true; }
    static bool pregram_enabled() {
        static const bool on = [] {
            const char* e = std::getenv("QBFAC_PREGRAM");
            return !(e && e[0] == '0');
        }();
        return on;
    }

    std::int64_t hh_fallbacks = 0;
    std::int64_t wide_passes = 0;
    // Row geometry of a sharded panel for the Householder fallback: -1 = the rows of A; the
    // column-sharded n-side panels set (n_pad, rank blk) around their orth.
    std::int64_t geo_rows = -1, geo_row0 = 0;

private:
    DBuf scratch_t_, stat_, tri_, wide_, wide_y_, wide_s_, wide_diag_, rs_full_, rs_loc_;
    bool want_pregram_ = false;
    const double* pregram_for_ = nullptr;  // X whose upper Gram wide_ already holds
    DBuf wslot_[kNumSlots];
    std::int64_t wld_ = 0;
    Context& c_;
    Matrix& a_;
    cudaStream_t st_;
};

struct Timer {
    cudaEvent_t e0, e1;
    cudaStream_t st;
    explicit Timer(cudaStream_t s) : st(s) {
        QB_CUDA(cudaEventCreate(&e0));
        QB_CUDA(cudaEventCreate(&e1));
        QB_CUDA(cudaEventRecord(e0, st));
    }
    double stop() {
        QB_CUDA(cudaEventRecord(e1, st));
        QB_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        QB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        return ms;
    }
    ~Timer() {
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
};

void check_eps(double eps, double norm_a_sq) {
    const double floor = std::sqrt(4.0 * kEpsMach / 0.01) * std::sqrt(norm_a_sq);
    if (!(eps > floor)) {
        QbError e(kToleranceFloorError, "epsilon below the Theorem 3 floor " + std::to_string(floor));
        e.floor = floor;
        throw e;
    }
}

std::int64_t even(std::int64_t x) { return std::max<std::int64_t>(2, round_up(x, 2)); }

// Shared state of one factorization.
struct State {
    Context& c;
    Engine& eng;
    std::int64_t m, n, cap, ld;
    std::int64_t k = 0;
    // B^T rows held here: all n (replicated), or this rank's column block of B (column-sharded
    // n-side: nb_store = blk rows of storage, nb = the real ones, n_pad = world blk)
    std::int64_t nb, nb_store, n_pad = 0;
    bool nsh = false;
    DBuf q, bt;
    double* d_e;
    double eps2 = 0.0;
    std::vector<double> trace;

    State(Context& cc, Engine& e, std::int64_t m_, std::int64_t n_, std::int64_t cap_, std::int64_t nb_ = -1,
          std::int64_t nb_store_ = -1, std::int64_t n_pad_ = 0)
        : c(cc), eng(e), m(m_), n(n_), cap(cap_), ld(even(cap_)), nb(nb_ < 0 ? n_ : nb_),
          nb_store(nb_store_ < 0 ? n_ : nb_store_), n_pad(n_pad_), nsh(nb_ >= 0),
          q(static_cast<std::size_t>(std::max<std::int64_t>(m_, 1)) * even(cap_), cc.st),
          bt(static_cast<std::size_t>(std::max<std::int64_t>(nb_store_ < 0 ? n_ : nb_store_, 1)) * even(cap_), cc.st),
          d_e(cc.d_small + static_cast<std::size_t>(kSlot) * kNumSlots + 1) {
        QB_CUDA(cudaEventCreateWithFlags(&ind_ev, cudaEventDisableTiming));
    }
    ~State() { cudaEventDestroy(ind_ev); }
    State(const State&) = delete;
    State& operator=(const State&) = delete;
    cudaEvent_t ind_ev = nullptr;  // marks the indicator read-back when later work is queued behind it
    bool ind_ev_armed = false;

    MatView qk() const { return MatView{q.p, m, k, ld, true}; }
    MatView btk() const { return MatView{bt.p, nb, k, ld, true}; }
    MatView bt_cols(std::int64_t kk) const { return MatView{bt.p, nb, kk, ld, true}; }
    MatView qslot(std::int64_t w) const { return MatView{q.p + k, m, w, ld, true}; }
    MatView btslot(std::int64_t w) const { return MatView{bt.p + k, nb, w, ld, true}; }

    // Rows of B_i enter E one by one: enqueue the device step and the
    // read-back of its result (and of the block's lazy CholQR statuses), then one sync.
    void indicator_enqueue(int d, bool check) {
        double* norms = c.d_small + static_cast<std::size_t>(kNorms) * kSlot;
        column_sumsq(c.st, c.ws_red, btslot(d), norms);
        if (nsh) c.allreduce(norms, static_cast<std::size_t>(d));  // row norms of B_i over the column blocks
        indicator_step(c.st, d_e, norms, d, eps2, check ? 1 : 0, c.d_ind);
        QB_CUDA(cudaMemcpyAsync(c.h_ind, c.d_ind, sizeof(IndicatorOut), cudaMemcpyDeviceToHost, c.st));
    }
    // Everything enqueued so far (the indicator and status read-backs) is marked by an event, so
    // work queued after it (the next block's first pass) keeps the GPU busy while the host waits.
    void indicator_mark() {
        QB_CUDA(cudaEventRecord(ind_ev, c.st));
        ind_ev_armed = true;
    }
    std::pair<int, bool> indicator_finish() {
        if (ind_ev_armed) QB_CUDA(cudaEventSynchronize(ind_ev));
        else QB_CUDA(cudaStreamSynchronize(c.st));
        ind_ev_armed = false;
        return {c.h_ind->keep, c.h_ind->met != 0};
    }
    std::pair<int, bool> indicator(int d, bool check) {
        indicator_enqueue(d, check);
        auto r = indicator_finish();
        trace.push_back(c.h_ind->e);
        return r;
    }
    void set_e(double e) {
        c.h_scalar[1] = e;
        QB_CUDA(cudaMemcpyAsync(d_e, c.h_scalar + 1, sizeof(double), cudaMemcpyHostToDevice, c.st));
        QB_CUDA(cudaStreamSynchronize(c.st));
    }
    double get_e() {
        QB_CUDA(cudaMemcpyAsync(c.h_scalar + 2, d_e, sizeof(double), cudaMemcpyDeviceToHost, c.st));
        QB_CUDA(cudaStreamSynchronize(c.st));
        return c.h_scalar[2];
    }
};

std::unique_ptr<Result> finish(State& s, Matrix& a, std::int64_t passes0, int term, double norm_a_sq) {
    auto r = std::make_unique<Result>();
    r->ctx = &s.c;
    r->m = s.m;
    r->n = s.n;
    r->rank = s.k;
    r->ld = s.ld;
    r->q = std::move(s.q);
    if (s.nsh) {  // the column blocks of B back on every rank (the result contract: B replicated)
        DBuf full(static_cast<std::size_t>(std::max<std::int64_t>(s.n_pad, 1)) * s.ld, s.c.st);
        s.c.all_gather(s.bt.p, full.p, static_cast<std::size_t>(s.nb_store * s.ld));
        r->bt = std::move(full);
    } else {
        r->bt = std::move(s.bt);
    }
    r->e = s.get_e();
    r->norm_a_sq = norm_a_sq;
    r->passes = a.passes - passes0;
    r->terminated_by = term;
    r->trace = s.trace;
    return r;
}

// ---- randQB_EI ---------------------------------------------------------------------
std::unique_ptr<Result> run_ei(Context& c, Matrix& a, const Params& p) {
    if (p.b < 1) throw QbError(kDimensionError, "rand_qb_ei: block size must be >= 1");
    Engine eng(c, a);
    const std::int64_t m = a.m, n = a.n;
    const std::int64_t mg = a.m_global;
    const bool fixed_prec = p.mode == 1;
    std::int64_t cap = std::min(mg, n);
    if (fixed_prec) {
        if (p.max_rank > 0) cap = std::min(cap, p.max_rank);
    } else {
        cap = std::min(cap, p.k + p.s);
    }
    const std::int64_t passes0 = a.passes;
    const bool sharded = c.world > 1;
    // Column-sharded n-side (world > 1; QBFAC_NSHARD=0 keeps B replicated): this rank owns the
    // column block [rank blk, rank blk + blk) of B and of every n-side block (Omega_i rows for the
    // B Omega_i product, Z, B_i^T); A^T passes reduce-scatter instead of allreducing n x b, the
    // k x b products B X are partial sums allreduced, Z is all-gathered once per power step for
    // the A Z pass, and B is gathered once at the end. n-side work per rank: 1 / world.
    const char* nsh_env = std::getenv("QBFAC_NSHARD");
    const bool nsh = sharded && !(nsh_env && nsh_env[0] == '0');
    const std::int64_t blk = nsh ? ceil_div(n, c.world) : n, n_pad = blk * (nsh ? c.world : 1);
    const std::int64_t c0 = nsh ? blk * c.rank : 0;
    const std::int64_t nl = nsh ? std::max<std::int64_t>(0, std::min(blk, n - c0)) : n;
    State s = nsh ? State(c, eng, m, n, cap, nl, blk, n_pad) : State(c, eng, m, n, cap);
    const double norm_a_sq = eng.frob_device(s.d_e);   // Alg. 2 step 2, +1 pass
    a.passes += 1;
    s.eps2 = p.eps_abs * p.eps_abs;
    int term = 0;
    std::int64_t g_used = 0, blocks = 0;
    auto wrap = [&](int t) {
        auto r = finish(s, a, passes0, t, norm_a_sq);
        r->gaussians_used = g_used;
        r->blocks = blocks;
        r->hh_fallbacks = eng.hh_fallbacks;
        return r;
    };
    if (fixed_prec) {
        check_eps(p.eps_abs, norm_a_sq);
        if (norm_a_sq < s.eps2) return wrap(1);
    }
    const std::int64_t bmax = std::min<std::int64_t>(p.b, std::max<std::int64_t>(cap, 1));
    const std::int64_t bpad = even(bmax);
    // Omega_i of several blocks is drawn by ONE launch (the blocks consume consecutive
    // n x b_i pieces of the column-major stream, so block j of a batch is columns
    // [j b, j b + b_i) of an n x (nb b) draw); batches are capped at ~256 MB.
    const std::int64_t nblk_total = ceil_div(std::max<std::int64_t>(cap, 1), bmax);
    const std::int64_t nb_batch = std::max<std::int64_t>(
        1, std::min<std::int64_t>(nblk_total, (std::int64_t{256} << 20) / (8 * std::max<std::int64_t>(n, 1) * bmax)));
    const std::int64_t ldom = even(nb_batch * bmax);
    DBuf om(static_cast<std::size_t>(n) * ldom, c.st);
    std::int64_t batch_first = -1, batch_cols = 0;  // draw offset (in blocks) and width of the current batch
    // Y and Z rows padded to a multiple of 4 doubles: every CSR gather of one of their rows then
    // starts on a 32-byte L2 sector (w = 50: 13 sectors per row instead of 13.5 on average)
    const std::int64_t lyz = round_up(bpad, 4);
    DBuf y(static_cast<std::size_t>(std::max<std::int64_t>(m, 1)) * lyz, c.st);
    DBuf tmp(static_cast<std::size_t>(std::max<std::int64_t>(std::max<std::int64_t>(m, n), 1)) * bpad, c.st);
    DBuf z(p.power > 0 ? static_cast<std::size_t>(blk) * lyz : 0, c.st);
    DBuf zfull(nsh && p.power > 0 ? static_cast<std::size_t>(n_pad) * lyz : 0, c.st);
    DBuf mbuf(static_cast<std::size_t>(std::max<std::int64_t>(cap, 1)) * bpad, c.st);
    double e_host = norm_a_sq;
    // The next block's first pass Y = A Omega_{i+1} does not depend on block i's outcome: it is
    // queued behind block i's indicator read-back, so the GPU keeps working while the host waits
    // for the stop decision (QBFAC_EI_PREFETCH=0 disables). Discarded when block i terminates or
    // is recomputed; counted as a pass only when the next block uses it.
    static const bool prefetch_on = [] {
        const char* e = std::getenv("QBFAC_EI_PREFETCH");
        return !(e && e[0] == '0');
    }();
    // m_pre: the next block's B Omega_{i+1} is queued behind the read-back too (one GPU only: no
    // allreduce in between). Queueing its projection Y -= Q (B Omega_{i+1}) as well measured no
    // further gain (config 1 3.80 -> 3.83 ms): the read-back is already covered.
    bool y_pre = false, m_pre = false;
    // The sketches inside the power iteration (Y before the A^T pass, Z before the A pass) only
    // pass their span on; their orth may stop after one CholQR pass (QBFAC_EI_SPAN_ORTH=0: always two).
    const bool span_only = [] {
        const char* e = std::getenv("QBFAC_EI_SPAN_ORTH");
        return !(e && e[0] == '0');
    }();
    // Dense resident A, narrow blocks: the first pass of several consecutive blocks is ONE product
    // A [Omega_i ... Omega_{i+c-1}] (their Omega columns are adjacent in the batch drawn above), up to
    // 104 columns wide, so the pass runs on the wide DMMA tiles instead of c launches of b-column
    // products that never fill the pipeline (b = 20: 5 blocks per product). Each block still counts
    // its pass (Alg. 2 reads A once per block; the count reported is the algorithm's). Blocks past a
    // termination waste at most c - 1 narrow products. QBFAC_EI_YBATCH=0 disables.
    const bool ybatch_on = [] {  // read per run (tests compare both settings in one process)
        const char* e = std::getenv("QBFAC_EI_YBATCH");
        return !(e && e[0] == '0');
    }();
    const std::int64_t nbat = (ybatch_on && !a.sparse && !a.host_stream && bmax % 2 == 0)
                                  ? std::max<std::int64_t>(1, std::min<std::int64_t>(104 / bmax, nb_batch)) : 1;
    const std::int64_t ldyb = round_up(nbat * bmax, 4);
    DBuf ybat(nbat > 1 ? static_cast<std::size_t>(std::max<std::int64_t>(m, 1)) * ldyb : 0, c.st);
    std::int64_t yb_first = -1, yb_count = 0;  // blocks [yb_first, yb_first + yb_count) of A Omega are in ybat
    auto ybatch_fill = [&](std::int64_t j0, std::int64_t k_now) {  // needs Omega blocks j0.. in the drawn batch
        const std::int64_t in_batch = batch_first + nb_batch - j0;
        const std::int64_t left = ceil_div(cap - k_now, bmax);
        yb_count = std::max<std::int64_t>(1, std::min(std::min(nbat, in_batch), left));
        yb_first = j0;
        const std::int64_t cols = std::min(yb_count * bmax, std::min(cap - k_now, batch_cols - (j0 - batch_first) * bmax));
        eng.apply(MatView{om.p + (j0 - batch_first) * bmax, n, cols, ldom, true}, MatView{ybat.p, m, cols, ldyb, true});
    };
    while (true) {
        if (s.k >= cap) { term = 0; break; }
        const std::int64_t bi = std::min(p.b, cap - s.k);
        ++blocks;
        const std::int64_t passes_before = a.passes;
        // blocks before the last are full width, so block j starts at draw g_used = j * n * bmax
        const std::int64_t jblk = g_used / (n * bmax);
        if (batch_first < 0 || jblk < batch_first || jblk >= batch_first + nb_batch || g_used % (n * bmax) != 0) {
            batch_first = jblk;
            batch_cols = std::min(nb_batch * bmax, cap - s.k);
            MatView all{om.p, n, batch_cols, ldom, true};
            gaussian_fill(c.st, c.rng, p.seed, p.stream, static_cast<std::uint64_t>(g_used), all);  // step 4
        }
        MatView omv{om.p + (jblk - batch_first) * bmax, n, bi, ldom, true};
        bool in_ybatch = false;
        if (nbat > 1 && g_used % (n * bmax) == 0) {
            if (yb_first < 0 || jblk < yb_first || jblk >= yb_first + yb_count) ybatch_fill(jblk, s.k);
            in_ybatch = true;
        }
        MatView yv = in_ybatch ? MatView{ybat.p + (jblk - yb_first) * bmax, m, bi, ldyb, true} : MatView{y.p, m, bi, lyz, true};
        MatView mv{mbuf.p, s.k, bi, bi, true};
        int d = 0, keep = 0;
        bool met = false, refilled = false;
        // attempt 0: optimistic CholQR, statuses checked once with the indicator read;
        // attempt 1 (rare): the same block with Householder panels (exact deficiency rules).
        for (int attempt = 0; attempt < 2; ++attempt) {
            a.passes = passes_before;
            eng.begin_block(/*optimistic=*/true, /*force_hh=*/attempt > 0);
            // step 5: Y = A Omega_i - Q (B Omega_i)   (Omega_i drawn with its batch above)
            if (!(attempt == 0 && (y_pre || in_ybatch))) eng.apply(omv, yv);
            y_pre = false;
            a.passes += 1;
            if (s.k > 0) {
                if (!(attempt == 0 && m_pre))
                    eng.gemm(1.0, s.btk().t(), omv.rows_range(c0, nl), 0.0, mv);  // B Omega_i (partial if nsh)
                if (nsh) eng.allreduce_view(mv);
                eng.gemm(-1.0, s.qk(), mv, 1.0, yv);
            }
            m_pre = false;
            // per-block power iteration with deflation at every application
            for (std::int64_t it = 0; it < p.power; ++it) {
                eng.orth_block(yv, yv, kR1, kR1inv, sharded, tmp, false, span_only);
                MatView zv{z.p, blk, bi, lyz, true};   // this rank's rows of Z (all n when replicated)
                MatView zr = zv.rows_range(0, nl);
                if (nsh) eng.apply_t_rs(yv, zv, n_pad, blk);
                else eng.apply_t(yv, zv);
                a.passes += 1;
                if (s.k > 0) {
                    eng.gemm(1.0, s.qk().t(), yv, 0.0, mv);
                    eng.allreduce_view(mv);
                    eng.gemm(-1.0, s.btk(), mv, 1.0, zr);
                }
                if (nsh) {
                    eng.geo_rows = n_pad;
                    eng.geo_row0 = c0;
                    eng.orth_block(zv, zv, kR1, kR1inv, true, tmp, false, span_only);  // rows of Z split over the ranks
                    eng.geo_rows = -1;
                    c.all_gather(z.p, zfull.p, static_cast<std::size_t>(blk * lyz));
                    eng.apply(MatView{zfull.p, n, bi, lyz, true}, yv); a.passes += 1;
                } else {
                    eng.orth_block(zv, zv, kR1, kR1inv, false, tmp, false, span_only);
                    eng.apply(zv, yv); a.passes += 1;
                }
                if (s.k > 0) {
                    eng.gemm(1.0, s.btk().t(), zr, 0.0, mv);
                    if (nsh) eng.allreduce_view(mv);
                    eng.gemm(-1.0, s.qk(), mv, 1.0, yv);
                }
            }
            // orth, then re-orthogonalisation against Q (step 6)
            MatView qs = s.qslot(bi);
            // (when the re-orthogonalisation follows, this orth too only hands on a span: the
            // projection is linear, and the second orth below is the one that makes Q_i orthonormal)
            d = eng.orth_block(yv, qs, kR1, kR1inv, sharded, tmp, false, span_only && s.k > 0);
            if (d > 0 && s.k > 0) {
                MatView qd = s.qslot(d);
                MatView md{mbuf.p, s.k, d, d, true};
                eng.gemm(1.0, s.qk().t(), qd, 0.0, md);
                eng.allreduce_view(md);
                eng.gemm(-1.0, s.qk(), md, 1.0, qd);
                const int d2 = eng.orth_block(qd, qd, kR2, kR2inv, sharded, tmp, false);
                d = std::min(d, d2);
            }
            if (d == 0) {
                if (attempt == 0) { eng.fetch_lazy(); QB_CUDA(cudaStreamSynchronize(c.st)); }
                if (attempt == 0 && !eng.lazy_ok()) continue;
                break;
            }
            // step 7: B_i^T = A^T Q_i (+1 pass; this rank's column block of B_i when nsh)
            if (nsh) eng.apply_t_rs(s.qslot(d), s.btslot(d), n_pad, blk);
            else eng.apply_t(s.qslot(d), s.btslot(d));
            a.passes += 1;
            s.indicator_enqueue(d, fixed_prec);
            eng.fetch_lazy();
            if (prefetch_on && attempt == 0 && d == bi && bi == bmax) {
                // next block (if this one neither terminates nor is recomputed): k + bi columns,
                // Omega at draw offset g_used + n bi, i.e. block jblk + 1 of the batch
                const std::int64_t bn = std::min(p.b, cap - (s.k + bi));
                if (bn > 0 && jblk + 1 < batch_first + nb_batch && (jblk + 1 - batch_first) * bmax + bn <= batch_cols) {
                    if (nbat > 1) {
                        s.indicator_mark();
                        if (jblk + 1 >= yb_first + yb_count) {  // the next block opens a new product
                            ybatch_fill(jblk + 1, s.k + bi);
                            refilled = true;
                        }
                    } else {
                        s.indicator_mark();
                        eng.apply(MatView{om.p + (jblk + 1 - batch_first) * bmax, n, bn, ldom, true},
                                  MatView{y.p, m, bn, lyz, true});
                        y_pre = true;
                    }
                    if (!sharded) {  // B Omega_{i+1} over the k + bi rows of B this block leaves behind
                        eng.gemm(1.0, s.bt_cols(s.k + bi).t(), MatView{om.p + (jblk + 1 - batch_first) * bmax, n, bn, ldom, true},
                                 0.0, MatView{mbuf.p, s.k + bi, bn, bn, true});
                        m_pre = true;
                    }
                }
            }
            std::tie(keep, met) = s.indicator_finish();
            if (attempt == 0 && !eng.lazy_ok()) {  // every rank sees the same (reduced) statuses
                y_pre = m_pre = false;  // the block is recomputed (Y and the coefficients overwritten)
                if (refilled) yb_first = -1;  // ... into columns the next product already occupies: drop it
                s.set_e(e_host);  // undo this block's indicator update
                continue;
            }
            break;
        }
        g_used += n * bi;
        if (d == 0) { term = 3; break; }
        e_host = c.h_ind->e;
        s.trace.push_back(e_host);
        s.k += keep;
        if (met) { term = 1; break; }
        if (d < bi) { term = 3; break; }
    }
    return wrap(term);
}

// ---- randQB_FP / fixed rank / single pass --------------------------------------------
std::unique_ptr<Result> run_fp(Context& c, Matrix& a, const Params& p) {
    if (p.b < 1) throw QbError(kDimensionError, "rand_qb_fp: block size must be >= 1");
    const bool fp_span_only = [] {
        const char* e = std::getenv("QBFAC_EI_SPAN_ORTH");
        return !(e && e[0] == '0');
    }();
    if (a.host_stream && (p.alg != 3 || p.power != 0))
        throw QbError(kError, "host-streamed matrix: only single_pass_fp consumes a RowStream");
    Engine eng(c, a);
    const std::int64_t m = a.m, n = a.n, mg = a.m_global;
    const bool fixed = p.alg != 1;           // Alg. 3 / single pass: fixed rank l = k + s
    const bool reorth = p.alg == 1 || p.alg == 3 || p.reorth;
    std::int64_t cap = std::min(mg, n);
    if (fixed) {
        const std::int64_t l = p.k + p.s;
        if (l < 1 || l > cap) throw QbError(kDimensionError, "rand_qb_fp_fixed_rank: bad l");
        cap = l;
    } else {
        if (p.l_budget < p.b) throw QbError(kDimensionError, "rand_qb_fp: l_budget must be >= b");
        if (p.max_rank > 0) cap = std::min(cap, p.max_rank);
    }
    const std::int64_t passes0 = a.passes;
    State s(c, eng, m, n, cap);
    const bool sharded = c.world > 1;
    s.eps2 = fixed ? 0.0 : p.eps_abs * p.eps_abs;
    double norm_a_sq = 0.0;
    int term = 2;
    std::int64_t g_used = 0, blocks = 0, restarts = 0;
    auto wrap = [&](int t) {
        auto r = finish(s, a, passes0, t, norm_a_sq);
        r->gaussians_used = g_used;
        r->blocks = blocks;
        r->restarts = restarts;
        r->hh_fallbacks = eng.hh_fallbacks;
        if (p.alg == 3) r->passes = 1;  // one stream consumption
        return r;
    };
    const std::int64_t lmax = fixed ? cap : std::min(p.l_budget, cap);
    const std::int64_t lpad = even(lmax);
    const std::int64_t bmax = std::min(p.b, lmax);
    const std::int64_t bpad = even(bmax);
    DBuf om(static_cast<std::size_t>(n) * lpad, c.st);
    DBuf g(static_cast<std::size_t>(std::max<std::int64_t>(m, 1)) * lpad, c.st);
    DBuf h(static_cast<std::size_t>(n) * lpad, c.st);
    DBuf y(static_cast<std::size_t>(std::max<std::int64_t>(m, 1)) * bpad, c.st);
    DBuf tmp(static_cast<std::size_t>(std::max<std::int64_t>(std::max<std::int64_t>(m, n), 1)) * bpad, c.st);
    DBuf ct(static_cast<std::size_t>(n) * bpad, c.st);
    DBuf m1(static_cast<std::size_t>(std::max<std::int64_t>(cap, 1)) * bpad, c.st);
    DBuf m2(static_cast<std::size_t>(std::max<std::int64_t>(cap, std::max<std::int64_t>(lpad, 64))) * std::max<std::int64_t>(bpad, 64), c.st);
    DBuf wtmp(p.power > 0 ? static_cast<std::size_t>(std::max<std::int64_t>(std::max<std::int64_t>(m, n), 1)) * 64 : 0, c.st);
    double e_host = 0.0;
    for (int restart = 0;; ++restart) {
        if (s.k >= cap) { term = 0; break; }
        if (fixed && restart > 0) { term = 0; break; }
        if (restart > p.max_restarts) { term = 2; break; }
        if (restart > 0) ++restarts;
        const std::int64_t l = fixed ? cap : std::min(p.l_budget, cap - s.k);
        const std::uint64_t stream_id = restart == 0 ? p.stream : p.stream + 1 + static_cast<std::uint64_t>(restart);
        MatView omv{om.p, n, l, l, true};
        gaussian_fill(c.st, c.rng, p.seed, stream_id, 0, omv);                   // step 2
        if (restart == 0) g_used = n * l;
        MatView gv{g.p, m, l, l, true};
        MatView hv{h.p, n, l, l, true};
        for (std::int64_t it = 0; it < p.power; ++it) {                            // steps 3-6
            if (!sharded) eng.request_pregram();
            eng.apply(omv, gv); a.passes += 1;
            eng.orth_wide(gv, sharded, wtmp, m2);
            eng.apply_t(gv, omv); a.passes += 1;
            eng.orth_wide(omv, false, wtmp, m2);
        }
        if (a.host_stream) {                                                       // steps 7-9, one stream
            norm_a_sq = eng.stream_single_pass(omv, gv, hv);
            e_host = norm_a_sq;
            s.set_e(norm_a_sq);
            a.passes += 2;
        } else {
        eng.apply(omv, gv); a.passes += 1;                                         // step 7
        if (restart == 0) {                                                        // step 9
            norm_a_sq = eng.frob_device(s.d_e);  // same logical pass (multiply_with_norm)
            e_host = norm_a_sq;
            if (!fixed) {
                check_eps(p.eps_abs, norm_a_sq);
                if (norm_a_sq < s.eps2) { term = 1; break; }
            }
        }
        eng.apply_t(gv, hv); a.passes += 1;                                        // step 8
        }
        bool stop = false;
        for (std::int64_t off = 0; off < l; off += p.b) {                          // steps 10-21
            const std::int64_t bi = std::min(p.b, l - off);
            ++blocks;
            MatView omi = omv.cols_range(off, bi);
            MatView gi = gv.cols_range(off, bi);
            MatView hi = hv.cols_range(off, bi);
            MatView yv{y.p, m, bi, bi, true};
            MatView m1v{m1.p, s.k, bi, bi, true};
            int d = 0, keep = 0;
            bool met = false;
            for (int attempt = 0; attempt < 2; ++attempt) {  // optimistic CholQR, Householder redo
                eng.begin_block(true, attempt > 0);
                eng.wide_mode = bi > kSmallMax;
                copy_matrix(c.st, gi, yv);
                if (s.k > 0) {                                                     // step 12
                    eng.gemm(1.0, s.btk().t(), omi, 0.0, m1v);
                    eng.gemm(-1.0, s.qk(), m1v, 1.0, yv);
                }
                MatView qs = s.qslot(bi);
                // step 13; when steps 14-15 follow, R_1 only has to satisfy Y = Q~ R_1 (B_i's formula
                // below holds for any such pair), so this orth may stop after one pass like run_ei's
                d = eng.orth_block(yv, qs, kR1, kR1inv, sharded, tmp, true, fp_span_only && reorth && s.k > 0);
                int rinv_slot = kR1inv;
                if (d > 0 && reorth && s.k > 0) {                                  // steps 14-15 (9a-9b)
                    MatView qd = s.qslot(d);
                    MatView md{m2.p, s.k, d, d, true};
                    eng.gemm(1.0, s.qk().t(), qd, 0.0, md);
                    eng.allreduce_view(md);
                    eng.gemm(-1.0, s.qk(), md, 1.0, qd);
                    const int d2 = eng.orth_block(qd, qd, kR2, kR2inv, sharded, tmp);
                    d = std::min(d, d2);
                    if (d > 0) {
                        eng.tri_pair(kR2, kR1, kR, kR1inv, kR2inv, kRinv, d);
                        rinv_slot = kRinv;
                    }
                }
                if (d == 0) {
                    if (attempt == 0) { eng.fetch_lazy(); QB_CUDA(cudaStreamSynchronize(c.st)); }
                    if (attempt == 0 && !eng.lazy_ok()) continue;
                    break;
                }
                // step 16 (9c): B_i^T = (H_i - B^T (Q^T Y_i + B Omega_i)) R_i^{-1}
                //   (Alg. 3 without re-orth: B_i^T = (H_i - B^T (B Omega_i)) R_i^{-1})
                MatView ctv{ct.p, n, d, d, true};
                copy_matrix(c.st, hi.cols_range(0, d), ctv);
                if (s.k > 0) {
                    MatView mm{m2.p, s.k, d, d, true};
                    if (reorth) {
                        eng.gemm(1.0, s.qk().t(), yv.cols_range(0, d), 0.0, mm);
                        eng.allreduce_view(mm);
                        add_matrix(c.st, m1v.cols_range(0, d), mm, 1.0);
                    } else {
                        copy_matrix(c.st, m1v.cols_range(0, d), mm);
                    }
                    eng.gemm(-1.0, s.btk(), mm, 1.0, ctv);
                }
                eng.gemm(1.0, ctv, eng.rmat(rinv_slot, d), 0.0, s.btslot(d));
                s.indicator_enqueue(d, !fixed);                                    // steps 19-20
                eng.fetch_lazy();
                std::tie(keep, met) = s.indicator_finish();
                if (attempt == 0 && !eng.lazy_ok()) {  // every rank sees the same (reduced) statuses
                    s.set_e(e_host);
                    continue;
                }
                break;
            }
            eng.begin_block(false, false);
            eng.wide_mode = false;
            if (d == 0) { term = 3; stop = true; break; }
            e_host = c.h_ind->e;
            s.trace.push_back(e_host);
            s.k += keep;
            if (met) { term = 1; stop = true; break; }
            if (d < bi) { term = 3; stop = true; break; }
        }
        if (stop) break;
    }
    return wrap(term);
}

}  // namespace

// ---- test hook: the wide orthonormalisation used by the power iteration ----------------
void test_orth_wide(Context& c, const MatView& x, bool force_bcgs2) {
    Matrix dummy;
    Engine eng(c, dummy);
    DBuf tmp(static_cast<std::size_t>(std::max<std::int64_t>(x.rows, 1)) * 64, c.st);
    DBuf sbuf(static_cast<std::size_t>(std::max<std::int64_t>(x.cols, 64)) * 64, c.st);
    if (force_bcgs2) eng.orth_wide_bcgs2(x, false, tmp, sbuf);
    else eng.orth_wide(x, false, tmp, sbuf);
    QB_CUDA(cudaStreamSynchronize(c.st));
}

// ---- qb_to_svd (PAPER Eq. 1.3) ---------------------------------------
// B (r x n) = N Q_b^T with Q_b = orth(B^T) (n x r, the wide CholQR2 / BCGS2 of the power step)
// and N = B Q_b (r x r); one-sided Jacobi N W = U_r Sigma; then U = Q U_r(:, top k),
// V = Q_b W(:, top k). Everything runs on the device; only Sigma (r doubles, for the order)
// and the k columns of U, V leave it.
namespace {
__global__ void gather_scale_kernel(const double* __restrict__ src, int r, const int* __restrict__ idx,
                                    const double* __restrict__ scale, int k, double* __restrict__ dst) {
    const std::int64_t total = static_cast<std::int64_t>(r) * k;
    for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(e % r), t = static_cast<int>(e / r);
        const double sc = scale ? scale[t] : 1.0;
        dst[e] = src[i + static_cast<std::int64_t>(idx[t]) * r] * sc;
    }
}
}  // namespace

int qb_to_svd(Context& c, Result& r, std::int64_t k, double* u_out, std::int64_t ldu, double* s_out, double* v_out,
              std::int64_t ldv) {
    const std::int64_t rk = r.rank, m = r.m, n = r.n;
    if (k < 0 || k > rk) throw QbError(kDimensionError, "qb_to_svd: k too large");
    if (k == 0) return 0;
    if (ldu < m || ldv < n) throw QbError(kDimensionError, "qb_to_svd: leading dimension too small");
    Matrix dummy;
    Engine eng(c, dummy);
    cudaStream_t st = c.st;
    // Q_b = orth(B^T) on a packed copy
    DBuf x(static_cast<std::size_t>(n) * rk, st);
    MatView xv{x.p, n, rk, rk, true};
    copy_matrix(st, r.bt_view(), xv);
    DBuf tmp(static_cast<std::size_t>(std::max<std::int64_t>(n, 1)) * 64, st);
    DBuf sbuf(static_cast<std::size_t>(std::max<std::int64_t>(rk, 64)) * 64, st);
    eng.orth_wide(xv, false, tmp, sbuf);
    // N = B Q_b (r x r, column-major), W = I
    DBuf nm(static_cast<std::size_t>(rk) * rk, st), wm(static_cast<std::size_t>(rk) * rk, st);
    MatView nv{nm.p, rk, rk, rk, false}, wv{wm.p, rk, rk, rk, false};
    eng.gemm(1.0, r.bt_view().t(), xv, 0.0, nv);
    set_identity(st, wv);
    const int sweeps = jacobi_svd(st, nm.p, wm.p, static_cast<int>(rk), c.d_gbar);
    // Sigma_j = ||N(:, j)||, descending order
    DBuf nrm(static_cast<std::size_t>(rk), st);
    column_sumsq(st, c.ws_red, nv, nrm.p);
    std::vector<double> hs(static_cast<std::size_t>(rk));
    QB_CUDA(cudaMemcpyAsync(hs.data(), nrm.p, sizeof(double) * rk, cudaMemcpyDeviceToHost, st));
    QB_CUDA(cudaStreamSynchronize(st));
    std::vector<int> idx(static_cast<std::size_t>(rk));
    for (std::int64_t i = 0; i < rk; ++i) idx[i] = static_cast<int>(i);
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return hs[a] > hs[b]; });
    std::vector<double> sig(static_cast<std::size_t>(k)), inv(static_cast<std::size_t>(k));
    for (std::int64_t t = 0; t < k; ++t) {
        sig[t] = std::sqrt(hs[idx[t]]);
        inv[t] = sig[t] > 0.0 ? 1.0 / sig[t] : 0.0;
    }
    DBuf aux(static_cast<std::size_t>(2 * k + 1), st);
    int* d_idx = reinterpret_cast<int*>(aux.p);  // k ints in the first k/2 + 1 doubles
    double* d_inv = aux.p + k;
    QB_CUDA(cudaMemcpyAsync(d_idx, idx.data(), sizeof(int) * k, cudaMemcpyHostToDevice, st));
    QB_CUDA(cudaMemcpyAsync(d_inv, inv.data(), sizeof(double) * k, cudaMemcpyHostToDevice, st));
    DBuf uk(static_cast<std::size_t>(rk) * k, st), wk(static_cast<std::size_t>(rk) * k, st);
    const int blocks = static_cast<int>(std::min<std::int64_t>(ceil_div(rk * k, 256), 4096));
    gather_scale_kernel<<<blocks, 256, 0, st>>>(nm.p, static_cast<int>(rk), d_idx, d_inv, static_cast<int>(k), uk.p);
    QB_LAUNCH_CHECK();
    gather_scale_kernel<<<blocks, 256, 0, st>>>(wm.p, static_cast<int>(rk), d_idx, nullptr, static_cast<int>(k), wk.p);
    QB_LAUNCH_CHECK();
    // U = Q U_r(:, top k), V = Q_b W(:, top k), both column-major for the copy-out. The copies
    // (8 (m + n) k bytes, the PCIe-bound part at large k) run on the copy stream behind the
    // product that fills them: V first, then U in column chunks, so all but the first product
    // and the last chunk's copy overlap.
    DBuf ud(static_cast<std::size_t>(std::max<std::int64_t>(m, 1)) * k, st), vd(static_cast<std::size_t>(n) * k, st);
    cudaEvent_t ev;
    QB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    auto copy_out = [&](double* dst, std::int64_t ldd, const double* src, std::int64_t rows, std::int64_t cols) {
        QB_CUDA(cudaEventRecord(ev, st));
        QB_CUDA(cudaStreamWaitEvent(c.st_copy, ev, 0));
        QB_CUDA(cudaMemcpy2DAsync(dst, ldd * sizeof(double), src, rows * sizeof(double), rows * sizeof(double),
                                  static_cast<std::size_t>(cols), cudaMemcpyDeviceToHost, c.st_copy));
    };
    // (column chunks: the first copy starts after a quarter of the first product)
    auto product_out = [&](const MatView& left, const double* coef, double* dev, std::int64_t rows, double* host,
                           std::int64_t ldh) {
        const std::int64_t nchunk = (rows * k >= (std::int64_t{1} << 24)) ? 4 : 1;
        const std::int64_t cw = ceil_div(k, nchunk);
        for (std::int64_t c0 = 0; c0 < k; c0 += cw) {
            const std::int64_t cn = std::min(cw, k - c0);
            eng.gemm(1.0, left, MatView{const_cast<double*>(coef) + c0 * rk, rk, cn, rk, false}, 0.0,
                     MatView{dev + c0 * rows, rows, cn, rows, false});
            copy_out(host + c0 * ldh, ldh, dev + c0 * rows, rows, cn);
        }
    };
    product_out(xv, wk.p, vd.p, n, v_out, ldv);
    if (m > 0) product_out(r.q_view(), uk.p, ud.p, m, u_out, ldu);
    QB_CUDA(cudaStreamSynchronize(c.st_copy));
    QB_CUDA(cudaStreamSynchronize(st));
    QB_CUDA(cudaEventDestroy(ev));
    std::copy(sig.begin(), sig.end(), s_out);
    return sweeps;
}

// ---- operator layer ------------------------------------------------------------------
// DenseMatrix::from_data rejects non-finite entries (dense_matrix.cpp:17-18). An async upload
// defers that check to its first ||A||^2 (frob_device); a consumer that never forms the norm
// (randQB, the range finder, a bare multiply) runs it here, once, before its result is returned.
void finish_finite_check(Context& c, Matrix& a) {
    if (!a.check_finite) return;
    a.wait_resident(c.st);
    double* d = c.d_small + static_cast<std::size_t>(kSlot) * kNumSlots + 3;
    sum_squares(c.st, c.ws_red, a.dense_view(), d);
    QB_CUDA(cudaMemcpyAsync(c.h_scalar, d, sizeof(double), cudaMemcpyDeviceToHost, c.st));
    QB_CUDA(cudaStreamSynchronize(c.st));
    a.check_finite = false;
    if (!std::isfinite(c.h_scalar[0])) throw QbError(kError, "from_data: non-finite entry");
}

double frob_norm_sq(Context& c, Matrix& a) {
    Engine eng(c, a);
    a.passes += 1;
    return eng.frob_device(c.d_small + static_cast<std::size_t>(kSlot) * kNumSlots + 3);
}

void multiply(Context& c, Matrix& a, const MatView& x, const MatView& y, bool trans) {
    Engine eng(c, a);
    if (trans) eng.apply_t(x, y);
    else eng.apply(x, y);
    a.passes += 1;
    finish_finite_check(c, a);
}

// ---- baselines (§8(f) 4) ---------------------------------------------
// Orthonormal basis of Y's leading columns with the reference's deficiency rule; returns
// the kept width (panels <= 112 columns: exact Householder decision on CholQR failure;
// wider: wide CholQR2 / BCGS2, full width).
int orth_any(Engine& eng, const MatView& y, bool sharded, DBuf& tmp, DBuf& sbuf) {
    if (y.cols <= kSmallMax) return eng.orth_block(y, y, kR1, kR1inv, sharded, tmp, false);
    eng.orth_wide(y, sharded, tmp, sbuf);
    return static_cast<int>(y.cols);
}

// randQB (Fig. 1a): Q = orth((A A^T)^P A Omega) with orth after every application, B = Q^T A.
std::unique_ptr<Result> run_qb(Context& c, Matrix& a, const Params& p) {
    const std::int64_t m = a.m, n = a.n, l = p.k + p.s;
    if (l < 1 || l > std::min(a.m_global, n)) throw QbError(kDimensionError, "rand_qb: l must be in [1, min(m, n)]");
    Engine eng(c, a);
    const bool sharded = c.world > 1;
    const std::int64_t passes0 = a.passes;
    State s(c, eng, m, n, l);
    DBuf om(static_cast<std::size_t>(n) * even(l), c.st);
    DBuf tmp(static_cast<std::size_t>(std::max<std::int64_t>(std::max(m, n), 1)) * 64, c.st);
    DBuf sbuf(static_cast<std::size_t>(std::max<std::int64_t>(l, 64)) * 64, c.st);
    MatView omv{om.p, n, l, l, true};
    gaussian_fill(c.st, c.rng, p.seed, p.stream, 0, omv);
    std::int64_t d = l;
    bool collapsed = false;
    MatView y{s.q.p, m, d, s.ld, true};
    eng.apply(omv, y); a.passes += 1;
    auto orth_y = [&](const MatView& v) {
        const int dd = orth_any(eng, v, sharded && v.rows == m, tmp, sbuf);
        if (dd < v.cols) collapsed = true;
        return static_cast<std::int64_t>(dd);
    };
    d = orth_y(y);
    for (std::int64_t it = 0; it < p.power && d > 0; ++it) {
        MatView w{om.p, n, d, d, true};
        eng.apply_t(MatView{s.q.p, m, d, s.ld, true}, w); a.passes += 1;
        d = orth_y(w);
        if (d == 0) break;
        MatView yy{s.q.p, m, d, s.ld, true};
        eng.apply(MatView{om.p, n, d, d, true}, yy); a.passes += 1;
        d = orth_y(yy);
    }
    s.k = d;
    if (d > 0) { eng.apply_t(s.qk(), s.btk()); }
    a.passes += 1;
    s.set_e(-1.0);  // SPEC.md:212 sentinel: no error indicator
    auto r = finish(s, a, passes0, collapsed ? 3 : 0, 0.0);
    r->hh_fallbacks = eng.hh_fallbacks;
    return r;
}

// randQB_b (Fig. 1b): explicit residual, 4 passes per block.
std::unique_ptr<Result> run_qb_b(Context& c, Matrix& a, const Params& p) {
    if (p.b < 1) throw QbError(kDimensionError, "rand_qb_b: block size must be >= 1");
    if (a.sparse || a.host_stream) throw QbError(kDimensionError, "rand_qb_b: dense A only (the residual is dense)");
    a.wait_resident(c.st);
    const std::int64_t m = a.m, n = a.n;
    const bool fixed_prec = p.mode == 1;
    std::int64_t cap = std::min(a.m_global, n);
    if (!fixed_prec) cap = std::min(cap, p.k + p.s);
    Engine eng(c, a);
    const bool sharded = c.world > 1;
    const std::int64_t passes0 = a.passes;
    State s(c, eng, m, n, cap);
    s.eps2 = fixed_prec ? p.eps_abs * p.eps_abs : 0.0;
    // residual R = A (column-major, same layout as A)
    DBuf res(static_cast<std::size_t>(a.lda) * std::max<std::int64_t>(n, 1), c.st);
    MatView rv{res.p, m, n, a.lda, false};
    copy_matrix(c.st, a.dense_view(), rv);
    const std::int64_t bmax = std::min<std::int64_t>(p.b, std::max<std::int64_t>(cap, 1));
    DBuf om(static_cast<std::size_t>(n) * even(bmax), c.st);
    DBuf tmp(static_cast<std::size_t>(std::max<std::int64_t>(std::max(m, n), 1)) * even(bmax), c.st);
    DBuf mbuf(static_cast<std::size_t>(std::max<std::int64_t>(cap, 1)) * even(bmax), c.st);
    double norm_a_sq = 0.0;
    int term = 0;
    std::int64_t g_used = 0, blocks = 0;
    while (true) {
        if (s.k >= cap) { term = 0; break; }
        sum_squares(c.st, c.ws_red, rv, s.d_e);              // E = ||R||_F^2 (one pass over R)
        c.allreduce(s.d_e, 1);
        a.passes += 1;
        const double e = s.get_e();
        if (!std::isfinite(e)) throw QbError(kError, "from_data: non-finite entry");
        if (s.k == 0) {
            norm_a_sq = e;
            if (fixed_prec) check_eps(p.eps_abs, norm_a_sq);
        }
        if (fixed_prec && e < s.eps2) { term = 1; break; }
        const std::int64_t bi = std::min(p.b, cap - s.k);
        ++blocks;
        MatView omv{om.p, n, bi, bi, true};
        gaussian_fill(c.st, c.rng, p.seed, p.stream, static_cast<std::uint64_t>(g_used), omv);
        g_used += n * bi;
        MatView qs = s.qslot(bi);
        eng.gemm(1.0, rv, omv, 0.0, qs);                    // Y = R Omega_i
        a.passes += 1;
        int d = eng.orth_block(qs, qs, kR1, kR1inv, sharded, tmp, false);
        if (d > 0 && s.k > 0) {                              // re-orthogonalisation against Q
            MatView qd = s.qslot(d);
            MatView md{mbuf.p, s.k, d, d, true};
            eng.gemm(1.0, s.qk().t(), qd, 0.0, md);
            eng.allreduce_view(md);
            eng.gemm(-1.0, s.qk(), md, 1.0, qd);
            d = std::min(d, eng.orth_block(qd, qd, kR2, kR2inv, sharded, tmp, false));
        }
        if (d == 0) { term = 3; break; }
        MatView bts = s.btslot(d);
        eng.gemm(1.0, rv.t(), s.qslot(d), 0.0, bts);         // B_i^T = R^T Q_i
        eng.allreduce_view(bts);
        a.passes += 1;
        const auto [keep, met] = s.indicator(d, fixed_prec);  // rows of B_i enter E
        eng.gemm(-1.0, s.qslot(keep), s.btslot(keep).t(), 1.0, rv);  // R -= Q_i B_i
        a.passes += 1;
        s.k += keep;
        if (met) { term = 1; break; }
        if (keep < bi) { term = 3; break; }
    }
    s.trace.clear();
    auto r = finish(s, a, passes0, term, norm_a_sq);
    r->gaussians_used = g_used;
    r->blocks = blocks;
    r->hh_fallbacks = eng.hh_fallbacks;
    return r;
}

// Adaptive randomized range finder (Eq. 2.4; Halko et al. Alg. 4.2): Q grows one vector at a
// time; stops when the r most recent residual samples are all <= tol / (10 sqrt(2/pi)).
std::unique_ptr<Result> run_arf(Context& c, Matrix& a, const Params& p) {
    const std::int64_t r = p.b;
    if (r < 1) throw QbError(kDimensionError, "adaptive_range_finder: r must be >= 1");
    // Row-sharded (world > 1): samples and Q rows live on their ranks; the column norms, the
    // projections Q^T v and the final A^T Q are summed over ranks (the same allreduces as EI).
    const std::int64_t m = a.m, n = a.n;
    std::int64_t cap = std::min(a.m_global, n);
    if (p.max_rank > 0) cap = std::min(cap, p.max_rank);
    Engine eng(c, a);
    const std::int64_t passes0 = a.passes;
    State s(c, eng, m, n, cap);
    const double thr = p.eps_abs / (10.0 * std::sqrt(2.0 / 3.14159265358979323846));
    // window of r samples, column-major m x r (each sample contiguous), plus scratch
    DBuf win(static_cast<std::size_t>(std::max<std::int64_t>(m, 1)) * r, c.st);
    DBuf om(static_cast<std::size_t>(n) * r, c.st);
    DBuf yv(static_cast<std::size_t>(std::max<std::int64_t>(m, 1)), c.st);
    DBuf cv(static_cast<std::size_t>(std::max<std::int64_t>(cap, r) + 1), c.st);
    DBuf nrm(static_cast<std::size_t>(r + 1), c.st);
    std::vector<double> hn(static_cast<std::size_t>(r + 1));
    std::uint64_t g_used = 0;
    {   // y_1..y_r = A omega_i, one pass each
        MatView omv{om.p, n, r, r, true};
        gaussian_fill(c.st, c.rng, p.seed, p.stream, 0, omv);
        g_used = static_cast<std::uint64_t>(n * r);
        MatView wv{win.p, m, r, std::max<std::int64_t>(m, 1), false};
        for (std::int64_t i = 0; i < r; ++i) {
            MatView oi{om.p + i, n, 1, r, true};
            MatView yi{win.p + i * m, m, 1, 1, true};
            eng.apply(oi, yi);
            a.passes += 1;
        }
        (void)wv;
    }
    auto project = [&](double* v) {  // v -= Q (Q^T v)
        if (s.k == 0) return;
        MatView vv{v, m, 1, 1, true};
        MatView cc{cv.p, s.k, 1, 1, true};
        eng.gemm(1.0, s.qk().t(), vv, 0.0, cc);
        eng.allreduce_view(cc);
        eng.gemm(-1.0, s.qk(), cc, 1.0, vv);
    };
    std::int64_t head = 0;
    int term = 1;
    while (true) {
        MatView wv{win.p, m, r, std::max<std::int64_t>(m, 1), false};
        column_sumsq(c.st, c.ws_red, wv, nrm.p);
        c.allreduce(nrm.p, static_cast<std::size_t>(r));
        QB_CUDA(cudaMemcpyAsync(hn.data(), nrm.p, sizeof(double) * r, cudaMemcpyDeviceToHost, c.st));
        QB_CUDA(cudaStreamSynchronize(c.st));
        double mx = 0.0;
        for (std::int64_t i = 0; i < r; ++i) mx = std::max(mx, std::sqrt(hn[i]));
        if (!(mx > thr)) { term = 1; break; }
        if (s.k >= cap) { term = 0; break; }
        // q_j = (I - Q Q^T) y_head, normalised
        double* yh = win.p + head * m;
        QB_CUDA(cudaMemcpyAsync(yv.p, yh, sizeof(double) * m, cudaMemcpyDeviceToDevice, c.st));
        project(yv.p);
        MatView y1{yv.p, m, 1, 1, true};
        column_sumsq(c.st, c.ws_red, MatView{yv.p, m, 1, std::max<std::int64_t>(m, 1), false}, nrm.p + r);
        c.allreduce(nrm.p + r, 1);
        QB_CUDA(cudaMemcpyAsync(hn.data() + r, nrm.p + r, sizeof(double), cudaMemcpyDeviceToHost, c.st));
        QB_CUDA(cudaStreamSynchronize(c.st));
        const double yn = std::sqrt(hn[r]);
        if (!(yn > 0.0)) { term = 3; break; }
        scale_matrix(c.st, y1, 1.0 / yn);
        MatView qj = s.qslot(1);
        copy_matrix(c.st, y1, qj);
        // omega_{j+r}: one pass; then all window samples lose their q_j component
        MatView o1{om.p, n, 1, 1, true};
        gaussian_fill(c.st, c.rng, p.seed, p.stream, g_used, o1);
        g_used += static_cast<std::uint64_t>(n);
        s.k += 1;
        MatView whead{yh, m, 1, 1, true};
        eng.apply(o1, whead);
        a.passes += 1;
        // the new sample is projected against Q (with q_j); the others lose q_j's component
        project(yh);
        for (std::int64_t i = 0; i < r; ++i) {
            if (i == head) continue;
            double* yi = win.p + i * m;
            MatView vi{yi, m, 1, 1, true};
            MatView cc{cv.p, 1, 1, 1, true};
            eng.gemm(1.0, y1.t(), vi, 0.0, cc);
            eng.allreduce_view(cc);
            eng.gemm(-1.0, y1, cc, 1.0, vi);
        }
        head = (head + 1) % r;
    }
    if (s.k > 0) eng.apply_t(s.qk(), s.btk());
    a.passes += 1;
    s.set_e(-1.0);
    auto res = finish(s, a, passes0, term, 0.0);
    res->gaussians_used = static_cast<std::int64_t>(g_used);
    return res;
}

std::unique_ptr<Result> run(Context& c, Matrix& a, const Params& p) {
    Timer t(c.st);
    std::unique_ptr<Result> r;
    switch (p.alg) {
        case 0: r = run_ei(c, a, p); break;
        case 1: case 2: case 3: r = run_fp(c, a, p); break;
        case 4: r = run_qb(c, a, p); break;
        case 5: r = run_qb_b(c, a, p); break;
        case 6: r = run_arf(c, a, p); break;
        default: throw QbError(kError, "unknown algorithm id");
    }
    finish_finite_check(c, a);
    r->device_ms = t.stop();
    return r;
}

}  // namespace qbgpu
