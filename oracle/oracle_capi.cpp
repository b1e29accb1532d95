// ORACLE — TEST INFRASTRUCTURE ONLY. Not part of the product path.
//
// extern "C" surface of oracle/_ref/libqbref.so for the Python checker
// (oracle/oracle.py). Links the reference's own translation units, compiled in
// place from /root/reference/proj/src (see oracle/Makefile), and the restated
// algorithm layer (qr_restated.cpp, qb_restated.cpp).
//
// Status codes mirror the product C-ABI (include/qbfac_gpu.h):
//   0 ok, 1 DimensionError, 2 SingularityError, 3 ToleranceFloorError,
//   4 FormatError, 5 ResourceError, 6 Error, 7 other.

#include <cstdint>
#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "qb_restated.hpp"
#include "qbfac/kernels.hpp"
#include "qbfac/qr.hpp"

using namespace qbfac;

extern "C" {

struct qbo_params {
    std::int32_t alg;          // 0 EI, 1 FP, 2 FP fixed rank, 3 single pass, 4 randQB, 5 randQB_b, 6 range finder
    std::int32_t mode;         // 0 fixed_rank, 1 fixed_precision
    std::int64_t b, power, k, s, max_rank, l_budget, max_restarts;
    double eps_abs;
    std::uint64_t seed, stream;
    std::int32_t reorth;
    std::int32_t pad_;
};

struct qbo_result {
    std::int64_t rank;
    double E;
    double norm_a_sq;
    std::int64_t passes;
    std::int32_t terminated_by;
    std::int32_t status;
    std::int64_t diag_index;
    double floor;
    std::int64_t m, n;
    std::int64_t n_trace;
    char msg[256];
    double seconds;  // steady_clock around the rand_qb_* call (matrix wrap excluded)
};

}  // extern "C"

namespace {

struct Handle {
    QBFactorization f;
};

void set_msg(qbo_result* r, const char* m) {
    std::strncpy(r->msg, m, sizeof(r->msg) - 1);
    r->msg[sizeof(r->msg) - 1] = 0;
}

template <class Fn>
int guard(qbo_result* res, Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const DimensionError& e) {
        if (res) set_msg(res, e.what());
        return 1;
    } catch (const SingularityError& e) {
        if (res) { set_msg(res, e.what()); res->diag_index = static_cast<std::int64_t>(e.diag_index()); }
        return 2;
    } catch (const ToleranceFloorError& e) {
        if (res) { set_msg(res, e.what()); res->floor = e.floor_value(); }
        return 3;
    } catch (const FormatError& e) {
        if (res) set_msg(res, e.what());
        return 4;
    } catch (const ResourceError& e) {
        if (res) set_msg(res, e.what());
        return 5;
    } catch (const Error& e) {
        if (res) set_msg(res, e.what());
        return 6;
    } catch (const std::bad_alloc&) {
        if (res) set_msg(res, "out of memory");
        return 5;
    } catch (const std::exception& e) {
        if (res) set_msg(res, e.what());
        return 7;
    }
}

QBFactorization run(const MatrixHandle& a, const qbo_params& p) {
    RngStream rng(p.seed, p.stream);
    switch (p.alg) {
        case 0: {
            StopRule stop = p.mode == 1 ? StopRule::fixed_precision(p.eps_abs)
                                        : StopRule::fixed_rank(p.k, p.s);
            return rand_qb_ei(a, stop, p.b, static_cast<int>(p.power), rng, p.max_rank);
        }
        case 1:
            return rand_qb_fp(a, p.eps_abs, p.b, static_cast<int>(p.power), p.l_budget, rng,
                              p.max_rank, static_cast<int>(p.max_restarts));
        case 2:
            return rand_qb_fp_fixed_rank(a, p.k, p.s, p.b, p.reorth != 0, rng);
        case 3: {
            auto rs = a.row_stream();
            QBFactorization f = single_pass_fp(*rs, p.k + p.s, p.b, rng);
            f.passes = a.passes();
            return f;
        }
        case 4:
            return rand_qb(a, p.k + p.s, static_cast<int>(p.power), rng);
        case 5: {
            StopRule stop = p.mode == 1 ? StopRule::fixed_precision(p.eps_abs)
                                        : StopRule::fixed_rank(p.k, p.s);
            return rand_qb_b(a, stop, p.b, rng);
        }
        case 6:
            return adaptive_range_finder(a, p.eps_abs, p.b, rng, p.max_rank);
        default:
            throw Error("unknown algorithm id");
    }
}

void fill(qbo_result* r, const QBFactorization& f, qbfac::index m, qbfac::index n) {
    r->rank = static_cast<std::int64_t>(f.Q.cols());
    r->E = f.error_indicator;
    r->norm_a_sq = f.norm_a_sq;
    r->passes = f.passes;
    r->terminated_by = static_cast<std::int32_t>(f.terminated_by);
    r->m = static_cast<std::int64_t>(m);
    r->n = static_cast<std::int64_t>(n);
    r->n_trace = static_cast<std::int64_t>(f.e_trace.size());
}

}  // namespace

extern "C" {

const char* qbo_lane_name() { return kernels::active_kernels().name; }

// ---- RNG pins (rng.cpp:28-79) ---------------------------------------------
int qbo_rng_u64(std::uint64_t seed, std::uint64_t stream, std::int64_t count, std::uint64_t* out) {
    RngStream r(seed, stream);
    for (std::int64_t i = 0; i < count; ++i) out[i] = r.next_u64();
    return 0;
}

int qbo_rng_double(std::uint64_t seed, std::uint64_t stream, std::int64_t count, double* out) {
    RngStream r(seed, stream);
    for (std::int64_t i = 0; i < count; ++i) out[i] = r.next_double();
    return 0;
}

// `skip` gaussians are drawn first (one next_gaussian() each), then gaussian(rows, cols).
int qbo_gaussian(std::uint64_t seed, std::uint64_t stream, std::int64_t skip, std::int64_t rows,
                 std::int64_t cols, double* out) {
    return guard(nullptr, [&] {
        RngStream r(seed, stream);
        for (std::int64_t i = 0; i < skip; ++i) r.next_gaussian();
        DenseMatrix g = gaussian(static_cast<qbfac::index>(rows), static_cast<qbfac::index>(cols), r);
        std::memcpy(out, g.data(), sizeof(double) * g.size());
    });
}

int qbo_substream_id(std::uint64_t seed, std::uint64_t stream, std::uint64_t id, std::uint64_t* out_stream) {
    RngStream r(seed, stream);
    *out_stream = r.substream(id).stream_id();
    return 0;
}

// ---- primitives ------------------------------------------------------------
int qbo_orth_qr(std::int64_t m, std::int64_t n, const double* a, double* q, double* r) {
    return guard(nullptr, [&] {
        DenseMatrix x = DenseMatrix::from_data(m, n, std::vector<double>(a, a + m * n));
        QrResult res = orth_qr(x);
        std::memcpy(q, res.q.data(), sizeof(double) * m * n);
        std::memcpy(r, res.r.data(), sizeof(double) * n * n);
    });
}

int qbo_rank_deficiency(std::int64_t n, const double* r, double thr, std::int64_t* out, std::int64_t* count) {
    return guard(nullptr, [&] {
        DenseMatrix x = DenseMatrix::from_data(n, n, std::vector<double>(r, r + n * n));
        auto d = rank_deficiency_report(x, thr);
        *count = static_cast<std::int64_t>(d.size());
        for (std::size_t i = 0; i < d.size(); ++i) out[i] = static_cast<std::int64_t>(d[i]);
    });
}

int qbo_tri_solve_t(std::int64_t b, std::int64_t ncols, const double* r, const double* c,
                    double* x, double thr, std::int64_t* diag_index) {
    qbo_result res{};
    int st = guard(&res, [&] {
        DenseMatrix rr = DenseMatrix::from_data(b, b, std::vector<double>(r, r + b * b));
        DenseMatrix cc = DenseMatrix::from_data(b, ncols, std::vector<double>(c, c + b * ncols));
        DenseMatrix xx = tri_solve_transposed(rr, cc, thr);
        std::memcpy(x, xx.data(), sizeof(double) * b * ncols);
    });
    *diag_index = res.diag_index;
    return st;
}

double qbo_orth_loss(std::int64_t m, std::int64_t n, const double* q) {
    DenseMatrix x = DenseMatrix::from_data(m, n, std::vector<double>(q, q + m * n));
    return orthogonality_loss(x);
}

int qbo_validate_epsilon(double eps, double frob_a, double delta, double* floor_out) {
    EpsilonCheck c = validate_epsilon(eps, frob_a, delta);
    *floor_out = c.floor;
    return c.valid ? 1 : 0;
}

// Reference dense / CSR products through MatrixHandle::multiply (matrix_handle.cpp:112-116).
int qbo_dense_multiply(std::int64_t m, std::int64_t n, const double* a, std::int64_t w,
                       const double* x, int trans, double* y) {
    return guard(nullptr, [&] {
        MatrixHandle h(DenseMatrix::from_data(m, n, std::vector<double>(a, a + m * n)));
        const qbfac::index xr = trans ? m : n;
        DenseMatrix xx = DenseMatrix::from_data(xr, w, std::vector<double>(x, x + xr * w));
        DenseMatrix yy = h.multiply(xx, trans != 0);
        std::memcpy(y, yy.data(), sizeof(double) * yy.size());
    });
}

int qbo_csr_multiply(std::int64_t m, std::int64_t n, std::int64_t nnz, const std::int64_t* rp,
                     const std::int32_t* ci, const double* v, std::int64_t w, const double* x,
                     int trans, double* y) {
    return guard(nullptr, [&] {
        MatrixHandle h(SparseCsrMatrix::from_parts(
            m, n, std::vector<std::int64_t>(rp, rp + m + 1), std::vector<std::int32_t>(ci, ci + nnz),
            std::vector<double>(v, v + nnz)));
        const qbfac::index xr = trans ? m : n;
        DenseMatrix xx = DenseMatrix::from_data(xr, w, std::vector<double>(x, x + xr * w));
        DenseMatrix yy = h.multiply(xx, trans != 0);
        std::memcpy(y, yy.data(), sizeof(double) * yy.size());
    });
}

double qbo_csr_frob_sq(std::int64_t m, std::int64_t n, std::int64_t nnz, const std::int64_t* rp,
                       const std::int32_t* ci, const double* v) {
    MatrixHandle h(SparseCsrMatrix::from_parts(
        m, n, std::vector<std::int64_t>(rp, rp + m + 1), std::vector<std::int32_t>(ci, ci + nnz),
        std::vector<double>(v, v + nnz)));
    return h.frob_norm_sq();
}

// Validation only (sparse_csr.cpp:10-40); returns the status code of from_parts.
int qbo_csr_validate(std::int64_t m, std::int64_t n, std::int64_t nnz, const std::int64_t* rp,
                     const std::int32_t* ci, const double* v, std::int64_t rp_len) {
    qbo_result res{};
    return guard(&res, [&] {
        SparseCsrMatrix::from_parts(m, n, std::vector<std::int64_t>(rp, rp + rp_len),
                                    std::vector<std::int32_t>(ci, ci + nnz),
                                    std::vector<double>(v, v + nnz));
    });
}

// SparseCsrMatrix::from_triplets (sparse_csr.cpp:42-64): sort by (row, col), reject duplicates
// and out-of-range coordinates, then from_parts validation. Outputs the CSR arrays.
int qbo_csr_from_triplets(std::int64_t m, std::int64_t n, std::int64_t nt, const std::int64_t* rows,
                          const std::int64_t* cols, const double* vals, std::int64_t* rp, std::int32_t* ci,
                          double* v) {
    qbo_result res{};
    return guard(&res, [&] {
        std::vector<SparseCsrMatrix::Triplet> t(static_cast<std::size_t>(nt));
        for (std::int64_t i = 0; i < nt; ++i)
            t[i] = SparseCsrMatrix::Triplet{static_cast<qbfac::index>(rows[i]), static_cast<qbfac::index>(cols[i]),
                                            vals[i]};
        SparseCsrMatrix a = SparseCsrMatrix::from_triplets(m, n, std::move(t));
        std::memcpy(rp, a.row_ptr().data(), sizeof(std::int64_t) * (m + 1));
        std::memcpy(ci, a.col_idx().data(), sizeof(std::int32_t) * a.nnz());
        std::memcpy(v, a.values().data(), sizeof(double) * a.nnz());
    });
}

// ---- algorithms --------------------------------------------------------------
void* qbo_run_dense(std::int64_t m, std::int64_t n, const double* a, const qbo_params* p,
                    qbo_result* res) {
    std::memset(res, 0, sizeof(*res));
    Handle* h = nullptr;
    res->status = guard(res, [&] {
        MatrixHandle mh(DenseMatrix::from_data(m, n, std::vector<double>(a, a + m * n)));
        auto hh = std::make_unique<Handle>();
        const auto t0 = std::chrono::steady_clock::now();
        hh->f = run(mh, *p);
        res->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        fill(res, hh->f, m, n);
        h = hh.release();
    });
    return h;
}

void* qbo_run_csr(std::int64_t m, std::int64_t n, std::int64_t nnz, const std::int64_t* rp,
                  const std::int32_t* ci, const double* v, const qbo_params* p, qbo_result* res) {
    std::memset(res, 0, sizeof(*res));
    Handle* h = nullptr;
    res->status = guard(res, [&] {
        MatrixHandle mh(SparseCsrMatrix::from_parts(
            m, n, std::vector<std::int64_t>(rp, rp + m + 1), std::vector<std::int32_t>(ci, ci + nnz),
            std::vector<double>(v, v + nnz)));
        auto hh = std::make_unique<Handle>();
        const auto t0 = std::chrono::steady_clock::now();
        hh->f = run(mh, *p);
        res->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        fill(res, hh->f, m, n);
        h = hh.release();
    });
    return h;
}

int qbo_copy_q(void* h, double* out) {
    auto* hh = static_cast<Handle*>(h);
    std::memcpy(out, hh->f.Q.data(), sizeof(double) * hh->f.Q.size());
    return 0;
}

int qbo_copy_b(void* h, double* out) {
    auto* hh = static_cast<Handle*>(h);
    std::memcpy(out, hh->f.B.data(), sizeof(double) * hh->f.B.size());
    return 0;
}

int qbo_copy_trace(void* h, double* out) {
    auto* hh = static_cast<Handle*>(h);
    std::memcpy(out, hh->f.e_trace.data(), sizeof(double) * hh->f.e_trace.size());
    return 0;
}

void qbo_free(void* h) { delete static_cast<Handle*>(h); }

double qbo_explicit_error_dense(std::int64_t m, std::int64_t n, const double* a, std::int64_t k,
                                const double* q, const double* b) {
    MatrixHandle mh(DenseMatrix::from_data(m, n, std::vector<double>(a, a + m * n)));
    DenseMatrix qq = DenseMatrix::from_data(m, k, std::vector<double>(q, q + m * k));
    DenseMatrix bb = DenseMatrix::from_data(k, n, std::vector<double>(b, b + k * n));
    return explicit_error(mh, qq, bb);
}

double qbo_explicit_error_csr(std::int64_t m, std::int64_t n, std::int64_t nnz, const std::int64_t* rp,
                              const std::int32_t* ci, const double* v, std::int64_t k,
                              const double* q, const double* b) {
    MatrixHandle mh(SparseCsrMatrix::from_parts(
        m, n, std::vector<std::int64_t>(rp, rp + m + 1), std::vector<std::int32_t>(ci, ci + nnz),
        std::vector<double>(v, v + nnz)));
    DenseMatrix qq = DenseMatrix::from_data(m, k, std::vector<double>(q, q + m * k));
    DenseMatrix bb = DenseMatrix::from_data(k, n, std::vector<double>(b, b + k * n));
    return explicit_error(mh, qq, bb);
}

}  // extern "C"
