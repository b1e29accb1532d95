// qbfac/qb_gpu.hpp — reference-side C++ binding of the B200 path (header-only).
//
// A maintainer of the reference library adds this header next to its own
// qbfac/qb.hpp (missing from the snapshot; types per SPEC.md:209-220) and links
// libqbfac_gpu.so. The functions keep the reference signatures
// and semantics:
//   * A is read through the reference MatrixHandle (matrix_handle.hpp:41-86):
//     dense() column-major data or sparse() CSR arrays are handed to the C-ABI;
//   * Omega comes from the same RngStream (seed(), stream_id(), rng.hpp:16-42) —
//     the stream must be at its initial position (checked: a stream that has already
//     been drawn from, including a cached Box-Muller half, throws qbfac::Error before
//     any device work); afterwards `rng` is advanced by exactly the draws the
//     reference would have consumed;
//   * the PassCounter of A is advanced by the passes the device made;
//   * status codes are rethrown as the reference exception types (types.hpp).
#pragma once

#include <bit>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "qbfac/dense_matrix.hpp"
#include "qbfac/matrix_handle.hpp"
#include "qbfac/qb.hpp"
#include "qbfac/rng.hpp"
#include "qbfac/types.hpp"
#include "qbfac_gpu.h"

namespace qbfac::gpu {

namespace detail {

inline void raise(int st, const char* msg, const qbfac_info* info) {
    switch (st) {
        case QBFAC_OK: return;
        case QBFAC_DIMENSION_ERROR: throw DimensionError(msg);
        case QBFAC_SINGULARITY_ERROR: throw SingularityError(msg, info ? static_cast<index>(info->diag_index) : 0);
        case QBFAC_TOLERANCE_FLOOR_ERROR: throw ToleranceFloorError(msg, info ? info->floor : 0.0);
        case QBFAC_FORMAT_ERROR: throw FormatError(msg);
        case QBFAC_RESOURCE_ERROR: throw ResourceError(msg);
        default: throw Error(msg);
    }
}

// One context per thread and device (a context is not re-entrant).
inline qbfac_gpu_ctx* context(int device = 0) {
    struct Holder {
        qbfac_gpu_ctx* c = nullptr;
        ~Holder() { if (c) qbfac_gpu_destroy(c); }
    };
    thread_local Holder h;
    if (!h.c) {
        const int st = qbfac_gpu_create(device, &h.c);
        if (st) raise(st, qbfac_gpu_last_error(nullptr), nullptr);
    }
    return h.c;
}

struct MatrixGuard {
    qbfac_gpu_matrix* m = nullptr;
    ~MatrixGuard() { qbfac_gpu_matrix_free(m); }
};
struct ResultGuard {
    qbfac_gpu_result* r = nullptr;
    ~ResultGuard() { qbfac_gpu_result_free(r); }
};

inline void upload(qbfac_gpu_ctx* c, const MatrixHandle& a, MatrixGuard& g) {
    int st;
    if (a.is_sparse()) {
        const SparseCsrMatrix& s = a.sparse();
        st = qbfac_gpu_matrix_csr(c, static_cast<int64_t>(s.rows()), static_cast<int64_t>(s.cols()),
                                  static_cast<int64_t>(s.nnz()), s.row_ptr().data(), s.col_idx().data(),
                                  s.values().data(), &g.m);
    } else {
        const DenseMatrix& d = a.dense();
        st = qbfac_gpu_matrix_dense(c, static_cast<int64_t>(d.rows()), static_cast<int64_t>(d.cols()), d.data(),
                                    static_cast<int64_t>(d.rows() ? d.rows() : 1), &g.m);
    }
    if (st) raise(st, qbfac_gpu_last_error(c), nullptr);
}

// Advance `rng` by `draws` next_gaussian() calls without evaluating the transform:
// a Box-Muller pair consumes two next_u64(); an odd count leaves the sin half cached.
inline void advance(RngStream& rng, std::int64_t draws) {
    for (std::int64_t p = 0; p < draws / 2; ++p) {
        rng.next_u64();
        rng.next_u64();
    }
    if (draws % 2) rng.next_gaussian();
}

// The device regenerates Omega from position 0 of (seed, stream). Compare the next draws of
// a copy of `rng` with those of a fresh RngStream(seed, stream): one next_gaussian() (a
// cached sin half shows here) and one next_u64() (the xoshiro state). Bitwise.
inline void require_fresh(const RngStream& rng) {
    RngStream used = rng;
    RngStream fresh(rng.seed(), rng.stream_id());
    const double g0 = used.next_gaussian(), g1 = fresh.next_gaussian();
    const std::uint64_t u0 = used.next_u64(), u1 = fresh.next_u64();
    if (std::bit_cast<std::uint64_t>(g0) != std::bit_cast<std::uint64_t>(g1) || u0 != u1)
        throw Error("qbfac::gpu: the RngStream has already been drawn from; the device path generates Omega "
                    "from the initial position of (seed, stream) — pass a fresh RngStream");
}

inline QBFactorization run(const MatrixHandle& a, qbfac_params p, RngStream& rng) {
    require_fresh(rng);
    qbfac_gpu_ctx* c = context();
    p.seed = rng.seed();
    p.stream = rng.stream_id();
    MatrixGuard mg;
    upload(c, a, mg);
    ResultGuard rg;
    qbfac_info info{};
    const int st = qbfac_gpu_run(c, mg.m, &p, &rg.r, &info);
    if (st) raise(st, qbfac_gpu_last_error(c), &info);
    const index r = static_cast<index>(info.rank), m = a.rows(), n = a.cols();
    std::vector<double> q(m * r), b(r * n);
    if (r) {
        if (int s2 = qbfac_gpu_result_copy_q(rg.r, q.data(), static_cast<int64_t>(m ? m : 1)))
            raise(s2, qbfac_gpu_last_error(c), nullptr);
        if (int s3 = qbfac_gpu_result_copy_b(rg.r, b.data(), static_cast<int64_t>(r)))
            raise(s3, qbfac_gpu_last_error(c), nullptr);
    }
    QBFactorization f;
    f.Q = DenseMatrix::from_data(m, r, std::move(q));
    f.B = DenseMatrix::from_data(r, n, std::move(b));
    f.error_indicator = info.error_indicator;
    f.passes = info.passes;
    f.terminated_by = static_cast<Termination>(info.terminated_by);
    a.pass_counter().add(info.passes);
    advance(rng, info.gaussians_used);
    return f;
}

}  // namespace detail

// SPEC.md:273-281
inline QBFactorization rand_qb_ei(const MatrixHandle& a, const StopRule& stop, index b, int power, RngStream& rng,
                                  index max_rank = 0) {
    qbfac_params p{};
    p.alg = QBFAC_ALG_EI;
    p.mode = stop.mode == StopRule::Mode::fixed_precision ? 1 : 0;
    p.b = static_cast<int64_t>(b);
    p.power = power;
    p.k = static_cast<int64_t>(stop.k);
    p.s = static_cast<int64_t>(stop.s);
    p.eps_abs = stop.eps;
    p.max_rank = static_cast<int64_t>(max_rank);
    return detail::run(a, p, rng);
}

// SPEC.md:291-299
inline QBFactorization rand_qb_fp(const MatrixHandle& a, double eps_abs, index b, int power, index l_budget,
                                  RngStream& rng, index max_rank = 0, int max_restarts = 8) {
    qbfac_params p{};
    p.alg = QBFAC_ALG_FP;
    p.mode = 1;
    p.b = static_cast<int64_t>(b);
    p.power = power;
    p.l_budget = static_cast<int64_t>(l_budget);
    p.eps_abs = eps_abs;
    p.max_rank = static_cast<int64_t>(max_rank);
    p.max_restarts = max_restarts;
    return detail::run(a, p, rng);
}

// SPEC.md:282-290
inline QBFactorization rand_qb_fp_fixed_rank(const MatrixHandle& a, index k, index s, index b, bool reorth,
                                             RngStream& rng) {
    qbfac_params p{};
    p.alg = QBFAC_ALG_FP_FIXED_RANK;
    p.mode = 0;
    p.b = static_cast<int64_t>(b);
    p.k = static_cast<int64_t>(k);
    p.s = static_cast<int64_t>(s);
    p.reorth = reorth ? 1 : 0;
    return detail::run(a, p, rng);
}

// SPEC.md:300-308 with A resident (one logical pass: G, H and ||A||_F^2 together).
inline QBFactorization single_pass_fp(const MatrixHandle& a, index l, index b, RngStream& rng) {
    qbfac_params p{};
    p.alg = QBFAC_ALG_SINGLE_PASS;
    p.mode = 0;
    p.b = static_cast<int64_t>(b);
    p.k = static_cast<int64_t>(l);
    return detail::run(a, p, rng);
}

}  // namespace qbfac::gpu
