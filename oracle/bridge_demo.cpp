// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Drop-in check of the reference-side binding (include/qbfac/qb_gpu.hpp): the same
// reference MatrixHandle / RngStream objects are factorized by the restated CPU
// algorithm (qbfac::rand_qb_ei / rand_qb_fp) and by qbfac::gpu::rand_qb_ei /
// rand_qb_fp (C-ABI -> libqbfac_gpu.so). Prints one JSON line per case.
#include <cmath>
#include <cstdio>
#include <string>

#include "qb_restated.hpp"
#include "qbfac/kernels.hpp"
#include "qbfac/qb_gpu.hpp"
#include "qbfac/qr.hpp"

using namespace qbfac;

static DenseMatrix synth(index n, double tau, std::uint64_t seed) {
    RngStream r(seed);
    DenseMatrix u = orth_qr(gaussian(n, n, r)).q;
    DenseMatrix v = orth_qr(gaussian(n, n, r)).q;
    for (index j = 0; j < n; ++j) {
        const double s = std::exp(-static_cast<double>(j + 1) / tau);
        for (index i = 0; i < n; ++i) u(i, j) *= s;
    }
    DenseMatrix vt = v.transposed();
    return multiply(u, vt);
}

static void report(const char* name, const MatrixHandle& a, const QBFactorization& c, const QBFactorization& g,
                   long long pc, long long pg, std::uint64_t u_cpu, std::uint64_t u_gpu) {
    const double ec = explicit_error(a, c.Q, c.B), eg = explicit_error(a, g.Q, g.B);
    std::printf("{\"case\": \"%s\", \"rank_cpu\": %zu, \"rank_gpu\": %zu, \"E_cpu\": %.17g, \"E_gpu\": %.17g, "
                "\"err_cpu\": %.17g, \"err_gpu\": %.17g, \"term_cpu\": %d, \"term_gpu\": %d, "
                "\"passes_cpu\": %lld, \"passes_gpu\": %lld, \"rng_next_cpu\": %llu, \"rng_next_gpu\": %llu}\n",
                name, c.Q.cols(), g.Q.cols(), c.error_indicator, g.error_indicator, ec, eg,
                static_cast<int>(c.terminated_by), static_cast<int>(g.terminated_by), pc, pg,
                static_cast<unsigned long long>(u_cpu), static_cast<unsigned long long>(u_gpu));
}

int main() {
    try {
        {
            MatrixHandle a(synth(300, 7.0, 9));
            const double eps = 1e-4 * std::sqrt(a.frob_norm_sq());
            RngStream r1(5), r2(5);
            const long long p0 = a.passes();
            QBFactorization c = rand_qb_ei(a, StopRule::fixed_precision(eps), 10, 1, r1);
            const long long p1 = a.passes();
            QBFactorization g = gpu::rand_qb_ei(a, StopRule::fixed_precision(eps), 10, 1, r2);
            const long long p2 = a.passes();
            report("ei_dense_300", a, c, g, p1 - p0, p2 - p1, r1.next_u64(), r2.next_u64());
        }
        {
            MatrixHandle a(synth(400, 20.0, 3));
            const double eps = 1e-3 * std::sqrt(a.frob_norm_sq());
            RngStream r1(6), r2(6);
            const long long p0 = a.passes();
            QBFactorization c = rand_qb_fp(a, eps, 10, 1, 200, r1);
            const long long p1 = a.passes();
            QBFactorization g = gpu::rand_qb_fp(a, eps, 10, 1, 200, r2);
            const long long p2 = a.passes();
            report("fp_dense_400", a, c, g, p1 - p0, p2 - p1, r1.next_u64(), r2.next_u64());
        }
        {
            std::vector<SparseCsrMatrix::Triplet> t;
            RngStream r(11);
            for (index i = 0; i < 2000; ++i)
                for (int q = 0; q < 8; ++q) t.push_back({i, (i * 37 + q * 211) % 1500, r.next_double()});
            MatrixHandle a(SparseCsrMatrix::from_triplets(2000, 1500, t));
            const double eps = 0.5 * std::sqrt(a.frob_norm_sq());
            RngStream r1(4), r2(4);
            const long long p0 = a.passes();
            QBFactorization c = rand_qb_ei(a, StopRule::fixed_precision(eps), 16, 1, r1, 300);
            const long long p1 = a.passes();
            QBFactorization g = gpu::rand_qb_ei(a, StopRule::fixed_precision(eps), 16, 1, r2, 300);
            const long long p2 = a.passes();
            report("ei_csr_2000x1500", a, c, g, p1 - p0, p2 - p1, r1.next_u64(), r2.next_u64());
        }
        {
            MatrixHandle a(synth(100, 7.0, 1));
            RngStream r2(1);
            try {
                gpu::rand_qb_ei(a, StopRule::fixed_precision(1e-9 * std::sqrt(a.frob_norm_sq())), 10, 0, r2);
                std::printf("{\"case\": \"floor\", \"thrown\": false}\n");
            } catch (const ToleranceFloorError& e) {
                std::printf("{\"case\": \"floor\", \"thrown\": true, \"floor\": %.17g}\n", e.floor_value());
            }
        }
        for (int draws : {1, 2}) {
            // a stream already drawn from (odd count: cached Box-Muller half; even: advanced state)
            MatrixHandle a(synth(100, 7.0, 1));
            RngStream r2(7);
            for (int d = 0; d < draws; ++d) r2.next_gaussian();
            const double eps = 1e-2 * std::sqrt(a.frob_norm_sq());
            const long long p0 = a.passes();
            bool thrown = false;
            try {
                gpu::rand_qb_ei(a, StopRule::fixed_precision(eps), 10, 0, r2);
            } catch (const Error&) {
                thrown = true;
            }
            std::printf("{\"case\": \"consumed_rng_%d\", \"thrown\": %s, \"passes\": %lld}\n", draws,
                        thrown ? "true" : "false", a.passes() - p0);
        }
    } catch (const std::exception& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
        return 1;
    }
    return 0;
}
