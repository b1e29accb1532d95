// ORACLE — TEST INFRASTRUCTURE ONLY. Not part of the product path.
//
// CPU restatement of the reference's missing `src/qr.cpp` (declared in
// /root/reference/proj/include/qbfac/qr.hpp:10-29, contract in SPEC.md:55-108).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
// the library this file is built into (oracle/_ref/libqbref.so).
//
// The inner loops call the reference's own SIMD lane (kernels::active_kernels(),
// proj/src/kernels_dispatch.cpp:38-50) so the arithmetic is the reference's.

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "qbfac/kernels.hpp"
#include "qbfac/qr.hpp"

namespace qbfac {

// Economic Householder QR with diag(R) >= 0 (qr.hpp:15-18).
// Unblocked LAPACK-style reflectors (beta = -sign(alpha)*||x||), Q formed by
// backward accumulation (dorg2r order), then the sign post-pass that makes the
// factorization unique.
QrResult orth_qr(const DenseMatrix& mtx) {
    const index m = mtx.rows(), n = mtx.cols();
    if (m < n) throw DimensionError("orth_qr: rows < cols");
    const auto& k = kernels::active_kernels();
    DenseMatrix w = mtx;  // reflectors stored below the diagonal, R above
    std::vector<double> tau(n, 0.0), rdiag(n, 0.0);
    for (index j = 0; j < n; ++j) {
        double* x = w.col(j) + j;
        const index len = m - j;
        const double alpha = x[0];
        const double sigma = len > 1 ? k.sum_sq(x + 1, len - 1) : 0.0;
        if (sigma == 0.0) {
            tau[j] = 0.0;
            rdiag[j] = alpha;
            x[0] = 1.0;
        } else {
            const double norm = std::sqrt(alpha * alpha + sigma);
            const double beta = alpha >= 0.0 ? -norm : norm;
            tau[j] = (beta - alpha) / beta;
            k.scal(1.0 / (alpha - beta), x + 1, len - 1);
            x[0] = 1.0;
            rdiag[j] = beta;
        }
        if (tau[j] != 0.0) {
            for (index c = j + 1; c < n; ++c) {
                double* y = w.col(c) + j;
                const double d = k.dot(x, y, len);
                k.axpy(-tau[j] * d, x, y, len);
            }
        }
    }
    DenseMatrix r(n, n);
    for (index c = 0; c < n; ++c) {
        for (index i = 0; i < c; ++i) r(i, c) = w(i, c);
        r(c, c) = rdiag[c];
    }
    DenseMatrix q(m, n);
    for (index i = 0; i < n; ++i) q(i, i) = 1.0;
    for (index jj = n; jj-- > 0;) {
        if (tau[jj] == 0.0) continue;
        const double* v = w.col(jj) + jj;  // v[0] == 1
        const index len = m - jj;
        for (index c = jj; c < n; ++c) {
            double* y = q.col(c) + jj;
            const double d = k.dot(v, y, len);
            k.axpy(-tau[jj] * d, v, y, len);
        }
    }
    for (index j = 0; j < n; ++j) {
        if (r(j, j) < 0.0) {
            for (index c = j; c < n; ++c) r(j, c) = -r(j, c);
            k.scal(-1.0, q.col(j), m);
        }
    }
    return QrResult{std::move(q), std::move(r)};
}

// qr.hpp:20-21.
std::vector<index> rank_deficiency_report(const DenseMatrix& r, double threshold) {
    const index n = std::min(r.rows(), r.cols());
    double mx = 0.0;
    for (index j = 0; j < n; ++j) mx = std::max(mx, std::fabs(r(j, j)));
    std::vector<index> out;
    for (index j = 0; j < n; ++j)
        if (std::fabs(r(j, j)) <= threshold * mx) out.push_back(j);
    return out;
}

// qr.hpp:23-26: R^T X = C by forward substitution, column by column.
DenseMatrix tri_solve_transposed(const DenseMatrix& r, const DenseMatrix& c, double threshold) {
    const index b = r.rows();
    if (r.cols() != b || c.rows() != b) throw DimensionError("tri_solve_transposed: shape");
    double mx = 0.0;
    for (index j = 0; j < b; ++j) mx = std::max(mx, std::fabs(r(j, j)));
    for (index j = 0; j < b; ++j)
        if (std::fabs(r(j, j)) <= threshold * mx)
            throw SingularityError("tri_solve_transposed: singular diagonal at index " +
                                       std::to_string(j), j);
    const auto& k = kernels::active_kernels();
    DenseMatrix x = c;
    for (index col = 0; col < c.cols(); ++col) {
        double* xc = x.col(col);
        for (index i = 0; i < b; ++i) {
            const double s = i > 0 ? k.dot(r.col(i), xc, i) : 0.0;
            xc[i] = (xc[i] - s) / r(i, i);
        }
    }
    return x;
}

// qr.hpp:28-29: ||Q^T Q - I||_inf.
double orthogonality_loss(const DenseMatrix& q) {
    DenseMatrix g = multiply_at_b(q, q);
    double worst = 0.0;
    for (index i = 0; i < g.rows(); ++i) {
        double s = 0.0;
        for (index j = 0; j < g.cols(); ++j) s += std::fabs(g(i, j) - (i == j ? 1.0 : 0.0));
        worst = std::max(worst, s);
    }
    return worst;
}

}  // namespace qbfac
