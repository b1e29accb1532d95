// ORACLE — TEST INFRASTRUCTURE ONLY. Not part of the product path.
//
// CPU restatement of the reference's missing `src/qb.cpp`
// (/root/reference/proj/CMakeLists.txt:26). The algorithms follow
//   Alg. 2 randQB_EI
//   row-by-row truncation      PAPER.md:206-220 (steps 7a-8e)
//   Alg. 3 / steps 9a-9c
//   Alg. 4 randQB_FP
//   single pass (Remark 4.2)
//   contracts and decisions
// on top of the reference's own operator layer (MatrixHandle::multiply etc.,
// proj/src/matrix_handle.cpp:104-132), dense products (dense_matrix.cpp:68-92)
// and RNG (rng.cpp:72-79), so pass arithmetic and Omega are the reference's.
//
// Interpretation decisions (mirrored by the GPU path and
// recorded in DESIGN.md):
//  * EI power iteration: deflate at every application,
//      Y = A W - Q (B W),  Z = A^T W - B^T (Q^T W),  orth between applications.
//  * RNG: EI draws gaussian(n, b_i) per block from `rng`; FP draws gaussian(n, l)
//    once from `rng`, restart r >= 1 draws from rng.substream(r).
//  * Rank collapse: if a QR of the block reports deficient diagonals
//    (rank_deficiency_report, threshold 1e-12) the block keeps its leading
//    columns before the first deficient index, its rows enter B and E as usual,
//    and the run ends with rank_collapse (unless the tolerance was met first).
//  * B is kept transposed (B^T, n x k) so blocks append as columns.

#include "qb_restated.hpp"

#include <algorithm>
#include <cmath>
#include <string>

#include "qbfac/kernels.hpp"
#include "qbfac/qr.hpp"

namespace qbfac {

namespace {

constexpr double kRankTol = 1e-12;

struct QBState {
    DenseMatrix q;   // m x k
    DenseMatrix bt;  // n x k  (B^T)
    index k = 0;
    double e = 0.0;
    std::vector<double> trace;

    QBState(index m, index n) : q(m, 0), bt(n, 0) {}

    // Alg. 1 steps 5-8 with the row-by-row refinement 7a-8e.
    // Returns true when E < eps^2 was reached inside this block.
    bool append(DenseMatrix qi, DenseMatrix bti, bool check_tol, double eps2) {
        const auto& kt = kernels::active_kernels();
        index keep = bti.cols();
        bool met = false;
        for (index j = 0; j < bti.cols(); ++j) {
            e -= kt.sum_sq(bti.col(j), bti.rows());
            if (check_tol && e < eps2) {
                keep = j + 1;
                met = true;
                break;
            }
        }
        if (keep < qi.cols()) {
            qi.truncate_columns(keep);
            bti.truncate_columns(keep);
        }
        q.append_columns(qi);
        bt.append_columns(bti);
        k += keep;
        trace.push_back(e);
        return met;
    }

    // (A - QB) X = A X - Q (B X), B X = (B^T)^T X.
    DenseMatrix apply(const MatrixHandle& a, const DenseMatrix& x) const {
        DenseMatrix y = a.multiply(x, false);
        if (k > 0) {
            DenseMatrix m = multiply_at_b(bt, x);
            multiply_acc(y, q, m, -1.0);
        }
        return y;
    }

    // (A - QB)^T W = A^T W - B^T (Q^T W).
    DenseMatrix apply_t(const MatrixHandle& a, const DenseMatrix& w) const {
        DenseMatrix z = a.multiply(w, true);
        if (k > 0) {
            DenseMatrix m = multiply_at_b(q, w);
            multiply_acc(z, bt, m, -1.0);
        }
        return z;
    }

    // Block Gram-Schmidt re-orthogonalisation Q_i - Q (Q^T Q_i) (Alg. 2 step 6).
    void project_out(DenseMatrix& qi) const {
        if (k == 0) return;
        DenseMatrix m = multiply_at_b(q, qi);
        multiply_acc(qi, q, m, -1.0);
    }
};

index leading_rank(const DenseMatrix& r) {
    auto d = rank_deficiency_report(r, kRankTol);
    return d.empty() ? r.cols() : d.front();
}

DenseMatrix leading_block(const DenseMatrix& r, index d) {
    DenseMatrix out(d, d);
    for (index j = 0; j < d; ++j)
        for (index i = 0; i <= j; ++i) out(i, j) = r(i, j);
    return out;
}

DenseMatrix upper_mul(const DenseMatrix& a, const DenseMatrix& b) {
    // product of two upper-triangular d x d matrices
    const index d = a.rows();
    DenseMatrix c(d, d);
    for (index j = 0; j < d; ++j)
        for (index i = 0; i <= j; ++i) {
            double s = 0.0;
            for (index p = i; p <= j; ++p) s += a(i, p) * b(p, j);
            c(i, j) = s;
        }
    return c;
}

QBFactorization finish(QBState& st, const MatrixHandle* a, std::int64_t passes0,
                       Termination t, double norm_a_sq) {
    QBFactorization f;
    f.Q = std::move(st.q);
    f.B = st.bt.transposed();
    f.error_indicator = st.e;
    f.passes = a ? a->passes() - passes0 : 0;
    f.terminated_by = t;
    f.norm_a_sq = norm_a_sq;
    f.e_trace = std::move(st.trace);
    return f;
}

void check_eps(double eps, double norm_a_sq) {
    EpsilonCheck c = validate_epsilon(eps, std::sqrt(norm_a_sq), 0.01);
    if (!c.valid)
        throw ToleranceFloorError("epsilon below the Theorem 3 floor " + std::to_string(c.floor),
                                  c.floor);
}

// One block of Alg. 3 with optional steps 9a-9c. `yi` is the deflated sketch
// G_I - Q (B Omega_i), `m1` = B Omega_i (k x bi, empty when k == 0).
// Returns the number of rows produced (leading rank); 0 on immediate collapse.
index fp_block(QBState& st, const DenseMatrix& yi, const DenseMatrix& hi, const DenseMatrix& m1,
               bool reorth, DenseMatrix& qi_out, DenseMatrix& bti_out) {
    QrResult qr1 = orth_qr(yi);
    index d = leading_rank(qr1.r);
    if (d == 0) return 0;
    DenseMatrix qi = qr1.q.leading_columns(d);
    DenseMatrix r = leading_block(qr1.r, d);
    if (reorth && st.k > 0) {
        st.project_out(qi);                       // step 9a
        QrResult qr2 = orth_qr(qi);
        index d2 = leading_rank(qr2.r);
        if (d2 == 0) return 0;
        r = upper_mul(qr2.r, r);                  // step 9b
        if (d2 < d) {
            r = leading_block(r, d2);
            d = d2;
        }
        qi = qr2.q.leading_columns(d);
    }
    // step 9c: C^T = H_i - B^T (Q^T Y_i + B Omega_i)   (n x d)
    DenseMatrix ct = hi.leading_columns(d);
    if (st.k > 0) {
        DenseMatrix ylead = yi.leading_columns(d);
        DenseMatrix m = multiply_at_b(st.q, ylead);
        if (reorth) {
            for (index j = 0; j < d; ++j)
                for (index i = 0; i < st.k; ++i) m(i, j) += m1(i, j);
        } else {
            // Alg. 3 step 9 (no re-orth): C = H_i^T - Omega_i^T B^T B.
            for (index j = 0; j < d; ++j)
                for (index i = 0; i < st.k; ++i) m(i, j) = m1(i, j);
        }
        multiply_acc(ct, st.bt, m, -1.0);
    }
    DenseMatrix x = tri_solve_transposed(r, ct.transposed(), kRankTol);  // R^T X = C
    qi_out = std::move(qi);
    bti_out = x.transposed();
    return d;
}

}  // namespace

// ---- baselines ----------------------------------------------------------------------
namespace {
// orth with the reference's deficiency rule: leading columns before the first |R_jj| <=
// 1e-12 max|R_jj| (qr.hpp:20-21); `collapsed` is set when columns were dropped.
DenseMatrix orth_leading(const DenseMatrix& y, bool& collapsed) {
    QrResult qr = orth_qr(y);
    const index d = leading_rank(qr.r);
    if (d < y.cols()) collapsed = true;
    return qr.q.leading_columns(d);
}
}  // namespace

QBFactorization rand_qb(const MatrixHandle& a, index l, int power, RngStream& rng) {
    const index m = a.rows(), n = a.cols();
    if (l == 0 || l > std::min(m, n)) throw DimensionError("rand_qb: l must be in [1, min(m, n)]");
    const std::int64_t p0 = a.passes();
    bool collapsed = false;
    DenseMatrix omega = gaussian(n, l, rng);
    DenseMatrix q = orth_leading(a.multiply(omega, false), collapsed);
    for (int p = 0; p < power; ++p) {
        DenseMatrix w = orth_leading(a.multiply(q, true), collapsed);
        q = orth_leading(a.multiply(w, false), collapsed);
    }
    DenseMatrix bt = a.multiply(q, true);
    QBState st(m, n);
    st.q = std::move(q);
    st.bt = std::move(bt);
    st.k = st.q.cols();
    st.e = -1.0;  // SPEC.md:212 sentinel: randQB keeps no error indicator
    return finish(st, &a, p0, collapsed ? Termination::rank_collapse : Termination::rank_reached, 0.0);
}

QBFactorization rand_qb_b(const MatrixHandle& a, const StopRule& stop, index b, RngStream& rng) {
    if (b == 0) throw DimensionError("rand_qb_b: block size must be >= 1");
    if (a.is_sparse()) throw DimensionError("rand_qb_b: dense A only (the residual is dense)");
    const index m = a.rows(), n = a.cols();
    const std::int64_t p0 = a.passes();
    const bool fixed_prec = stop.mode == StopRule::Mode::fixed_precision;
    const index cap = fixed_prec ? std::min(m, n) : std::min(std::min(m, n), stop.k + stop.s);
    const double eps2 = stop.eps * stop.eps;
    DenseMatrix res = a.dense();  // explicit residual R = A - Q B
    QBState st(m, n);
    double norm_a_sq = 0.0;
    Termination term = Termination::rank_reached;
    while (true) {
        if (st.k >= cap) { term = Termination::rank_reached; break; }
        st.e = frob_norm_sq(res);                       // ||R||_F^2 (one pass over R)
        a.pass_counter().add(1);
        if (st.k == 0) {
            norm_a_sq = st.e;
            if (fixed_prec) check_eps(stop.eps, norm_a_sq);
        }
        if (fixed_prec && st.e < eps2) { term = Termination::tolerance_met; break; }
        const index bi = std::min(b, cap - st.k);
        DenseMatrix omega = gaussian(n, bi, rng);
        DenseMatrix y = multiply(res, omega);           // R Omega_i
        a.pass_counter().add(1);
        QrResult qr1 = orth_qr(y);
        index d = leading_rank(qr1.r);
        if (d == 0) { term = Termination::rank_collapse; break; }
        DenseMatrix qi = qr1.q.leading_columns(d);
        if (st.k > 0) {                                  // re-orthogonalisation against Q
            st.project_out(qi);
            QrResult qr2 = orth_qr(qi);
            const index d2 = leading_rank(qr2.r);
            if (d2 == 0) { term = Termination::rank_collapse; break; }
            d = std::min(d, d2);
            qi = qr2.q.leading_columns(d);
        }
        DenseMatrix bti = multiply_at_b(res, qi);       // B_i^T = R^T Q_i
        a.pass_counter().add(1);
        const index k0 = st.k;
        const bool met = st.append(qi, bti, fixed_prec, eps2);
        const index kept = st.k - k0;
        DenseMatrix qk = st.q.column_range(k0, st.k), bk = st.bt.column_range(k0, st.k);
        multiply_acc(res, qk, bk.transposed(), -1.0);   // R -= Q_i B_i
        a.pass_counter().add(1);
        if (met) { term = Termination::tolerance_met; break; }
        if (kept < bi) { term = Termination::rank_collapse; break; }
    }
    st.trace.clear();
    return finish(st, &a, p0, term, norm_a_sq);
}

QBFactorization adaptive_range_finder(const MatrixHandle& a, double tol_spectral, index r, RngStream& rng,
                                      index max_rank) {
    if (r == 0) throw DimensionError("adaptive_range_finder: r must be >= 1");
    const index m = a.rows(), n = a.cols();
    const std::int64_t p0 = a.passes();
    index cap = std::min(m, n);
    if (max_rank > 0) cap = std::min(cap, max_rank);
    const double thr = tol_spectral / (10.0 * std::sqrt(2.0 / 3.14159265358979323846));
    const auto& kt = kernels::active_kernels();
    auto nrm = [&](const DenseMatrix& v) { return std::sqrt(kt.sum_sq(v.data(), v.rows())); };
    QBState st(m, n);
    // y_1..y_r = A omega_i (r passes)
    std::vector<DenseMatrix> ys;
    {
        DenseMatrix om = gaussian(n, r, rng);
        for (index i = 0; i < r; ++i) ys.push_back(a.multiply(om.column_range(i, i + 1), false));
    }
    auto project = [&](DenseMatrix& v) {  // v - Q (Q^T v)
        if (st.k == 0) return;
        DenseMatrix c = multiply_at_b(st.q, v);
        multiply_acc(v, st.q, c, -1.0);
    };
    index head = 0;  // ys[head .. head + r) is the current window
    Termination term = Termination::tolerance_met;
    while (true) {
        double mx = 0.0;
        for (index i = 0; i < r; ++i) mx = std::max(mx, nrm(ys[head + i]));
        if (!(mx > thr)) { term = Termination::tolerance_met; break; }
        if (st.k >= cap) { term = Termination::rank_reached; break; }
        DenseMatrix y = ys[head];
        project(y);                                      // y_j = (I - Q Q^T) y_j
        const double yn = nrm(y);
        if (!(yn > 0.0)) { term = Termination::rank_collapse; break; }
        for (index i = 0; i < m; ++i) y(i, 0) /= yn;    // q_j
        st.q.append_columns(y);
        st.k += 1;
        DenseMatrix om = gaussian(n, 1, rng);            // omega_{j+r}
        DenseMatrix ynew = a.multiply(om, false);        // one pass
        project(ynew);
        for (index i = 1; i < r; ++i) {                  // y_i -= q_j (q_j^T y_i)
            DenseMatrix& v = ys[head + i];
            double c = 0.0;
            for (index t = 0; t < m; ++t) c += y(t, 0) * v(t, 0);
            for (index t = 0; t < m; ++t) v(t, 0) -= c * y(t, 0);
        }
        ys.push_back(std::move(ynew));
        ++head;
    }
    st.bt = a.multiply(st.q, true);                      // B = Q^T A (one pass)
    st.e = -1.0;
    return finish(st, &a, p0, term, 0.0);
}

EpsilonCheck validate_epsilon(double eps, double frob_a, double delta) {
    const double floor = std::sqrt(4.0 * kEpsMach / delta) * frob_a;
    return {eps > floor, floor};
}

QBFactorization rand_qb_ei(const MatrixHandle& a, const StopRule& stop, index b, int power,
                           RngStream& rng, index max_rank) {
    if (b == 0) throw DimensionError("rand_qb_ei: block size must be >= 1");
    const index m = a.rows(), n = a.cols();
    const std::int64_t p0 = a.passes();
    const bool fixed_prec = stop.mode == StopRule::Mode::fixed_precision;
    index cap = std::min(m, n);
    if (fixed_prec) {
        if (max_rank > 0) cap = std::min(cap, max_rank);
    } else {
        cap = std::min(cap, stop.k + stop.s);
    }
    QBState st(m, n);
    const double norm_a_sq = a.frob_norm_sq();  // Alg. 2 step 2 (+1 pass)
    st.e = norm_a_sq;
    const double eps2 = stop.eps * stop.eps;
    if (fixed_prec) {
        check_eps(stop.eps, norm_a_sq);
        if (st.e < eps2) return finish(st, &a, p0, Termination::tolerance_met, norm_a_sq);
    }
    Termination term = Termination::rank_reached;
    while (true) {
        if (st.k >= cap) {
            term = Termination::rank_reached;
            break;
        }
        const index bi = std::min(b, cap - st.k);
        DenseMatrix omega = gaussian(n, bi, rng);         // step 4
        DenseMatrix y = st.apply(a, omega);               // step 5 (A Omega_i - Q (B Omega_i))
        for (int p = 0; p < power; ++p) {
            DenseMatrix w = orth_qr(y).q;
            DenseMatrix z = st.apply_t(a, w);
            DenseMatrix zq = orth_qr(z).q;
            y = st.apply(a, zq);
        }
        QrResult qr1 = orth_qr(y);
        index d = leading_rank(qr1.r);
        if (d == 0) {
            term = Termination::rank_collapse;
            break;
        }
        DenseMatrix qi = qr1.q.leading_columns(d);
        if (st.k > 0) {                                   // step 6 re-orthogonalisation
            st.project_out(qi);
            QrResult qr2 = orth_qr(qi);
            index d2 = leading_rank(qr2.r);
            if (d2 == 0) {
                term = Termination::rank_collapse;
                break;
            }
            d = std::min(d, d2);
            qi = qr2.q.leading_columns(d);
        }
        DenseMatrix bti = a.multiply(qi, true);           // step 7: B_i^T = A^T Q_i
        if (st.append(std::move(qi), std::move(bti), fixed_prec, eps2)) {
            term = Termination::tolerance_met;
            break;
        }
        if (d < bi) {
            term = Termination::rank_collapse;
            break;
        }
    }
    return finish(st, &a, p0, term, norm_a_sq);
}

QBFactorization rand_qb_fp(const MatrixHandle& a, double eps_abs, index b, int power,
                           index l_budget, RngStream& rng, index max_rank, int max_restarts) {
    if (b == 0) throw DimensionError("rand_qb_fp: block size must be >= 1");
    if (l_budget < b) throw DimensionError("rand_qb_fp: l_budget must be >= b");
    const index m = a.rows(), n = a.cols();
    const std::int64_t p0 = a.passes();
    index cap = std::min(m, n);
    if (max_rank > 0) cap = std::min(cap, max_rank);
    const double eps2 = eps_abs * eps_abs;
    QBState st(m, n);
    double norm_a_sq = 0.0;
    Termination term = Termination::sketch_exhausted;
    for (int restart = 0;; ++restart) {
        if (st.k >= cap) {
            term = Termination::rank_reached;
            break;
        }
        if (restart > max_restarts) {
            term = Termination::sketch_exhausted;
            break;
        }
        const index l = std::min(l_budget, cap - st.k);
        RngStream sub = restart == 0 ? rng : rng.substream(static_cast<std::uint64_t>(restart));
        RngStream& r = restart == 0 ? rng : sub;
        DenseMatrix omega = gaussian(n, l, r);                     // step 2
        for (int p = 0; p < power; ++p) {                          // steps 3-6
            DenseMatrix g = orth_qr(a.multiply(omega, false)).q;
            omega = orth_qr(a.multiply(g, true)).q;
        }
        DenseMatrix g;
        if (restart == 0) {                                        // steps 7 + 9
            g = a.multiply_with_norm(omega, false, norm_a_sq);
            st.e = norm_a_sq;
            check_eps(eps_abs, norm_a_sq);
            if (st.e < eps2) {
                term = Termination::tolerance_met;
                break;
            }
        } else {
            g = a.multiply(omega, false);
        }
        DenseMatrix h = a.multiply(g, true);                       // step 8
        bool stop = false;
        for (index off = 0; off < l; off += b) {                   // steps 10-21
            const index bi = std::min(b, l - off);
            DenseMatrix om_i = omega.column_range(off, off + bi);
            DenseMatrix yi = g.column_range(off, off + bi);
            DenseMatrix hi = h.column_range(off, off + bi);
            DenseMatrix m1;
            if (st.k > 0) {
                m1 = multiply_at_b(st.bt, om_i);                   // B Omega_i
                multiply_acc(yi, st.q, m1, -1.0);                  // step 12
            }
            DenseMatrix qi, bti;
            const index d = fp_block(st, yi, hi, m1, true, qi, bti);
            if (d == 0) {
                term = Termination::rank_collapse;
                stop = true;
                break;
            }
            if (st.append(std::move(qi), std::move(bti), true, eps2)) {
                term = Termination::tolerance_met;
                stop = true;
                break;
            }
            if (d < bi) {
                term = Termination::rank_collapse;
                stop = true;
                break;
            }
        }
        if (stop) break;
    }
    return finish(st, &a, p0, term, norm_a_sq);
}

QBFactorization rand_qb_fp_fixed_rank(const MatrixHandle& a, index k, index s, index b,
                                      bool reorth, RngStream& rng) {
    if (b == 0) throw DimensionError("rand_qb_fp_fixed_rank: block size must be >= 1");
    const index m = a.rows(), n = a.cols();
    const index l = k + s;
    if (l == 0 || l > std::min(m, n)) throw DimensionError("rand_qb_fp_fixed_rank: bad l");
    const std::int64_t p0 = a.passes();
    QBState st(m, n);
    DenseMatrix omega = gaussian(n, l, rng);
    double norm_a_sq = 0.0;
    DenseMatrix g = a.multiply_with_norm(omega, false, norm_a_sq);
    st.e = norm_a_sq;
    DenseMatrix h = a.multiply(g, true);
    Termination term = Termination::rank_reached;
    for (index off = 0; off < l; off += b) {
        const index bi = std::min(b, l - off);
        DenseMatrix om_i = omega.column_range(off, off + bi);
        DenseMatrix yi = g.column_range(off, off + bi);
        DenseMatrix hi = h.column_range(off, off + bi);
        DenseMatrix m1;
        if (st.k > 0) {
            m1 = multiply_at_b(st.bt, om_i);
            multiply_acc(yi, st.q, m1, -1.0);
        }
        DenseMatrix qi, bti;
        const index d = fp_block(st, yi, hi, m1, reorth, qi, bti);
        if (d == 0) {
            term = Termination::rank_collapse;
            break;
        }
        st.append(std::move(qi), std::move(bti), false, 0.0);
        if (d < bi) {
            term = Termination::rank_collapse;
            break;
        }
    }
    return finish(st, &a, p0, term, norm_a_sq);
}

QBFactorization single_pass_fp(RowStream& stream, index l, index b, RngStream& rng) {
    if (b == 0) throw DimensionError("single_pass_fp: block size must be >= 1");
    const index m = stream.rows(), n = stream.cols();
    if (l == 0 || l > std::min(m, n)) throw DimensionError("single_pass_fp: bad l");
    const auto& kt = kernels::active_kernels();
    DenseMatrix omega = gaussian(n, l, rng);
    DenseMatrix g(m, l), h(n, l);
    std::vector<double> row(n);
    double norm_a_sq = 0.0;
    for (index i = 0; i < m; ++i) {                 // the one pass (matrix_handle.cpp:45-50, 66-73)
        stream.next_row(row);
        norm_a_sq += kt.sum_sq(row.data(), n);
        for (index j = 0; j < l; ++j) {
            const double gij = kt.dot(row.data(), omega.col(j), n);   // G(i,:) = A(i,:) Omega
            g(i, j) = gij;
            if (gij != 0.0) kt.axpy(gij, row.data(), h.col(j), n);    // H += A(i,:)^T G(i,:)
        }
    }
    QBState st(m, n);
    st.e = norm_a_sq;
    Termination term = Termination::rank_reached;
    for (index off = 0; off < l; off += b) {
        const index bi = std::min(b, l - off);
        DenseMatrix om_i = omega.column_range(off, off + bi);
        DenseMatrix yi = g.column_range(off, off + bi);
        DenseMatrix hi = h.column_range(off, off + bi);
        DenseMatrix m1;
        if (st.k > 0) {
            m1 = multiply_at_b(st.bt, om_i);
            multiply_acc(yi, st.q, m1, -1.0);
        }
        DenseMatrix qi, bti;
        const index d = fp_block(st, yi, hi, m1, true, qi, bti);
        if (d == 0) {
            term = Termination::rank_collapse;
            break;
        }
        st.append(std::move(qi), std::move(bti), false, 0.0);
        if (d < bi) {
            term = Termination::rank_collapse;
            break;
        }
    }
    QBFactorization f = finish(st, nullptr, 0, term, norm_a_sq);
    f.passes = 1;
    return f;
}

double explicit_error(const MatrixHandle& a, const DenseMatrix& q, const DenseMatrix& b) {
    const auto& kt = kernels::active_kernels();
    double acc = 0.0;
    a.for_each_column_block(256, [&](index j0, const DenseMatrix& blk) {
        DenseMatrix r = blk;
        if (q.cols() > 0) {
            DenseMatrix bb(b.rows(), blk.cols());
            for (index j = 0; j < blk.cols(); ++j)
                for (index i = 0; i < b.rows(); ++i) bb(i, j) = b(i, j0 + j);
            multiply_acc(r, q, bb, -1.0);
        }
        acc += kt.sum_sq(r.data(), r.size());
    });
    return std::sqrt(acc);
}

}  // namespace qbfac
