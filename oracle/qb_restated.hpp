// ORACLE — TEST INFRASTRUCTURE ONLY. Not part of the product path.
//
// Restated declarations of the reference's missing algorithm header (the
// reference ships no qb.hpp; the types and signatures survive only in
// /root/reference/SPEC.md:209-335). Built on the reference's own public API
// (MatrixHandle, DenseMatrix, RngStream) from /root/reference/proj/include.

#pragma once

#include <cstdint>
#include <vector>

#include "qbfac/dense_matrix.hpp"
#include "qbfac/matrix_handle.hpp"
#include "qbfac/rng.hpp"
#include "qbfac/types.hpp"

namespace qbfac {

// SPEC.md:210 terminated_by.
enum class Termination : int {
    rank_reached = 0,
    tolerance_met = 1,
    sketch_exhausted = 2,
    rank_collapse = 3,
};

// SPEC.md:216-220.
struct StopRule {
    enum class Mode : int { fixed_rank = 0, fixed_precision = 1 };
    Mode mode = Mode::fixed_precision;
    index k = 0;
    index s = 0;
    double eps = 0.0;  // absolute Frobenius tolerance

    static StopRule fixed_rank(index k, index s) { return {Mode::fixed_rank, k, s, 0.0}; }
    static StopRule fixed_precision(double eps) { return {Mode::fixed_precision, 0, 0, eps}; }
};

// SPEC.md:209-215. B is rank x n. `e_trace` (oracle extra) holds E after every
// block boundary for the Theorem-2 checks.
struct QBFactorization {
    DenseMatrix Q;
    DenseMatrix B;
    double error_indicator = -1.0;
    std::int64_t passes = 0;
    Termination terminated_by = Termination::rank_reached;
    double norm_a_sq = 0.0;
    std::vector<double> e_trace;
};

struct EpsilonCheck {
    bool valid;
    double floor;
};

// SPEC.md:327-335 (Theorem 3): valid iff eps > sqrt(4*u/delta)*||A||_F, u = kEpsMach (types.hpp:14).
EpsilonCheck validate_epsilon(double eps, double frob_a, double delta = 0.01);

// Alg. 2 + per-block power iteration + row
// truncation. max_rank == 0 means min(m, n).
QBFactorization rand_qb_ei(const MatrixHandle& a, const StopRule& stop, index b, int power,
                           RngStream& rng, index max_rank = 0);

// Alg. 4 with steps 9a-9c and restart on
// sketch exhaustion.
QBFactorization rand_qb_fp(const MatrixHandle& a, double eps_abs, index b, int power,
                           index l_budget, RngStream& rng, index max_rank = 0,
                           int max_restarts = 8);

// Alg. 3, optionally with steps 9a-9c.
QBFactorization rand_qb_fp_fixed_rank(const MatrixHandle& a, index k, index s, index b,
                                      bool reorth, RngStream& rng);

// Remark 4.2.
QBFactorization single_pass_fp(RowStream& stream, index l, index b, RngStream& rng);

// ---- baselines (§8(f) 4) ----
// randQB (Fig. 1a): Q = orth of the power-iterated sketch (orth after every application of
// A and A^T), B = Q^T A; passes = 2 + 2P; E is the -1 sentinel; a deficient QR keeps the
// leading columns and ends rank_collapse.
QBFactorization rand_qb(const MatrixHandle& a, index l, int power, RngStream& rng);
// randQB_b (Fig. 1b): explicit residual R (dense A only); per block: E = ||R||_F^2 (pass),
// Y = R Omega_i (pass), Q_i = orth(Y) re-orthogonalised against Q, B_i = Q_i^T R (pass) with the
// row-by-row truncation of PAPER.md:206-220 on E, R -= Q_i B_i (pass): 4 passes per block.
QBFactorization rand_qb_b(const MatrixHandle& a, const StopRule& stop, index b, RngStream& rng);
// Adaptive randomized range finder (Eq. 2.4, Halko et al. Alg. 4.2): Q grows one vector at a
// time until the last r residual samples are all below tol / (10 sqrt(2/pi)); B = Q^T A.
QBFactorization adaptive_range_finder(const MatrixHandle& a, double tol_spectral, index r, RngStream& rng,
                                      index max_rank = 0);

// ||A - QB||_F streamed over column blocks of 256 (+1 pass).
double explicit_error(const MatrixHandle& a, const DenseMatrix& q, const DenseMatrix& b);

}  // namespace qbfac
