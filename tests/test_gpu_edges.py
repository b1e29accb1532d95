"""Edge cases of the hot path against the oracle: ragged / degenerate shapes, empty rows and
columns in CSR, one-row matrices, b larger than the matrix, wide and tall dense shapes."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cmp(got, ref, tol=1e-10):
    assert got.rank == ref.rank and got.terminated_by == ref.terminated_by and got.passes == ref.passes
    if got.rank:
        sg = np.linalg.svd(got.B, compute_uv=False)
        sr = np.linalg.svd(ref.B, compute_uv=False)
        sel = sr > 1e-8 * sr[0]
        assert np.max(np.abs(sg - sr)[sel] / sr[sel]) <= tol


def _csr_with_holes(m, n, seed):
    """Rows with 0..9 entries (many empty) over columns restricted to a subset (empty columns)."""
    rs = np.random.default_rng(seed)
    live_cols = np.sort(rs.choice(n, n // 2, replace=False))
    rp = [0]
    ci, v = [], []
    for i in range(m):
        k = int(rs.integers(0, 10)) if i % 3 else 0
        cols = np.sort(rs.choice(live_cols, k, replace=False))
        ci.extend(cols.tolist())
        v.extend(rs.standard_normal(k).tolist())
        rp.append(len(ci))
    return (m, n, np.array(rp, dtype=np.int64), np.array(ci, dtype=np.int32), np.array(v))


@pytest.mark.parametrize("P", [0, 1])
def test_csr_empty_rows_and_columns(ctx, oracle, P):
    from paper_1606_09402_b200 import qbfac
    csr = _csr_with_holes(700, 400, 3)
    eps = 0.3 * np.sqrt((csr[4] ** 2).sum())
    ref = oracle.run("ei", csr=csr, b=16, power=P, eps_abs=eps, max_rank=150, seed=2)
    got = qbfac.rand_qb_ei(qbfac.MatrixHandle.csr(*csr, ctx=ctx), qbfac.StopRule.fixed_precision(eps), 16, P,
                           qbfac.RngStream(2), max_rank=150)
    _cmp(got, ref)
    assert abs(got.error_indicator - ref.E) <= 1e-10 * ref.E + 2e-13 * ref.norm_a_sq


def test_one_row_matrix(ctx, oracle):
    """SPEC single_pass_fp: one-row matrix -> rank-1 exact recovery; EI on it stops at rank 1."""
    from paper_1606_09402_b200 import qbfac
    a = np.asfortranarray(np.random.default_rng(1).standard_normal((1, 40)))
    got = qbfac.single_pass_fp(qbfac.MatrixHandle.dense(a, ctx), 1, 1, qbfac.RngStream(3))
    assert got.rank == 1 and np.linalg.norm(a - got.Q @ got.B) <= 1e-12 * np.linalg.norm(a)
    ref = oracle.run("ei", a, b=5, power=0, eps_abs=1e-6 * np.linalg.norm(a), seed=4)
    ei = qbfac.rand_qb_ei(qbfac.MatrixHandle.dense(a, ctx), qbfac.StopRule.fixed_precision(1e-6 * np.linalg.norm(a)),
                          5, 0, qbfac.RngStream(4))
    _cmp(ei, ref)


@pytest.mark.parametrize("m,n,b", [(30, 500, 40), (700, 25, 10), (64, 64, 64), (129, 65, 33)])
def test_ragged_shapes_fixed_rank(ctx, oracle, m, n, b):
    """b larger than the matrix, wide / tall shapes, sizes one past a tile boundary."""
    from paper_1606_09402_b200 import qbfac
    rs = np.random.default_rng(m * n)
    a = np.asfortranarray(rs.standard_normal((m, n)) * np.logspace(0, -3, n)[None, :])
    k = min(m, n) - 3
    ref = oracle.run("ei", a, b=b, power=1, fixed_rank=(k, 2), seed=7)
    got = qbfac.rand_qb_ei(qbfac.MatrixHandle.dense(a, ctx), qbfac.StopRule.fixed_rank(k, 2), b, 1,
                           qbfac.RngStream(7))
    _cmp(got, ref, tol=1e-9)
    assert np.abs(got.Q.T @ got.Q - np.eye(got.rank)).max() < 1e-12


def test_zero_matrix(ctx):
    """A = 0: any positive tolerance is met immediately (E = 0 < eps^2) with empty factors; the
    Theorem-3 floor is 0 so validate_epsilon accepts it."""
    from paper_1606_09402_b200 import qbfac
    a = np.zeros((50, 40), order="F")
    got = qbfac.rand_qb_ei(qbfac.MatrixHandle.dense(a, ctx), qbfac.StopRule.fixed_precision(1e-3), 10, 0,
                           qbfac.RngStream(1))
    assert got.rank == 0 and got.terminated_by == "tolerance_met"


def test_fp_budget_equals_block(ctx, oracle):
    """l_budget == b: one block per sketch, restarts on exhaustion."""
    from paper_1606_09402_b200 import matgen, qbfac
    a = matgen.synthesize(200, 200, matgen.spectrum("exp_decay", 200, tau=7.0), 5)
    eps = 1e-2 * np.linalg.norm(a)
    ref = oracle.run("fp", a, b=10, power=0, eps_abs=eps, l_budget=10, max_rank=100, seed=6)
    got = qbfac.rand_qb_fp(qbfac.MatrixHandle.dense(a, ctx), eps, 10, 0, 10, qbfac.RngStream(6), max_rank=100)
    assert got.rank == ref.rank and got.terminated_by == ref.terminated_by and got.passes == ref.passes
