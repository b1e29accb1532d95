"""Baselines on the device (§8(f) 4) against the oracle restatement
(oracle/qb_restated.cpp rand_qb / rand_qb_b / adaptive_range_finder on the reference's kernels)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _m2(n, seed=9):
    from paper_1606_09402_b200 import matgen
    return matgen.synthesize(n, n, matgen.spectrum("exp_decay", n, tau=7.0), seed)


def _sv(b):
    return np.linalg.svd(b, compute_uv=False) if b.shape[0] else np.zeros(0)


@pytest.mark.parametrize("l,P", [(60, 0), (60, 2), (130, 1)])
def test_rand_qb_vs_oracle(ctx, oracle, l, P):
    from paper_1606_09402_b200 import qbfac
    a = _m2(300)
    ref = oracle.run("qb", a, fixed_rank=(l, 0), power=P, seed=3)
    got = qbfac.rand_qb(qbfac.MatrixHandle.dense(a, ctx), l, P, qbfac.RngStream(3))
    assert got.rank == ref.rank == l and got.passes == ref.passes == 2 + 2 * P
    assert got.error_indicator == -1.0 and got.terminated_by == ref.terminated_by == "rank_reached"
    s_g, s_r = _sv(got.B), _sv(ref.B)
    sel = s_r > 1e-6 * s_r[0]
    assert np.max(np.abs(s_g - s_r)[sel] / s_r[sel]) <= 1e-10
    e_g, e_r = np.linalg.norm(a - got.Q @ got.B), np.linalg.norm(a - ref.Q @ ref.B)
    assert abs(e_g - e_r) <= 1e-10 * e_r + 1e-14 * np.linalg.norm(a)


def test_rand_qb_exact_rank_and_collapse(ctx, oracle):
    """SPEC: exact rank r, l >= r, P=0 -> ||A - QB|| <= 1e-10 ||A||; the deficient sketch keeps its
    leading columns and ends rank_collapse (same decision as the reference's QR)."""
    from paper_1606_09402_b200 import qbfac
    rs = np.random.default_rng(1)
    a = np.asfortranarray(rs.standard_normal((200, 30)) @ rs.standard_normal((30, 150)))
    ref = oracle.run("qb", a, fixed_rank=(40, 0), power=0, seed=2)
    got = qbfac.rand_qb(qbfac.MatrixHandle.dense(a, ctx), 40, 0, qbfac.RngStream(2))
    assert got.rank == ref.rank == 30 and got.terminated_by == ref.terminated_by == "rank_collapse"
    assert np.linalg.norm(a - got.Q @ got.B) <= 1e-10 * np.linalg.norm(a)


@pytest.mark.parametrize("mode", ["precision", "rank"])
def test_rand_qb_b_vs_oracle_and_ei(ctx, oracle, mode):
    """SPEC: same seed as rand_qb_ei on Matrix 2 (n=300, eps=1e-4 ||A||, b=10) -> identical rank
    and ||Q_b - Q_ei|| <= 1e-8; fixed_rank(40, 0), b=10 -> 16 passes."""
    from paper_1606_09402_b200 import qbfac
    a = _m2(300)
    if mode == "precision":
        eps = 1e-4 * np.linalg.norm(a)
        stop = qbfac.StopRule.fixed_precision(eps)
        ref = oracle.run("qb_b", a, b=10, eps_abs=eps, seed=5)
    else:
        stop = qbfac.StopRule.fixed_rank(40, 0)
        ref = oracle.run("qb_b", a, b=10, fixed_rank=(40, 0), seed=5)
    got = qbfac.rand_qb_b(qbfac.MatrixHandle.dense(a, ctx), stop, 10, qbfac.RngStream(5))
    assert got.rank == ref.rank and got.passes == ref.passes and got.terminated_by == ref.terminated_by
    if mode == "rank":
        assert got.passes == 16 and got.rank == 40
    assert abs(got.error_indicator - ref.E) <= 1e-10 * abs(ref.E) + 2e-13 * ref.norm_a_sq
    assert np.linalg.norm(got.Q - ref.Q) <= 1e-8
    if mode == "precision":
        ei = qbfac.rand_qb_ei(qbfac.MatrixHandle.dense(a, ctx), stop, 10, 0, qbfac.RngStream(5))
        assert ei.rank == got.rank and np.linalg.norm(ei.Q - got.Q) <= 1e-8


def test_rand_qb_b_rejects_sparse(ctx):
    from paper_1606_09402_b200 import matgen, qbfac
    csr = matgen.csr_uniform(300, 200, 5, seed=1)
    with pytest.raises(qbfac.DimensionError):
        qbfac.rand_qb_b(qbfac.MatrixHandle.csr(*csr, ctx=ctx), qbfac.StopRule.fixed_rank(10, 0), 5,
                        qbfac.RngStream(1))


@pytest.mark.parametrize("sparse", [False, True])
def test_range_finder_vs_oracle(ctx, oracle, sparse):
    from paper_1606_09402_b200 import matgen, qbfac
    if sparse:
        csr = matgen.csr_uniform(400, 300, 8, seed=2)
        h = qbfac.MatrixHandle.csr(*csr, ctx=ctx)
        tol = 0.6 * np.sqrt((csr[4] ** 2).sum())
        ref = oracle.run("arf", csr=csr, b=10, eps_abs=tol, max_rank=120, seed=3)
    else:
        a = _m2(300)
        h = qbfac.MatrixHandle.dense(a, ctx)
        tol = 1e-2 * np.linalg.norm(a)
        ref = oracle.run("arf", a, b=10, eps_abs=tol, seed=3)
    got = qbfac.adaptive_range_finder(h, tol, 10, qbfac.RngStream(3), max_rank=120 if sparse else 0)
    assert got.rank == ref.rank and got.passes == ref.passes and got.terminated_by == ref.terminated_by
    s_g, s_r = _sv(got.B), _sv(ref.B)
    assert np.max(np.abs(s_g - s_r) / s_r) <= 1e-9


def test_range_finder_exact_rank_and_trivial(ctx):
    """SPEC: exact rank-k A, tiny tol -> between k and k + r columns; tol >= 10 sqrt(2/pi) ||A||_F ->
    immediate termination, near-empty Q."""
    from paper_1606_09402_b200 import qbfac
    rs = np.random.default_rng(4)
    a = np.asfortranarray(rs.standard_normal((150, 12)) @ rs.standard_normal((12, 120)))
    got = qbfac.adaptive_range_finder(qbfac.MatrixHandle.dense(a, ctx), 1e-9 * np.linalg.norm(a), 10,
                                      qbfac.RngStream(1))
    assert 12 <= got.rank <= 22
    big = 10 * np.sqrt(2 / np.pi) * np.linalg.norm(a)
    got2 = qbfac.adaptive_range_finder(qbfac.MatrixHandle.dense(a, ctx), big, 10, qbfac.RngStream(1))
    assert got2.rank <= 10 and got2.terminated_by == "tolerance_met"  # 'near-empty'
