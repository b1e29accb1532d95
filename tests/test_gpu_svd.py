"""qb_to_svd on the device (§8(f) 1): orth(B^T) + one-sided Jacobi."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_diag_exact(ctx):
    """SPEC: A = diag(3, 2, 1), exact QB with l = 3 -> S = (3, 2, 1) to 1e-12."""
    from paper_1606_09402_b200 import qbfac
    a = np.diag([3.0, 2.0, 1.0])
    r = qbfac.run_device(qbfac.MatrixHandle.dense(a, ctx), alg=0, mode=0, b=3, k=3, s=0, seed=1)
    t = r.svd(3)
    assert np.max(np.abs(t.S - [3.0, 2.0, 1.0])) <= 1e-12
    assert np.linalg.norm(t.U @ np.diag(t.S) @ t.V.T - a) <= 1e-12


@pytest.mark.parametrize("n,l,P,k", [(300, 60, 1, 50), (400, 130, 0, 120)])
def test_matrix2_top_k(ctx, n, l, P, k):
    """SPEC: Matrix 2 (n=300, l=60, P=1, k=50): max_j |S_j - sigma_j| / sigma_j <= 1e-3 against the
    SVD of A; U, V orthonormality loss <= 1e-10; S equals the SVD of B (1e-12) and U S V^T = Q B
    restricted to the top k."""
    from paper_1606_09402_b200 import matgen, qbfac
    sig = matgen.spectrum("exp_decay", n, tau=7.0)
    a = matgen.synthesize(n, n, sig, 9)
    r = qbfac.run_device(qbfac.MatrixHandle.dense(a, ctx), alg=0, mode=0, b=10, power=P, k=l, s=0, seed=3)
    t = r.svd(k)
    assert np.all(np.diff(t.S) <= 0)
    if (n, l, P, k) == (300, 60, 1, 50):  # the SPEC example; the other case checks the SVD of B only
        assert np.max(np.abs(t.S - sig[:k]) / sig[:k]) <= 1e-3
    assert np.abs(t.U.T @ t.U - np.eye(k)).max() <= 1e-10
    assert np.abs(t.V.T @ t.V - np.eye(k)).max() <= 1e-10
    q, b = r.q(), r.b()
    sb = np.linalg.svd(b, compute_uv=False)
    assert np.max(np.abs(t.S - sb[:k]) / sb[:k]) <= 1e-12
    uu, ss, vvt = np.linalg.svd(q @ b, full_matrices=False)
    ref = uu[:, :k] @ np.diag(ss[:k]) @ vvt[:k]
    assert np.linalg.norm(t.U @ np.diag(t.S) @ t.V.T - ref) <= 1e-10 * np.linalg.norm(ref)


def test_sparse_and_wide_rank(ctx):
    """CSR input, rank 150 (> the 112-column panel limit: wide CholQR2 path for orth(B^T))."""
    from paper_1606_09402_b200 import matgen, qbfac
    csr = matgen.csr_uniform(2000, 900, 20, seed=4)
    r = qbfac.run_device(qbfac.MatrixHandle.csr(*csr, ctx=ctx), alg=0, mode=0, b=25, power=1, k=150, s=0, seed=5)
    t = r.svd(150)
    b = r.b()
    sb = np.linalg.svd(b, compute_uv=False)
    assert np.max(np.abs(t.S - sb) / sb) <= 1e-11
    assert np.abs(t.V.T @ t.V - np.eye(150)).max() <= 1e-10


def test_k_too_large(ctx):
    from paper_1606_09402_b200 import qbfac
    a = np.random.default_rng(0).standard_normal((50, 40))
    r = qbfac.run_device(qbfac.MatrixHandle.dense(a, ctx), alg=0, mode=0, b=10, k=20, s=0, seed=1)
    with pytest.raises(qbfac.DimensionError):
        r.svd(21)


@pytest.mark.parametrize("rank", [333, 600, 1000, 1450, 1568, 1600])
def test_block_jacobi_large_rank(ctx, rank):
    """qb_to_svd at rank 333 (odd: plain column loads) / 600 / 1000 / 1450 and 1568 (more block pairs than
    2-CTA clusters fit; 1568 is the largest rank whose column slices fit shared memory) through the
    Gram-based block one-sided Jacobi (nb = 8 column blocks, one 2-CTA cluster per block pair), and
    1600 through the column-rotating block kernel that remains above it: S equals the SVD of B to 1e-12 relative, U and V orthonormal,
    U S V^T = Q B, and the scalar Jacobi (QBFAC_JACOBI_SCALAR=1) agrees."""
    import os
    from paper_1606_09402_b200 import matgen, qbfac
    csr = matgen.csr_uniform(6000, 3000, 30, seed=8)
    r = qbfac.run_device(qbfac.MatrixHandle.csr(*csr, ctx=ctx), alg=0, mode=0, b=50, power=1, k=rank, s=0, seed=2)
    t = r.svd(rank)
    b = r.b()
    sb = np.linalg.svd(b, compute_uv=False)
    assert np.max(np.abs(t.S - sb) / sb) <= 1e-12
    assert np.abs(t.U.T @ t.U - np.eye(rank)).max() <= 1e-10
    assert np.abs(t.V.T @ t.V - np.eye(rank)).max() <= 1e-10
    qb = r.q() @ b
    assert np.linalg.norm(t.U @ np.diag(t.S) @ t.V.T - qb) <= 1e-10 * np.linalg.norm(qb)
    os.environ["QBFAC_JACOBI_SCALAR"] = "1"
    try:
        t2 = r.svd(rank)
    finally:
        os.environ.pop("QBFAC_JACOBI_SCALAR")
    assert np.max(np.abs(t2.S - t.S) / t.S) <= 1e-12
