"""Matrix Market ingest / export against the reference's own CSR builder
SparseCsrMatrix::from_triplets (sparse_csr.cpp:42-64, compiled into the oracle). The host
parser needs no GPU; the device upload test is marked gpu."""
import numpy as np
import pytest

from paper_1606_09402_b200 import matgen, qbfac


def _sparse_random(n, density, seed):
    rs = np.random.default_rng(seed)
    mask = rs.random((n, n)) < density
    rows, cols = np.nonzero(mask)
    vals = rs.standard_normal(len(rows)) * 10.0 ** rs.integers(-300, 300, len(rows))
    return rows, cols, vals


def test_dense_round_trip_bitwise(tmp_path):
    """SPEC: 2x2 dense round trip -> bitwise-equal values."""
    a = np.array([[1.0 / 3.0, -2.5e-308], [np.pi * 1e300, 5e-324]], order="F")
    p = str(tmp_path / "d.mtx")
    qbfac.write_matrix_market(p, a=a)
    kind, b = qbfac.read_matrix_market(p)
    assert kind == "dense" and np.array_equal(a.view(np.int64), b.view(np.int64))


def test_sparse_round_trip_matches_reference_from_triplets(tmp_path, oracle):
    """SPEC: sparse_random(n=500, 0.003) round trip -> identical pattern and values; the parsed
    CSR equals the reference's from_triplets on the same triplets, bit for bit."""
    n = 500
    rows, cols, vals = _sparse_random(n, 0.003, 1)
    perm = np.random.default_rng(2).permutation(len(rows))  # from_triplets sorts
    st, rp, ci, v = oracle.csr_from_triplets(n, n, rows[perm], cols[perm], vals[perm])
    assert st == "ok"
    p = str(tmp_path / "s.mtx")
    qbfac.write_matrix_market(p, csr=(n, n, rp, ci, v))
    kind, m2, n2, rp2, ci2, v2 = qbfac.read_matrix_market(p)
    assert kind == "csr" and (m2, n2) == (n, n)
    assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2) and np.array_equal(v.view(np.int64), v2.view(np.int64))


def test_unsorted_file_equals_from_triplets(tmp_path, oracle):
    """Entries in arbitrary order, comment lines, blank lines, '+' signs, exponents."""
    m, n = 40, 70
    rs = np.random.default_rng(5)
    flat = rs.choice(m * n, 300, replace=False)
    rows, cols = flat // n, flat % n
    vals = rs.standard_normal(300)
    lines = ["%%MatrixMarket matrix coordinate real general", "% a comment", "", f"{m} {n} {len(vals)}"]
    for r, c, x in zip(rows, cols, vals):
        lines.append(f"{r + 1} {c + 1} {float(x)!r}" if r % 3 else f"  +{r + 1}\t{c + 1}   {x:.17e}  ")
        if r % 7 == 0:
            lines.append("% interleaved comment")
    p = tmp_path / "u.mtx"
    p.write_text("\n".join(lines) + "\n")
    st, rp, ci, v = oracle.csr_from_triplets(m, n, rows, cols, vals)
    kind, m2, n2, rp2, ci2, v2 = qbfac.read_matrix_market(str(p))
    assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2) and np.array_equal(v, v2)


@pytest.mark.parametrize("banner", ["%%MatrixMarket matrix coordinate complex general",
                                    "%%MatrixMarket matrix coordinate real symmetric",
                                    "%%MatrixMarket matrix coordinate pattern general",
                                    "%%MatrixMarket vector coordinate real general",
                                    "MatrixMarket matrix coordinate real general"])
def test_unsupported_banners(tmp_path, banner):
    """SPEC: complex banner (and any non real/general flag) -> unsupported-format error."""
    p = tmp_path / "b.mtx"
    p.write_text(banner + "\n2 2 1\n1 1 1.0\n")
    with pytest.raises(qbfac.FormatError):
        qbfac.read_matrix_market(str(p))


@pytest.mark.parametrize("body,exc,ref", [("3 3 2\n1 1 1.0\n1 1 2.0\n", qbfac.FormatError, "FormatError"),
                                          ("3 3 1\n4 1 1.0\n", qbfac.FormatError, "FormatError"),
                                          ("3 3 1\n0 1 1.0\n", qbfac.FormatError, "FormatError"),
                                          ("3 3 2\n1 1 1.0\n", qbfac.FormatError, None),
                                          ("3 3 1\n1 1 nan\n", qbfac.Error, "Error"),
                                          ("3 3 1\n1 x 1.0\n", qbfac.FormatError, None)])
def test_invalid_entries(tmp_path, oracle, body, exc, ref):
    """Duplicates / out-of-range coordinates are FormatError as in from_triplets; non-finite
    values are Error as in from_parts; count mismatches and garbage are FormatError."""
    p = tmp_path / "e.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n" + body)
    with pytest.raises(exc):
        qbfac.read_matrix_market(str(p))
    if ref is not None:
        lines = body.strip().split("\n")[1:]
        trip = [line.split() for line in lines]
        rows = [int(t[0]) - 1 for t in trip]
        cols = [int(t[1]) - 1 for t in trip]
        vals = [float(t[2]) for t in trip]
        if min(rows) >= 0:
            assert oracle.csr_from_triplets(3, 3, rows, cols, vals)[0] == ref


def test_empty_and_wide(tmp_path):
    p = tmp_path / "z.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n5 1000000 0\n")
    kind, m, n, rp, ci, v = qbfac.read_matrix_market(str(p))
    assert (m, n, len(v)) == (5, 1000000, 0) and np.array_equal(rp, np.zeros(6))


@pytest.mark.gpu
def test_device_ingest_equals_in_memory(tmp_path, ctx, oracle):
    """read_matrix_market -> MatrixHandle on the device: the device CSR is the parsed CSR, and
    randQB_EI on it equals randQB_EI on the in-memory handle (same seed) bit for bit."""
    csr = matgen.csr_uniform(3000, 1500, 20, seed=11)
    p = str(tmp_path / "c.mtx")
    qbfac.write_matrix_market(p, csr=csr)
    h_file = qbfac.MatrixHandle.from_mtx(p, ctx)
    assert h_file.sparse and (h_file.m, h_file.n) == (3000, 1500)
    rp, ci, v = h_file.export()
    assert np.array_equal(rp, csr[2]) and np.array_equal(ci, csr[3]) and np.array_equal(v, csr[4])
    h_mem = qbfac.MatrixHandle.csr(*csr, ctx=ctx)
    eps = 0.5 * np.sqrt((csr[4] ** 2).sum())
    f1 = qbfac.rand_qb_ei(h_file, qbfac.StopRule.fixed_precision(eps), 20, 1, qbfac.RngStream(3), max_rank=200)
    f2 = qbfac.rand_qb_ei(h_mem, qbfac.StopRule.fixed_precision(eps), 20, 1, qbfac.RngStream(3), max_rank=200)
    assert f1.rank == f2.rank and np.array_equal(f1.B, f2.B) and np.array_equal(f1.Q, f2.Q)
    a = np.asfortranarray(np.random.default_rng(0).standard_normal((70, 30)))
    pd = str(tmp_path / "d.mtx")
    qbfac.write_matrix_market(pd, a=a)
    hd = qbfac.MatrixHandle.from_mtx(pd, ctx)
    assert not hd.sparse and np.array_equal(hd.export(), a)
