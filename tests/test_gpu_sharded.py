"""Row-sharded engine on one GPU: `world` contexts form an in-process rank
group (qbfac_gpu_test_create_local_group), each driven by its own host thread; the engine's
collectives — the n x w allreduce after every A^T pass, the b x b / k x b Gram allreduces and
||A||^2 — meet at a host barrier and are summed in rank order. Every rank must reproduce the
unsharded factorization: same rank, passes and termination, bitwise-identical replicated B across
ranks, σ(B) and ||A - QB|| of the stacked row shards of Q against the single-context run."""
import ctypes as C
import threading

import numpy as np
import pytest

from paper_1606_09402_b200 import dist, matgen, qbfac

pytestmark = pytest.mark.gpu


def _local_group(world):
    L = qbfac.lib()
    L.qbfac_gpu_test_create_local_group.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    arr = (C.c_void_p * world)()
    st = L.qbfac_gpu_test_create_local_group(0, world, arr)
    assert st == 0, L.qbfac_gpu_last_error(None).decode()
    ctxs = []
    for r in range(world):
        c = qbfac.Context.__new__(qbfac.Context)
        c._h = C.c_void_p(arr[r])
        c.device, c.rank, c.world = 0, r, world
        ctxs.append(c)
    return ctxs


def _run_ranks(handles, **kw):
    out, errs = [None] * len(handles), []

    def work(r):
        try:
            res = qbfac.run_device(handles[r], **kw)
            out[r] = (res.rank, int(res.info.passes), int(res.info.terminated_by), float(res.info.error_indicator),
                      res.q(), res.b())
            res.free()
        except Exception as ex:  # pragma: no cover - surfaced below
            errs.append(repr(ex))

    ths = [threading.Thread(target=work, args=(r,)) for r in range(len(handles))]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=300)
    assert not errs, errs
    return out


def _single(h, **kw):
    res = qbfac.run_device(h, **kw)
    o = (res.rank, int(res.info.passes), int(res.info.terminated_by), float(res.info.error_indicator), res.q(), res.b())
    res.free()
    return o


def _check(a_dense, ref, shards, sig_tol):
    rank, passes, term, e, q, b = ref
    for r, s in enumerate(shards):
        assert s[0] == rank and s[1] == passes and s[2] == term, (r, s[:3], ref[:3])
        assert np.array_equal(s[5], shards[0][5]), "replicated B differs across ranks"
    qs = np.vstack([s[4] for s in shards])
    bs = shards[0][5]
    sg = np.linalg.svd(bs, compute_uv=False)
    sr = np.linalg.svd(b, compute_uv=False)
    # relative tolerance, with the absolute rounding floor u ||B|| for singular values far below sigma_1
    assert np.all(np.abs(sg - sr) <= sig_tol * sr + 1e-15 * sr[0]), np.max(np.abs(sg - sr) / sr)
    err_s = np.linalg.norm(a_dense - qs @ bs)
    err_r = np.linalg.norm(a_dense - q @ b)
    assert abs(err_s - err_r) <= 1e-8 * np.linalg.norm(a_dense) + 1e-6 * err_r
    if e >= 0:
        assert abs(shards[0][3] - e) <= 1e-10 * e + 1e-13 * np.linalg.norm(a_dense) ** 2
    assert np.linalg.norm(qs.T @ qs - np.eye(qs.shape[1])) < 1e-10


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("alg,kw", [(0, dict(b=10, power=1, max_rank=200)),
                                    (1, dict(b=10, power=1, max_rank=200, l_budget=120)),
                                    (3, dict(mode=0, b=16, k=60, s=0))])
def test_sharded_dense_matches_single(world, alg, kw):
    a = matgen.synthesize(901, 300, matgen.spectrum("exp_decay", 300, tau=12.0), 21)
    eps = 1e-3 * np.linalg.norm(a)
    run = dict(alg=alg, eps_abs=eps, seed=7, **kw)
    ref = _single(qbfac.MatrixHandle.dense(a, qbfac.default_context()), **run)
    ctxs = _local_group(world)
    plan = dist.plan_dense_rows(a.shape[0], world)
    hs = [qbfac.MatrixHandle.dense_shard(dist.shard_dense(a, r0, rows), a.shape[0], r0, ctxs[g])
          for g, (r0, rows) in enumerate(plan)]
    shards = _run_ranks(hs, **run)
    _check(a, ref, shards, 1e-10 if alg == 0 else 1e-8)


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_csr_ei_matches_single(world):
    csr = matgen.csr_uniform(1200, 500, 13, seed=11)
    a = matgen.csr_to_dense(csr)
    eps = 0.6 * np.linalg.norm(a)
    run = dict(alg=0, b=20, power=1, max_rank=120, eps_abs=eps, seed=3)
    ref = _single(qbfac.MatrixHandle.csr(*csr, ctx=qbfac.default_context()), **run)
    ctxs = _local_group(world)
    plan = dist.plan_csr_rows(csr[2], world)
    hs = []
    for g, (r0, rows) in enumerate(plan):
        loc = dist.shard_csr(csr, r0, rows)
        hs.append(qbfac.MatrixHandle.csr_shard(csr[0], r0, csr[1], loc[2], loc[3], loc[4], ctxs[g]))
    shards = _run_ranks(hs, **run)
    _check(a, ref, shards, 1e-10)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("alg", [0, 1])
def test_sharded_rank_collapse_householder(world, alg, oracle):
    """Exact rank-15 A with a tiny tolerance: the second block's sketch is numerically rank
    deficient, its CholQR panels fail and the block is redone with Householder panels. Under
    row sharding the Householder fallback assembles the panel on every rank (exact sum over
    ranks of zero-padded row blocks), factors it redundantly and keeps the local rows: rank,
    passes and termination equal the unsharded device run (and, for EI, the oracle's)."""
    rs = np.random.default_rng(0)
    a = np.asfortranarray(rs.standard_normal((120, 15)) @ rs.standard_normal((15, 90)))
    eps = 1e-6 * np.linalg.norm(a)
    run = dict(alg=alg, b=10, power=0, eps_abs=eps, seed=8, max_rank=90)
    if alg == 1:
        run["l_budget"] = 40
    ref = _single(qbfac.MatrixHandle.dense(a, qbfac.default_context()), **run)
    if alg == 0:
        o = oracle.run("ei", a, b=10, power=0, eps_abs=eps, seed=8, max_rank=90)
        assert (ref[0], qbfac.TERMINATION[ref[2]]) == (o.rank, o.terminated_by)
    r = qbfac.run_device(qbfac.MatrixHandle.dense(a, qbfac.default_context()), **run)
    assert int(r.info.householder_fallbacks) > 0  # the deficient block took the Householder path
    r.free()
    ctxs = _local_group(world)
    plan = dist.plan_dense_rows(a.shape[0], world, align=8)
    hs = [qbfac.MatrixHandle.dense_shard(dist.shard_dense(a, r0, rows), a.shape[0], r0, ctxs[g])
          for g, (r0, rows) in enumerate(plan)]
    shards = _run_ranks(hs, **run)
    for s in shards:
        assert (s[0], s[1], s[2]) == ref[:3]
        assert np.array_equal(s[5], shards[0][5])
    qs = np.vstack([s[4] for s in shards])
    assert np.linalg.norm(a - qs @ shards[0][5]) <= 1e-10 * np.linalg.norm(a)


@pytest.mark.parametrize("alg", [0, 1])
def test_sharded_wide_block(alg):
    """b = 130 > 112 under row sharding (world 2): the wide BCGS2 panels allreduce their
    projections and Grams; every rank matches the unsharded run."""
    a = matgen.synthesize(700, 500, matgen.spectrum("exp_decay", 500, tau=20.0), 23)
    eps = 1e-6 * np.linalg.norm(a)
    run = dict(alg=alg, b=130, power=1, eps_abs=eps, seed=5, max_rank=400)
    if alg == 1:
        run["l_budget"] = 390  # no restart: FP's B_i update stays well conditioned
    ref = _single(qbfac.MatrixHandle.dense(a, qbfac.default_context()), **run)
    ctxs = _local_group(2)
    plan = dist.plan_dense_rows(a.shape[0], 2)
    hs = [qbfac.MatrixHandle.dense_shard(dist.shard_dense(a, r0, rows), a.shape[0], r0, ctxs[g])
          for g, (r0, rows) in enumerate(plan)]
    shards = _run_ranks(hs, **run)
    _check(a, ref, shards, 1e-10 if alg == 0 else 1e-8)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_range_finder(world):
    """The adaptive range finder row-sharded: window norms, projections Q^T v and
    A^T Q summed over ranks; every rank matches the unsharded device run."""
    a = matgen.synthesize(400, 300, matgen.spectrum("exp_decay", 300, tau=6.0), 31)
    run = dict(alg=6, b=8, eps_abs=1e-6 * np.linalg.norm(a, 2), seed=12, max_rank=200)
    ref = _single(qbfac.MatrixHandle.dense(a, qbfac.default_context()), **run)
    ctxs = _local_group(world)
    plan = dist.plan_dense_rows(a.shape[0], world, align=8)
    hs = [qbfac.MatrixHandle.dense_shard(dist.shard_dense(a, r0, rows), a.shape[0], r0, ctxs[g])
          for g, (r0, rows) in enumerate(plan)]
    shards = _run_ranks(hs, **run)
    for s in shards:
        assert (s[0], s[1], s[2]) == ref[:3]
        assert np.array_equal(s[5], shards[0][5])
    qs = np.vstack([s[4] for s in shards])
    assert np.abs(qs.T @ qs - np.eye(qs.shape[1])).max() < 1e-10
    sg, sr = np.linalg.svd(shards[0][5], compute_uv=False), np.linalg.svd(ref[5], compute_uv=False)
    assert np.max(np.abs(sg - sr) / sr) < 1e-8


def test_sharded_qb_to_svd():
    """qb_to_svd on a row-sharded result: B^T is replicated, so every rank forms the same
    r x r factor and Jacobi rotations (deterministic) and returns its own rows of U; stacked,
    they equal the unsharded U S V^T."""
    a = matgen.synthesize(600, 300, matgen.spectrum("exp_decay", 300, tau=9.0), 41)
    run = dict(alg=0, mode=0, b=20, power=1, k=60, s=0, seed=3)
    single = qbfac.run_device(qbfac.MatrixHandle.dense(a, qbfac.default_context()), **run)
    ref = single.svd(40)
    single.free()
    ctxs = _local_group(2)
    plan = dist.plan_dense_rows(a.shape[0], 2, align=8)
    hs = [qbfac.MatrixHandle.dense_shard(dist.shard_dense(a, r0, rows), a.shape[0], r0, ctxs[g])
          for g, (r0, rows) in enumerate(plan)]
    out, errs = [None, None], []

    def work(r):
        try:
            res = qbfac.run_device(hs[r], **run)
            out[r] = res.svd(40)
            res.free()
        except Exception as ex:  # pragma: no cover
            errs.append(repr(ex))
    ths = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=300)
    assert not errs, errs
    assert np.array_equal(out[0].S, out[1].S) and np.array_equal(out[0].V, out[1].V)
    u = np.vstack([out[0].U, out[1].U])
    np.testing.assert_allclose(out[0].S, ref.S, rtol=1e-10)
    lr = ref.U @ np.diag(ref.S) @ ref.V.T
    assert np.linalg.norm(u @ np.diag(out[0].S) @ out[0].V.T - lr) <= 1e-9 * np.linalg.norm(lr)
    assert np.abs(u.T @ u - np.eye(40)).max() < 1e-10


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("P", [0, 2])
def test_column_sharded_n_side_matches_replicated(world, P, monkeypatch):
    """randQB_EI at world > 1 keeps B (and every n-side block) column-sharded: A^T passes
    reduce-scatter, B X products are partial sums allreduced, Z is all-gathered for the A Z pass,
    B is gathered at the end. Same rank / passes / termination as the replicated-B run
    (QBFAC_NSHARD=0) and as the unsharded run, B bitwise identical on every rank, sigma(B) and
    ||A - QB|| as the unsharded run. Zipf CSR with a hybrid (dense rows / columns) split, as config 5."""
    csr = matgen.csr_zipf(6000, 1500, alpha=1.1, target_nnz=90000, seed=17)
    a = matgen.csr_to_dense(csr)
    eps = 0.6 * np.linalg.norm(a)
    run = dict(alg=0, b=20, power=P, max_rank=300, eps_abs=eps, seed=7)
    ref = _single(qbfac.MatrixHandle.csr(*csr, ctx=qbfac.default_context()), **run)
    plan = dist.plan_csr_rows(csr[2], world)

    def sharded(nsh):
        monkeypatch.setenv("QBFAC_NSHARD", nsh)
        ctxs = _local_group(world)
        hs = []
        for g, (r0, rows) in enumerate(plan):
            loc = dist.shard_csr(csr, r0, rows)
            hs.append(qbfac.MatrixHandle.csr_shard(csr[0], r0, csr[1], loc[2], loc[3], loc[4], ctxs[g]))
        return _run_ranks(hs, **run)
    col = sharded("1")
    rep = sharded("0")
    _check(a, ref, col, 1e-10)
    assert (col[0][0], col[0][1], col[0][2]) == (rep[0][0], rep[0][1], rep[0][2])
    sc = np.linalg.svd(col[0][5], compute_uv=False)
    sr = np.linalg.svd(rep[0][5], compute_uv=False)
    assert np.max(np.abs(sc - sr) / sr) < 1e-10
