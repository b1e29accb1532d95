"""Host-side checks that run without a GPU: the C-ABI library loads and exports every
symbol its headers declare, compute entry points fail loudly without a device (no CPU
fallback), the harness generators, and the row-sharding plan + collective pattern of
the multi-GPU path on a world_size-2 gloo group.
"""
import ctypes as C
import os
import re
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(qbfac_gpu_\w+)\s*\(", txt)))


@pytest.mark.parametrize("header", ["qbfac_gpu.h", "qbfac_gpu_testing.h"])
def test_library_exports_every_declared_symbol(header):
    from paper_1606_09402_b200 import qbfac
    lib = C.CDLL(qbfac.library_path())
    names = _declared(header)
    assert len(names) >= 5
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_only():
    import subprocess
    from paper_1606_09402_b200 import qbfac
    out = subprocess.run(["cuobjdump", "--list-elf", qbfac.library_path()], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1606_09402_b200 import qbfac
    with pytest.raises(qbfac.Error):
        qbfac.Context(0)


def test_validate_epsilon_c_abi_matches_oracle(oracle):
    from paper_1606_09402_b200 import qbfac
    for eps, fa, d in [(2.2e-7, 1.0, 0.01), (1e-8, 1.0, 0.01), (1.0, 3.0, 1.0), (5e-7, 2.5, 0.01)]:
        assert qbfac.validate_epsilon(eps, fa, d) == oracle.validate_epsilon(eps, fa, d)


def test_nccl_unique_id_on_host():
    from paper_1606_09402_b200 import qbfac
    a = qbfac.Context.nccl_unique_id()
    b = qbfac.Context.nccl_unique_id()
    assert len(a) == 128 and a != b


def test_matgen_csr_uniform_valid(oracle):
    from paper_1606_09402_b200 import matgen
    csr = matgen.csr_uniform(500, 300, 17, seed=3)
    m, n, rp, ci, v = csr
    assert oracle.csr_validate(m, n, rp, ci, v) == "ok"
    assert np.all(np.diff(rp) == 17) and np.all((v >= 0) & (v < 1))


def test_matgen_csr_zipf_small(oracle):
    from paper_1606_09402_b200 import matgen
    csr = matgen.csr_zipf(2000, 800, alpha=1.1, target_nnz=30000, seed=5)
    m, n, rp, ci, v = csr
    assert oracle.csr_validate(m, n, rp, ci, v) == "ok"
    lens = np.diff(rp)
    assert lens.min() >= 1 and lens.max() == n          # densest rows take every column
    assert np.all(v > 0)                                 # log(1+k), k >= 1: no explicit zeros
    assert 0.5 * 30000 < len(v) < 1.1 * 30000


# ---- row sharding ------------------------------------------------------------------------
def test_plan_dense_rows():
    from paper_1606_09402_b200 import dist
    for m, w in [(40000, 8), (40000, 3), (100, 4), (7, 2)]:
        plan = dist.plan_dense_rows(m, w)
        assert sum(r for _, r in plan) == m and plan[0][0] == 0
        for (r0, r), (r1, _) in zip(plan, plan[1:]):
            assert r0 + r == r1
        if m >= 32 * w:
            assert all(r0 % 32 == 0 for r0, _ in plan)


def test_plan_csr_rows_balances_nnz():
    from paper_1606_09402_b200 import dist, matgen
    csr = matgen.csr_zipf(20000, 3000, alpha=1.1, target_nnz=200000, seed=2)
    plan = dist.plan_csr_rows(csr[2], 8)
    nnz = [int(csr[2][r0 + r] - csr[2][r0]) for r0, r in plan]
    assert sum(nnz) == len(csr[4])
    heavy = int(np.diff(csr[2]).max())
    assert max(nnz) <= sum(nnz) / 8 + heavy + 20000 / 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as tdist

    from paper_1606_09402_b200 import dist, matgen
    try:
        tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        csr = matgen.csr_uniform(900, 400, 11, seed=9)
        m, n = csr[0], csr[1]
        plan = dist.plan_csr_rows(csr[2], world)
        r0, rows = plan[rank]
        loc = dist.shard_csr(csr, r0, rows)
        a_loc = matgen.csr_to_dense(loc)
        a = matgen.csr_to_dense(csr)
        rs = np.random.default_rng(0)
        omega = rs.standard_normal((n, 7))          # replicated (same seed on every rank)
        y_glob = rs.standard_normal((m, 7))
        y_loc = y_glob[r0:r0 + rows]
        # the device engine's exchange steps, emulated with gloo on host tensors:
        g_loc = a_loc @ omega                                   # A_g Omega: no collective
        h = torch.from_numpy(a_loc.T @ y_loc)                   # A^T Y: allreduce n x w
        gram = torch.from_numpy(y_loc.T @ y_loc)                # Y^T Y: allreduce b x b
        fro = torch.tensor([float((loc[4] ** 2).sum())], dtype=torch.float64)
        for t in (h, gram, fro):
            tdist.all_reduce(t)
        ok = (np.allclose(g_loc, (a @ omega)[r0:r0 + rows], rtol=0, atol=1e-12)
              and np.abs(h.numpy() - a.T @ y_glob).max() < 1e-12
              and np.abs(gram.numpy() - y_glob.T @ y_glob).max() < 1e-11
              and abs(fro.item() - float((csr[4] ** 2).sum())) < 1e-10)
        # NCCL id bootstrap through the process group (rank 0 creates, all receive)
        nid = dist.nccl_bootstrap(rank)
        ids = [None] * world
        tdist.all_gather_object(ids, nid)
        ok = ok and len(nid) == 128 and all(x == ids[0] for x in ids)
        rows_all = [None] * world
        tdist.all_gather_object(rows_all, (r0, rows))
        ok = ok and sorted(rows_all)[0][0] == 0 and sum(r for _, r in rows_all) == m
        q.put((rank, bool(ok)))
        tdist.destroy_process_group()
    except Exception as ex:  # pragma: no cover
        q.put((rank, repr(ex)))


def test_row_sharded_exchange_pattern_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res
