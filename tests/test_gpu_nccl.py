"""The NCCL transport of the row-sharded engine, on real hardware.

* One GPU: a one-rank NCCL communicator (qbfac_gpu_create_dist(dev, 0, 1, id), bootstrapped
  through torch.distributed exactly as bench.py does) — ncclCommInitRank and ncclAllReduce
  run on the device; a factorization through that context equals the plain one.
* Two or more GPUs (skipped otherwise): two processes, one GPU each, NCCL over NVLink, the
  config-1 recipe row-sharded; both ranks must match the oracle and agree bitwise on B.
"""
import ctypes as C
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_one_rank_communicator():
    import torch
    from paper_1606_09402_b200 import matgen, qbfac
    uid = qbfac.Context.nccl_unique_id()
    assert len(uid) == 128
    ctx = qbfac.Context(0, 0, 1, uid)
    L = qbfac.lib()
    L.qbfac_gpu_test_allreduce.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    x = torch.arange(1000, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ctx.check(L.qbfac_gpu_test_allreduce(ctx.handle, C.c_void_p(x.data_ptr()), 1000))
    assert torch.equal(x, torch.arange(1000, dtype=torch.float64, device="cuda"))
    L.qbfac_gpu_test_collective.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int64]
    for op in (1, 2):  # ncclReduceScatter / ncclAllGather on the one-rank communicator: identity
        y = torch.zeros(1000, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        ctx.check(L.qbfac_gpu_test_collective(ctx.handle, op, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), 1000))
        assert torch.equal(x, y)
    a = matgen.synthesize(400, 300, matgen.spectrum("exp_decay", 300, tau=9.0), 3)
    eps = 1e-5 * np.linalg.norm(a)
    plain = qbfac.rand_qb_ei(qbfac.MatrixHandle.dense(a, qbfac.default_context()),
                             qbfac.StopRule.fixed_precision(eps), 10, 1, qbfac.RngStream(8))
    nccl = qbfac.rand_qb_ei(qbfac.MatrixHandle.dense_shard(a, 400, 0, ctx), qbfac.StopRule.fixed_precision(eps),
                            10, 1, qbfac.RngStream(8))
    assert nccl.rank == plain.rank and nccl.passes == plain.passes
    assert np.array_equal(nccl.B, plain.B) and np.array_equal(nccl.Q, plain.Q)
    ctx.close()


_WORKER = r"""
import os, sys, json
import numpy as np
sys.path.insert(0, {root!r})
import torch, torch.distributed as dist
from paper_1606_09402_b200 import dist as qd, matgen, qbfac
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
ctx = qd.sharded_context(rank)
a = matgen.cfg1_matrix()
eps = 1e-2 * np.linalg.norm(a)
row0, rows = qd.plan_dense_rows(a.shape[0], world)[rank]
h = qbfac.MatrixHandle.dense_shard(a[row0:row0 + rows], a.shape[0], row0, ctx)
r = qbfac.rand_qb_ei(h, qbfac.StopRule.fixed_precision(eps), 20, 0, qbfac.RngStream(42), max_rank=1000)
np.save(os.path.join({out!r}, f"q{{rank}}.npy"), r.Q)
np.save(os.path.join({out!r}, f"b{{rank}}.npy"), r.B)
json.dump({{"rank": r.rank, "passes": r.passes, "E": r.error_indicator, "term": r.terminated_by, "row0": row0}},
          open(os.path.join({out!r}, f"r{{rank}}.json"), "w"))
dist.destroy_process_group()
"""


def test_nccl_two_ranks_cfg1(oracle, tmp_path):
    import json
    import subprocess

    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (NCCL over NVLink); the one-rank test covers the transport on one GPU")
    from paper_1606_09402_b200 import matgen
    port = _free_port()
    code = _WORKER.format(root=ROOT, out=str(tmp_path))
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", code], env=env))
    for p in procs:
        assert p.wait(timeout=600) == 0
    res = [json.load(open(tmp_path / f"r{r}.json")) for r in range(2)]
    a = matgen.cfg1_matrix()
    eps = 1e-2 * np.linalg.norm(a)
    ref = oracle.run("ei", a, b=20, power=0, eps_abs=eps, max_rank=1000, seed=42)
    b0, b1 = np.load(tmp_path / "b0.npy"), np.load(tmp_path / "b1.npy")
    assert np.array_equal(b0, b1)  # replicated B bitwise identical on every rank
    for r in res:
        assert r["rank"] == ref.rank and r["passes"] == ref.passes and r["term"] == ref.terminated_by
    q = np.vstack([np.load(tmp_path / "q0.npy"), np.load(tmp_path / "q1.npy")])
    s, sr = np.linalg.svd(b0, compute_uv=False), np.linalg.svd(ref.B, compute_uv=False)
    assert np.max(np.abs(s - sr) / sr) < 1e-10
    e_g, e_r = oracle.explicit_error(q, b0, a=a), oracle.explicit_error(ref.Q, ref.B, a=a)
    assert abs(e_g - e_r) <= 1e-10 * e_r
