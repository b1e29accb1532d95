"""qb_to_svd at cfg3 rank 1000 and cfg2 rank 259: Gram-based block Jacobi (QBFAC_JACOBI_GRAM, inner
sweeps QBFAC_JACOBI_INNER) against the column-rotating block kernel; sigma compared with numpy."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1606_09402_b200 import matgen, qbfac
ctx = qbfac.default_context()
os.environ["QBFAC_JACOBI_TRACE"] = "1"
def run(r3, tag):
    k = r3.rank
    ub = torch.empty((k, r3.info.m), dtype=torch.float64, pin_memory=True).numpy().T
    vb = torch.empty((k, r3.info.n), dtype=torch.float64, pin_memory=True).numpy().T
    sb = np.linalg.svd(r3.b(), compute_uv=False)
    for gram, inner in (("0", "1"), ("1", "1"), ("1", "2")):
        os.environ["QBFAC_JACOBI_GRAM"] = gram
        os.environ["QBFAC_JACOBI_INNER"] = inner
        ts = []
        for _ in range(2):
            t0 = time.perf_counter(); t = r3.svd(k, ub, vb); t1 = time.perf_counter(); ts.append(t1 - t0)
        v = np.asarray(t.V)
        print(f"{tag} gram={gram} inner={inner}: qb_to_svd {1e3*min(ts):.1f} ms, {t.sweeps} sweeps, "
              f"max rel dS vs numpy {np.max(np.abs(t.S-sb)/sb):.2e}, |V^T V - I| {np.abs(v.T @ v - np.eye(k)).max():.2e}", flush=True)
csr = matgen.csr_uniform(100000, 50000, 50, seed=3)
h3 = qbfac.MatrixHandle.csr(*csr, ctx=ctx)
eps3 = 0.5 * float(np.sqrt((csr[4] ** 2).sum()))
run(qbfac.run_device(h3, alg=0, b=50, power=1, max_rank=1000, eps_abs=eps3, seed=42), "cfg3 r=1000")
n = 8000
at = matgen.synthesize_torch(n, n, matgen.spectrum("inv", n), 2)
h = qbfac.MatrixHandle.dense_device(at.data_ptr(), n, n, n, ctx)
eps = 5e-2 * float(torch.linalg.norm(at))
run(qbfac.run_device(h, alg=1, b=50, power=1, max_rank=2000, l_budget=2000, eps_abs=eps, seed=42), "cfg2 r=259")
