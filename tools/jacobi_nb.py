"""qb_to_svd device time vs the Jacobi block width (QBFAC_JACOBI_NB, read per call), cfg3 rank 1000."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1606_09402_b200 import matgen, qbfac
ctx = qbfac.default_context()
csr = matgen.csr_uniform(100000, 50000, 50, seed=3)
h3 = qbfac.MatrixHandle.csr(*csr, ctx=ctx)
eps3 = 0.5 * float(np.sqrt((csr[4] ** 2).sum()))
r3 = qbfac.run_device(h3, alg=0, b=50, power=1, max_rank=1000, eps_abs=eps3, seed=42)
k = r3.rank
ub = torch.empty((k, r3.info.m), dtype=torch.float64, pin_memory=True).numpy().T
vb = torch.empty((k, r3.info.n), dtype=torch.float64, pin_memory=True).numpy().T
ref = None
for nb in ("8", "4", "2", "1"):
    os.environ["QBFAC_JACOBI_NB"] = nb
    ts = []
    for _ in range(2):
        t0 = time.perf_counter(); t = r3.svd(k, ub, vb); t1 = time.perf_counter(); ts.append(t1 - t0)
    if ref is None:
        ref = t.S.copy()
    print(f"nb={nb}: qb_to_svd {1e3*min(ts):.1f} ms, {t.sweeps} sweeps, max rel dS vs nb=8 {np.max(np.abs(t.S-ref)/ref):.2e}", flush=True)
