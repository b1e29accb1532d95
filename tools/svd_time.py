"""Time qb_to_svd on the device for config 2 (rank 259) and config 3 (rank 1000)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1606_09402_b200 import matgen, qbfac
ctx = qbfac.default_context()
n = 8000
at = matgen.synthesize_torch(n, n, matgen.spectrum("inv", n), 2)
h = qbfac.MatrixHandle.dense_device(at.data_ptr(), n, n, n, ctx)
eps = 5e-2 * float(torch.linalg.norm(at))
r = qbfac.run_device(h, alg=1, b=50, power=1, max_rank=2000, l_budget=2000, eps_abs=eps, seed=42)
for _ in range(3):
    t0 = time.perf_counter(); t = r.svd(r.rank); t1 = time.perf_counter()
print(f"cfg2 rank {r.rank}: qb_to_svd {1e3*(t1-t0):.1f} ms, {t.sweeps} Jacobi sweeps, S[0]={t.S[0]:.6f} S[-1]={t.S[-1]:.3e} (1/j: {1/r.rank:.3e})")
csr = matgen.csr_uniform(100000, 50000, 50, seed=3)
h3 = qbfac.MatrixHandle.csr(*csr, ctx=ctx)
eps3 = 0.5 * float(np.sqrt((csr[4] ** 2).sum()))
r3 = qbfac.run_device(h3, alg=0, b=50, power=1, max_rank=1000, eps_abs=eps3, seed=42)
for _ in range(2):
    t0 = time.perf_counter(); t = r3.svd(r3.rank); t1 = time.perf_counter()
print(f"cfg3 rank {r3.rank}: qb_to_svd {1e3*(t1-t0):.1f} ms, {t.sweeps} Jacobi sweeps (pageable outputs)")
# pinned outputs: the 1.2 GB of U and V leave at the PCIe rate
k = r3.rank
ub = torch.empty((k, r3.info.m), dtype=torch.float64, pin_memory=True).numpy().T
vb = torch.empty((k, r3.info.n), dtype=torch.float64, pin_memory=True).numpy().T
for _ in range(2):
    t0 = time.perf_counter(); t = r3.svd(k, ub, vb); t1 = time.perf_counter()
gb = 8 * (r3.info.m + r3.info.n) * k / 1e9
print(f"cfg3 rank {k}: qb_to_svd {1e3*(t1-t0):.1f} ms with pinned outputs ({gb:.2f} GB of U, V to the host), "
      f"{t.sweeps} sweeps")
