"""One qb_to_svd of config 3's rank-1000 factorization between cudaProfilerStart/Stop (for an ncu launch list):
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file out.csv python tools/svd_profile.py"""
import os, sys
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
r3.svd(k, ub, vb)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
t = r3.svd(k, ub, vb)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("sweeps", t.sweeps)
