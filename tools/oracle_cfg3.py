"""Full-size config-3 oracle run (CPU, reference kernels + restated EI): writes
tests/golden/cfg3_full_oracle.json (rank, E, ||A||^2, passes, sigma(B), explicit error)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from oracle import oracle as O  # noqa: E402
from paper_1606_09402_b200 import matgen  # noqa: E402
from run_configs import csr_explicit_error  # noqa: E402

csr = matgen.csr_uniform(100000, 50000, 50, seed=3)
eps = 0.5 * float(np.sqrt((csr[4] ** 2).sum()))
t0 = time.time()
r = O.run("ei", csr=csr, b=50, power=1, eps_abs=eps, max_rank=1000, seed=42)
t = time.time() - t0
s = np.linalg.svd(r.B, compute_uv=False)
out = {"config": "cfg3 full: EI CSR 1e5x5e4 (50/row, seed 3), b=50, P=1, eps=0.5 rel, cap 1000, Omega seed 42",
       "rank": r.rank, "E": r.E, "norm_a_sq": r.norm_a_sq, "passes": r.passes, "terminated_by": r.terminated_by,
       "sigma": s.tolist(), "explicit_error": csr_explicit_error(csr, r.Q, r.B), "e_trace": r.e_trace.tolist(),
       "oracle_seconds": t, "lane": O.lane_name()}
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "cfg3_full_oracle.json"), "w"))
print("done", t)
