"""Config-2 e2e (pinned host A -> Q, B on the host) against the row-chunk size of the asynchronous
upload (qbfac_gpu_matrix_dense_async): python tools/e2e_chunk_sweep.py [chunk_rows ...]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import pinned_inputs  # noqa: E402
from paper_1606_09402_b200 import qbfac  # noqa: E402

chunks = [int(x) for x in sys.argv[1:]] or [0, 512, 640, 768, 896, 1024, 1152, 1280, 1536, 2048]
a, _ = pinned_inputs.matrix(2)
n = a.shape[0]
eps = 5e-2 * float(np.linalg.norm(a))
ctx = qbfac.Context(0)
host_a = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
host_a.numpy()[:] = np.asarray(a).T
a_view = host_a.numpy().T
q_out = torch.empty(n * 2000, dtype=torch.float64, pin_memory=True).numpy()
b_out = torch.empty(n * 2000, dtype=torch.float64, pin_memory=True).numpy()


def once(chunk):
    ctx.synchronize()
    t0 = time.perf_counter()
    h = qbfac.MatrixHandle.dense_async(a_view, ctx, chunk_rows=chunk)
    r = qbfac.run_device(h, alg=1, b=50, power=1, max_rank=2000, l_budget=2000, eps_abs=eps, seed=42)
    r.q(q_out)
    r.b(b_out)
    rank = qbfac.info_dict(r.info)["rank"]
    r.free()
    h.free()
    ctx.synchronize()
    return time.perf_counter() - t0, rank


for rep in range(2):
    for c in chunks:
        ts = [once(c) for _ in range(6)]
        print(f"chunk_rows {c:5d}: e2e median {np.median([t for t, _ in ts[1:]]) * 1e3:.3f} ms "
              f"(min {min(t for t, _ in ts[1:]) * 1e3:.3f}), rank {ts[-1][1]}", flush=True)
