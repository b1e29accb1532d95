"""One factorization of a BASELINE config between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists and captures.

  python tools/profile_run.py --config 2 [--warmup 1] [--pass-only]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--pass-only", action="store_true", help="profile one dense pass only")
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_1606_09402_b200 import matgen, qbfac

    ctx = qbfac.default_context()
    if args.config == 2:
        n = 8000
        at = matgen.synthesize_torch(n, n, matgen.spectrum("inv", n), 2)
        h = qbfac.MatrixHandle.dense_device(at.data_ptr(), n, n, n, ctx)
        eps = 5e-2 * float(torch.linalg.norm(at))
        run = lambda: qbfac.run_device(h, alg=1, b=50, power=1, max_rank=2000, l_budget=2000, eps_abs=eps, seed=42)
        w = 2000
    elif args.config == 1:
        a = matgen.cfg1_matrix()
        h = qbfac.MatrixHandle.dense(a, ctx)
        eps = 1e-2 * float(np.linalg.norm(a))
        n = 2000
        run = lambda: qbfac.run_device(h, alg=0, b=20, power=0, max_rank=1000, eps_abs=eps, seed=42)
        w = 20
    elif args.config == 3:
        csr = matgen.csr_uniform(100000, 50000, 50, seed=3)
        h = qbfac.MatrixHandle.csr(*csr, ctx=ctx)
        eps = 0.5 * float(np.sqrt((csr[4] ** 2).sum()))
        n = 50000
        run = lambda: qbfac.run_device(h, alg=0, b=50, power=1, max_rank=1000, eps_abs=eps, seed=42)
        w = 50
    elif args.config == 4:
        m, n = 40000, 20000
        sig = np.exp(-np.arange(1, 401) / 60.0)
        at = matgen.synthesize_torch(m, n, sig, 4, noise=1e-6)
        h = qbfac.MatrixHandle.dense_device(at.data_ptr(), m, n, m, ctx)
        run = lambda: qbfac.run_device(h, alg=3, mode=0, b=100, k=400, s=0, seed=42)
        w = 400
    else:
        csr = matgen.csr_zipf(2_000_000, 500_000, alpha=1.1, target_nnz=2e8, seed=5)
        h = qbfac.MatrixHandle.csr(*csr, ctx=ctx)
        eps = 0.6 * float(np.sqrt((csr[4] ** 2).sum()))
        run = lambda: qbfac.run_device(h, alg=0, b=100, power=2, max_rank=2000, eps_abs=eps, seed=42)
        w = 100
    if args.pass_only:
        x = torch.randn((h.n, w), dtype=torch.float64, device="cuda")
        y = torch.empty((h.m, w), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        run = lambda: h.multiply_device(x.data_ptr(), w, w, False, y.data_ptr(), w)
    for _ in range(args.warmup):
        r = run()
        if r is not None:
            r.free()
    ctx.synchronize()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    t0 = time.perf_counter()
    r = run()
    ctx.synchronize()
    t1 = time.perf_counter()
    torch.cuda.profiler.stop()
    if r is not None:
        print("info", qbfac.info_dict(r.info))
    print(f"wall {1e3 * (t1 - t0):.3f} ms")


if __name__ == "__main__":
    main()
