import time, numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
from paper_1606_09402_b200 import qbfac, matgen
n = 8000
ctx = qbfac.default_context()
at = matgen.synthesize_torch(n, n, matgen.spectrum("inv", n), 2)
host = torch.empty((n, n), dtype=torch.float64, pin_memory=True); host.copy_(at.cpu())
dev = torch.empty_like(at)
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); dev.copy_(host, non_blocking=True); torch.cuda.synchronize()
    print("H2D 512MB pinned: %.2f ms (%.1f GB/s)" % ((time.perf_counter()-t0)*1e3, 512e6/(time.perf_counter()-t0)/1e9))
a_view = host.numpy().T
eps = 5e-2 * float(torch.linalg.norm(at))
for mode in ("dense", "dense_async"):
    for _ in range(3):
        ctx.synchronize(); t0 = time.perf_counter()
        h = getattr(qbfac.MatrixHandle, mode)(a_view, ctx); t1 = time.perf_counter()
        r = qbfac.run_device(h, alg=1, b=50, power=1, max_rank=2000, l_budget=2000, eps_abs=eps, seed=42); t2 = time.perf_counter()
        q = r.q(); b = r.b(); t3 = time.perf_counter()
        r.free(); h.free(); ctx.synchronize(); t4 = time.perf_counter()
        print(f"{mode}: handle {1e3*(t1-t0):.1f} run {1e3*(t2-t1):.1f} (device {qbfac.info_dict(r.info)['device_ms']:.1f}) d2h {1e3*(t3-t2):.1f} free {1e3*(t4-t3):.1f} total {1e3*(t4-t0):.1f} ms")
