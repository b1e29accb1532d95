"""Fixed cost of the skinny NN update Y (m x 50) = beta Y - Q (m x k) M (k x 50): time vs k and beta.
  python tools/gemm_nn_probe.py"""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1606_09402_b200 import qbfac
L = qbfac.lib()
P, I64, D, I = C.c_void_p, C.c_int64, C.c_double, C.c_int
L.qbfac_gpu_test_gemm.argtypes = [P, D, P, I64, I64, I64, I, P, I64, I64, I, D, P, I64, I]
ctx = qbfac.default_context()
stream = torch.cuda.ExternalStream(ctx.stream())
N, ldq = 50, 1000
q = torch.randn(400000 * ldq, dtype=torch.float64, device="cuda")
def run(k, beta, ldc, reps=20, M=100000, ldq=1000):
    m = torch.randn(k * N, dtype=torch.float64, device="cuda")
    y = torch.zeros(M * ldc, dtype=torch.float64, device="cuda")
    call = lambda: L.qbfac_gpu_test_gemm(ctx.handle, -1.0, C.c_void_p(q.data_ptr()), M, k, ldq, 1, C.c_void_p(m.data_ptr()), N, N, 1,
                                         beta, C.c_void_p(y.data_ptr()), ldc, 1)
    for _ in range(3): assert call() == 0
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps): call()
    e1.record(stream)
    ctx.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
for beta in (1.0, 0.0):
    print(f"ldc=52 beta={beta}: " + "  ".join(f"k={k}: {run(k, beta, 52):6.1f} us" for k in (32, 64, 128, 250, 500, 1000)), flush=True)
# per launch or per tile? rows scaled at k = 32 and 128 (beta = 0)
for k in (32, 128):
    print(f"k={k} beta=0: " + "  ".join(f"M={M}: {run(k, 0.0, 52, M=M):6.1f} us" for M in (18944, 50000, 100000, 200000, 400000)), flush=True)

# row stride of Q: packed (ld = k) vs the engine's ld = cap = 1000, beta = 0
for k in (32, 128, 500):
    print(f"k={k} beta=0: " + "  ".join(f"ldq={l}: {run(k, 0.0, 52, ldq=l):6.1f} us" for l in (k, 512 if k < 512 else 504, 1000, 1024)), flush=True)
