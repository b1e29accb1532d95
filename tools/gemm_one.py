"""Run one GEMM shape (for ncu): python tools/gemm_one.py M N K a_row b_row c_row [reps]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1606_09402_b200 import qbfac  # noqa: E402

M, N, K, ar, br, cr = (int(x) for x in sys.argv[1:7])
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 2
L = qbfac.lib()
P, I64, D, I = C.c_void_p, C.c_int64, C.c_double, C.c_int
L.qbfac_gpu_test_gemm.argtypes = [P, D, P, I64, I64, I64, I, P, I64, I64, I, D, P, I64, I]
ctx = qbfac.default_context()
a = torch.randn(M * K, dtype=torch.float64, device="cuda")
b = torch.randn(K * N, dtype=torch.float64, device="cuda")
c = torch.zeros(M * N, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for _ in range(reps):
    st = L.qbfac_gpu_test_gemm(ctx.handle, 1.0, C.c_void_p(a.data_ptr()), M, K, K if ar else M, ar,
                               C.c_void_p(b.data_ptr()), N, N if br else K, br, 0.0, C.c_void_p(c.data_ptr()),
                               N if cr else M, cr)
    assert st == 0
print("ok")
