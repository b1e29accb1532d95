"""Run the fused CholQR2 panel kernel on rows x b (for traces / ncu): python tools/panel_one.py rows b [reps]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1606_09402_b200 import qbfac  # noqa: E402

rows, b = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
L = qbfac.lib()
L.qbfac_gpu_test_cholqr2.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_void_p,
                                     C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
ctx = qbfac.default_context()
y = torch.randn((rows, b), dtype=torch.float64, device="cuda")
q = torch.empty_like(y)
r = torch.zeros((112, 112), dtype=torch.float64, device="cuda")
ri = torch.zeros_like(r)
st = C.c_int(0)
for _ in range(reps):
    torch.cuda.synchronize()
    assert L.qbfac_gpu_test_cholqr2(ctx.handle, C.c_void_p(y.data_ptr()), rows, b, b, C.c_void_p(q.data_ptr()), b,
                                    C.c_void_p(r.data_ptr()), C.c_void_p(ri.data_ptr()), C.byref(st)) == 0
print("ok")
