"""Run the cooperative blocked Cholesky once at l (for ncu): python tools/chol_wide_one.py [l] [reps]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1606_09402_b200 import qbfac  # noqa: E402

l = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
L = qbfac.lib()
L.qbfac_gpu_test_chol_wide.argtypes = [C.c_void_p] * 2 + [C.c_int] + [C.c_void_p] * 3
ctx = qbfac.default_context()
y = torch.randn((3 * l, l), dtype=torch.float64, device="cuda")
g0 = (y.T @ y).contiguous()
r = torch.zeros((l, l), dtype=torch.float64, device="cuda")
ri = torch.zeros((l, l), dtype=torch.float64, device="cuda")
bd = C.c_int(0)
st = torch.cuda.ExternalStream(ctx.stream())
for i in range(reps):
    g = g0.clone()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    assert L.qbfac_gpu_test_chol_wide(ctx.handle, C.c_void_p(g.data_ptr()), l, C.c_void_p(r.data_ptr()),
                                      C.c_void_p(ri.data_ptr()), C.byref(bd)) == 0
    e1.record(st)
    torch.cuda.synchronize()
    print(f"l={l} chol_wide {e0.elapsed_time(e1):.3f} ms (incl. memsets + status read)")
rr = r.cpu().numpy().T
print("resid", np.linalg.norm(rr.T @ rr - g0.cpu().numpy()) / np.linalg.norm(g0.cpu().numpy()))
