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
# per-step breakdown of the last launch (CTA 0 %globaltimer stamps)
L.qbfac_gpu_test_chol_wide_trace.argtypes = [C.c_void_p, C.c_void_p]
tr = np.zeros((64, 4), dtype=np.uint64)
assert L.qbfac_gpu_test_chol_wide_trace(ctx.handle, tr.ctypes.data) == 0
t = tr.astype(np.int64)
nt = (l + 63) // 64
ph2 = [(t[k, 1] - t[k, 0]) / 1e3 for k in range(nt)]
ph3 = [(t[k, 2] - t[k, 1]) / 1e3 for k in range(nt - 1)]
syn = [(t[k, 3] - t[k, 2]) / 1e3 for k in range(nt - 1)]
print(f"steps {nt}: phase2 sum {sum(ph2):.1f} us (first {ph2[0]:.1f}), phase3(CTA0) sum {sum(ph3):.1f} us "
      f"(first {ph3[0]:.1f}, last {ph3[-1]:.1f}), wait-for-grid sum {sum(syn):.1f} us, "
      f"total {(t[nt - 1, 1] - t[0, 0]) / 1e3:.1f} us")
