"""Per-phase breakdown of the fused CholQR2 panel kernel (%globaltimer stamps of CTA 0).

  python tools/panel_trace.py [rows b [reps]]   (default: the config-3 and config-1 shapes)
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1606_09402_b200 import qbfac  # noqa: E402

L = qbfac.lib()
L.qbfac_gpu_test_cholqr2.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_void_p,
                                     C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
L.qbfac_gpu_test_panel_trace.argtypes = [C.c_void_p, C.c_void_p]
NAMES = ["gramA", "write_part", "reduceA", "cholA", "barrier", "phaseB", "reduceB", "cholB", "barrier", "phaseD"]


def run(rows, b, reps, near_identity=False):
    ctx = qbfac.default_context()
    y = torch.randn((rows, b), dtype=torch.float64, device="cuda")
    if near_identity:
        y = torch.linalg.qr(y)[0].contiguous()
    q = torch.empty_like(y)
    r = torch.zeros((112, 112), dtype=torch.float64, device="cuda")
    ri = torch.zeros_like(r)
    st = C.c_int(0)
    tr = np.zeros(44, dtype=np.uint64)
    rows_out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        assert L.qbfac_gpu_test_cholqr2(ctx.handle, C.c_void_p(y.data_ptr()), rows, b, b, C.c_void_p(q.data_ptr()),
                                        b, C.c_void_p(r.data_ptr()), C.c_void_p(ri.data_ptr()), C.byref(st)) == 0
        assert L.qbfac_gpu_test_panel_trace(ctx.handle, tr.ctypes.data) == 0
        t = tr.astype(np.int64)
        if near_identity:
            rows_out.append([(t[1] - t[0]) / 1e3, (t[5] - t[1]) / 1e3, (t[11] - t[5]) / 1e3, (t[11] - t[0]) / 1e3])
        else:
            rows_out.append([(t[i + 1] - t[i]) / 1e3 for i in range(10)] + [(t[10] - t[0]) / 1e3])
    med = np.median(np.array(rows_out[1:] or rows_out), axis=0)
    names = ["gramA", "reduce+cholA", "phaseB(one pass)", "total"] if near_identity else NAMES + ["total"]
    print(f"panel {rows}x{b}{' near-identity' if near_identity else ''}: " +
          " ".join(f"{n}={v:.1f}" for n, v in zip(names, med)) + " us", flush=True)
    if not near_identity:
        print(f"  in-panel chol A (clk): " + fmt_chol(tr, b), flush=True)


def chol(b, reps=5):
    """clock64 breakdown of the in-CTA Cholesky (chol_small kernel, one CTA) on a Gaussian Gram."""
    ctx = qbfac.default_context()
    L.qbfac_gpu_test_chol.argtypes = [C.c_void_p] * 2 + [C.c_int] + [C.c_void_p] * 3
    y = np.random.default_rng(b).standard_normal((100000, b))
    g = torch.as_tensor(np.ascontiguousarray((y.T @ y).T), device="cuda")
    r = torch.zeros((b, b), dtype=torch.float64, device="cuda")
    ri = torch.zeros_like(r)
    st = C.c_int(0)
    tr = np.zeros(44, dtype=np.uint64)
    for _ in range(reps):
        L.qbfac_gpu_test_chol(ctx.handle, C.c_void_p(g.data_ptr()), b, C.c_void_p(r.data_ptr()),
                              C.c_void_p(ri.data_ptr()), C.byref(st))
    assert L.qbfac_gpu_test_panel_trace(ctx.handle, tr.ctypes.data) == 0
    print(f"chol b={b} (clk): " + fmt_chol(tr, b), flush=True)


def fmt_chol(tr, b):
    t = tr[12:].astype(np.int64)
    P = (b + 15) // 16
    parts = [("load", t[1] - t[0])]
    prev = t[1]
    for p in range(P):
        for k, nm in ((2, "elim"), (3, "row"), (4, "trail")):
            sl = k + 3 * p
            if t[sl] > prev:
                parts.append((f"{nm}{p}", t[sl] - prev))
                prev = t[sl]
    parts.append(("Rout", t[23] - prev))
    prev = t[23]
    for jb in range(P):
        parts.append((f"inv{jb}", t[24 + jb] - prev))
        prev = t[24 + jb]
    parts.append(("end", t[31] - prev))
    parts.append(("total", t[31] - t[0]))
    return " ".join(f"{n}={v}" for n, v in parts)


if __name__ == "__main__":
    if len(sys.argv) > 2:
        run(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 5)
    else:
        for b in (20, 50, 100):
            chol(b)
        for rows, b in ((100000, 50), (2000, 20), (2000000, 100), (100000, 100)):
            run(rows, b, 6)
            run(rows, b, 6, near_identity=True)
