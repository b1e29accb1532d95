"""Launch chol_small for several block widths (for ncu launch lists / captures)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_1606_09402_b200 import qbfac
    L = qbfac.lib()
    L.qbfac_gpu_test_chol.argtypes = [C.c_void_p] * 2 + [C.c_int] + [C.c_void_p] * 3
    ctx = qbfac.default_context()
    for b in (20, 50, 64, 112):
        y = np.random.default_rng(b).standard_normal((4 * b, b))
        g = torch.as_tensor(np.ascontiguousarray((y.T @ y).T), device="cuda")
        r = torch.zeros((b, b), dtype=torch.float64, device="cuda")
        ri = torch.zeros((b, b), dtype=torch.float64, device="cuda")
        st = C.c_int(0)
        torch.cuda.synchronize()
        for _ in range(3):
            L.qbfac_gpu_test_chol(ctx.handle, C.c_void_p(g.data_ptr()), b, C.c_void_p(r.data_ptr()),
                                  C.c_void_p(ri.data_ptr()), C.byref(st))
    print("done")


if __name__ == "__main__":
    main()
