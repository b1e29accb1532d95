"""Time the DMMA GEMM on the shapes of the hot path (CUDA events, warm, L2 > input).

  python tools/gemm_bench.py
"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1606_09402_b200 import qbfac
    L = qbfac.lib()
    P, I64, D, I = C.c_void_p, C.c_int64, C.c_double, C.c_int
    L.qbfac_gpu_test_gemm.argtypes = [P, D, P, I64, I64, I64, I, P, I64, I64, I, D, P, I64, I]
    ctx = qbfac.default_context()
    stream = torch.cuda.ExternalStream(ctx.stream())
    shapes = [
        # name, M, N, K, a_row, b_row, c_row
        ("cfg2 G=A*Om  (NN)", 8000, 2000, 8000, 0, 1, 1),
        ("cfg2 H=A^T*G (TN)", 8000, 2000, 8000, 1, 1, 1),
        ("cfg4 G=A*Om", 40000, 400, 20000, 0, 1, 1),
        ("cfg4 H=A^T*G", 20000, 400, 40000, 1, 1, 1),
        ("gram 8000x2000", 2000, 2000, 8000, 0, 1, 0),
        ("X*Rinv 8000x2000", 8000, 2000, 2000, 1, 0, 1),
        ("Q*M 1e5x1000x50", 100000, 50, 1000, 1, 1, 1),
        ("Q^T*Y 1e5x1000x50", 1000, 50, 100000, 0, 1, 1),
        ("cfg1 A*Om 2000x20", 2000, 20, 2000, 0, 1, 1),
        ("Bt^T*Om 5e4x500x50", 500, 50, 50000, 0, 1, 1),
        ("Bt*M 5e4x500x50", 50000, 50, 500, 1, 1, 1),
        ("Y*Rinv 1e5x50x50", 100000, 50, 50, 1, 0, 1),
        ("gram Y^T Y 1e5x50", 50, 50, 100000, 0, 1, 0),
        ("Q*M 1e6x500x100", 1000000, 100, 500, 1, 1, 1),
        ("Q^T*Y 1e6x500x100", 500, 100, 1000000, 0, 1, 1),
        ("Bt^T*Om 5e5x500x100", 500, 100, 500000, 0, 1, 1),
        ("Bt*M 5e5x500x100", 500000, 100, 500, 1, 1, 1),
    ]
    res = {}
    for name, M, N, K, ar, br, cr in shapes:
        a = torch.randn(M * K, dtype=torch.float64, device="cuda")
        b = torch.randn(K * N, dtype=torch.float64, device="cuda")
        c = torch.zeros(M * N, dtype=torch.float64, device="cuda")
        lda = K if ar else M
        ldb = N if br else K
        ldc = N if cr else M
        torch.cuda.synchronize()

        def call():
            st = L.qbfac_gpu_test_gemm(ctx.handle, 1.0, C.c_void_p(a.data_ptr()), M, K, lda, ar,
                                       C.c_void_p(b.data_ptr()), N, ldb, br, 0.0, C.c_void_p(c.data_ptr()), ldc, cr)
            assert st == 0, L.qbfac_gpu_last_error(ctx.handle)
        for _ in range(2):
            call()
        reps = 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            call()
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / reps
        res[name] = {"ms": t * 1e3, "tflops": 2.0 * M * N * K / t / 1e12}
        print(f"{name:24s} {t * 1e3:9.3f} ms {2.0 * M * N * K / t / 1e12:7.2f} TF/s", flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", "gemm_bench.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
