"""The skinny DMMA products of config 3's EI block loop (m = 1e5, n = 5e4, b = 50) with the
engine's exact layouts (Q: m x cap row-major, B^T: n x cap row-major, blocks row-major), timed
with CUDA events at several ranks k:
  A  M = Q^T Y      (k x b, K = m)   2 per block
  B  Y -= Q M       (m x b, K = k)   3 per block
  C  M = B Omega    (k x b, K = n)   2 per block
  D  Z -= B^T M     (n x b, K = k)   1 per block

  python tools/gemm_cfg3.py [--b 50] [--m 100000] [--n 50000]
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b", type=int, default=50)
    ap.add_argument("--m", type=int, default=100000)
    ap.add_argument("--n", type=int, default=50000)
    ap.add_argument("--cap", type=int, default=1000)
    ap.add_argument("--only", default="ABCD")
    ap.add_argument("--k", type=int, default=0, help="one rank k only")
    args = ap.parse_args()
    import torch

    from paper_1606_09402_b200 import qbfac
    L = qbfac.lib()
    P, I64, D, I = C.c_void_p, C.c_int64, C.c_double, C.c_int
    L.qbfac_gpu_test_gemm.argtypes = [P, D, P, I64, I64, I64, I, P, I64, I64, I, D, P, I64, I]
    ctx = qbfac.default_context()
    stream = torch.cuda.ExternalStream(ctx.stream())
    m, n, b, cap = args.m, args.n, args.b, args.cap
    lyz = (b + 3) // 4 * 4
    q = torch.randn(m * cap, dtype=torch.float64, device="cuda")
    bt = torch.randn(n * cap, dtype=torch.float64, device="cuda")
    y = torch.randn(m * lyz, dtype=torch.float64, device="cuda")
    z = torch.randn(n * lyz, dtype=torch.float64, device="cuda")
    mv = torch.zeros(cap * b, dtype=torch.float64, device="cuda")

    def ptr(t):
        return C.c_void_p(t.data_ptr())

    def gemm(alpha, a, M, K, lda, ar, bb, N, ldb, br, beta, c, ldc, cr):
        st = L.qbfac_gpu_test_gemm(ctx.handle, alpha, ptr(a), M, K, lda, ar, ptr(bb), N, ldb, br, beta, ptr(c), ldc, cr)
        assert st == 0, L.qbfac_gpu_last_error(ctx.handle)

    def timed(fn, reps=5):
        fn()
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3 / reps

    peak_tf = 35.4
    tot = {"A": 0.0, "B": 0.0, "C": 0.0, "D": 0.0, "E": 0.0}
    ideal = {"A": 0.0, "B": 0.0, "C": 0.0, "D": 0.0, "E": 0.0}
    print(f"m={m} n={n} b={b}: time (us) and TFLOP/s per product", flush=True)
    for k in ([args.k] if args.k else range(50, cap, 50)):
        ops = {
            # Q^T Y: A = Q^T (k x m col-major view of row-major Q, ld cap)
            "A": (lambda: gemm(1.0, q, k, m, cap, 0, y, b, lyz, 1, 0.0, mv, b, 1), 2.0 * m * k * b, 2),
            # Y -= Q M
            "B": (lambda: gemm(-1.0, q, m, k, cap, 1, mv, b, b, 1, 1.0, y, lyz, 1), 2.0 * m * k * b, 3),
            # Y = -Q M (beta = 0: no read of Y)
            "E": (lambda: gemm(-1.0, q, m, k, cap, 1, mv, b, b, 1, 0.0, y, lyz, 1), 2.0 * m * k * b, 0),
            # M = (B^T)^T Omega: A = B^T^T (k x n col-major view, ld cap)
            "C": (lambda: gemm(1.0, bt, k, n, cap, 0, z, b, lyz, 1, 0.0, mv, b, 1), 2.0 * n * k * b, 2),
            # Z -= B^T M
            "D": (lambda: gemm(-1.0, bt, n, k, cap, 1, mv, b, b, 1, 1.0, z, lyz, 1), 2.0 * n * k * b, 1),
        }
        line = []
        for name, (fn, fl, per_block) in ops.items():
            if name not in args.only:
                continue
            t = timed(fn)
            tot[name] += per_block * t
            ideal[name] += per_block * fl / (peak_tf * 1e12)
            line.append(f"{name} {t * 1e6:7.1f} us {fl / t / 1e12:5.1f} TF")
        print(f"k={k:4d}: " + " | ".join(line), flush=True)
    print("per factorization (19 blocks with k > 0): " +
          ", ".join(f"{k} {1e3 * v:.2f} ms (peak {1e3 * ideal[k]:.2f})" for k, v in tot.items()), flush=True)


if __name__ == "__main__":
    main()
