"""CSR pass A*X / A^T*X of configs 3 and 5 under each L2 eviction-hint mode
(QBFAC_SPMM_HINT = 0..3, read at every launch): CUDA events, warm, same inputs.

  python tools/spmm_hints.py [--configs 3,5] [--modes 0,1,2,3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="3,5")
    ap.add_argument("--modes", default="0,1,2,3")
    args = ap.parse_args()
    import torch

    from paper_1606_09402_b200 import matgen, qbfac
    ctx = qbfac.default_context()
    stream = torch.cuda.ExternalStream(ctx.stream())
    for cfg in (int(c) for c in args.configs.split(",")):
        if cfg == 3:
            csr, w = matgen.csr_uniform(100000, 50000, 50, seed=3), 50
        else:
            csr, w = matgen.csr_zipf(2_000_000, 500_000, alpha=1.1, target_nnz=2e8, seed=5), 100
        h = qbfac.MatrixHandle.csr(*csr, ctx=ctx)
        m, n = h.m, h.n
        for trans in (False, True):
            rin, rout = (m, n) if trans else (n, m)
            torch.manual_seed(cfg + 10 * trans)
            x = torch.randn((rin, w), dtype=torch.float64, device="cuda")
            y = torch.empty((rout, w), dtype=torch.float64, device="cuda")
            ref = None
            for mode in args.modes.split(","):
                os.environ["QBFAC_SPMM_HINT"] = mode
                torch.cuda.synchronize()
                for _ in range(2):
                    h.multiply_device(x.data_ptr(), w, w, trans, y.data_ptr(), w)
                ctx.synchronize()
                reps = 5
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(reps):
                    h.multiply_device(x.data_ptr(), w, w, trans, y.data_ptr(), w)
                e1.record(stream)
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / 1e3 / reps
                same = "" if ref is None else ("bitwise-equal" if torch.equal(ref, y) else "DIFFERENT")
                if ref is None:
                    ref = y.clone()
                print(f"cfg{cfg} {'A^T' if trans else 'A  '}*X w={w} hint={mode}: {t * 1e3:8.3f} ms {same}", flush=True)
        os.environ["QBFAC_SPMM_HINT"] = "0"


if __name__ == "__main__":
    main()
