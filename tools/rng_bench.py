"""Time the device Gaussian generator for several sizes (CUDA events on the library stream)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1606_09402_b200 import qbfac
    ctx = qbfac.default_context()
    L = qbfac.lib()
    stream = torch.cuda.ExternalStream(ctx.stream())
    for rows, cols in [(2000, 20), (20000, 20), (50000, 50), (200000, 50), (8000, 2000)]:
        out = torch.empty((cols, rows), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        for _ in range(2):
            L.qbfac_gpu_gaussian_device(ctx.handle, 42, 0, 12345, rows, cols, C.c_void_p(out.data_ptr()), rows)
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            L.qbfac_gpu_gaussian_device(ctx.handle, 42, 0, 12345, rows, cols, C.c_void_p(out.data_ptr()), rows)
        e1.record(stream)
        ctx.synchronize()
        t = e0.elapsed_time(e1) / 5 * 1e3
        print(f"{rows}x{cols}: {t:8.1f} us  {rows * cols / t / 1e3:8.2f} Gnormal/s", flush=True)


if __name__ == "__main__":
    main()
