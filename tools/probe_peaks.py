"""Probe FP64 peaks on the B200 box (cuBLAS DGEMM = the FP64 roofline denominator).

Writes gpurun_out/fp64_peaks.json. Not part of the product path.
"""
import json, os, subprocess, time
import torch

def bench(fn, iters=10):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(iters):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best

out = {"gpu": torch.cuda.get_device_name(0)}
p = torch.cuda.get_device_properties(0)
out["sms"] = p.multi_processor_count
out["mem_gb"] = p.total_memory / 1e9
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    t = bench(lambda: a @ b)
    out[f"dgemm_{n}_tflops"] = 2 * n**3 / t / 1e12
# sustained: back to back 3 s
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); t0 = time.time(); k = 0
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True); s.record()
while time.time() - t0 < 3.0:
    a @ b; k += 1
    if k % 4 == 0: torch.cuda.synchronize()
e.record(); torch.cuda.synchronize()
out["dgemm_8192_sustained_tflops"] = 2 * 8192**3 * k / (s.elapsed_time(e) / 1e3) / 1e12
# tall-skinny shapes on the path
for (m, n, w) in ((8000, 8000, 2000), (40000, 20000, 400), (2000, 2000, 20)):
    A = torch.randn(n, m, dtype=torch.float64, device="cuda").t()  # col-major m x n
    X = torch.randn(w, n, dtype=torch.float64, device="cuda").t()
    t = bench(lambda: A @ X)
    out[f"dgemm_nn_{m}x{n}x{w}_tflops"] = 2 * m * n * w / t / 1e12
    G = torch.randn(w, m, dtype=torch.float64, device="cuda").t()
    t = bench(lambda: A.t() @ G)
    out[f"dgemm_tn_{m}x{n}x{w}_tflops"] = 2 * m * n * w / t / 1e12
x = torch.empty(2 * 1024**3 // 8, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
t = bench(lambda: y.copy_(x))
out["copy_gbs"] = 2 * x.numel() * 8 / t / 1e9
out["nproc"] = os.cpu_count()
try:
    out["lscpu_model"] = [l for l in subprocess.check_output(["lscpu"], text=True).splitlines() if "Model name" in l][0]
except Exception as ex:
    out["lscpu_model"] = str(ex)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/fp64_peaks.json", "w"), indent=1)
print(json.dumps(out, indent=1))
