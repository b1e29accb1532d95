"""Why do the bench's config-4/5 sub-measurements run slower than tools/run_configs.py? Replays
the bench's steps and times config 4 after each."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
from paper_1606_09402_b200 import qbfac
D = bench.Dist()
ctx = qbfac.Context(0)
def c4(tag):
    r = bench.config_dense4(D, ctx)
    print(tag, "cfg4", round(r["time_to_eps_s"] * 1e3, 2), "ms", flush=True)
c4("start")
r3 = bench.config_sparse(D, ctx, 3)
print("cfg3", r3["time_to_eps_s"], flush=True)
c4("after cfg3")
pa = torch.randn((8192, 8192), dtype=torch.float64, device="cuda")
pb = torch.randn((8192, 8192), dtype=torch.float64, device="cuda")
for _ in range(6):
    pa @ pb
torch.cuda.synchronize()
del pa, pb
c4("after cublas")
torch.cuda.empty_cache()
c4("after empty_cache")
host = torch.empty((8000, 8000), dtype=torch.float64, pin_memory=True)
c4("after pinned 512MB")
