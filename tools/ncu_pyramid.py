"""C3 pyramid workload for ncu: a few device pyramids (dwt_into) of one 16384^2 image.

Launch order per pyramid: L0 band 0, L0 band 1, L1, L2, L3 (stream_kernel), L4 (tile_kernel).
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF97, Transform, build_scheme
n = int(os.environ.get("N", "16384"))
fast = os.environ.get("FAST", "1") == "1"
reps = int(os.environ.get("REPS", "3"))
tr = Transform(build_scheme(os.environ.get("SCHEME", "non-separable-split"), CDF97), "single", fast=fast)
x = torch.rand((n, n), device="cuda")
for _ in range(reps):
    ll, det = tr.dwt(x, 5)
torch.cuda.synchronize()
print("ok", tr.fwd_plan.key, fast)
