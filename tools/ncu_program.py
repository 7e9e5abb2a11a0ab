"""One 8192^2 forward of one program (ncu target): SCHEME, WAVELET, FAST env."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF53, CDF97, Transform, build_scheme
plan = CDF97 if os.environ.get("WAVELET", "cdf97") == "cdf97" else CDF53
tr = Transform(build_scheme(os.environ.get("SCHEME", "separable-convolution"), plan), "single",
               fast=os.environ.get("FAST", "1") == "1", tile=False)
x = torch.rand((8192, 8192), device="cuda")
q = tr.forward(x)
for _ in range(3):
    tr.forward(x, out=q)
torch.cuda.synchronize()
print("ok", tr.fwd_plan.key)
