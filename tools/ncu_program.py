"""ncu target: one forward or inverse of one built-in program on an N x N f32 image.
    python tools/ncu_program.py <wavelet> <scheme> <fwd|inv> [N]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF53, CDF97, Transform, build_scheme

wavelet, scheme, direction = sys.argv[1:4]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 8192
tr = Transform(build_scheme(scheme, {"cdf53": CDF53, "cdf97": CDF97}[wavelet]), "single", fast=True)
x = torch.rand((n, n), device="cuda")
q = tr.forward(x)
torch.cuda.synchronize()
if direction == "fwd":
    tr.forward(x, out=q)
else:
    tr.inverse(*q, out=x)
torch.cuda.synchronize()
print("ok", tr.fwd_plan.key if direction == "fwd" else tr.inv_plan.key)
