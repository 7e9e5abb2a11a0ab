"""Small fixed workload for ncu captures: N forward launches of one config."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF53, CDF97, Transform, build_scheme
scheme = sys.argv[1] if len(sys.argv) > 1 else "non-separable-split"
fast = (sys.argv[2] == "fast") if len(sys.argv) > 2 else False
n = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
tr = Transform(build_scheme(scheme, CDF97), "single", fast=fast)
x = torch.rand((n, n), device="cuda")
outs = tr.forward(x)
for _ in range(4):
    tr.forward(x, out=outs)
torch.cuda.synchronize()
print("ok", tr.fwd_plan.key, fast)
