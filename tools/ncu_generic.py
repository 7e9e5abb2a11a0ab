"""ncu target: the fused generic interpreter (K10) on the reference tests' ASYMMETRIC plan, 4096^2."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fractions import Fraction as F
import torch
from paper_1705_08266_b200 import LiftingPlan, Transform, build_scheme, poly1

asym = LiftingPlan("asym", ((poly1({0: F(-3, 4), -1: F(-1, 4)}), poly1({0: F(1, 8), 1: F(3, 8)})),))
tr = Transform(build_scheme("non-separable-split", asym), "single")
x = torch.rand((4096, 4096), device="cuda")
out = tr.forward(x)
for _ in range(3):
    tr.forward(x, out=out)
torch.cuda.synchronize()
print("ok", tr.fwd_plan.key)
