"""Tiny check of the fused generic interpreter against the per-sub-step one."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fractions import Fraction as F
import torch
from paper_1705_08266_b200 import CDF97, LiftingPlan, Transform, build_scheme, poly1

asym = LiftingPlan("asym", ((poly1({0: F(-3, 4), -1: F(-1, 4)}), poly1({0: F(1, 8), 1: F(3, 8)})),))
for n in (34, 130):
    x = torch.rand((n, n + 4), device="cuda")
    for plan in (asym, CDF97):
        s = build_scheme("non-separable-split", plan)
        a = Transform(s, "single", force_generic=True)          # fused generic tile
        b = Transform(s, "single", force_generic=True, tile=False)  # per-sub-step
        ya, yb = a.forward(x), b.forward(x)
        torch.cuda.synchronize()
        print(n, plan.name, all(torch.equal(u, v) for u, v in zip(ya, yb)), flush=True)
