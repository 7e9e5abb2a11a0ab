"""Generic interpreter (K0) vs fused kernels: a custom plan and a built-in one at 4096^2."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fractions import Fraction as F
import torch
from paper_1705_08266_b200 import CDF97, LiftingPlan, Transform, build_scheme, poly1


def timed(fn, reps=20):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    return statistics.median(ts)


n = 4096
x = torch.rand((n, n), device="cuda")
asym = LiftingPlan("asym", ((poly1({0: F(-3, 4), -1: F(-1, 4)}), poly1({0: F(1, 8), 1: F(3, 8)})),))
for name, plan in (("cdf97", CDF97), ("asym", asym)):
    for scheme in ("non-separable-split", "separable-lifting"):
        for kw in (dict(), dict(force_generic=True)):
            tr = Transform(build_scheme(scheme, plan), "single", **kw)
            out = tr.forward(x)
            ms = timed(lambda: tr.forward(x, out=out))
            print(f"{name} {scheme} {'generic' if kw else ('fused' if tr.fwd_plan.fused else 'generic(auto)')}: "
                  f"{ms*1e3:.1f} us = {n*n/ms/1e6:.1f} Gpx/s", flush=True)
