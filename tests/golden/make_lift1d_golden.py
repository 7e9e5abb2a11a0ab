"""1-D lifting fixtures from the REAL reference (liftfuse.schemes.apply_plan_1d /
invert_plan_1d).  Run in the build container:  python tests/golden/make_lift1d_golden.py"""
import os
import sys
from fractions import Fraction as F

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from liftfuse import schemes as S  # noqa: E402
from liftfuse.laurent import LaurentPoly1  # noqa: E402
from liftfuse.wavelets import CDF53, CDF97  # noqa: E402

P1 = LaurentPoly1
PLANS = {
    "cdf53": CDF53,
    "cdf97": CDF97,
    # wider supports than the CDF family (the reference tests' shapes)
    "asym": S.LiftingPlan("asym", ((P1({0: F(-3, 4), -1: F(-1, 4)}), P1({0: F(1, 8), 1: F(3, 8)})),)),
    "wide": S.LiftingPlan("wide", ((P1({1: F(1, 16), 0: F(-9, 16), -1: F(-9, 16), -2: F(1, 16)}),
                                    P1({0: F(1, 4), 1: F(1, 4)})),), scale=(F(2, 3), F(3, 2))),
}
LENGTHS = (2, 4, 6, 10, 34, 130)
out = {}
rng = np.random.default_rng(11)
for name, plan in PLANS.items():
    for n in LENGTHS:
        x = rng.random(n)
        lo, hi = S.apply_plan_1d(plan, list(x))
        out[f"{name}/{n}/x"] = x
        out[f"{name}/{n}/low"] = np.array(lo)
        out[f"{name}/{n}/high"] = np.array(hi)
        out[f"{name}/{n}/rec"] = np.array(S.invert_plan_1d(plan, lo, hi))
np.savez(os.path.join(os.path.dirname(os.path.abspath(__file__)), "lift1d.npz"), **out)
print(len(out), "arrays")
