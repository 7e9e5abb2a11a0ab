"""The 1-D plans of tests/golden/make_lift1d_golden.py, built with this package."""
from fractions import Fraction as F

from paper_1705_08266_b200 import CDF53, CDF97, LiftingPlan, poly1

PLANS = {
    "cdf53": CDF53,
    "cdf97": CDF97,
    "asym": LiftingPlan("asym", ((poly1({0: F(-3, 4), -1: F(-1, 4)}), poly1({0: F(1, 8), 1: F(3, 8)})),)),
    "wide": LiftingPlan("wide", ((poly1({1: F(1, 16), 0: F(-9, 16), -1: F(-9, 16), -2: F(1, 16)}),
                                  poly1({0: F(1, 4), 1: F(1, 4)})),), scale=(F(2, 3), F(3, 2))),
}
LENGTHS = (2, 4, 6, 10, 34, 130)
