"""Median-of-N timing of one forward level (default: C3 level 0, 9/7 split) for A/B tests."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF97, Transform, build_scheme

n = int(os.environ.get("N", "16384"))
scheme = os.environ.get("SCHEME", "non-separable-split")
x = torch.rand((n, n), device="cuda")
res = []
for fast in (False, True):
    tr = Transform(build_scheme(scheme, CDF97), "single", fast=fast)
    o = tr.forward(x)
    for _ in range(5):
        tr.forward(x, out=o)
    ts = []
    for _ in range(30):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); tr.forward(x, out=o); e.record(); e.synchronize()
        ts.append(s.elapsed_time(e))
    res.append(f"{'fast' if fast else 'strict'} med {statistics.median(ts):.4f} min {min(ts):.4f} ms")
print(os.environ.get("TAG", ""), n, " | ".join(res))
