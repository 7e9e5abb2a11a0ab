"""Locate mismatches between the two-level fused kernel and two single-level launches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF97, Transform, build_scheme
shapes = [tuple(int(v) for v in s.split("x")) for s in os.environ.get("SHAPES", "16384x16384,4096x4096,8192x8192").split(",")]
tr = Transform(build_scheme(os.environ.get("SCHEME", "non-separable-split"), CDF97), "single",
               fast=os.environ.get("FAST") == "1")
for (h, w) in shapes:
    x = torch.rand((h, w), device="cuda", generator=torch.Generator(device="cuda").manual_seed(h + w))
    got = tr.forward2(x)
    ll0, hl0, lh0, hh0 = tr.forward(x)
    want = (hl0, lh0, hh0) + tuple(tr.forward(ll0.contiguous()))
    for name, g, wv in zip(("hl0", "lh0", "hh0", "ll1", "hl1", "lh1", "hh1"), got[0] + got[1], want):
        d = (g != wv).nonzero()
        if d.numel():
            rows = d[:, 0].unique(); cols = d[:, 1].unique()
            print((h, w), name, d.shape[0], "px rows", rows[:8].tolist(), "..", rows[-4:].tolist(),
                  "cols", cols[:8].tolist(), "..", cols[-4:].tolist(), flush=True)
    print((h, w), "checked", flush=True)
