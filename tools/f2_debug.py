"""Locate mismatches between the two-level fused kernel and two single-level launches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF53, CDF97, SCHEME_NAMES, Transform, build_scheme
shapes = [(1024, 1024), (1032, 1544), (600, 1000), (48, 256), (4096, 8192)]
for wname, plan in (("cdf53", CDF53), ("cdf97", CDF97)):
    for sname in SCHEME_NAMES:
        if wname == "cdf97" and sname == "separable-convolution":
            continue
        tr = Transform(build_scheme(sname, plan), "single")
        for (h, w) in shapes:
            x = torch.rand((h, w), device="cuda", generator=torch.Generator(device="cuda").manual_seed(h + w))
            got = tr.forward2(x)
            ll0, hl0, lh0, hh0 = tr.forward(x)
            want = (hl0, lh0, hh0) + tuple(tr.forward(ll0.contiguous()))
            bad = []
            for name, g, wv in zip(("hl0", "lh0", "hh0", "ll1", "hl1", "lh1", "hh1"), got[0] + got[1], want):
                d = (g != wv).nonzero()
                if d.numel():
                    rows = d[:, 0].unique()
                    cols = d[:, 1].unique()
                    bad.append(f"{name}: {d.shape[0]} px rows {rows[:6].tolist()}..{rows[-3:].tolist()} cols {cols[:6].tolist()}..{cols[-3:].tolist()}")
            print(wname, sname, (h, w), "OK" if not bad else bad, flush=True)
