"""Does cutting one huge launch into row-band launches help?  (TLB reach / footprint test)"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF97, Transform, build_scheme

tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=True)


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    return statistics.median(ts)


N = 65536
y = torch.empty((N, N), device="cuda")
for i in range(0, N, 4096):
    y[i:i + 4096].uniform_()
o = tuple(torch.empty((N // 2, N // 2), device="cuda") for _ in range(4))
R = N // 2
for nb in (1, 2, 4, 8, 16, 32, 64):
    def step():
        for b in range(nb):
            r0, r1 = R * b // nb, R * (b + 1) // nb
            tr.forward_rows(y, 0, N, r0, r1, out=tuple(t[r0:r1] for t in o))
    ms = timed(step)
    print(f"C5 in {nb} row bands: {ms:.3f} ms = {N*N/ms/1e6:.1f} Gpx/s, {8*N*N/ms/1e6/6512.3:.3f} of copy", flush=True)
