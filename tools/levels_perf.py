"""Per-level and graph timing of the C3 pyramid (medians), for tuning small levels."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF97, Transform, build_scheme
n = 16384
fast = os.environ.get("FAST", "0") == "1"
tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=fast)
x = torch.rand((n, n), device="cuda")
src, lv = x, []
for l in range(5):
    o = tr.forward(src)
    for _ in range(3): tr.forward(src, out=o)
    ts = []
    for _ in range(20):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); tr.forward(src, out=o); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    lv.append(statistics.median(ts)); src = o[0]
g = tr.capture_dwt(x, 5)
for _ in range(3): g.replay()
ts = []
for _ in range(20):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); g.replay(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
gm = statistics.median(ts)
print(os.environ.get("TAG", ""), "fast" if fast else "strict", "levels", " ".join(f"{v*1e3:.1f}" for v in lv), "us | graph", f"{gm:.4f} ms = {n*n/gm/1e6:.1f} Gpx/s")
