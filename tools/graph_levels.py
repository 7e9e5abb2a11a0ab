"""C3 pyramid timing inside the CUDA graph: per-level (event nodes) and whole-graph medians."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF97, Transform, build_scheme
n = int(os.environ.get("N", "16384"))
fast = os.environ.get("FAST", "1") == "1"
tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=fast)
x = torch.rand((n, n), device="cuda")


def timed(g, reps=30):
    for _ in range(3): g.replay()
    ts, lv = [], []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); g.replay(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
        if g.events is not None: lv.append(g.level_ms())
    return statistics.median(ts), [statistics.median(c) for c in zip(*lv)] if lv else []


ge = tr.capture_dwt(x, 5, level_events=True)
_, lv = timed(ge)
g = tr.capture_dwt(x, 5)
gm, _ = timed(g)
print(os.environ.get("TAG", ""), "levels", " ".join(f"{v*1e3:.1f}" for v in lv), "us | graph", f"{gm:.4f} ms = {n*n/gm/1e6:.1f} Gpx/s", flush=True)
