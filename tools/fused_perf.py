"""C3 pyramid graph time with two-level fused kernels vs one launch per level
(B2DWT_FUSE2_MIN_QUADS / fuse=False), plus per-launch-group event times."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF97, Transform, build_scheme
n = int(os.environ.get("N", "16384"))
levels = int(os.environ.get("LEVELS", "5"))
x = torch.rand((n, n), device="cuda")


def timed(g, reps=30):
    for _ in range(5): g.replay()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): g.replay()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / reps


# MODES: comma list of fast:fuse pairs, e.g. "1:1,0:1" (default: all four)
modes = [tuple(bool(int(v)) for v in m.split(":")) for m in os.environ.get("MODES", "1:1,1:0,0:1,0:0").split(",")]
for fast, fuse in modes:
    if True:
        tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=fast, fuse=fuse)
        g = tr.capture_dwt(x, levels)
        ms = timed(g)
        del g
        ge = tr.capture_dwt(x, levels, level_events=True)
        runs = []
        for _ in range(20):
            ge.replay(); torch.cuda.synchronize(); runs.append(ge.level_ms())
        groups = ge.groups
        per = [statistics.median(r[i] for r in runs[5:]) for i in range(len(groups))]
        del ge
        print(f"fast={fast} fuse={fuse}: graph {ms:.4f} ms = {n*n/ms/1e6:.1f} Gpx/s | groups",
              " ".join(f"{a}-{b}:{p*1e3:.1f}us" for (a, b), p in zip(groups, per)), flush=True)
