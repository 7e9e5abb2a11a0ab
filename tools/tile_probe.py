"""Small-level kernels side by side: tile vs stream on one pyramid-level size
(N x N input, default 2048 = C3 level 3).  Prints median CUDA-event times;
under ncu, profile with -k regex:tile_kernel or -k regex:stream_kernel."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF97, Transform, build_scheme

n = int(os.environ.get("N", "2048"))
reps = int(os.environ.get("REPS", "50"))
x = torch.rand((n, n), device="cuda")
for tile in (True, False):
    tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=True, tile=tile)
    out = tr.forward(x)
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); tr.forward(x, out=out); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    print(f"N={n} {'tile' if tile else 'stream'}: {statistics.median(ts)*1e3:.1f} us", flush=True)
