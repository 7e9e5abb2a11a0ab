"""C3-size INVERSE pyramid: 5-level idwt of a 16384^2 f32 pyramid (one launch per
level; torch CUDA graph of the eager calls), fast and strict, beside the forward
graph -- the reconstruction side a user of the reference also runs."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF97, Transform, build_scheme

n, levels = int(os.environ.get("N", "16384")), 5
x = torch.rand((n, n), device="cuda")
for fast in (True, False):
    tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=fast)
    ll, det = tr.dwt(x, levels)
    out = torch.empty_like(x)
    for _ in range(3):
        tr.idwt(ll, det, out=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        tr.idwt(ll, det, out=out)
    ts = []
    for _ in range(5):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            g.replay()
        e.record(); e.synchronize(); ts.append(s.elapsed_time(e) / 20)
    ms = statistics.median(ts)
    err = (out - x).abs().max().item()
    print(f"idwt fast={fast}: {ms:.4f} ms = {n * n / ms / 1e6:.1f} Gpx/s, 8 B/px/level bytes "
          f"{8 * sum((n >> l) ** 2 for l in range(levels)) / (ms * 1e-3) / 1e9:.0f} GB/s, max |rec - x| {err:.2e}",
          flush=True)
