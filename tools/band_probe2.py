"""Row-band splitting at C3 size, and batch chunking at C4 (footprint test, part 2)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF97, Transform, build_scheme

tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=True)


def timed(fn, reps=10):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    return statistics.median(ts)


N = 16384
y = torch.rand((N, N), device="cuda")
o = tuple(torch.empty((N // 2, N // 2), device="cuda") for _ in range(4))
R = N // 2
for nb in (1, 2, 4, 8, 16):
    g = torch.cuda.CUDAGraph()
    def step():
        for b in range(nb):
            r0, r1 = R * b // nb, R * (b + 1) // nb
            tr.forward_rows(y, 0, N, r0, r1, out=tuple(t[r0:r1] for t in o))
    step(); torch.cuda.synchronize()
    with torch.cuda.graph(g):
        step()
    ms = timed(g.replay)
    print(f"C3 L0 in {nb} row bands (graph): {ms*1e3:.1f} us, {8*N*N/ms/1e6/6512.3:.3f} of copy", flush=True)
n_img, n = 1024, 2048
x = torch.empty((n_img, n, n), device="cuda")
for i in range(0, n_img, 64):
    x[i:i + 64].uniform_()
outs = tuple(torch.empty((n_img, n // 2, n // 2), device="cuda") for _ in range(4))
for chunk in (4, 8, 16, 32):
    def step():
        for i in range(0, n_img, chunk):
            tr.forward(x[i:i + chunk], out=tuple(t[i:i + chunk] for t in outs))
    ms = timed(step, reps=5)
    print(f"C4 chunk {chunk}: {ms:.3f} ms = {n_img*n*n/ms/1e6:.1f} Gpx/s, {8*n_img*n*n/ms/1e6/6512.3:.3f} of copy", flush=True)
