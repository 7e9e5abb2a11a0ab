"""C4 / C5 shape experiments: launch chunking for the batch and the 65536^2 image."""
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


n_img, n = 1024, 2048
x = torch.empty((n_img, n, n), device="cuda")
for i in range(0, n_img, 64):
    x[i:i + 64].uniform_()
outs = tuple(torch.empty((n_img, n // 2, n // 2), device="cuda") for _ in range(4))
for chunk in (32, 64, 128, 256, 512, 1024):
    def step():
        for i in range(0, n_img, chunk):
            tr.forward(x[i:i + chunk], out=tuple(o[i:i + chunk] for o in outs))
    ms = timed(step)
    print(f"C4 chunk {chunk}: {ms:.3f} ms = {n_img*n*n/ms/1e6:.1f} Gpx/s, {8*n_img*n*n/ms/1e6/6512.3:.3f} of copy", flush=True)
del x, outs
torch.cuda.empty_cache()
N = 65536
y = torch.empty((N, N), device="cuda")
for i in range(0, N, 4096):
    y[i:i + 4096].uniform_()
o = tuple(torch.empty((N // 2, N // 2), device="cuda") for _ in range(4))
ms = timed(lambda: tr.forward(y, out=o))
print(f"C5 65536^2 forward: {ms:.3f} ms = {N*N/ms/1e6:.1f} Gpx/s, {8*N*N/ms/1e6/6512.3:.3f} of copy", flush=True)
ms = timed(lambda: tr.forward_rows(y, 0, N, 0, N // 2, out=o))
print(f"C5 65536^2 forward_rows: {ms:.3f} ms = {N*N/ms/1e6:.1f} Gpx/s", flush=True)
for rows in (16384, 32768):
    yy = y[:rows]
    oo = tuple(t[:rows // 2] for t in o)
    ms = timed(lambda: tr.forward(yy, out=oo))
    print(f"{rows}x65536 forward: {ms:.3f} ms, {8*rows*N/ms/1e6/6512.3:.3f} of copy", flush=True)
z = y.view(-1)[:16384 * 16384].view(16384, 16384)
oz = tuple(t.reshape(-1)[:8192 * 8192].view(8192, 8192) for t in o)
ms = timed(lambda: tr.forward(z, out=oz))
print(f"16384^2 forward: {ms:.3f} ms, {8*16384*16384/ms/1e6/6512.3:.3f} of copy", flush=True)
