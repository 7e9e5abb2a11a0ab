"""Device timing of the fused kernels (development aid, not the bench contract)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF53, CDF97, SCHEME_NAMES, Transform, build_scheme

def t_events(fn, reps=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    times = []
    for _ in range(reps):
        s.record(); fn(); e.record(); e.synchronize(); times.append(s.elapsed_time(e))
    times.sort()
    return times[len(times)//2]

peak = 6512.3
n = 16384
x = torch.rand((n, n), device="cuda")
for fast in (False, True):
  for tma in (True, False):
    tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=fast, tma=tma)
    lv = []
    src = x
    for l in range(5):
        outs = tr.forward(src)
        ms = t_events(lambda: tr.forward(src, out=outs))
        lv.append(ms)
        src = outs[0]
    gbs = 8 * n * n / lv[0] / 1e6
    g = tr.capture_dwt(x, 5)
    msg = t_events(g.replay, reps=20)
    byts = 8 * n * n * sum(4.0 ** -l for l in range(5))
    print(f"fast={fast} tma={tma}: L0 {lv[0]:.3f} ms {gbs:.0f} GB/s ({gbs/peak:.2f} of copy); levels(ms) "
          + " ".join(f"{v:.4f}" for v in lv)
          + f" | graph 5-level {msg:.3f} ms {byts/msg/1e6:.0f} GB/s {n*n/msg/1e6:.1f} Gpx/s")
for wname, plan in (("cdf53", CDF53), ("cdf97", CDF97)):
    for name in SCHEME_NAMES:
        tr = Transform(build_scheme(name, plan), "single")
        x4 = torch.rand((8192, 8192), device="cuda")
        outs = tr.forward(x4)
        rec = torch.empty_like(x4)
        ms = t_events(lambda: tr.forward(x4, out=outs), reps=20)
        msi = t_events(lambda: tr.inverse(*outs, out=rec), reps=20)
        b = 8 * 8192**2
        print(f"8192^2 {wname} {name}: fwd {ms*1e3:.1f} us ({b/ms/1e6:.0f} GB/s) inv {msi*1e3:.1f} us ({b/msi/1e6:.0f} GB/s)")
y = torch.empty_like(x)
ms = t_events(lambda: y.copy_(x))
print(f"torch copy 1 GiB: {ms:.3f} ms {8*n*n/ms/1e6:.0f} GB/s")
