"""Quick device timing of the fused kernels (development aid, not the bench contract)."""
import sys, os, time
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
x = torch.rand((16384, 16384), device="cuda")
for fast in (False, True):
  for tma in (True, False):
    tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=fast, tma=tma)
    outs = tr.forward(x)
    ms = t_events(lambda: tr.forward(x, out=outs))
    gbs = 8 * 16384**2 / ms / 1e6
    print(f"L1 16384^2 nssplit97 fast={fast} tma={tma}: {ms:.3f} ms  {gbs:.0f} GB/s  {gbs/peak:.2f} of copy")
    ll, det = tr.dwt(x, 5)
    scratch = torch.empty(((16384//2)**2 + (16384//4)**2,), device="cuda")
    ms = t_events(lambda: tr.dwt_into(x, 5, det, ll, scratch))
    byts = 8 * 16384**2 * sum(4.0**-l for l in range(5))
    print(f"   5-level: {ms:.3f} ms  {byts/ms/1e6:.0f} GB/s  {16384**2/ms/1e6:.1f} Gpx/s")
for wname, plan in (("cdf53", CDF53), ("cdf97", CDF97)):
    for name in SCHEME_NAMES:
        tr = Transform(build_scheme(name, plan), "single")
        x4 = torch.rand((4096, 4096), device="cuda")
        outs = tr.forward(x4)
        ms = t_events(lambda: tr.forward(x4, out=outs), reps=20)
        msi = t_events(lambda: tr.inverse(*outs), reps=20)
        print(f"C2 {wname} {name}: fwd {ms*1e3:.1f} us ({8*4096**2/ms/1e6:.0f} GB/s) inv {msi*1e3:.1f} us")
# copy reference
y = torch.empty_like(x)
ms = t_events(lambda: y.copy_(x))
print(f"torch copy 1 GiB: {ms:.3f} ms {8*16384**2/ms/1e6:.0f} GB/s")
