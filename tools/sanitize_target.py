"""compute-sanitizer workload: every kernel family once, small sizes (the tools
slow kernels down 10-100x).  Exits non-zero if any result is wrong.

  stream kernel (TMA and cp.async fills) forward + inverse, tile kernel, generic
  tile (K10) and per-sub-step (K0) interpreters, the two-level fused kernel, the
  PDL-chained device pyramid (b2dwt_dwt) and both host pipelines.
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF97, Transform, build_scheme

n = int(os.environ.get("N", "2048"))
s = build_scheme("non-separable-split", CDF97)
x = torch.rand((n, n), device="cuda")
ok = True


def same(a, b):
    global ok
    ok &= bool(torch.equal(a, b))


ref = Transform(s, "single", tile=False)
q = ref.forward(x)
rec = ref.inverse(*q)
for kw in (dict(tile=False, tma=False), dict(tile=True), dict(force_generic=True), dict(force_generic=True, tile=False)):
    tr = Transform(s, "single", **kw)
    xs = x[:512, :512].contiguous() if kw.get("force_generic") else x
    want = ref.forward(xs)
    got = tr.forward(xs)
    for a, b in zip(got, want):
        same(a, b)
    same(tr.inverse(*got), ref.inverse(*want))
for fast in (False, True):
    tr = Transform(s, "single", fast=fast)
    got = tr.forward2(x)
    ll0, hl0, lh0, hh0 = tr.forward(x)
    want = (hl0, lh0, hh0) + tuple(tr.forward(ll0.contiguous()))
    for a, b in zip(got[0] + got[1], want):
        same(a, b)
    ll, det = tr.dwt(x, 5)
    llh, deth = tr.dwt_host(x.cpu().pin_memory(), 5, bands=8)
    same(llh, ll.cpu())
    for d, e in zip(det, deth):
        for a, b in zip(d, e):
            same(a.cpu(), b)
    back = tr.idwt_host(llh, deth, bands=8)
    same(back, tr.idwt(ll, det).cpu())
torch.cuda.synchronize()
print("sanitize target", "ok" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
