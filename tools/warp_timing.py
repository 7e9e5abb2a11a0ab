"""Per-warp cycle records of the fused kernel (debug hook) -> work-split tuning."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1705_08266_b200 import CDF97, Transform, build_scheme, _native

lib = _native.load()
lib.b2dwt_debug_enable.argtypes = [ctypes.c_int64]
lib.b2dwt_debug_fetch.argtypes = [ctypes.c_void_p, ctypes.c_int64]
N = 4096
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
fast = len(sys.argv) > 2 and sys.argv[2] == "fast"
tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=fast)
x = torch.rand((n, n), device="cuda")
o = tr.forward(x)
for _ in range(3):
    tr.forward(x, out=o)
torch.cuda.synchronize()
lib.b2dwt_debug_enable(N)
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record(); tr.forward(x, out=o); e.record(); e.synchronize()
buf = np.zeros((N, 4), dtype=np.int64)
lib.b2dwt_debug_fetch(buf.ctypes.data, N)
lib.b2dwt_debug_enable(0)
rec = buf[buf[:, 1] > 0]
cyc, rows, erows, sm = rec.T
print(f"n={n} fast={fast} kernel {s.elapsed_time(e):.3f} ms, warps {len(rec)}, SMs {len(set(sm))}")
inter = erows == 0
print(f"interior warps {inter.sum()}: rows {rows[inter].mean():.1f}, cycles mean {cyc[inter].mean():.0f} max {cyc[inter].max()}, "
      f"cycles/row {np.mean(cyc[inter] / rows[inter]):.1f}")
if (~inter).any():
    ed = ~inter
    print(f"edge-touching warps {ed.sum()}: rows {rows[ed].mean():.1f} (edge rows {erows[ed].mean():.1f}), cycles mean {cyc[ed].mean():.0f} max {cyc[ed].max()}")
    pure = erows == rows
    if pure.any():
        print(f"   pure-edge warps: cycles/row {np.mean(cyc[pure] / rows[pure]):.1f}")
order = np.argsort(-cyc)[:8]
print("slowest:", [(int(cyc[i]), int(rows[i]), int(erows[i]), int(sm[i])) for i in order])
per_sm = {}
for c, m in zip(cyc, sm):
    per_sm.setdefault(int(m), []).append(int(c))
mx = sorted((max(v), k, len(v)) for k, v in per_sm.items())
print("per-SM max cycles: min", mx[0], "median", mx[len(mx)//2], "max", mx[-1])
