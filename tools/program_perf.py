"""All 16 built-in programs: one 8192^2 forward / inverse launch each (f32), median
of CUDA-event timings, fast and strict, as a fraction of the measured copy bandwidth
(8 B/px).  Also the C3-relevant pyramid-pair times per scheme."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF53, CDF97, SCHEME_NAMES, Transform, build_scheme

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
n = int(os.environ.get("N", "8192"))
x = torch.rand((n, n), device="cuda")


def t(fn, reps=15, per_graph=10):
    """ms per call: a CUDA graph of `per_graph` back-to-back calls (no host gaps)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(per_graph):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); g.replay(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e) / per_graph)
    return statistics.median(ts)


only = os.environ.get("PROGRAMS")  # e.g. "cdf97/separable-convolution,cdf97/non-separable-split"
arith = os.environ.get("ARITH", "fast,strict").split(",")
for fast in [a == "fast" for a in arith]:
    for wname, plan in (("cdf53", CDF53), ("cdf97", CDF97)):
        for sname in SCHEME_NAMES:
            if only and f"{wname}/{sname}" not in only.split(","):
                continue
            tr = Transform(build_scheme(sname, plan), "single", fast=fast)
            q = tr.forward(x)
            rec = torch.empty_like(x)
            f = t(lambda: tr.forward(x, out=q))
            i = t(lambda: tr.inverse(*q, out=rec))
            print(json.dumps({"program": f"{wname}/{sname}", "arith": "fast" if fast else "strict", "n": n,
                              "fwd_us": round(f * 1e3, 1), "inv_us": round(i * 1e3, 1),
                              "fwd_frac": round(8 * n * n / (f * 1e-3) / 1e9 / peak, 3),
                              "inv_frac": round(8 * n * n / (i * 1e-3) / 1e9 / peak, 3)}), flush=True)
