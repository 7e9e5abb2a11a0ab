"""Scheme ordering on the C3 workload itself: the 16384^2 5-level pyramid (CUDA
graph, fused pairs where built) for every forward scheme of both wavelets,
fast and strict -- the paper's comparison at the north-star
size, beside tools/program_perf.py's single-level table."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF53, CDF97, SCHEME_NAMES, Transform, build_scheme

n = int(os.environ.get("N", "16384"))
levels = int(os.environ.get("LEVELS", "5"))
x = torch.rand((n, n), device="cuda")


def timed(g, reps=20):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            g.replay()
        e.record(); e.synchronize(); ts.append(s.elapsed_time(e) / reps)
    return statistics.median(ts)


for fast in (True, False):
    for wname, plan in (("cdf53", CDF53), ("cdf97", CDF97)):
        for sname in SCHEME_NAMES:
            tr = Transform(build_scheme(sname, plan), "single", fast=fast)
            g = tr.capture_dwt(x, levels)
            ms = timed(g)
            groups = g.groups if hasattr(g, "groups") else None
            del g
            print(json.dumps({"program": f"{wname}/{sname}", "arith": "fast" if fast else "strict", "n": n,
                              "levels": levels, "ms": round(ms, 4), "gpix_per_s": round(n * n / ms / 1e6, 1),
                              "groups": groups}), flush=True)
