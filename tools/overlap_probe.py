"""Experiment: overlap pyramid levels on two streams inside one CUDA graph
(level 1's top band runs while level 0's bottom band still streams)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF97, Transform, build_scheme

tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=True)
N, L = 16384, 5
x = torch.rand((N, N), device="cuda")
up, down = tr.cone[0], tr.cone[1]
lls = [torch.empty((N >> (l + 1), N >> (l + 1)), device="cuda") for l in range(L)]
det = [tuple(torch.empty((N >> (l + 1), N >> (l + 1)), device="cuda") for _ in range(3)) for l in range(L)]


def outs(l, r0, r1):
    return (lls[l][r0:r1],) + tuple(d[r0:r1] for d in det[l])


def timed(g, reps=30):
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); g.replay(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    return statistics.median(ts)


def pyramid_serial():
    src = x
    for l in range(L):
        tr.forward(src, out=outs(l, 0, N >> (l + 1)))
        src = lls[l]


def pyramid_overlap(nb0, nb1):
    main = torch.cuda.current_stream()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    s1.wait_stream(main); s2.wait_stream(main)
    R0, R1 = N // 2, N // 4
    evs = []
    with torch.cuda.stream(s1):
        for b in range(nb0):
            r0, r1 = R0 * b // nb0, R0 * (b + 1) // nb0
            tr.forward_rows(x, 0, N, r0, r1, out=outs(0, r0, r1))
            ev = torch.cuda.Event(); ev.record(s1); evs.append((r1, ev))
    with torch.cuda.stream(s2):
        prev = 0
        for b in range(nb1):
            end = R1 if b == nb1 - 1 else R1 * (b + 1) // nb1
            need = 2 * min(R1, end + down)  # LL0 rows needed
            for r1, ev in evs:
                if r1 >= need:
                    s2.wait_event(ev)
                    break
            else:
                s2.wait_event(evs[-1][1])
            if end > prev:
                tr.forward_rows(lls[0], 0, N // 2, prev, end, out=outs(1, prev, end))
            prev = end
        src = lls[1]
        for l in range(2, L):
            tr.forward(src, out=outs(l, 0, N >> (l + 1)))
            src = lls[l]
    main.wait_stream(s1); main.wait_stream(s2)


for name, fn in [("serial", pyramid_serial)] + [(f"overlap {a}x{b}", (lambda a=a, b=b: pyramid_overlap(a, b)))
                                               for a, b in ((2, 2), (4, 2), (4, 4), (8, 4))]:
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ms = timed(g)
    print(f"{name}: {ms*1e3:.1f} us = {N*N/ms/1e6:.1f} Gpx/s", flush=True)
g2 = tr.capture_dwt(x, L)
print(f"capture_dwt: {timed(g2)*1e3:.1f} us", flush=True)
