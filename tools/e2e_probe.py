"""Host-buffer pyramid (b2dwt_dwt_host) timing vs band count, beside the
PCIe floor (1 GiB H2D and 1 GiB D2H on two streams at once)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_08266_b200 import CDF97, Transform, build_scheme

n, levels = 16384, 5
tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=True)
host = torch.empty((n, n)).pin_memory()
host.uniform_()
det = [tuple(torch.empty((n >> (l + 1), n >> (l + 1))).pin_memory() for _ in range(3)) for l in range(levels)]
ll = torch.empty((n >> levels, n >> levels)).pin_memory()


def timed(fn, reps=5):
    fn(); fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    return statistics.median(ts)


d_in = torch.empty((n, n), device="cuda"); d_out = torch.empty((n, n), device="cuda")
h_out = torch.empty((n, n)).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def floor():
    cur = torch.cuda.current_stream(); s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(host, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)


print(f"PCIe floor (1 GiB each way, concurrent): {timed(floor):.2f} ms", flush=True)
for b in [int(x) for x in os.environ.get("BANDS", "4 8 16 32 64").split()]:
    ms = timed(lambda: tr.dwt_host(host, levels, details=det, ll=ll, bands=b, sync=False))
    print(f"bands={b}: {ms:.2f} ms = {n * n / ms / 1e6:.2f} Gpx/s", flush=True)

# inverse: host pyramid -> host image
rec = torch.empty((n, n)).pin_memory()
tr.dwt_host(host, levels, details=det, ll=ll, bands=16)
for b in (8, 16, 32):
    ms = timed(lambda: tr.idwt_host(ll, det, out=rec, bands=b, sync=False))
    print(f"idwt_host bands={b}: {ms:.2f} ms = {n * n / ms / 1e6:.2f} Gpx/s", flush=True)
