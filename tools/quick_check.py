"""Fast GPU spot check of one program against the oracle (dev builds with a program subset)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle
from paper_1705_08266_b200 import CDF97, Transform, build_scheme
from paper_1705_08266_b200.program import compile_scheme
scheme = build_scheme(os.environ.get("SCHEME", "non-separable-split"), CDF97)
prog = compile_scheme(scheme)
bad = 0
for tma in (True, False):
    tr = Transform(scheme, "single", tma=tma)
    for h, w in [(64, 64), (130, 262), (520, 8200), (2050, 3074), (4096, 4096)]:
        img = np.random.default_rng(h * 7 + w).random((h, w)).astype(np.float32)
        got = [c.cpu().numpy() for c in tr.forward(torch.from_numpy(img).cuda())]
        want = oracle.forward(img, prog)
        ok = all(np.array_equal(g, v) for g, v in zip(got, want))
        bad += not ok
        print("tma" if tma else "cpasync", (h, w), "OK" if ok else "MISMATCH", flush=True)
print("FAIL" if bad else "ALL OK")
