"""Fixtures of the reference's barrier-free fault model (liftfuse.engine.
run_without_barriers), for the GPU witness test.  Run in the build container:
    python tests/golden/make_nobarrier_golden.py"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from liftfuse.engine import Image2D, TileConfig, compile_scheme, deinterleave, run_without_barriers  # noqa: E402
from liftfuse.schemes import build_scheme  # noqa: E402
from liftfuse.wavelets import CDF53, CDF97  # noqa: E402

out = {}
for wname, plan in (("cdf53", CDF53), ("cdf97", CDF97)):
    for scheme in ("separable-lifting", "non-separable-split"):
        for tile in ((8, 8), (16, 4), None):
            img = Image2D.random(64, 48, seed=21)
            comps = deinterleave(img)
            res = run_without_barriers(compile_scheme(build_scheme(scheme, plan)), comps, TileConfig(tile=tile))
            key = f"{wname}/{scheme}/{'full' if tile is None else f'{tile[0]}x{tile[1]}'}"
            for c, name in enumerate(("ll", "hl", "lh", "hh")):
                out[f"{key}/{name}"] = res[c]
np.savez(os.path.join(os.path.dirname(os.path.abspath(__file__)), "nobarrier.npz"), **out)
print(len(out), "arrays")
