"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run in the build container (where the read-only reference lives):

    python tests/golden/make_golden.py

It imports ``liftfuse`` from /root/reference/pkg/src and records, with the
reference's own code paths:

* ``programs.json``  -- ``compile_scheme(build_scheme(...))`` and
  ``compile_scheme(invert_scheme(...))`` term tables (coefficients as
  ``float.hex``) for CDF 5/3, CDF 9/7 and the custom plans of the
  reference's tests (HAAR_LIKE / ASYMMETRIC from tests/test_schemes.py:386-396,
  TRIVIAL from tests/test_engine.py:26-28);
* ``vectors.npz``    -- full outputs of ``liftfuse.engine.forward`` and
  ``inverse`` on ``Image2D.random(w, h, seed, precision)`` inputs for small
  sizes (incl. 2x2, odd component sizes, and widths whose row pitch is not a
  multiple of 16 B);
* ``hashes.json``    -- SHA-256 of the output bytes for larger sizes (up to
  the C1 config, 1024x1024 CDF 9/7 separable lifting), so GPU tests can check
  bit-exactness at size without shipping megabytes;
* ``pyramid.npz``    -- multi-level goldens: the reference's single-level
  ``forward`` iterated on ``ll`` (the reference itself has no
  multi-level API).

Nothing on the GPU box reads /root/reference; only these files travel.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from fractions import Fraction as F

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from liftfuse.engine import (  # noqa: E402
    Image2D,
    SubbandQuad,
    compile_scheme,
    deinterleave,
    forward,
    inverse,
    run_reference,
)
from liftfuse.laurent import LaurentPoly1  # noqa: E402
from liftfuse.schemes import SCHEME_NAMES, LiftingPlan, build_scheme, invert_scheme  # noqa: E402
from liftfuse.wavelets import CDF53, CDF97  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle.oracle import program_to_json  # noqa: E402

PLANS = {
    "cdf53": CDF53,
    "cdf97": CDF97,
    "haar-like": LiftingPlan(name="haar-like", pairs=((LaurentPoly1({0: F(-1)}), LaurentPoly1({0: F(1, 2)})),)),
    "asym": LiftingPlan(
        name="asym",
        pairs=((LaurentPoly1({0: F(-3, 4), -1: F(-1, 4)}), LaurentPoly1({0: F(1, 8), 1: F(3, 8)})),),
    ),
    "trivial": LiftingPlan(name="trivial", pairs=((LaurentPoly1.zero(), LaurentPoly1.zero()),)),
}

# (width, height, seed): small sizes stored in full
SMALL = [(2, 2, 0), (4, 2, 1), (6, 6, 2), (12, 10, 13), (14, 10, 3), (30, 46, 1), (34, 34, 9)]
# larger sizes stored as hashes: acceptance-corpus shapes incl. W*4 % 16 == 8
LARGE = [(64, 48, 9), (130, 62, 4), (250, 110, 8), (256, 256, 7), (66, 254, 10)]
C1 = (1024, 1024, 0)


def key(wavelet, scheme, direction, w, h, seed, precision):
    return f"{wavelet}/{scheme}/{direction}/{w}x{h}/s{seed}/{precision}"


def sha(arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).astype(a.dtype.newbyteorder("<")).tobytes())
    return h.hexdigest()


def main():
    programs = {}
    for wname, plan in PLANS.items():
        for sname in SCHEME_NAMES:
            s = build_scheme(sname, plan)
            programs[f"{wname}/{sname}/fwd"] = program_to_json(compile_scheme(s))
            programs[f"{wname}/{sname}/inv"] = program_to_json(compile_scheme(invert_scheme(s)))
    with open(os.path.join(HERE, "programs.json"), "w") as fh:
        json.dump(programs, fh, indent=0, sort_keys=True)

    vectors = {}
    hashes = {}
    for wname, plan in PLANS.items():
        for sname in SCHEME_NAMES:
            scheme = build_scheme(sname, plan)
            for precision in ("single", "double"):
                for (w, h, seed) in SMALL + LARGE:
                    img = Image2D.random(w, h, seed=seed, precision=precision)
                    q = forward(img, scheme)
                    rec = inverse(q, scheme)
                    kf = key(wname, sname, "fwd", w, h, seed, precision)
                    ki = key(wname, sname, "inv", w, h, seed, precision)
                    hashes[kf] = sha(q.components())
                    hashes[ki] = sha([rec.data])
                    if (w, h, seed) in SMALL:
                        for c, name in enumerate(("ll", "hl", "lh", "hh")):
                            vectors[kf + "/" + name] = q.components()[c]
                        vectors[ki + "/img"] = rec.data
    # C1: the reference CPU path config (BASELINE.json configs[0])
    w, h, seed = C1
    img = Image2D.random(w, h, seed=seed, precision="single")
    for sname in SCHEME_NAMES:
        for wname in ("cdf53", "cdf97"):
            scheme = build_scheme(sname, PLANS[wname])
            q = forward(img, scheme)
            hashes[key(wname, sname, "fwd", w, h, seed, "single")] = sha(q.components())
            hashes[key(wname, sname, "inv", w, h, seed, "single")] = sha([inverse(q, scheme).data])
    np.savez_compressed(os.path.join(HERE, "vectors.npz"), **vectors)

    # multi-level pyramids: forward iterated on ll
    pyr = {}
    for wname, sname, (w, h, seed), levels in [
        ("cdf97", "non-separable-split", (64, 64, 5), 3),
        ("cdf53", "non-separable-lifting", (96, 40, 6), 3),
        ("cdf97", "separable-convolution", (48, 80, 7), 2),
        ("cdf97", "separable-lifting", (32, 32, 8), 4),
    ]:
        scheme = build_scheme(sname, PLANS[wname])
        for precision in ("single", "double"):
            img = Image2D.random(w, h, seed=seed, precision=precision)
            base = f"{wname}/{sname}/{w}x{h}/s{seed}/L{levels}/{precision}"
            ll = img
            for lvl in range(levels):
                q = forward(ll, scheme)
                pyr[f"{base}/{lvl}/hl"] = q.hl.data
                pyr[f"{base}/{lvl}/lh"] = q.lh.data
                pyr[f"{base}/{lvl}/hh"] = q.hh.data
                ll = q.ll
            pyr[f"{base}/ll"] = ll.data
            # reconstruction through the reference's inverse, level by level
            cur = ll
            for lvl in reversed(range(levels)):
                cur = inverse(SubbandQuad(cur, Image2D(pyr[f"{base}/{lvl}/hl"]), Image2D(pyr[f"{base}/{lvl}/lh"]),
                                          Image2D(pyr[f"{base}/{lvl}/hh"])), scheme)
            pyr[f"{base}/rec"] = cur.data
    np.savez_compressed(os.path.join(HERE, "pyramid.npz"), **pyr)

    meta = {
        "generator": "tests/golden/make_golden.py",
        "reference": "liftfuse 0.1.0 at /root/reference/pkg (read-only)",
        "numpy": np.__version__,
        "inputs": "Image2D.random(w, h, seed, precision) = default_rng(seed).random((h, w), float64).astype(T)",
        "hashes": hashes,
    }
    with open(os.path.join(HERE, "hashes.json"), "w") as fh:
        json.dump(meta, fh, indent=0, sort_keys=True)
    # sanity: run_reference on deinterleaved comps == forward (engine.py:481-487)
    img = Image2D.random(12, 10, seed=13)
    prog = compile_scheme(build_scheme("non-separable-split", CDF97))
    a = run_reference(prog, deinterleave(img))
    b = forward(img, build_scheme("non-separable-split", CDF97)).components()
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    print(f"programs: {len(programs)}  vectors: {len(vectors)}  hashes: {len(hashes)}  pyramid: {len(pyr)}")


if __name__ == "__main__":
    main()
