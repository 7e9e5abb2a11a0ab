"""Pin the CPU oracle (oracle/dwt_oracle.c) to the reference's own outputs.

Every golden output under tests/golden/ was produced by the real reference
(tests/golden/make_golden.py).  The oracle must reproduce all of them bit for
bit before any GPU parity claim is trusted.
"""

import numpy as np
import pytest

from oracle import oracle
from tests import golden_data as G


def _forward_inputs(wavelet, scheme, w, h, seed, precision):
    img = G.random_image(w, h, seed, precision)
    return img, oracle.deinterleave(img)


def test_oracle_matches_reference_vectors_bitwise():
    progs = G.programs()
    vec = G.vectors()
    checked = 0
    for k in G.hashes():
        wavelet, scheme, direction, w, h, seed, precision = G.parse_key(k)
        if f"{k}/img" not in vec and f"{k}/ll" not in vec:
            continue
        img, comps = _forward_inputs(wavelet, scheme, w, h, seed, precision)
        fwd = oracle.run_reference(progs[f"{wavelet}/{scheme}/fwd"], comps, threads=2)
        if direction == "fwd":
            for c, name in enumerate(("ll", "hl", "lh", "hh")):
                assert np.array_equal(fwd[c], vec[f"{k}/{name}"]), (k, name)
        else:
            rec = oracle.inverse(fwd, progs[f"{wavelet}/{scheme}/inv"], threads=3)
            assert np.array_equal(rec, vec[f"{k}/img"]), k
        checked += 1
    assert checked >= 500


@pytest.mark.parametrize("threads", [1, 4])
def test_oracle_matches_reference_hashes(threads):
    progs = G.programs()
    checked = 0
    for k, digest in G.hashes().items():
        wavelet, scheme, direction, w, h, seed, precision = G.parse_key(k)
        if w * h > 70000 and threads == 1:
            continue
        img, comps = _forward_inputs(wavelet, scheme, w, h, seed, precision)
        fwd = oracle.run_reference(progs[f"{wavelet}/{scheme}/fwd"], comps, threads=threads)
        if direction == "fwd":
            assert G.sha(fwd) == digest, k
        else:
            rec = oracle.inverse(fwd, progs[f"{wavelet}/{scheme}/inv"], threads=threads)
            assert G.sha([rec]) == digest, k
        checked += 1
    assert checked > 300


def test_oracle_multilevel_matches_iterated_reference():
    progs = G.programs()
    pyr = G.pyramids()
    bases = sorted({k.rsplit("/", 1)[0] if k.endswith(("/ll", "/rec")) else k.rsplit("/", 2)[0] for k in pyr})
    for base in bases:
        wavelet, scheme, dims, seed, lv, precision = base.split("/")
        w, h = (int(x) for x in dims.split("x"))
        levels = int(lv[1:])
        img = G.random_image(w, h, int(seed[1:]), precision)
        ll, details = oracle.dwt(img, progs[f"{wavelet}/{scheme}/fwd"], levels)
        assert np.array_equal(ll, pyr[f"{base}/ll"]), base
        for lvl, (hl, lh, hh) in enumerate(details):
            assert np.array_equal(hl, pyr[f"{base}/{lvl}/hl"])
            assert np.array_equal(lh, pyr[f"{base}/{lvl}/lh"])
            assert np.array_equal(hh, pyr[f"{base}/{lvl}/hh"])
        rec = oracle.idwt(ll, details, progs[f"{wavelet}/{scheme}/inv"])
        assert np.array_equal(rec, pyr[f"{base}/rec"]), base


def test_oracle_against_live_reference(liftfuse):
    """In the build container: oracle == reference run_reference on fresh inputs."""
    from liftfuse.engine import Image2D, compile_scheme, deinterleave, run_reference
    from liftfuse.schemes import SCHEME_NAMES, build_scheme, invert_scheme
    from liftfuse.wavelets import CDF53, CDF97

    for plan in (CDF53, CDF97):
        for name in SCHEME_NAMES:
            for (w, h, seed) in [(18, 22, 3), (40, 8, 4), (2, 6, 5)]:
                img = Image2D.random(w, h, seed=seed, precision="single")
                s = build_scheme(name, plan)
                for prog in (compile_scheme(s), compile_scheme(invert_scheme(s))):
                    comps = deinterleave(img)
                    ref = run_reference(prog, comps)
                    got = oracle.run_reference(prog, comps, threads=2)
                    assert all(np.array_equal(a, b) for a, b in zip(ref, got)), (plan.name, name)
