"""GPU parity at C2 size (BASELINE.json configs[1]: 4096^2, CDF 5/3 and 9/7, all
four schemes, forward and inverse) for EVERY built-in program.

SURVEY.md section 8(c) parity policy:

1. strict mode is bit-identical to ``run_reference`` -- f32 (the TMA stream
   kernel, the product's main variant) and f64 (the cp.async variant), forward
   and inverse; the inverse consumes the oracle's own forward output;
2. fast (FMA) mode stays within max|err| <= 1e-4 x (max - min of the input) of
   the f64 oracle (the north star's float32 tolerance), forward and inverse, with
   identical subband layout and edges.

The oracle (oracle/dwt_oracle.c) is pinned to the reference's own golden vectors
by tests/test_oracle.py; the reference tolerances these mirror are in
liftfuse tests/test_engine.py:156-183.
"""

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1705_08266_b200 import (CDF53, CDF97, SCHEME_NAMES, Transform, build_scheme,  # noqa: E402
                                   compile_scheme, invert_scheme)

N = 4096
PLANS = {"cdf53": CDF53, "cdf97": CDF97}
NAMES = ("ll", "hl", "lh", "hh")
PROGRAMS = [(w, s) for w in PLANS for s in SCHEME_NAMES]
IDS = [f"{w}-{s}" for w, s in PROGRAMS]

_IMAGES = {}


def _image(dtype):
    if dtype not in _IMAGES:
        # Image2D.random(N, N, seed=0, precision) (engine.py:125-129)
        _IMAGES[dtype] = np.random.default_rng(0).random((N, N), dtype=np.float64).astype(dtype)
    return _IMAGES[dtype]


def _programs(wavelet, scheme):
    s = build_scheme(scheme, PLANS[wavelet])
    return s, compile_scheme(s), compile_scheme(invert_scheme(s))


def _first_diff(g, w):
    idx = np.argwhere(g != w)
    return idx[:3].tolist(), int(idx.shape[0])


@pytest.mark.parametrize("precision", ["single", "double"])
@pytest.mark.parametrize("wavelet,scheme", PROGRAMS, ids=IDS)
def test_c2_strict_forward_and_inverse_bit_exact(wavelet, scheme, precision):
    dtype = np.float32 if precision == "single" else np.float64
    img = _image(dtype)
    s, fwd, inv = _programs(wavelet, scheme)
    tr = Transform(s, precision)
    assert tr.fwd_plan.fused and tr.inv_plan.fused
    want = oracle.forward(img, fwd)
    got = [c.cpu().numpy() for c in tr.forward(torch.from_numpy(img).cuda())]
    for g, w, n in zip(got, want, NAMES):
        assert g.shape == w.shape and g.dtype == w.dtype
        assert np.array_equal(g, w), (n, _first_diff(g, w))
    want_rec = oracle.inverse(want, inv)
    rec = tr.inverse(*[torch.from_numpy(c).cuda() for c in want]).cpu().numpy()
    assert np.array_equal(rec, want_rec), _first_diff(rec, want_rec)


@pytest.mark.parametrize("wavelet,scheme", PROGRAMS, ids=IDS)
def test_c2_fast_forward_and_inverse_within_tolerance(wavelet, scheme):
    img = _image(np.float32)
    s, fwd, inv = _programs(wavelet, scheme)
    tr = Transform(s, "single", fast=True)
    # forward: f32 FMA kernel vs the f64 oracle on the same (f32-valued) image
    want = oracle.forward(img.astype(np.float64), fwd)
    tol = 1e-4 * float(img.max() - img.min())
    got = [c.cpu().numpy() for c in tr.forward(torch.from_numpy(img).cuda())]
    for g, w, n in zip(got, want, NAMES):
        assert g.shape == w.shape
        err = float(np.abs(g.astype(np.float64) - w).max())
        assert err <= tol, (n, err, tol)
    # inverse: f32 subbands (the f64 reference's, rounded) in, f64 oracle inverse of the same values
    sub32 = [w.astype(np.float32) for w in want]
    want_rec = oracle.inverse([c.astype(np.float64) for c in sub32], inv)
    rec = tr.inverse(*[torch.from_numpy(c).cuda() for c in sub32]).cpu().numpy()
    tol_rec = 1e-4 * float(want_rec.max() - want_rec.min())
    err = float(np.abs(rec.astype(np.float64) - want_rec).max())
    assert err <= tol_rec, (err, tol_rec)
    # and the round trip closes on the original image
    assert float(np.abs(rec.astype(np.float64) - img).max()) <= 1e-4 * float(img.max() - img.min()) * 10
