"""GPU: the reference's own engine and acceptance checks (liftfuse tests/
test_engine.py, tests/test_acceptance.py) restated against this
package's drop-in API, so every check runs on the sm_100a kernels with the
reference's tolerances.  Exact array fixtures live in tests/golden/ and are
checked in test_gpu_parity.py; these are the known-answer and invariant tests.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1705_08266_b200 import (  # noqa: E402
    CDF53,
    CDF97,
    SCHEME_NAMES,
    Image2D,
    LiftingPlan,
    SubbandQuad,
    TileConfig,
    build_scheme,
    compile_scheme,
    deinterleave,
    forward,
    inverse,
    poly1,
    run_reference,
    run_tiled,
)

PLANS = {"cdf53": CDF53, "cdf97": CDF97}
TRIVIAL = LiftingPlan("trivial", ((poly1({}), poly1({})),))
# the acceptance corpus geometry: (seed, (width, height)), even sizes up to 256^2,
# including widths whose f32 row pitch is 8 (mod 16) bytes
SIZES = [(64, 64), (96, 64), (64, 96), (128, 128), (130, 62), (192, 128), (56, 200), (256, 256), (250, 110),
         (34, 34), (66, 254), (128, 256), (222, 222), (100, 100), (48, 16), (16, 48), (254, 254), (200, 200),
         (88, 120), (256, 128)]
CORPUS = list(enumerate(SIZES))


def _transfer(scheme):
    acc = None
    for p in scheme.passes:
        for m in p.matrices:
            acc = m if acc is None else m @ acc
    return acc


@pytest.mark.parametrize("name", SCHEME_NAMES)
def test_constant_image_has_zero_detail_cdf53(name):
    q = forward(Image2D.constant(32, 16, value=0.7), build_scheme(name, CDF53))
    for band in (q.hl, q.lh, q.hh):
        assert np.abs(band.data).max() <= 1e-15
    assert np.allclose(q.ll.data, 0.7, atol=1e-15)


def test_trivial_plan_returns_deinterleaved_input():
    q = forward(Image2D(np.arange(4.0).reshape(2, 2)), build_scheme("non-separable-lifting", TRIVIAL))
    assert [float(b.data[0, 0]) for b in (q.ll, q.hl, q.lh, q.hh)] == [0.0, 1.0, 2.0, 3.0]


def test_zero_round_trip_exact_and_linearity():
    s = build_scheme("non-separable-split", CDF97)
    rec = inverse(forward(Image2D(np.zeros((16, 16))), s), s)
    assert np.all(rec.data == 0.0)
    x, y = Image2D.random(32, 32, seed=1), Image2D.random(32, 32, seed=2)
    a, b = 0.75, -1.5
    s = build_scheme("non-separable-lifting", CDF97)
    fc = forward(Image2D(a * x.data + b * y.data), s).components()
    fx, fy = forward(x, s).components(), forward(y, s).components()
    for cc, cx, cy in zip(fc, fx, fy):
        assert np.abs(cc - (a * cx + b * cy)).max() <= 1e-12


def test_cross_scheme_equivalence_and_perfect_reconstruction():
    tol_rec = {"cdf53": 1e-12, "cdf97": 1e-9}
    for wavelet, plan in PLANS.items():
        schemes = {n: build_scheme(n, plan) for n in SCHEME_NAMES}
        for seed, (w, h) in CORPUS:
            img = Image2D.random(w, h, seed=seed)
            quads = {n: forward(img, s) for n, s in schemes.items()}
            base = quads[SCHEME_NAMES[0]].components()
            for n in SCHEME_NAMES[1:]:
                d = max(float(np.abs(u - v).max()) for u, v in zip(base, quads[n].components()))
                assert d <= 1e-9, (wavelet, n, (w, h), d)
            for n, s in schemes.items():
                err = float(np.abs(inverse(quads[n], s).data - img.data).max())
                assert err <= tol_rec[wavelet], (wavelet, n, (w, h), err)
        for seed, (w, h) in CORPUS[:6]:  # single precision
            img = Image2D.random(w, h, seed=seed, precision="single")
            for n, s in schemes.items():
                rec = inverse(forward(img, s), s)
                assert rec.data.dtype == np.float32
                assert float(np.abs(rec.data - img.data).max()) <= 1e-3


def test_tiling_and_thread_invariance():
    img = Image2D.random(128, 96, seed=31)
    comps = deinterleave(img)
    for plan in PLANS.values():
        for n in SCHEME_NAMES:
            prog = compile_scheme(build_scheme(n, plan))
            ref = run_reference(prog, comps)
            for tile in ((8, 8), (16, 16), (32, 32), None):
                for threads in (1, 2, 8):
                    out = run_tiled(prog, comps, TileConfig(tile=tile, threads=threads))
                    assert all(np.array_equal(r, o) for r, o in zip(ref, out)), (n, tile, threads)


def test_impulse_response_matches_transfer_matrix():
    size, centre = 32, 8
    for plan in PLANS.values():
        transfer = _transfer(build_scheme("separable-convolution", plan))
        for n in SCHEME_NAMES:
            s = build_scheme(n, plan)
            for j, (pr, pc) in enumerate(((0, 0), (0, 1), (1, 0), (1, 1))):
                comps = forward(Image2D.delta(size, size, 2 * centre + pr, 2 * centre + pc), s).components()
                for i in range(4):
                    want = np.zeros((size // 2, size // 2))
                    for (km, kn), c in transfer.entries[i][j].terms.items():
                        want[centre + kn, centre + km] = float(c)
                    assert float(np.abs(comps[i] - want).max()) <= 1e-12, (n, i, j)


def test_subband_shape_errors():
    with pytest.raises(ValueError, match="all four subbands must share dimensions"):
        SubbandQuad(*(Image2D(np.zeros(s)) for s in ((2, 2), (2, 2), (2, 2), (2, 4))))


def test_missing_barrier_witness_matches_reference_fault_model():
    """run_without_barriers (engine.py:454-475): the barrier-free fault model is
    bit-identical to the reference's, corrupts tiled runs, and is harmless
    with one tile (tests/test_engine.py:241-259 witnesses)."""
    import os

    from paper_1705_08266_b200 import Image2D as I2, run_without_barriers

    gold = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "nobarrier.npz"))
    comps = deinterleave(I2.random(64, 48, seed=21))
    for wname, plan in PLANS.items():
        for scheme in ("separable-lifting", "non-separable-split"):
            prog = compile_scheme(build_scheme(scheme, plan))
            good = run_reference(prog, comps)
            for tile in ((8, 8), (16, 4), None):
                key = f"{wname}/{scheme}/{'full' if tile is None else f'{tile[0]}x{tile[1]}'}"
                got = run_without_barriers(prog, comps, TileConfig(tile=tile))
                for c, name in enumerate(("ll", "hl", "lh", "hh")):
                    assert np.array_equal(got[c], gold[f"{key}/{name}"]), (key, name)
                worst = max(float(np.abs(g - b).max()) for g, b in zip(good, got))
                if tile is None:
                    assert worst == 0.0, key
                else:
                    assert worst > 1e-6, key
