"""GPU: seeded random shapes through every built-in program and both host
pipelines, strict mode bit-exact against the oracle (tiny, thin, odd
component counts, widths with 8-byte row pitch, sizes that straddle the
stream / tile kernel switch and strip / segment / tile boundaries)."""

import zlib

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1705_08266_b200 import (  # noqa: E402
    CDF53,
    CDF97,
    SCHEME_NAMES,
    Transform,
    build_scheme,
    compile_scheme,
    invert_scheme,
)


def _shapes(seed, count):
    rng = np.random.default_rng(seed)
    fixed = [(2, 2), (2, 64), (64, 2), (4, 6), (6, 130), (130, 6), (34, 1026), (1026, 34)]
    rand = [(2 * int(rng.integers(1, 700)), 2 * int(rng.integers(1, 700))) for _ in range(count)]
    return fixed + rand


@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
def test_random_shapes_all_programs_bit_exact(wavelet):
    plan = {"cdf53": CDF53, "cdf97": CDF97}[wavelet]
    rng = np.random.default_rng(123)
    for name in SCHEME_NAMES:
        scheme = build_scheme(name, plan)
        fwd, inv = compile_scheme(scheme), compile_scheme(invert_scheme(scheme))
        for tile in (None, False):
            tr = Transform(scheme, "single", tile=tile)
            for h, w in _shapes(zlib.crc32(name.encode()), 6):
                img = rng.random((h, w), dtype=np.float32)
                got = [c.cpu().numpy() for c in tr.forward(torch.from_numpy(img).cuda())]
                want = oracle.forward(img, fwd)
                for g, wv in zip(got, want):
                    assert np.array_equal(g, wv), (wavelet, name, tile, (h, w))
                rec = tr.inverse(*[torch.from_numpy(c).cuda() for c in want]).cpu().numpy()
                assert np.array_equal(rec, oracle.inverse(want, inv)), (wavelet, name, tile, (h, w))


def test_random_pyramids_host_pipelines_bit_exact():
    rng = np.random.default_rng(7)
    scheme = build_scheme("non-separable-split", CDF97)
    tr = Transform(scheme, "single")
    fwd, inv = compile_scheme(scheme), compile_scheme(invert_scheme(scheme))
    for _ in range(6):
        levels = int(rng.integers(1, 5))
        h = (1 << levels) * int(rng.integers(1, 96))
        w = (1 << levels) * int(rng.integers(1, 96))
        img = rng.random((h, w), dtype=np.float32)
        want_ll, want_det = oracle.dwt(img, fwd, levels)
        ll, det = tr.dwt_host(img, levels, bands=int(rng.integers(1, 24)))
        assert np.array_equal(ll.numpy(), want_ll), (h, w, levels)
        for lvl in range(levels):
            for g, wv in zip(det[lvl], want_det[lvl]):
                assert np.array_equal(g.numpy(), wv), (h, w, levels, lvl)
        rec = tr.idwt_host(ll, det, bands=int(rng.integers(1, 24)))
        assert np.array_equal(rec.numpy(), oracle.idwt(want_ll, want_det, inv)), (h, w, levels)
