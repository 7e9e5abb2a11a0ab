"""Two-level fused kernel (csrc/fused2_kernel.cuh): levels l and l+1 of the
pyramid in one launch, level l's LL band kept on chip.

It must be invisible in the results: bit-identical to two single-level launches
(strict and fast), hence to the iterated reference (strict, against the oracle),
for every fusable built-in program, at shapes that exercise partial
super-strips, the checked top / bottom units, tiny images (edge units only),
padded pitches, the dynamic tail and footprint-split launches.
"""

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1705_08266_b200 import (CDF53, CDF97, SCHEME_NAMES, Transform, build_scheme,  # noqa: E402
                                   compile_scheme)

PLANS = {"cdf53": CDF53, "cdf97": CDF97}
FUSABLE = [(w, s) for w in PLANS for s in SCHEME_NAMES if not (w == "cdf97" and s == "separable-convolution")]


def _two_launches(tr, x):
    ll0, hl0, lh0, hh0 = tr.forward(x)
    return (hl0, lh0, hh0), tr.forward(ll0.contiguous())


@pytest.mark.parametrize("fast", [False, True], ids=["strict", "fast"])
@pytest.mark.parametrize("shape", [(1024, 1024), (600, 1000), (48, 256), (1028, 2060), (4096, 8192)])
def test_forward2_equals_two_launches(shape, fast):
    tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=fast)
    h, w = shape
    x = torch.rand((h, w), device="cuda", generator=torch.Generator(device="cuda").manual_seed(h * 7 + w))
    got = tr.forward2(x)
    assert got is not None, "fused kernel refused a fusable request"
    want = _two_launches(tr, x)
    for g, wv, n in zip(got[0] + got[1], want[0] + want[1], ("hl0", "lh0", "hh0", "ll1", "hl1", "lh1", "hh1")):
        assert torch.equal(g, wv), (shape, n, (g != wv).nonzero()[:5].tolist())


@pytest.mark.parametrize("wavelet,scheme", FUSABLE, ids=[f"{w}-{s}" for w, s in FUSABLE])
def test_fused_pyramid_equals_unfused_and_oracle(wavelet, scheme, monkeypatch):
    monkeypatch.setenv("B2DWT_FUSE2_MIN_QUADS", "1")  # fuse every pair b2dwt_dwt can

    s = build_scheme(scheme, PLANS[wavelet])
    h, w = 1032, 1544  # ragged super-strips at both fused pairs; 3 levels: pair + single
    img = np.random.default_rng(9).random((h, w)).astype(np.float32)
    x = torch.from_numpy(img).cuda()
    for fast in (False, True):
        fused = Transform(s, "single", fast=fast)
        plain = Transform(s, "single", fast=fast, fuse=False)
        assert fused.forward2(x) is not None, (wavelet, scheme)
        a_ll, a_det = fused.dwt(x, 3)
        b_ll, b_det = plain.dwt(x, 3)
        assert torch.equal(a_ll, b_ll), (wavelet, scheme, fast)
        for lvl in range(3):
            for u, v in zip(a_det[lvl], b_det[lvl]):
                assert torch.equal(u, v), (wavelet, scheme, fast, lvl)
        if not fast:
            want_ll, want_det = oracle.dwt(img, compile_scheme(s), 3)
            assert np.array_equal(a_ll.cpu().numpy(), want_ll)
            for lvl in range(3):
                for u, v in zip(a_det[lvl], want_det[lvl]):
                    assert np.array_equal(u.cpu().numpy(), v), (wavelet, scheme, lvl)


def test_fused_footprint_bands_padded_pitch_and_dynamic_tail(monkeypatch):
    """Row-band launches (small B2DWT_MAX_LAUNCH_BYTES), a padded image pitch,
    and an image large enough for the dynamic tail: still bit-identical."""
    tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=True)
    h, w = 4100, 6000
    base = torch.rand((h, w + 24), device="cuda")
    x = base[:, :w]  # row pitch w + 24 (16-B aligned)
    want = _two_launches(tr, x.contiguous())
    got = tr.forward2(x)
    assert got is not None
    for g, wv in zip(got[0] + got[1], want[0] + want[1]):
        assert torch.equal(g, wv)
    monkeypatch.setenv("B2DWT_MAX_LAUNCH_BYTES", str(16 << 20))
    got = tr.forward2(x)
    for g, wv in zip(got[0] + got[1], want[0] + want[1]):
        assert torch.equal(g, wv)


@pytest.mark.parametrize("fast", [False, True], ids=["strict", "fast"])
def test_two_fused_pairs_in_one_pyramid(fast, monkeypatch):
    """5 levels = pairs (0,1) and (2,3) plus level 4: the second pair reads one
    scratch half and must write its LL into the other (b2dwt_dwt), also inside
    the captured graph and its per-group event variant."""
    monkeypatch.setenv("B2DWT_FUSE2_MIN_QUADS", "1")
    s = build_scheme("non-separable-split", CDF97)
    img = np.random.default_rng(2).random((1024, 1536)).astype(np.float32)
    x = torch.from_numpy(img).cuda()
    fused = Transform(s, "single", fast=fast)
    plain = Transform(s, "single", fast=fast, fuse=False)
    a_ll, a_det = fused.dwt(x, 5)
    b_ll, b_det = plain.dwt(x, 5)
    assert torch.equal(a_ll, b_ll)
    for lvl in range(5):
        for u, v in zip(a_det[lvl], b_det[lvl]):
            assert torch.equal(u, v), lvl
    for events in (False, True):
        g = fused.capture_dwt(x, 5, level_events=events)
        assert g.groups == [(0, 1), (2, 3), (4, 4)]
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(g.ll, b_ll), events
        for lvl in range(5):
            for u, v in zip(g.details[lvl], b_det[lvl]):
                assert torch.equal(u, v), (events, lvl)
    if not fast:
        want_ll, _ = oracle.dwt(img, compile_scheme(s), 5)
        assert np.array_equal(a_ll.cpu().numpy(), want_ll)


def test_fusion_policy(monkeypatch):
    x = torch.rand((2048, 2048), device="cuda")
    s = build_scheme("non-separable-split", CDF97)
    assert Transform(s, "single", fast=True).capture_dwt(x, 3).groups == [(0, 1), (2, 2)]
    assert Transform(s, "single").capture_dwt(x, 3).groups == [(0, 1), (2, 2)]
    assert Transform(s, "single", fast=True, fuse=False).capture_dwt(x, 3).groups == [(0, 0), (1, 1), (2, 2)]
    monkeypatch.setenv("B2DWT_FUSE2_STRICT", "0")
    assert Transform(s, "single").capture_dwt(x, 3).groups == [(0, 0), (1, 1), (2, 2)]


def test_unfusable_requests_fall_back():
    s = build_scheme("separable-convolution", CDF97)  # per-sub-step reach 2: no fused kernel
    tr = Transform(s, "single")
    assert tr.forward2(torch.rand((512, 512), device="cuda")) is None
    narrow = Transform(build_scheme("non-separable-split", CDF97), "single")
    assert narrow.forward2(torch.rand((512, 128), device="cuda")) is None  # W < 256
    assert Transform(build_scheme("non-separable-split", CDF97), "double").forward2(
        torch.rand((512, 512), device="cuda", dtype=torch.float64)) is None
    # the pyramid still works (separate launches) and matches the oracle
    img = np.random.default_rng(1).random((256, 128)).astype(np.float32)
    ll, det = narrow.dwt(torch.from_numpy(img).cuda(), 2)
    want_ll, _ = oracle.dwt(img, compile_scheme(build_scheme("non-separable-split", CDF97)), 2)
    assert np.array_equal(ll.cpu().numpy(), want_ll)


def test_graph_replay_concurrent_with_other_stream_launches():
    """Dynamic-tail counters are per stream / per captured launch: a captured
    pyramid replayed while hundreds of eager launches run on another stream
    stays bit-exact (shared counter slots)."""
    tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=True)
    x = torch.rand((4096, 4096), device="cuda")
    g = tr.capture_dwt(x, 4)
    g.replay()
    torch.cuda.synchronize()
    want_ll = g.ll.clone()
    want_det = [tuple(t.clone() for t in d) for d in g.details]
    other = torch.cuda.Stream()
    y = torch.rand((2048, 2048), device="cuda")
    torch.cuda.synchronize()
    with torch.cuda.stream(other):
        outs = tr.forward(y)
    for _ in range(4):
        with torch.cuda.stream(other):
            for _ in range(80):
                tr.forward(y, out=outs)
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(g.ll, want_ll)
    for a, b in zip(g.details, want_det):
        for u, v in zip(a, b):
            assert torch.equal(u, v)


@pytest.mark.parametrize("seed", range(3))
def test_random_shapes_fused_pair_equals_two_launches(seed):
    """Random geometry: heights from the edge-units-only regime to many static
    units, widths across partial super-strips, padded pitches, both modes."""
    rng = np.random.default_rng(100 + seed)
    for trial in range(8):
        h = 4 * int(rng.integers(4, 400))
        w = 4 * int(rng.integers(64, 800))
        pad = 4 * int(rng.integers(0, 9))
        fast = bool(rng.integers(0, 2))
        wavelet, scheme = FUSABLE[int(rng.integers(0, len(FUSABLE)))]
        tr = Transform(build_scheme(scheme, PLANS[wavelet]), "single", fast=fast)
        base = torch.rand((h, w + pad), device="cuda", generator=torch.Generator(device="cuda").manual_seed(trial))
        x = base[:, :w]
        got = tr.forward2(x)
        assert got is not None, (h, w)
        want = _two_launches(tr, x.contiguous())
        for g, wv in zip(got[0] + got[1], want[0] + want[1]):
            assert torch.equal(g, wv), (seed, trial, h, w, pad, fast, wavelet, scheme)
