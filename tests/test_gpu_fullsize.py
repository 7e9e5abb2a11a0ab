"""GPU parity at the BASELINE.json configuration sizes:

* C3 (16384^2 f32, 9/7 non-separable-split, 5 levels): strict mode bit-exact
  against the CPU oracle for the whole pyramid, and fast mode within the north
  star's 1e-4 x input range;
* C4 (1024 x 2048^2, batch): batched launches (footprint-split into chunks)
  equal per-image launches bit for bit on a sample of items, and items match
  the oracle;
* C5 (65536^2): row bands computed from band buffers (the multi-GPU strip
  building block) equal the whole-image transform bit for bit; the fast
  whole-image output matches the f64 oracle on ~4100 x 65536 band buffers at
  both global edges and in the interior; forward + inverse reconstructs within
  1e-4 x range.
"""

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1705_08266_b200 import CDF97, Transform, build_scheme, compile_scheme  # noqa: E402

SCHEME = build_scheme("non-separable-split", CDF97)


def test_c3_pyramid_strict_bit_exact_and_fast_within_tolerance():
    n, levels = 16384, 5
    img = np.random.default_rng(0).random((n, n), dtype=np.float32)
    want_ll, want_det = oracle.dwt(img, compile_scheme(SCHEME), levels)
    x = torch.from_numpy(img).cuda()
    ll, det = Transform(SCHEME, "single").dwt(x, levels)
    assert np.array_equal(ll.cpu().numpy(), want_ll)
    for lvl in range(levels):
        for got, want in zip(det[lvl], want_det[lvl]):
            assert np.array_equal(got.cpu().numpy(), want), lvl
    fll, fdet = Transform(SCHEME, "single", fast=True).dwt(x, levels)
    tol = 1e-4 * float(img.max() - img.min())
    assert float(np.abs(fll.cpu().numpy() - want_ll).max()) <= tol
    for lvl in range(levels):
        for got, want in zip(fdet[lvl], want_det[lvl]):
            assert float(np.abs(got.cpu().numpy() - want).max()) <= tol


def test_c4_batch_equals_items_and_oracle():
    n_img, n = 1024, 2048
    tr = Transform(SCHEME, "single", fast=True)
    x = torch.empty((n_img, n, n), device="cuda")
    gen = torch.Generator(device="cuda").manual_seed(3)
    for i in range(0, n_img, 128):
        x[i:i + 128].uniform_(generator=gen)
    outs = tr.forward(x)  # 16 GiB in: runs as footprint-bounded batch chunks
    strict = Transform(SCHEME, "single")
    for b in (0, 1, 31, 32, 33, 511, 1023):
        single = tr.forward(x[b].contiguous())
        for cb, cs in zip(outs, single):
            assert torch.equal(cb[b], cs), b
    for b in (0, 777):
        img = x[b].cpu().numpy()
        want = oracle.forward(img, compile_scheme(SCHEME))
        got = strict.forward(x[b].contiguous())
        for g, w in zip(got, want):
            assert np.array_equal(g.cpu().numpy(), w), b
    # the benchmarked (fast, FMA) batched outputs against the f64 oracle
    for b in (5, 1000):
        img = x[b].cpu().numpy()
        want = oracle.forward(img.astype(np.float64), compile_scheme(SCHEME))
        tol = 1e-4 * float(img.max() - img.min())
        for c, w in zip(outs, want):
            err = float(np.abs(c[b].cpu().numpy().astype(np.float64) - w).max())
            assert err <= tol, (b, err)


def test_c5_row_bands_and_round_trip():
    n = 65536
    tr = Transform(SCHEME, "single", fast=True)
    x = torch.empty((n, n), device="cuda")
    gen = torch.Generator(device="cuda").manual_seed(5)
    for i in range(0, n, 4096):
        x[i:i + 4096].uniform_(generator=gen)
    full = tr.forward(x)  # 16 GiB: footprint-split into row bands inside the library
    up, down = tr.cone[0], tr.cone[1]
    rows = n // 2
    for r0, r1 in ((0, 4096), (8191, 8200), (rows // 2 - 3, rows // 2 + 5), (rows - 4096, rows)):
        b0, b1 = max(0, r0 - up), min(rows, r1 + down)
        out = tr.forward_rows(x[2 * b0:2 * b1], 2 * b0, n, r0, r1)
        for o, f in zip(out, full):
            assert torch.equal(o, f[r0:r1]), (r0, r1)
    # fast bands against the f64 oracle run on a band buffer (~4100 x 65536):
    # both global edges and one interior band.  The oracle reflects at the
    # buffer's own cut edges too, which reaches at most `up`/`down` quad rows
    # in from a cut, so the compared rows keep that margin from every cut.
    prog = compile_scheme(SCHEME)
    margin = 4
    for r0, r1 in ((0, 2048), (rows // 2 - 1024, rows // 2 + 1024), (rows - 2048, rows)):
        b0, b1 = max(0, r0 - up - margin), min(rows, r1 + down + margin)
        band = x[2 * b0:2 * b1].cpu().numpy()
        want = oracle.forward(band.astype(np.float64), prog)
        tol = 1e-4 * float(band.max() - band.min())
        for c, w in zip(full, want):
            err = float(np.abs(c[r0:r1].cpu().numpy().astype(np.float64) - w[r0 - b0:r1 - b0]).max())
            assert err <= tol, (r0, r1, err)
        del band, want
    rec = tr.inverse(*full)
    del full
    err = 0.0
    for i in range(0, n, 4096):
        err = max(err, float((rec[i:i + 4096] - x[i:i + 4096]).abs().max()))
    assert err <= 1e-4, err
