"""Memory-safety checks without compute-sanitizer (closed on this GPU pool: runs
under it left GPUs needing a reset), for every kernel family:

* out-of-bounds READS: every input sits inside a larger buffer whose padding
  (extra columns and rows on all sides) holds NaN; a read outside the image or
  its row band would put NaN into some output, so all outputs must be finite;
* out-of-bounds WRITES and unwritten outputs: every output plane sits inside a
  padded buffer filled with a sentinel bit pattern; afterwards the padding must
  still hold the sentinel and the plane itself none of it (initcheck's question
  for outputs), and the plane must equal the reference result;
* shared-memory races (racecheck's question): repeated runs, on the TMA and
  mbarrier rings and the fused kernel's LL ring, must be bit-identical.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1705_08266_b200 import CDF53, CDF97, Transform, build_scheme  # noqa: E402

SENTINEL = -1.2345678e30
PAD = 40  # elements of padding on every side (beyond any cone)


def padded(shape, fill, dtype=torch.float32):
    """A view of `shape` inside a buffer padded by PAD rows/columns of `fill`
    (row pitch rounded to 16 B so the TMA paths stay eligible)."""
    h, w = shape
    pitch = w + 2 * PAD
    pitch += (-pitch) % (16 // torch.tensor([], dtype=dtype).element_size())
    buf = torch.full((h + 2 * PAD, pitch), fill, dtype=dtype, device="cuda")
    return buf, buf[PAD:PAD + h, PAD:PAD + w]


def padded_input(img):
    buf, view = padded(img.shape, float("nan"), img.dtype)
    view.copy_(img)
    return buf, view


def check_guard(buf, view, ref):
    inner = torch.zeros_like(buf, dtype=torch.bool)
    h, w = view.shape
    inner[PAD:PAD + h, PAD:PAD + w] = True
    assert bool((buf[~inner] == SENTINEL).all()), "write outside the output plane"
    assert not bool((view == SENTINEL).any()), "output element never written"
    assert bool(torch.isfinite(view).all()), "NaN from a read outside the input"
    assert torch.equal(view, ref)


VARIANTS = [dict(tile=False), dict(tile=False, tma=False), dict(tile=True), dict(force_generic=True),
            dict(force_generic=True, tile=False)]


@pytest.mark.parametrize("variant", VARIANTS, ids=["stream-tma", "stream-cpasync", "tile", "gtile", "gsubstep"])
@pytest.mark.parametrize("shape", [(6, 10), (66, 130), (520, 1040), (1030, 2050)])
def test_forward_inverse_guard_bands(variant, shape):
    if variant.get("force_generic") and shape[0] > 600:
        shape = (258, 386)  # the interpreters are slow; their edge logic is size-independent
    for plan in (CDF97, CDF53):
        s = build_scheme("non-separable-split", plan)
        ref = Transform(s, "single")
        tr = Transform(s, "single", **variant)
        img = torch.rand(shape, device="cuda")
        want = ref.forward(img)
        _, xin = padded_input(img)
        outs = [padded((shape[0] // 2, shape[1] // 2), SENTINEL) for _ in range(4)]
        tr.forward(xin, out=tuple(v for _, v in outs))
        for (b, v), r in zip(outs, want):
            check_guard(b, v, r)
        # inverse from padded NaN-guarded planes into a sentinel-guarded image
        planes = [padded_input(c)[1] for c in want]
        ob, ov = padded(shape, SENTINEL)
        tr.inverse(*planes, out=ov)
        check_guard(ob, ov, ref.inverse(*want))


@pytest.mark.parametrize("fast", [False, True], ids=["strict", "fast"])
def test_fused_pair_guard_bands(fast):
    tr = Transform(build_scheme("non-separable-split", CDF97), "single", fast=fast)
    for shape in ((48, 256), (1032, 1544), (2048, 4096)):
        img = torch.rand(shape, device="cuda")
        ll0, hl0, lh0, hh0 = tr.forward(img)
        want = (hl0, lh0, hh0) + tuple(tr.forward(ll0.contiguous()))
        _, xin = padded_input(img)
        d0 = [padded((shape[0] // 2, shape[1] // 2), SENTINEL) for _ in range(3)]
        d1 = [padded((shape[0] // 4, shape[1] // 4), SENTINEL) for _ in range(4)]
        got = tr.forward2(xin, tuple(v for _, v in d0), tuple(v for _, v in d1))
        assert got is not None
        for (b, v), r in zip(d0 + d1, want):
            check_guard(b, v, r)


def test_row_band_guard_bands():
    tr = Transform(build_scheme("non-separable-split", CDF97), "single")
    h, w = 512, 300
    x = torch.rand((h, w), device="cuda")
    full = tr.forward(x)
    up, down = tr.cone[0], tr.cone[1]
    for r0, r1 in ((0, 64), (17, 93), (200, 256)):
        b0, b1 = max(0, r0 - up), min(h // 2, r1 + down)
        _, band = padded_input(x[2 * b0:2 * b1])
        outs = [padded((r1 - r0, w // 2), SENTINEL) for _ in range(4)]
        tr.forward_rows(band, 2 * b0, h, r0, r1, out=tuple(v for _, v in outs))
        for (b, v), f in zip(outs, full):
            check_guard(b, v, f[r0:r1])


def test_repeated_runs_bit_identical():
    """Shared-memory rings (TMA + mbarriers, the fused kernel's LL ring, the tile
    kernel's double buffers): 20 runs of each must agree bit for bit."""
    x = torch.rand((4096, 4096), device="cuda")
    s = build_scheme("non-separable-split", CDF97)
    for kw in (dict(tile=False), dict(tile=False, tma=False), dict(tile=True), dict(fast=True)):
        tr = Transform(s, "single", **kw)
        first = [t.clone() for t in tr.forward(x)]
        pair = tr.forward2(x) if kw.get("fast") else None
        pair0 = [t.clone() for t in (pair[0] + pair[1])] if pair else None
        for _ in range(20):
            for a, b in zip(tr.forward(x), first):
                assert torch.equal(a, b), kw
            if pair0 is not None:
                p = tr.forward2(x)
                for a, b in zip(p[0] + p[1], pair0):
                    assert torch.equal(a, b), kw


def test_host_pipelines_guard_host_buffers():
    """The host pipelines write HOST memory with 2-D copies: padded pinned
    planes must keep their sentinel padding."""
    tr = Transform(build_scheme("non-separable-split", CDF97), "single")
    h, w, levels = 1024, 768, 3
    x = torch.rand((h, w)).pin_memory()
    ll_d, det_d = tr.dwt(x.cuda(), levels)

    def host_padded(shape):
        buf = torch.full((shape[0] + 2 * PAD, shape[1] + 2 * PAD), SENTINEL).pin_memory()
        return buf, buf[PAD:PAD + shape[0], PAD:PAD + shape[1]]

    dets = [[host_padded((h >> (l + 1), w >> (l + 1))) for _ in range(3)] for l in range(levels)]
    llb, llv = host_padded((h >> levels, w >> levels))
    tr.dwt_host(x, levels, details=[tuple(v for _, v in d) for d in dets], ll=llv, bands=8)
    for l in range(levels):
        for (b, v), r in zip(dets[l], det_d[l]):
            assert bool((b[:PAD] == SENTINEL).all()) and bool((b[PAD + v.shape[0]:] == SENTINEL).all())
            assert bool((b[:, :PAD] == SENTINEL).all()) and bool((b[:, PAD + v.shape[1]:] == SENTINEL).all())
            assert torch.equal(v, r.cpu())
    assert torch.equal(llv, ll_d.cpu()) and bool((llb[:PAD] == SENTINEL).all())
    ob = torch.full((h + 2 * PAD, w + 2 * PAD), SENTINEL).pin_memory()
    ov = ob[PAD:PAD + h, PAD:PAD + w]
    tr.idwt_host(llv, [tuple(v for _, v in d) for d in dets], out=ov, bands=8)
    assert torch.equal(ov, tr.idwt(ll_d, det_d).cpu())
    assert bool((ob[:PAD] == SENTINEL).all()) and bool((ob[:, :PAD] == SENTINEL).all())
    assert bool((ob[PAD + h:] == SENTINEL).all()) and bool((ob[:, PAD + w:] == SENTINEL).all())
    assert np.isfinite(ov.numpy()).all()
