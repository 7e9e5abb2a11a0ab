"""Caller-buffer validation of the device API:
a wrong ``out=`` / input plane must raise before any pointer reaches the C ABI
(out-of-bounds device writes or host corruption otherwise)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1705_08266_b200 import CDF97, Transform, build_scheme  # noqa: E402

S = build_scheme("non-separable-split", CDF97)


def _planes(shape, **kw):
    return tuple(torch.empty(shape, device="cuda", **kw) for _ in range(4))


def test_forward_out_checked():
    tr = Transform(S, "single")
    x = torch.rand((64, 96), device="cuda")
    tr.forward(x, out=_planes((32, 48)))  # fine
    with pytest.raises(ValueError, match="shape"):
        tr.forward(x, out=_planes((32, 40)))
    with pytest.raises(TypeError):
        tr.forward(x, out=_planes((32, 48), dtype=torch.float64))
    with pytest.raises(TypeError):
        tr.forward(x, out=tuple(torch.empty((32, 48)) for _ in range(4)))  # host tensors
    with pytest.raises(ValueError):
        tr.forward(x, out=_planes((32, 48))[:3])
    wide = torch.empty((32, 96), device="cuda")
    with pytest.raises(ValueError, match="contiguous"):
        tr.forward(x, out=(wide[:, ::2],) + _planes((32, 48))[1:])
    xb = torch.rand((3, 64, 96), device="cuda")
    bad = (torch.empty((3, 32, 48), device="cuda"), torch.empty((3, 32, 48), device="cuda"),
           torch.empty((3, 32, 64), device="cuda")[:, :, :48], torch.empty((3, 32, 48), device="cuda"))
    with pytest.raises(ValueError, match="batch stride"):
        tr.forward(xb, out=bad)


def test_inverse_and_components_inputs_checked():
    tr = Transform(S, "single")
    ll, hl, lh, hh = tr.forward(torch.rand((64, 96), device="cuda"))
    with pytest.raises(TypeError):
        tr.inverse(ll, hl.cpu(), lh, hh)
    with pytest.raises(ValueError, match="share dimensions"):
        tr.inverse(ll, hl[:, :40], lh, hh)
    with pytest.raises(ValueError, match="shape"):
        tr.inverse(ll, hl, lh, hh, out=torch.empty((64, 90), device="cuda"))
    with pytest.raises(ValueError):
        tr.run_components([ll, hl, lh])
    with pytest.raises(ValueError, match="shape"):
        tr.run_components([ll, hl, lh, hh], out=_planes((32, 40)))


def test_pyramid_and_host_buffers_checked():
    tr = Transform(S, "single")
    x = torch.rand((128, 128), device="cuda")
    ll, det = tr.dwt(x, 3)
    with pytest.raises(ValueError):
        tr.idwt(ll, det[:2] + [(det[2][0], det[2][1], det[2][2][:, :8])])
    hx = torch.rand((128, 128))
    with pytest.raises(ValueError, match="shape"):
        tr.dwt_host(hx, 2, details=[tuple(torch.empty((64, 64)) for _ in range(3)),
                                    tuple(torch.empty((32, 30)) for _ in range(3))])
    with pytest.raises(ValueError, match="host"):
        tr.dwt_host(hx, 1, details=[tuple(torch.empty((64, 64), device="cuda") for _ in range(3))])
    with pytest.raises(ValueError, match="scratch"):
        tr.dwt_into(x, 2, [tuple(torch.empty((64, 64), device="cuda") for _ in range(3)),
                           tuple(torch.empty((32, 32), device="cuda") for _ in range(3))],
                    torch.empty((32, 32), device="cuda"), torch.empty((10,), device="cuda"))


def test_reference_api_cache_is_bounded():
    from paper_1705_08266_b200 import Image2D, engine, forward

    img = Image2D.random(32, 32, seed=0, precision="single")
    forward(img, build_scheme("non-separable-split", CDF97))
    before = len(engine._TRANSFORMS)
    for _ in range(40):  # a fresh scheme object per call, as the reference API invites
        forward(img, build_scheme("non-separable-split", CDF97))
    assert len(engine._TRANSFORMS) == before  # keyed by the compiled programs, not the object
    assert len(engine._TRANSFORMS) <= engine._TRANSFORMS_MAX
    assert np.isfinite(forward(img, S).ll.data).all()
