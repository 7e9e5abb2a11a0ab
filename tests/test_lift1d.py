"""1-D lifting: the CPU oracle against fixtures from the real reference, and
the GPU kernels (b2dwt_lift1d) against both."""

import os

import numpy as np
import pytest

from oracle import lift1d_oracle as O
from tests.lift1d_plans import LENGTHS, PLANS

GOLD = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "lift1d.npz"))


@pytest.mark.parametrize("name", sorted(PLANS))
def test_oracle_matches_reference_fixtures(name):
    plan = PLANS[name]
    for n in LENGTHS:
        x = GOLD[f"{name}/{n}/x"]
        lo, hi = O.apply_plan_1d(plan, list(x))
        assert np.array_equal(lo, GOLD[f"{name}/{n}/low"]) and np.array_equal(hi, GOLD[f"{name}/{n}/high"])
        assert np.array_equal(O.invert_plan_1d(plan, lo, hi), GOLD[f"{name}/{n}/rec"])
    with pytest.raises(ValueError, match="signal length must be even"):
        O.apply_plan_1d(plan, [1.0, 2.0, 3.0])


def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return torch


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(PLANS))
def test_gpu_matches_reference_fixtures(name):
    _cuda()
    from paper_1705_08266_b200.lift1d import apply_plan_1d, invert_plan_1d

    plan = PLANS[name]
    for n in LENGTHS:
        lo, hi = apply_plan_1d(plan, list(GOLD[f"{name}/{n}/x"]))
        assert np.array_equal(lo, GOLD[f"{name}/{n}/low"]) and np.array_equal(hi, GOLD[f"{name}/{n}/high"]), n
        assert np.array_equal(invert_plan_1d(plan, lo, hi), GOLD[f"{name}/{n}/rec"]), n


@pytest.mark.gpu
def test_gpu_batch_vs_oracle():
    torch = _cuda()
    from paper_1705_08266_b200.lift1d import Lift1D

    rng = np.random.default_rng(4)
    for name in ("cdf97", "wide"):
        plan = PLANS[name]
        x = rng.random((7, 1030))
        lo, hi = Lift1D(plan).forward(torch.from_numpy(x).cuda())
        for b in range(7):
            wl, wh = O.apply_plan_1d(plan, list(x[b]))
            assert np.array_equal(lo[b].cpu().numpy(), wl) and np.array_equal(hi[b].cpu().numpy(), wh)
        rec = Lift1D(plan).inverse(lo, hi)
        assert float((rec.cpu() - torch.from_numpy(x)).abs().max()) < 1e-12
        # f32: rounded in f32, within the north-star tolerance of the f64 result
        lo32, hi32 = Lift1D(plan).forward(torch.from_numpy(x.astype(np.float32)).cuda())
        assert float((lo32.double().cpu() - lo.cpu()).abs().max()) < 1e-4
        with pytest.raises(ValueError, match="signal length must be even"):
            Lift1D(plan).forward(torch.zeros((2, 7), device="cuda", dtype=torch.float64))
