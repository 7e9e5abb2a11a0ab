"""CPU: the selector layer (lifting.py / program.py) reproduces the reference's
compiled StencilPrograms bit for bit, and the generated kernel structures are
current."""

import pytest

from paper_1705_08266_b200 import CDF53, CDF97, SCHEME_NAMES, build_scheme, compile_scheme, get_plan, invert_scheme
from paper_1705_08266_b200 import codegen
from paper_1705_08266_b200.lifting import LiftingPlan, poly1
from paper_1705_08266_b200.program import component_index, extend
from tests import golden_data as G
from fractions import Fraction as F

PLANS = {
    "cdf53": CDF53,
    "cdf97": CDF97,
    "haar-like": LiftingPlan("haar-like", ((poly1({0: F(-1)}), poly1({0: F(1, 2)})),)),
    "asym": LiftingPlan("asym", ((poly1({0: F(-3, 4), -1: F(-1, 4)}), poly1({0: F(1, 8), 1: F(3, 8)})),)),
    "trivial": LiftingPlan("trivial", ((poly1({}), poly1({})),)),
}


def _dump(prog):
    return [
        (s.reach, tuple(tuple((a, b, c, float(d).hex()) for (a, b, c, d) in t) for t in s.terms))
        for p in prog.passes
        for s in p.substeps
    ]


@pytest.mark.parametrize("wavelet", sorted(PLANS))
@pytest.mark.parametrize("scheme", SCHEME_NAMES)
def test_compiled_programs_match_reference_goldens(wavelet, scheme):
    progs = G.programs()
    s = build_scheme(scheme, PLANS[wavelet])
    assert _dump(compile_scheme(s)) == _dump(progs[f"{wavelet}/{scheme}/fwd"])
    assert _dump(compile_scheme(invert_scheme(s))) == _dump(progs[f"{wavelet}/{scheme}/inv"])


def test_double_inversion_is_forward():
    for name in SCHEME_NAMES:
        s = build_scheme(name, CDF97)
        assert _dump(compile_scheme(invert_scheme(invert_scheme(s)))) == _dump(compile_scheme(s))


def test_live_reference_schemes_compile_identically(liftfuse):
    """Duck typing: the reference's own Scheme objects compile to the same tables."""
    from liftfuse.engine import compile_scheme as ref_compile
    from liftfuse.schemes import build_scheme as ref_build
    from liftfuse.wavelets import CDF53 as R53, CDF97 as R97

    from paper_1705_08266_b200.engine import _programs

    for plan in (R53, R97):
        for name in SCHEME_NAMES:
            rs = ref_build(name, plan)
            fwd, inv = _programs(rs)
            assert _dump(fwd) == _dump(ref_compile(rs))


def test_step_counts_and_halo():
    # reference tests/test_acceptance.py:84-99 and tests/test_engine.py:101-107
    steps = {("cdf53", n): v for n, v in zip(SCHEME_NAMES, (2, 4, 2, 2))}
    steps.update({("cdf97", n): v for n, v in zip(SCHEME_NAMES, (2, 8, 4, 4))})
    for (w, n), v in steps.items():
        assert build_scheme(n, get_plan(w)).steps == v
    assert compile_scheme(build_scheme("non-separable-split", CDF97)).halo == 1
    assert compile_scheme(build_scheme("separable-convolution", CDF97)).halo == 2


def test_compiled_offsets_follow_exponent_convention():
    # reference tests/test_engine.py:90-98
    predict_h = compile_scheme(build_scheme("separable-lifting", CDF53)).passes[0].substeps[0]
    assert predict_h.terms[1] == ((0, 0, 0, -0.5), (1, 0, 0, 1.0), (0, 1, 0, -0.5))


def test_extend_known_answers():
    # reference tests/test_engine.py:34-57
    assert extend(-1, 8) == 1 and extend(8, 8) == 6 and extend(3, 8) == 3
    assert extend(-3, 8) == 3 and extend(9, 8) == 5 and extend(14, 8) == 0 and extend(-14, 8) == 0
    assert extend(5, 1) == 0 and extend(-2, 2) == 0
    with pytest.raises(ValueError):
        extend(0, 0)
    # App. B table: component-index reflection by phase
    for cs in (3, 5, 8):
        assert component_index(-1, 0, cs) == 1 and component_index(-1, 1, cs) == 0
        assert component_index(cs, 0, cs) == cs - 1 and component_index(cs, 1, cs) == cs - 2
        assert component_index(-2, 0, cs) == 2 and component_index(-2, 1, cs) == 1


def test_unknown_names_rejected():
    with pytest.raises(ValueError, match="unknown scheme"):
        build_scheme("nope", CDF53)
    with pytest.raises(ValueError, match="unknown wavelet"):
        get_plan("db4")


def test_codegen_is_current():
    import os

    with open(codegen.OUT) as fh:
        assert fh.read() == codegen.render(), "run python -m paper_1705_08266_b200.codegen"
