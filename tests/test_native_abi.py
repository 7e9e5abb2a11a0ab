"""CPU: the C-ABI library loads, exports every symbol include/b2dwt.h declares,
and its host-side logic (plan matching, validation, error codes) works without
a GPU.  No pixel is computed here."""

import ctypes
import os
import re

import pytest

from paper_1705_08266_b200 import CDF53, CDF97, SCHEME_NAMES, _native, build_scheme, compile_scheme, invert_scheme
from paper_1705_08266_b200.lifting import LiftingPlan, poly1
from fractions import Fraction as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_native.LIB_PATH):
        import __graft_entry__

        __graft_entry__.build()
    return _native.load()


def test_exports_every_declared_symbol(lib):
    with open(os.path.join(ROOT, "include", "b2dwt.h")) as fh:
        header = fh.read()
    declared = set(re.findall(r"\b(b2dwt_[a-z0-9_]+)\s*\(", header))
    assert declared == set(_native.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.b2dwt_abi_version() == 1


def test_builtin_programs_select_fused_kernel(lib):
    keys = set()
    for plan in (CDF53, CDF97):
        for name in SCHEME_NAMES:
            s = build_scheme(name, plan)
            for direction, prog in (("fwd", compile_scheme(s)), ("inv", compile_scheme(invert_scheme(s)))):
                for dtype in (_native.F32, _native.F64):
                    p = _native.Plan(prog, dtype)
                    assert p.fused, (plan.name, name, direction)
                    assert p.key == f"{plan.name}/{name}/{direction}"
                    keys.add(p.key)
    assert len(keys) == 16


def test_other_coefficients_use_generic_interpreter(lib):
    # the fused kernels have the built-in coefficients compiled in as immediates
    asym = LiftingPlan("asym", ((poly1({0: F(-3, 4), -1: F(-1, 4)}), poly1({0: F(1, 8), 1: F(3, 8)})),))
    p = _native.Plan(compile_scheme(build_scheme("non-separable-split", asym)), _native.F32)
    assert not p.fused and p.key == "generic"


def test_other_supports_use_generic_interpreter(lib):
    haar = LiftingPlan("haar-like", ((poly1({0: F(-1)}), poly1({0: F(1, 2)})),))
    p = _native.Plan(compile_scheme(build_scheme("non-separable-lifting", haar)), _native.F32)
    assert not p.fused and p.key == "generic"
    forced = _native.Plan(compile_scheme(build_scheme("non-separable-split", CDF97)), _native.F32,
                          _native.FORCE_GENERIC)
    assert not forced.fused


def test_cone_of_fused_programs(lib):
    p97 = _native.Plan(compile_scheme(build_scheme("non-separable-split", CDF97)), _native.F32)
    p53 = _native.Plan(compile_scheme(build_scheme("non-separable-split", CDF53)), _native.F32)
    # measured fused cone: 2 quads per side for 9/7, 1 for 5/3
    assert p97.cone == (2, 2, 2, 2)
    assert p53.cone == (1, 1, 1, 1)


def test_validation_errors_without_gpu(lib):
    p = _native.Plan(compile_scheme(build_scheme("non-separable-split", CDF97)), _native.F32)
    pl = _native.planes([1, 1, 1, 1], [4, 4, 4, 4])
    rc = lib.b2dwt_forward(p.handle, ctypes.c_void_p(1), 8, 0, 5, 8, ctypes.byref(pl), 1, None)
    assert rc == _native.B2DWT_EINVAL
    assert lib.b2dwt_last_error().decode() == "dimensions must be even, got 8x5"
    with pytest.raises(ValueError, match="dimensions must be even"):
        _native.check(rc)
    bad = _native.Program(7, 0, None, None)
    h = ctypes.c_void_p()
    assert lib.b2dwt_plan_create(ctypes.byref(bad), 0, 0, ctypes.byref(h)) == _native.B2DWT_EINVAL


def test_no_cpu_fallback_without_device(lib):
    """On a host without a GPU every compute call must fail loudly."""
    if lib.b2dwt_device_count() > 0:
        pytest.skip("a CUDA device is present")
    p = _native.Plan(compile_scheme(build_scheme("non-separable-split", CDF97)), _native.F32)
    pl = _native.planes([8, 8, 8, 8], [4, 4, 4, 4])
    rc = lib.b2dwt_forward(p.handle, ctypes.c_void_p(16), 8, 0, 8, 8, ctypes.byref(pl), 1, None)
    assert rc == _native.B2DWT_ECUDA


def test_dwt_host_workspace_and_validation(lib):
    """b2dwt_dwt_host: workspace sizing and argument checks are host logic."""
    p = _native.Plan(compile_scheme(build_scheme("non-separable-split", CDF97)), _native.F32)
    n, levels = 16384, 5

    def up(x):
        return (x + 255) // 256 * 256

    want = up(n * n * 4)
    for lvl in range(levels):
        q = (n >> (lvl + 1)) ** 2 * 4
        want = up(want + q)
        want = up(want + 3 * up(q))
    assert lib.b2dwt_dwt_host_workspace(p.handle, n, n, levels) == want
    assert lib.b2dwt_dwt_host_workspace(p.handle, n, n, 0) == -1
    det = (_native.Planes * levels)()
    args = (ctypes.c_void_p(4096), n, n, n, levels, det, ctypes.c_void_p(4096), n >> levels)
    assert lib.b2dwt_dwt_host(p.handle, *args, None, want, 16, None) == _native.B2DWT_EINVAL
    assert lib.b2dwt_dwt_host(p.handle, *args, ctypes.c_void_p(4096), want - 1, 16, None) == _native.B2DWT_EINVAL
    assert "workspace too small" in lib.b2dwt_last_error().decode()
    bad = (ctypes.c_void_p(4096), n, n + 2, n, levels, det, ctypes.c_void_p(4096), n >> levels)
    assert lib.b2dwt_dwt_host(p.handle, *bad, ctypes.c_void_p(4096), want, 16, None) == _native.B2DWT_EINVAL
    inv = _native.Plan(compile_scheme(invert_scheme(build_scheme("non-separable-split", CDF97))), _native.F32)
    assert lib.b2dwt_dwt_host(inv.handle, *args, ctypes.c_void_p(4096), want, 16, None) == \
        _native.B2DWT_EUNSUPPORTED
    if lib.b2dwt_device_count() == 0:
        # valid request, no device: fails loudly, never computes on the CPU
        assert lib.b2dwt_dwt_host(p.handle, *args, ctypes.c_void_p(4096), want, 16, None) == _native.B2DWT_ECUDA
