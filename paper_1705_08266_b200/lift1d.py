"""Batched 1-D lifting on the GPU.

Drop-in for the reference's 1-D executor ``apply_plan_1d`` / ``invert_plan_1d``
(liftfuse/schemes.py:806-856) -- same arguments, same (low, high) lists, same
"signal length must be even" error, bit-identical results (the reference lifts
in Python floats; the f64 kernels round every product and sum separately in
the same ascending-shift order) -- plus :class:`Lift1D`, which lifts a whole
``[B, N]`` batch of device-resident signals per call (``b2dwt_lift1d``).
Plans may be this package's or the reference's own ``LiftingPlan`` objects.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native

__all__ = ["Lift1D", "apply_plan_1d", "invert_plan_1d"]


def _terms(poly, sign=1.0):
    items = sorted(poly.terms.items())
    return [int(k) for k, _ in items], [sign * float(c) for _, c in items]


def _step_arrays(plan, inverse: bool):
    """Flattened (target, count, shifts, coefs) for the C ABI.  Forward: for
    each pair, odd += P(even) then even += U(odd); inverse: the pairs reversed,
    even -= U(odd) then odd -= P(even) (schemes.py:822-852)."""
    steps = []
    if not inverse:
        for p, u in plan.pairs:
            steps += [(1, *_terms(p)), (0, *_terms(u))]
    else:
        for p, u in reversed(plan.pairs):
            steps += [(0, *_terms(u, -1.0)), (1, *_terms(p, -1.0))]
    target = (ctypes.c_int32 * max(1, len(steps)))(*[s[0] for s in steps])
    count = (ctypes.c_int32 * max(1, len(steps)))(*[len(s[1]) for s in steps])
    flat_k = [k for s in steps for k in s[1]]
    flat_c = [c for s in steps for c in s[2]]
    shifts = (ctypes.c_int32 * max(1, len(flat_k)))(*flat_k)
    coefs = (ctypes.c_double * max(1, len(flat_c)))(*flat_c)
    scale = None
    if plan.scale is not None:
        scale = (ctypes.c_double * 2)(float(plan.scale[0]), float(plan.scale[1]))
    return len(steps), target, count, shifts, coefs, scale


class Lift1D:
    """1-D lifting of ``plan`` on CUDA tensors ``[B, N]`` (or ``[N]``), f32 or f64."""

    def __init__(self, plan):
        self.plan = plan
        self._fwd = _step_arrays(plan, inverse=False)
        self._inv = _step_arrays(plan, inverse=True)

    @staticmethod
    def _dtype(t):
        import torch

        if t.dtype == torch.float32:
            return _native.F32
        if t.dtype == torch.float64:
            return _native.F64
        raise TypeError("signals must be float32 or float64")

    def forward(self, x, stream=None):
        import torch

        from .engine import _ptr, _stream_handle

        squeeze = x.dim() == 1
        x2 = x.unsqueeze(0) if squeeze else x
        if x2.dim() != 2 or not x2.is_cuda or x2.stride(1) != 1:
            raise ValueError("forward takes a CUDA [B, N] (or [N]) tensor with contiguous rows")
        b, n = x2.shape
        if n % 2:
            raise ValueError("signal length must be even")
        low = torch.empty((b, n // 2), dtype=x2.dtype, device=x2.device)
        high = torch.empty_like(low)
        k, tgt, cnt, sh, cf, sc = self._fwd
        _native.check(
            _native.load().b2dwt_lift1d(self._dtype(x2), k, tgt, cnt, sh, cf, sc, _ptr(x2), x2.stride(0), _ptr(low),
                                        _ptr(high), low.stride(0), n, b, _stream_handle(torch, stream)),
            "lift1d",
        )
        return (low[0], high[0]) if squeeze else (low, high)

    def inverse(self, low, high, stream=None):
        import torch

        from .engine import _ptr, _stream_handle

        squeeze = low.dim() == 1
        lo = (low.unsqueeze(0) if squeeze else low).contiguous().clone()
        hi = (high.unsqueeze(0) if squeeze else high).contiguous().clone()
        if lo.shape != hi.shape or not lo.is_cuda:
            raise ValueError("low and high must be CUDA tensors of one shape")
        b, h = lo.shape
        out = torch.empty((b, 2 * h), dtype=lo.dtype, device=lo.device)
        k, tgt, cnt, sh, cf, sc = self._inv
        _native.check(
            _native.load().b2dwt_unlift1d(self._dtype(lo), k, tgt, cnt, sh, cf, sc, _ptr(lo), _ptr(hi), lo.stride(0),
                                          _ptr(out), out.stride(0), 2 * h, b, _stream_handle(torch, stream)),
            "unlift1d",
        )
        return out[0] if squeeze else out


def apply_plan_1d(plan, samples):
    """Forward 1-D transform of an even-length signal; returns (low, high) lists."""
    if len(samples) % 2:
        raise ValueError("signal length must be even")
    import torch

    x = torch.tensor(np.asarray(samples, dtype=np.float64), device="cuda")
    low, high = Lift1D(plan).forward(x)
    return low.cpu().tolist(), high.cpu().tolist()


def invert_plan_1d(plan, low, high):
    """Inverse of :func:`apply_plan_1d`."""
    import torch

    lo = torch.tensor(np.asarray(low, dtype=np.float64), device="cuda")
    hi = torch.tensor(np.asarray(high, dtype=np.float64), device="cuda")
    return Lift1D(plan).inverse(lo, hi).cpu().tolist()
