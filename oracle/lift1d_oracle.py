"""CPU oracle for the batched 1-D lifting kernels (b2dwt_lift1d).

TEST INFRASTRUCTURE ONLY -- imported by tests/, never by the product package.

A plain-Python restatement of the reference's 1-D executor
(liftfuse/schemes.py:796-856): even/odd split, for each (P, U) pair
``odd[i] += sum_k p_k even[ext_even(i-k)]`` then ``even[i] += sum_k u_k
odd[ext_odd(i-k)]`` with terms in ascending k (schemes.py:796-803), the
whole-sample symmetric extension of engine.py:55-71, then the (lo, hi) gains;
the inverse divides by the gains and runs the pairs backwards with negated
polynomials.  Pinned to outputs of the real reference
(tests/golden/lift1d.npz, tests/golden/make_lift1d_golden.py).
"""

from __future__ import annotations


def extend(i: int, n: int) -> int:
    """Whole-sample symmetric extension (engine.py:55-71)."""
    if n == 1:
        return 0
    period = 2 * n - 2
    r = i % period
    return period - r if r >= n else r


def _conv(target, source, terms, ext):
    for i in range(len(target)):
        acc = target[i]
        for k, c in terms:
            acc += c * source[ext(i - k)]
        target[i] = acc
    return target


def _sorted(poly, sign=1.0):
    return [(k, sign * float(c)) for k, c in sorted(poly.terms.items())]


def apply_plan_1d(plan, samples):
    if len(samples) % 2:
        raise ValueError("signal length must be even")
    n = len(samples)
    even = [float(samples[2 * i]) for i in range(n // 2)]
    odd = [float(samples[2 * i + 1]) for i in range(n // 2)]
    ext_e = lambda i: extend(2 * i, n) // 2  # noqa: E731
    ext_o = lambda i: (extend(2 * i + 1, n) - 1) // 2  # noqa: E731
    for p, u in plan.pairs:
        odd = _conv(odd, even, _sorted(p), ext_e)
        even = _conv(even, odd, _sorted(u), ext_o)
    if plan.scale is not None:
        lo, hi = float(plan.scale[0]), float(plan.scale[1])
        even = [lo * v for v in even]
        odd = [hi * v for v in odd]
    return even, odd


def invert_plan_1d(plan, low, high):
    even = [float(v) for v in low]
    odd = [float(v) for v in high]
    n = 2 * len(even)
    ext_e = lambda i: extend(2 * i, n) // 2  # noqa: E731
    ext_o = lambda i: (extend(2 * i + 1, n) - 1) // 2  # noqa: E731
    if plan.scale is not None:
        lo, hi = float(plan.scale[0]), float(plan.scale[1])
        even = [v / lo for v in even]
        odd = [v / hi for v in odd]
    for p, u in reversed(plan.pairs):
        even = _conv(even, odd, _sorted(u, -1.0), ext_o)
        odd = _conv(odd, even, _sorted(p, -1.0), ext_e)
    out = [0.0] * n
    out[0::2] = even
    out[1::2] = odd
    return out
