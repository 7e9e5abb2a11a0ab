"""Wavelet lifting plans and the four 2-D transform schedules (selector layer).

This module is the construction-time half of the drop-in: it turns a 1-D
lifting plan into one of the four 2-D schedules of arXiv 1705.08266 and
lowers it (see :mod:`.program`) to the multiply-accumulate term tables that
the sm_100a kernels execute.  It runs on the host in microseconds; no pixel
ever passes through it.

It restates, for the GPU box where the reference package is absent, the
algebra the reference uses to derive those tables:

* sparse Laurent polynomials with insertion-ordered accumulation
  (reference ``liftfuse/laurent.py:72-277``) -- the accumulation order is
  kept because it fixes the floating-point bits of derived coefficients
  (``P*P`` cross terms, inverse back-substitution, convolution taps);
* 4x4 step matrices with product and unit-triangular inversion
  (``liftfuse/schemes.py:111-251``);
* the scheme builders (``schemes.py:328-421``, ``:544-591``, ``:597-714``)
  and ``invert_scheme`` (``schemes.py:738-787``);
* the built-in plans CDF 5/3 and CDF 9/7 (``liftfuse/wavelets.py:26-71``).

Symbolic proofs, pretty printers and consistency guards of the reference are
deliberately not restated (out of scope).  The CPU test
``tests/test_programs.py`` pins every compiled table produced here against the
reference's own compiled tables, bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

__all__ = [
    "EXACT",
    "FLOAT",
    "Laurent",
    "LiftingPlan",
    "StepMatrix",
    "Pass",
    "Scheme",
    "SCHEME_NAMES",
    "CDF53",
    "CDF97",
    "WAVELETS",
    "get_plan",
    "poly1",
    "build_scheme",
    "invert_scheme",
]

EXACT = "exact"
FLOAT = "float"

SCHEME_NAMES = (
    "separable-convolution",
    "separable-lifting",
    "non-separable-lifting",
    "non-separable-split",
)


# -- sparse Laurent polynomials -------------------------------------------------


def _key_add(a, b):
    if isinstance(a, tuple):
        return (a[0] + b[0], a[1] + b[1])
    return a + b


def _coerce(c, mode):
    if mode == EXACT:
        return c if isinstance(c, Fraction) else Fraction(c)
    return float(c)


class Laurent:
    """Sparse Laurent polynomial ``sum_k c_k z^{-k}``.

    Keys are ints (1-D) or ``(k_m, k_n)`` tuples (2-D, ``m`` horizontal).
    Coefficients are ``Fraction`` (exact mode) or ``float``.  Zero
    coefficients are dropped and the remaining terms keep insertion order,
    which is the order every product and sum below accumulates in
    (mirrors ``liftfuse/laurent.py:99-127``, ``:193-214``).
    """

    __slots__ = ("terms", "mode")

    def __init__(self, terms, mode=EXACT):
        self.mode = mode
        self.terms = {k: _coerce(c, mode) for k, c in terms.items() if c != 0}

    # ring operations ------------------------------------------------------------
    def __add__(self, other):
        acc = dict(self.terms)
        for k, c in other.terms.items():
            acc[k] = acc.get(k, 0) + c
        return Laurent(acc, self.mode)

    def __neg__(self):
        return Laurent({k: -c for k, c in self.terms.items()}, self.mode)

    def __sub__(self, other):
        return self + (-other)

    def __mul__(self, other):
        acc = {}
        for ka, ca in self.terms.items():
            for kb, cb in other.terms.items():
                k = _key_add(ka, kb)
                acc[k] = acc.get(k, 0) + ca * cb
        return Laurent(acc, self.mode)

    # helpers -----------------------------------------------------------------------
    def is_zero(self):
        return not self.terms

    def is_one(self):
        return len(self.terms) == 1 and self.terms.get((0, 0), None) == 1

    def constant_term(self):
        return self.terms.get(0, _coerce(0, self.mode))

    def reach(self):
        best = 0
        for k in self.terms:
            r = max(abs(k[0]), abs(k[1])) if isinstance(k, tuple) else abs(k)
            best = max(best, r)
        return best

    def horizontal(self):
        """Embed a 1-D polynomial along the image's horizontal axis."""
        return Laurent({(k, 0): c for k, c in self.terms.items()}, self.mode)

    def vertical(self):
        """Embed a 1-D polynomial along the image's vertical axis."""
        return Laurent({(0, k): c for k, c in self.terms.items()}, self.mode)

    def transpose(self):
        return Laurent({(k[1], k[0]): c for k, c in self.terms.items()}, self.mode)

    def __eq__(self, other):
        return isinstance(other, Laurent) and self.mode == other.mode and self.terms == other.terms

    def __repr__(self):
        return f"Laurent({self.terms!r}, {self.mode})"


def poly1(terms, mode=EXACT) -> Laurent:
    """A 1-D lifting polynomial, e.g. ``poly1({0: a, -1: a})`` for ``a(1 + z)``."""
    return Laurent(dict(terms), mode)


def _zero2(mode):
    return Laurent({}, mode)


def _one2(mode):
    return Laurent({(0, 0): 1}, mode)


def _const2(c, mode):
    return Laurent({(0, 0): c}, mode)


# -- lifting plans ------------------------------------------------------------------


@dataclass(frozen=True)
class LiftingPlan:
    """Ordered predict/update pairs plus optional final ``(low, high)`` gains.

    Same meaning as ``liftfuse.schemes.LiftingPlan`` (``schemes.py:87-108``).
    """

    name: str
    pairs: tuple
    scale: tuple | None = None
    mode: str = EXACT

    def __post_init__(self):
        object.__setattr__(self, "pairs", tuple(tuple(pu) for pu in self.pairs))
        if len(self.pairs) < 1:
            raise ValueError("a lifting plan needs at least one predict/update pair")
        for p, u in self.pairs:
            if p.mode != self.mode or u.mode != self.mode:
                raise ValueError("lifting filters must match the plan's coefficient mode")


# CDF 5/3: predict reads even[m], even[m+1]; update reads odd[m-1], odd[m]
# (``wavelets.py:23-36``).
CDF53 = LiftingPlan(
    name="cdf53",
    pairs=((poly1({0: Fraction(-1, 2), -1: Fraction(-1, 2)}), poly1({0: Fraction(1, 4), 1: Fraction(1, 4)})),),
    scale=None,
    mode=EXACT,
)

# CDF 9/7 lifting constants and gains (``wavelets.py:38-60``).
_A, _B, _G, _D, _K = (
    -1.586134342059924,
    -0.052980118572961,
    0.882911075530934,
    0.443506852043971,
    1.230174104914001,
)
CDF97 = LiftingPlan(
    name="cdf97",
    pairs=(
        (poly1({0: _A, -1: _A}, FLOAT), poly1({0: _B, 1: _B}, FLOAT)),
        (poly1({0: _G, -1: _G}, FLOAT), poly1({0: _D, 1: _D}, FLOAT)),
    ),
    scale=(1.0 / _K, _K),
    mode=FLOAT,
)

WAVELETS = {"cdf53": CDF53, "cdf97": CDF97}


def get_plan(name: str) -> LiftingPlan:
    try:
        return WAVELETS[name]
    except KeyError:
        raise ValueError(
            f"unknown wavelet {name!r}; expected one of {', '.join(sorted(WAVELETS))}"
        ) from None


# -- step matrices ------------------------------------------------------------------


class StepMatrix:
    """4x4 matrix of 2-D Laurent polynomials acting on the quadruple.

    Component order 1..4 = (even row, even col), (even, odd), (odd, even),
    (odd, odd) (``schemes.py:3-14``).
    """

    __slots__ = ("entries", "label")

    def __init__(self, entries, label):
        self.entries = tuple(tuple(r) for r in entries)
        self.label = label

    @property
    def mode(self):
        return self.entries[0][0].mode

    @classmethod
    def diagonal(cls, gains, mode, label):
        z = _zero2(mode)
        return cls([[_const2(gains[i], mode) if i == j else z for j in range(4)] for i in range(4)], label)

    def __matmul__(self, other):
        zero = _zero2(self.mode)
        rows = []
        for i in range(4):
            row = []
            for j in range(4):
                acc = zero
                for k in range(4):
                    a, b = self.entries[i][k], other.entries[k][j]
                    if a.is_zero() or b.is_zero():
                        continue
                    acc = acc + a * b
                row.append(acc)
            rows.append(row)
        return StepMatrix(rows, f"{self.label}*{other.label}")

    def relabel(self, label):
        return StepMatrix(self.entries, label)

    def reach(self):
        return max(e.reach() for row in self.entries for e in row)

    def _is_diagonal(self):
        return all(self.entries[i][j].is_zero() for i in range(4) for j in range(4) if i != j)

    def _unit_triangular(self, lower):
        if not all(self.entries[i][i].is_one() for i in range(4)):
            return False
        if lower:
            return all(self.entries[i][j].is_zero() for i in range(4) for j in range(i + 1, 4))
        return all(self.entries[i][j].is_zero() for i in range(4) for j in range(i))

    def inverse(self):
        """Inverse of a constant-diagonal or unit-triangular step matrix.

        Restates ``StepMatrix.inverse`` (``schemes.py:208-251``): reciprocal
        gains, or column-by-column symbolic back-substitution (which keeps the
        float accumulation order of the reference).
        """
        mode = self.mode
        if self._is_diagonal():
            gains = []
            for i in range(4):
                e = self.entries[i][i]
                if set(e.terms) != {(0, 0)}:
                    raise ValueError(f"cannot invert non-constant diagonal pass {self.label!r}")
                c = e.terms[(0, 0)]
                gains.append(Fraction(1, 1) / c if mode == EXACT else 1.0 / c)
            return StepMatrix.diagonal(gains, mode, f"inv({self.label})")
        if self._unit_triangular(lower=True):
            order = range(4)
        elif self._unit_triangular(lower=False):
            order = range(3, -1, -1)
        else:
            raise ValueError(f"pass {self.label!r} is not unit triangular; no symbolic inverse")
        zero, one = _zero2(mode), _one2(mode)
        inv = [[one if i == j else zero for j in range(4)] for i in range(4)]
        for j in range(4):
            for i in order:
                acc = one if i == j else zero
                for k in range(4):
                    if k == i:
                        continue
                    a = self.entries[i][k]
                    if a.is_zero() or inv[k][j].is_zero():
                        continue
                    acc = acc - a * inv[k][j]
                inv[i][j] = acc
        return StepMatrix(inv, f"inv({self.label})")


@dataclass(frozen=True)
class Pass:
    """A barrier-delimited pass: fused sub-step matrices applied left to right."""

    matrices: tuple
    barrier_before: bool = True
    kind: str = "lift"

    @property
    def label(self):
        return "+".join(m.label for m in self.matrices)

    def reach(self):
        return sum(m.reach() for m in self.matrices)


@dataclass(frozen=True)
class Scheme:
    """An ordered list of passes realizing one 2-D transform schedule."""

    name: str
    wavelet: str
    passes: tuple
    plan: LiftingPlan
    inverted: bool = False

    @property
    def mode(self):
        return self.plan.mode

    @property
    def steps(self):
        return sum(1 for p in self.passes if p.barrier_before)


# -- builders -------------------------------------------------------------------------


def _lift_1axis(pair):
    """(predict_h, predict_v, update_h, update_v) of one pair (``schemes.py:328-383``)."""
    p, u = pair
    mode = p.mode
    z, o = _zero2(mode), _one2(mode)
    ph = p.horizontal()
    pv = p.horizontal().transpose()
    uh = u.horizontal()
    uv = u.horizontal().transpose()
    return (
        StepMatrix([[o, z, z, z], [ph, o, z, z], [z, z, o, z], [z, z, ph, o]], "predict-h"),
        StepMatrix([[o, z, z, z], [z, o, z, z], [pv, z, o, z], [z, pv, z, o]], "predict-v"),
        StepMatrix([[o, uh, z, z], [z, o, z, z], [z, z, o, uh], [z, z, z, o]], "update-h"),
        StepMatrix([[o, z, uv, z], [z, o, z, uv], [z, z, o, z], [z, z, z, o]], "update-v"),
    )


def _lift_2d(pair):
    """Fused spatial predict/update of one pair (``schemes.py:386-421``)."""
    p, u = pair
    mode = p.mode
    z, o = _zero2(mode), _one2(mode)
    ph, uh = p.horizontal(), u.horizontal()
    pv, uv = ph.transpose(), uh.transpose()
    ppt, uut = ph * pv, uh * uv
    return (
        StepMatrix([[o, z, z, z], [ph, o, z, z], [pv, z, o, z], [ppt, pv, ph, o]], "predict-2d"),
        StepMatrix([[o, uh, uv, uut], [z, o, z, uv], [z, z, o, uh], [z, z, z, o]], "update-2d"),
    )


def _polyphase_1d(plan, inverse=False):
    """2x2 polyphase matrix of the whole plan (``schemes.py:444-496``)."""
    mode = plan.mode
    z, o = Laurent({}, mode), Laurent({0: 1}, mode)
    steps = []
    for p, u in plan.pairs:
        steps.append(("p", p))
        steps.append(("u", u))
    if plan.scale is not None:
        steps.append(("s", plan.scale))
    if inverse:
        rev = []
        for kind, arg in reversed(steps):
            if kind == "s":
                lo, hi = arg
                if mode == EXACT:
                    rev.append(("s", (Fraction(1, 1) / lo, Fraction(1, 1) / hi)))
                else:
                    rev.append(("s", (1.0 / lo, 1.0 / hi)))
            else:
                rev.append((kind, -arg))
        steps = rev
    acc = ((o, z), (z, o))
    for kind, arg in steps:
        if kind == "p":
            f = ((o, z), (arg, o))
        elif kind == "u":
            f = ((o, arg), (z, o))
        else:
            f = ((Laurent({0: arg[0]}, mode), z), (z, Laurent({0: arg[1]}, mode)))
        acc = tuple(
            tuple(f[i][0] * acc[0][j] + f[i][1] * acc[1][j] for j in range(2)) for i in range(2)
        )
    return acc


def _conv_matrices(poly, mode):
    (a, b), (c, d) = poly
    z = _zero2(mode)
    ah, bh, ch, dh = (f.horizontal() for f in (a, b, c, d))
    av, bv, cv, dv = (f.vertical() for f in (a, b, c, d))
    conv_h = StepMatrix([[ah, bh, z, z], [ch, dh, z, z], [z, z, ah, bh], [z, z, ch, dh]], "conv-h")
    conv_v = StepMatrix([[av, z, bv, z], [z, av, z, bv], [cv, z, dv, z], [z, cv, z, dv]], "conv-v")
    return conv_h, conv_v


def _scale_pass(plan):
    if plan.scale is None:
        return None
    lo, hi = plan.scale
    if plan.mode == EXACT:
        gains = (Fraction(lo) * Fraction(lo), Fraction(1, 1), Fraction(1, 1), Fraction(hi) * Fraction(hi))
    else:
        gains = (lo * lo, 1.0, 1.0, hi * hi)
    return Pass((StepMatrix.diagonal(gains, plan.mode, "scale"),), barrier_before=False, kind="scale")


def _suffix(plan, k):
    return f"#{k + 1}" if len(plan.pairs) > 1 else ""


def _separable_lifting(plan):
    passes = []
    for k, pair in enumerate(plan.pairs):
        for m in _lift_1axis(pair):
            passes.append(Pass((m.relabel(m.label + _suffix(plan, k)),)))
    sp = _scale_pass(plan)
    if sp is not None:
        passes.append(sp)
    return Scheme("separable-lifting", plan.name, tuple(passes), plan)


def _nonseparable(plan):
    passes = []
    for k, pair in enumerate(plan.pairs):
        for m in _lift_2d(pair):
            passes.append(Pass((m.relabel(m.label + _suffix(plan, k)),)))
    sp = _scale_pass(plan)
    if sp is not None:
        passes.append(sp)
    return Scheme("non-separable-lifting", plan.name, tuple(passes), plan)


def _split(plan):
    """Operation-reduced variant: remainder step, then constant h/v sub-steps."""
    mode = plan.mode
    passes = []
    for k, (p, u) in enumerate(plan.pairs):
        sfx = _suffix(plan, k)
        p0 = Laurent({0: p.constant_term()}, mode)
        u0 = Laurent({0: u.constant_term()}, mode)
        p1 = Laurent({e: c for e, c in p.terms.items() if e != 0}, mode)
        u1 = Laurent({e: c for e, c in u.terms.items() if e != 0}, mode)
        t_rem, s_rem = _lift_2d((p1, u1))
        th0, tv0, sh0, sv0 = _lift_1axis((p0, u0))
        passes.append(Pass((t_rem.relabel("predict-rest" + sfx), th0.relabel("predict-const-h" + sfx),
                            tv0.relabel("predict-const-v" + sfx))))
        passes.append(Pass((s_rem.relabel("update-rest" + sfx), sh0.relabel("update-const-h" + sfx),
                            sv0.relabel("update-const-v" + sfx))))
    sp = _scale_pass(plan)
    if sp is not None:
        passes.append(sp)
    return Scheme("non-separable-split", plan.name, tuple(passes), plan)


def _convolution(plan):
    conv_h, conv_v = _conv_matrices(_polyphase_1d(plan), plan.mode)
    return Scheme("separable-convolution", plan.name,
                  (Pass((conv_h,), kind="conv"), Pass((conv_v,), kind="conv")), plan)


_BUILDERS = {
    "separable-convolution": _convolution,
    "separable-lifting": _separable_lifting,
    "non-separable-lifting": _nonseparable,
    "non-separable-split": _split,
}


def build_scheme(name: str, plan: LiftingPlan) -> Scheme:
    """Build one of :data:`SCHEME_NAMES` for ``plan`` (``schemes.py:725-732``)."""
    try:
        builder = _BUILDERS[name]
    except KeyError:
        raise ValueError(f"unknown scheme {name!r}; expected one of {', '.join(SCHEME_NAMES)}") from None
    return builder(plan)


def invert_scheme(scheme: Scheme) -> Scheme:
    """Scheme computing the inverse transform (``schemes.py:738-787``).

    Lifting passes are reversed, their fused chains reversed, each matrix
    inverted; the convolution scheme is rebuilt from the inverse polyphase
    product with the vertical pass first.
    """
    if any(p.kind == "conv" for p in scheme.passes):
        now_inverted = not scheme.inverted
        conv_h, conv_v = _conv_matrices(_polyphase_1d(scheme.plan, inverse=now_inverted), scheme.mode)
        ordered = (conv_v, conv_h) if now_inverted else (conv_h, conv_v)
        return Scheme(scheme.name, scheme.wavelet, tuple(Pass((m,), kind="conv") for m in ordered),
                      scheme.plan, inverted=now_inverted)
    passes = tuple(
        Pass(tuple(m.inverse() for m in reversed(p.matrices)), barrier_before=p.barrier_before, kind=p.kind)
        for p in reversed(scheme.passes)
    )
    return Scheme(scheme.name, scheme.wavelet, passes, scheme.plan, inverted=not scheme.inverted)
