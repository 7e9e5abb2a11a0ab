"""Stencil programs: the per-sub-step multiply-accumulate term tables.

A scheme is lowered to a :class:`StencilProgram` exactly as the reference
does (``liftfuse/engine.py:224-282``): per pass, per fused sub-step, per
target component, a tuple of terms ``(src, dm, dn, coeff)`` meaning

    out[target][n, m] += coeff * in[src][n + dn, m + dm]

with ``(dm, dn)`` the negated stored exponents and the terms sorted by
``(dm, dn, src)`` (``engine.py:267``).  That sorted order is the
floating-point evaluation order every kernel in ``csrc/`` reproduces, which is
what makes the GPU results bit-identical to the reference in strict mode.

:func:`compile_scheme` accepts this package's schemes and also, by duck
typing, the reference's own ``liftfuse.schemes.Scheme`` objects (same
attribute names: ``passes[].matrices[].entries[i][j].terms``).
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = [
    "SubStepProgram",
    "PassProgram",
    "StencilProgram",
    "compile_scheme",
    "extend",
    "component_index",
    "PARITIES",
]

# (row, column) pixel parity of quad components 1..4 (``engine.py:52``).
PARITIES = ((0, 0), (0, 1), (1, 0), (1, 1))


def extend(index: int, size: int) -> int:
    """Whole-sample symmetric extension into ``[0, size)`` (``engine.py:55-71``).

    ``extend(-1, 8) == 1``, ``extend(8, 8) == 6``; period ``2*size - 2``; a
    single-sample signal extends to its only value.
    """
    if size < 1:
        raise ValueError("size must be >= 1")
    if size == 1:
        return 0
    period = 2 * size - 2
    i = index % period
    return period - i if i >= size else i


def component_index(i: int, parity: int, comp_size: int) -> int:
    """Quad-grid index read for component index ``i`` of a phase-``parity``
    component of length ``comp_size`` (``engine.py:82-92``): reflect in pixel
    coordinates, map back to the component."""
    return (extend(2 * i + parity, 2 * comp_size) - parity) >> 1


@dataclass(frozen=True)
class SubStepProgram:
    label: str
    terms: tuple  # per target: ((src, dm, dn, coeff), ...)
    reach: int


@dataclass(frozen=True)
class PassProgram:
    label: str
    kind: str
    barrier_before: bool
    substeps: tuple

    @property
    def reach(self) -> int:
        return sum(s.reach for s in self.substeps)


@dataclass(frozen=True)
class StencilProgram:
    scheme_name: str
    wavelet: str
    passes: tuple

    @property
    def halo(self) -> int:
        return max(p.reach for p in self.passes)

    def substeps(self):
        """All sub-steps in execution order (pass boundaries only matter to a
        tiled executor; the result is the plain composition)."""
        return [s for p in self.passes for s in p.substeps]


def _poly_reach(poly) -> int:
    best = 0
    for k in poly.terms:
        best = max(best, abs(k[0]), abs(k[1]))
    return best


def _compile_matrix(m) -> SubStepProgram:
    per_target = []
    reach = 0
    for i in range(4):
        terms = []
        for j in range(4):
            entry = m.entries[i][j]
            reach = max(reach, _poly_reach(entry))
            for (km, kn), c in entry.terms.items():
                terms.append((j, -km, -kn, float(c)))
        terms.sort(key=lambda t: (t[1], t[2], t[0]))
        per_target.append(tuple(terms))
    return SubStepProgram(m.label, tuple(per_target), reach)


def compile_scheme(scheme) -> StencilProgram:
    """Lower a scheme to its term tables (``engine.py:259-282``)."""
    passes = tuple(
        PassProgram(
            label="+".join(m.label for m in p.matrices),
            kind=p.kind,
            barrier_before=p.barrier_before,
            substeps=tuple(_compile_matrix(m) for m in p.matrices),
        )
        for p in scheme.passes
    )
    return StencilProgram(scheme.name, scheme.wavelet, passes)
