"""ctypes driver for the CPU parity checker ``libdwt_oracle.so``.

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline leg, never by the product package.

The functions mirror the reference's executor entry points so parity tests
read like the reference's own tests:

* :func:`run_reference`  ~ ``liftfuse.engine.run_reference`` (engine.py:442-451)
* :func:`forward` / :func:`inverse` ~ ``liftfuse.engine.forward/inverse``
  (engine.py:481-495) on plain NumPy arrays
* :func:`dwt` / :func:`idwt` -- the multi-level composition the north star
  adds: ``forward`` applied to the previous level's LL.

Programs are anything shaped like a ``StencilProgram`` (``.passes[].substeps[]
.terms``): the reference's own, this repo's, or the JSON fixtures under
tests/golden/ (see :func:`program_from_json`).
"""

from __future__ import annotations

import ctypes
import json
import os
import subprocess
from types import SimpleNamespace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libdwt_oracle.so")
_lib = None


class _Term(ctypes.Structure):
    _fields_ = [
        ("src", ctypes.c_int32),
        ("dm", ctypes.c_int32),
        ("dn", ctypes.c_int32),
        ("pad", ctypes.c_int32),
        ("coeff", ctypes.c_double),
    ]


def build(force: bool = False) -> str:
    """Compile the checker with its Makefile (gcc only)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        try:
            lib = ctypes.CDLL(_LIB_PATH)
        except OSError:
            # Host without the ISA the prebuilt .so assumed: rebuild portable.
            subprocess.run(["make", "-s", "-C", _HERE, "clean"], check=True)
            subprocess.run(["make", "-s", "-C", _HERE,
                            "CFLAGS=-O3 -ffp-contract=off -fno-fast-math -fPIC"], check=True)
            lib = ctypes.CDLL(_LIB_PATH)
        lib.oracle_run.restype = ctypes.c_int
        lib.oracle_run.argtypes = [
            ctypes.c_int, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(_Term),
            ctypes.c_void_p * 4, ctypes.c_void_p * 4, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
        ]
        _lib = lib
    return _lib


def _substeps(program):
    return [s for p in program.passes for s in p.substeps]


def _flatten(program):
    subs = _substeps(program)
    counts = (ctypes.c_int32 * max(1, 4 * len(subs)))()
    flat = []
    for si, sub in enumerate(subs):
        for t in range(4):
            counts[4 * si + t] = len(sub.terms[t])
            for (src, dm, dn, c) in sub.terms[t]:
                flat.append((src, dm, dn, 0, float(c)))
    terms = (_Term * max(1, len(flat)))(*[_Term(*x) for x in flat])
    return len(subs), counts, terms


def run_reference(program, comps, threads: int | None = None):
    """Run ``program`` over 4 component planes; returns 4 new planes."""
    comps = [np.ascontiguousarray(c) for c in comps]
    dtype = comps[0].dtype
    if dtype not in (np.float32, np.float64):
        raise TypeError("components must be float32 or float64")
    rows, cols = comps[0].shape
    if threads is None:
        threads = min(os.cpu_count() or 1, max(1, rows // 16))
    out = [np.empty_like(comps[0]) for _ in range(4)]
    nsub, counts, terms = _flatten(program)
    ins = (ctypes.c_void_p * 4)(*[c.ctypes.data for c in comps])
    outs = (ctypes.c_void_p * 4)(*[o.ctypes.data for o in out])
    rc = _load().oracle_run(0 if dtype == np.float32 else 1, nsub, counts, terms, ins, outs,
                            rows, cols, threads)
    if rc != 0:
        raise RuntimeError("oracle_run failed")
    return out


def deinterleave(a: np.ndarray):
    if a.shape[0] % 2 or a.shape[1] % 2:
        raise ValueError(f"dimensions must be even, got {a.shape[1]}x{a.shape[0]}")
    return [np.ascontiguousarray(a[0::2, 0::2]), np.ascontiguousarray(a[0::2, 1::2]),
            np.ascontiguousarray(a[1::2, 0::2]), np.ascontiguousarray(a[1::2, 1::2])]


def interleave(comps) -> np.ndarray:
    rows, cols = comps[0].shape
    out = np.empty((2 * rows, 2 * cols), dtype=comps[0].dtype)
    out[0::2, 0::2], out[0::2, 1::2], out[1::2, 0::2], out[1::2, 1::2] = comps
    return out


def forward(image: np.ndarray, program, threads=None):
    """(ll, hl, lh, hh) of one level; ``program`` is the compiled forward scheme."""
    return run_reference(program, deinterleave(image), threads)


def inverse(comps, inverse_program, threads=None) -> np.ndarray:
    """Interleaved image from 4 subbands; ``inverse_program`` is compiled from
    ``invert_scheme(scheme)``."""
    return interleave(run_reference(inverse_program, comps, threads))


def dwt(image: np.ndarray, program, levels: int, threads=None):
    """Multi-level forward: returns (ll_final, [(hl, lh, hh) per level, finest first])."""
    details = []
    ll = image
    for _ in range(levels):
        q = forward(ll, program, threads)
        details.append((q[1], q[2], q[3]))
        ll = q[0]
    return ll, details


def idwt(ll: np.ndarray, details, inverse_program, threads=None) -> np.ndarray:
    for hl, lh, hh in reversed(details):
        ll = inverse([ll, hl, lh, hh], inverse_program, threads)
    return ll


# -- JSON program fixtures -------------------------------------------------------


def program_to_json(program) -> dict:
    return {
        "scheme_name": program.scheme_name,
        "wavelet": program.wavelet,
        "passes": [
            {
                "label": p.label,
                "kind": p.kind,
                "barrier_before": bool(p.barrier_before),
                "substeps": [
                    {
                        "label": s.label,
                        "reach": int(s.reach),
                        "terms": [[[int(a), int(b), int(c), float(d).hex()] for (a, b, c, d) in t]
                                  for t in s.terms],
                    }
                    for s in p.substeps
                ],
            }
            for p in program.passes
        ],
    }


def program_from_json(d: dict):
    passes = []
    for p in d["passes"]:
        subs = tuple(
            SimpleNamespace(
                label=s["label"],
                reach=s["reach"],
                terms=tuple(tuple((a, b, c, float.fromhex(h)) for (a, b, c, h) in t) for t in s["terms"]),
            )
            for s in p["substeps"]
        )
        passes.append(SimpleNamespace(label=p["label"], kind=p["kind"], barrier_before=p["barrier_before"],
                                      substeps=subs))
    return SimpleNamespace(scheme_name=d["scheme_name"], wavelet=d["wavelet"], passes=tuple(passes))


def load_programs(path: str) -> dict:
    with open(path) as fh:
        raw = json.load(fh)
    return {k: program_from_json(v) for k, v in raw.items()}
