"""Public transform API -- a drop-in for ``liftfuse.engine`` backed by sm_100a kernels.

Same names, argument meaning and error behaviour as the reference
(``liftfuse/engine.py``):

==========================  =====================================================
reference                   here
==========================  =====================================================
``forward`` :481-487        :func:`forward` -- one fused kernel (deinterleave +
                            all passes + subband stores), ``b2dwt_forward``
``inverse`` :490-495        :func:`inverse` -- fused ``b2dwt_inverse``
``run_tiled`` :404-439      :func:`run_tiled` -- ``b2dwt_run_components``;
                            ``TileConfig`` is validated like the reference
                            (tile >= halo) and then ignored: GPU tiling is
                            internal and results do not depend on it
``run_reference`` :442-451  :func:`run_reference` (same device path)
``Image2D`` / ``SubbandQuad`` / ``TileConfig`` / ``deinterleave`` /
``interleave_quad`` / ``extend`` / ``compile_scheme`` -- same data types
==========================  =====================================================

New (north star): :func:`dwt` / :func:`idwt` multi-level pyramids, and the
device-tensor API :class:`Transform` that the benchmarks and multi-GPU paths
use (inputs stay resident in HBM; no host round trip).

Schemes may be this package's (:func:`.lifting.build_scheme`) or the
reference's own ``liftfuse.schemes.Scheme`` objects (duck-typed).
Arithmetic is "strict" by default: bit-identical to the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .lifting import EXACT, Laurent, LiftingPlan, Scheme, build_scheme, invert_scheme
from .program import StencilProgram, compile_scheme, extend

__all__ = [
    "PRECISION_DTYPES",
    "Image2D",
    "SubbandQuad",
    "Pyramid",
    "TileConfig",
    "StencilProgram",
    "Transform",
    "extend",
    "compile_scheme",
    "forward",
    "inverse",
    "dwt",
    "idwt",
    "run_tiled",
    "run_reference",
    "run_without_barriers",
    "deinterleave",
    "interleave_quad",
]

PRECISION_DTYPES = {"single": np.float32, "double": np.float64}


# -- data types (engine.py:95-197) ----------------------------------------------------


@dataclass(frozen=True)
class Image2D:
    """Row-major real-valued raster (engine.py:95-144)."""

    data: np.ndarray

    def __post_init__(self):
        arr = np.asarray(self.data)
        if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] < 1:
            raise ValueError("image data must be a non-empty 2-D array")
        if arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float64)
        object.__setattr__(self, "data", arr)

    @property
    def width(self) -> int:
        return self.data.shape[1]

    @property
    def height(self) -> int:
        return self.data.shape[0]

    @property
    def precision(self) -> str:
        return "single" if self.data.dtype == np.float32 else "double"

    @classmethod
    def random(cls, width: int, height: int, seed: int, precision: str = "double") -> "Image2D":
        rng = np.random.default_rng(seed)
        return cls(rng.random((height, width), dtype=np.float64).astype(PRECISION_DTYPES[precision]))

    @classmethod
    def constant(cls, width: int, height: int, value: float = 1.0, precision: str = "double") -> "Image2D":
        return cls(np.full((height, width), value, dtype=PRECISION_DTYPES[precision]))

    @classmethod
    def delta(cls, width: int, height: int, row: int, col: int, precision: str = "double") -> "Image2D":
        data = np.zeros((height, width), dtype=PRECISION_DTYPES[precision])
        data[row, col] = 1.0
        return cls(data)

    def astype(self, precision: str) -> "Image2D":
        return Image2D(self.data.astype(PRECISION_DTYPES[precision]))


@dataclass(frozen=True)
class SubbandQuad:
    """The four polyphase subbands of one level (engine.py:147-176)."""

    ll: Image2D
    hl: Image2D
    lh: Image2D
    hh: Image2D

    def __post_init__(self):
        shape = self.ll.data.shape
        for band in (self.hl, self.lh, self.hh):
            if band.data.shape != shape:
                raise ValueError("all four subbands must share dimensions")

    def components(self) -> list:
        return [self.ll.data, self.hl.data, self.lh.data, self.hh.data]

    def interleave(self) -> Image2D:
        return Image2D(interleave_quad(self.components()))

    @classmethod
    def from_components(cls, comps) -> "SubbandQuad":
        ll, hl, lh, hh = (Image2D(c) for c in comps)
        return cls(ll, hl, lh, hh)


@dataclass(frozen=True)
class Pyramid:
    """Multi-level result: ``details[l] = (hl, lh, hh)`` of level l (finest
    first) and the coarsest ``ll``.  Level l transforms level l-1's LL."""

    ll: Image2D
    details: tuple

    @property
    def levels(self) -> int:
        return len(self.details)


@dataclass(frozen=True)
class TileConfig:
    """Accepted and validated like the reference (engine.py:179-197); the GPU
    decomposition is internal and the result is independent of it."""

    tile: tuple | None = None
    threads: int = 1

    def __post_init__(self):
        if self.tile is not None:
            tw, th = self.tile
            if tw < 1 or th < 1:
                raise ValueError("tile dimensions must be positive")
        if self.threads < 1:
            raise ValueError("thread count must be positive")


def deinterleave(image: Image2D) -> list:
    """Host-side polyphase split (engine.py:200-211); the GPU path fuses it."""
    a = image.data
    if a.shape[0] % 2 or a.shape[1] % 2:
        raise ValueError(f"dimensions must be even, got {a.shape[1]}x{a.shape[0]}")
    return [np.ascontiguousarray(a[r::2, c::2]) for r, c in ((0, 0), (0, 1), (1, 0), (1, 1))]


def interleave_quad(comps) -> np.ndarray:
    """Host-side polyphase merge (engine.py:214-221); the GPU path fuses it."""
    rows, cols = comps[0].shape
    out = np.empty((2 * rows, 2 * cols), dtype=comps[0].dtype)
    out[0::2, 0::2], out[0::2, 1::2], out[1::2, 0::2], out[1::2, 1::2] = comps
    return out


# -- scheme adoption ----------------------------------------------------------------


def _adopt_plan(plan) -> LiftingPlan:
    if isinstance(plan, LiftingPlan):
        return plan
    mode = getattr(plan, "mode", EXACT)
    pairs = tuple((Laurent(dict(p.terms), mode), Laurent(dict(u.terms), mode)) for p, u in plan.pairs)
    return LiftingPlan(plan.name, pairs, plan.scale, mode)


def _adopt_scheme(scheme) -> Scheme:
    """This package's Scheme for a (possibly foreign, duck-typed) scheme."""
    if isinstance(scheme, Scheme):
        return scheme
    s = build_scheme(scheme.name, _adopt_plan(scheme.plan))
    return invert_scheme(s) if getattr(scheme, "inverted", False) else s


def _programs(scheme):
    """(forward program, inverse program) of a scheme."""
    fwd = compile_scheme(scheme)
    inv = compile_scheme(invert_scheme(_adopt_scheme(scheme)))
    return fwd, inv


def _check_tile(cfg: TileConfig, program) -> None:
    if cfg.tile is not None:
        tw, th = cfg.tile
        halo = program.halo
        if tw < halo or th < halo:
            raise ValueError(f"tile {tw}x{th} is smaller than the scheme halo {halo}")


# -- device plumbing ------------------------------------------------------------------


def _torch():
    import torch

    return torch


def _require_cuda():
    torch = _torch()
    _native.load()
    if not torch.cuda.is_available():
        raise _native.NativeError("no CUDA device visible: the b2dwt kernels need a B200 (no CPU fallback)")
    return torch


_NP2NATIVE = {np.dtype(np.float32): _native.F32, np.dtype(np.float64): _native.F64}


def _signature(program):
    return tuple(tuple(sub.terms) for p in program.passes for sub in p.substeps)


_PLAN_CACHE: dict = {}


def plan_for(program, dtype: int, flags: int = 0) -> _native.Plan:
    """Cached native plan for a compiled program."""
    key = (_signature(program), dtype, flags)
    plan = _PLAN_CACHE.get(key)
    if plan is None:
        plan = _native.Plan(program, dtype, flags)
        _PLAN_CACHE[key] = plan
    return plan


def _stream_handle(torch, stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes_void(s.cuda_stream)


def ctypes_void(x):
    import ctypes

    return ctypes.c_void_p(int(x))


def _ptr(t) -> int:
    return int(t.data_ptr())


def _check_buffer(torch, t, name, shape, dtype, device=None, host=False):
    """Validate a caller-supplied buffer before its pointer reaches the C ABI:
    a tensor of ``dtype`` and exactly ``shape``, on ``device`` (CUDA) or on the
    host, with unit element stride and non-overlapping rows (and batch items).
    A wrong buffer would otherwise become out-of-bounds device writes, or host
    corruption through the pipelines' 2-D copies."""
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if host:
        if t.device.type != "cpu":
            raise ValueError(f"{name} must be a host (CPU) tensor")
    elif not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    elif device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if t.numel() == 0:
        return t
    if t.stride(-1) != 1:
        raise ValueError(f"{name} rows must be contiguous")
    if t.dim() >= 2 and t.stride(-2) < t.shape[-1]:
        raise ValueError(f"{name} rows overlap (row stride {t.stride(-2)} < {t.shape[-1]})")
    if t.dim() == 3 and t.shape[0] > 1 and t.stride(0) < t.shape[1] * t.stride(1):
        raise ValueError(f"{name} batch items overlap")
    return t


def _same_batch_stride(planes, name):
    """The C ABI takes one batch stride for all four planes."""
    if planes[0].shape[0] > 1 and any(p.stride(0) != planes[0].stride(0) for p in planes[1:]):
        raise ValueError(f"{name}: the four planes must share one batch stride")


class Transform:
    """Device-resident transform for one scheme at one precision.

    All tensors are CUDA tensors; calls are asynchronous on the current torch
    stream (or ``stream``).  ``x`` is ``[H, W]`` or ``[B, H, W]`` (contiguous
    rows; any row pitch via ``stride``).
    """

    def __init__(self, scheme, precision: str = "single", fast: bool = False, tma: bool = True,
                 force_generic: bool = False, tile: bool | None = None, fuse: bool = True):
        self.scheme = scheme
        self.precision = precision
        self.np_dtype = np.dtype(PRECISION_DTYPES[precision])
        self.dtype = _NP2NATIVE[self.np_dtype]
        flags = _native.FAST if fast else 0
        if not tma:
            flags |= _native.NO_TMA
        if force_generic:
            flags |= _native.FORCE_GENERIC
        if tile is not None:  # None: small levels tile, large ones stream
            flags |= _native.FORCE_TILE if tile else _native.NO_TILE
        if not fuse:  # pyramids: one launch per level instead of fused level pairs
            flags |= _native.NO_FUSE
        self.flags = flags
        self.fwd_program, self.inv_program = _programs(scheme)
        self.fwd_plan = plan_for(self.fwd_program, self.dtype, flags)
        self.inv_plan = plan_for(self.inv_program, self.dtype, flags)

    @property
    def torch_dtype(self):
        torch = _torch()
        return torch.float32 if self.dtype == _native.F32 else torch.float64

    def _check(self, t, name):
        torch = _require_cuda()
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise TypeError(f"{name} must be a CUDA tensor")
        if t.dtype != self.torch_dtype:
            raise TypeError(f"{name} must be {self.torch_dtype}, got {t.dtype}")
        if t.stride(-1) != 1:
            raise ValueError(f"{name} rows must be contiguous")
        return torch

    # single level --------------------------------------------------------------------
    def forward(self, x, out=None, stream=None):
        """Return (ll, hl, lh, hh), each ``[..., H/2, W/2]``."""
        torch = self._check(x, "x")
        batched = x.dim() == 3
        xb = x if batched else x.unsqueeze(0)
        b, h, w = xb.shape
        if h % 2 or w % 2:
            raise ValueError(f"dimensions must be even, got {w}x{h}")
        if out is None:
            out = tuple(torch.empty((b, h // 2, w // 2), dtype=x.dtype, device=x.device) for _ in range(4))
        else:
            out = self._check_out_planes(torch, out, (b, h // 2, w // 2), x.device, batched)
        pl = _native.planes([_ptr(o) for o in out], [o.stride(1) for o in out], out[0].stride(0))
        _native.check(
            _native.load().b2dwt_forward(self.fwd_plan.handle, _ptr(xb), xb.stride(1), xb.stride(0), h, w, pl, b,
                                         _stream_handle(torch, stream)),
            "forward",
        )
        return out if batched else tuple(o[0] for o in out)

    def _check_out_planes(self, torch, out, shape3, device, batched):
        """Four caller-supplied output planes of ``shape3`` = (B, rows, cols)
        (or (rows, cols) each for an unbatched call); returns 3-D views."""
        if not isinstance(out, (tuple, list)) or len(out) != 4:
            raise ValueError("out must be four planes (ll, hl, lh, hh)")
        want = shape3 if batched else shape3[1:]
        planes = []
        for o, n in zip(out, ("ll", "hl", "lh", "hh")):
            _check_buffer(torch, o, f"out[{n}]", want, self.torch_dtype, device)
            planes.append(o if o.dim() == 3 else o.unsqueeze(0))
        _same_batch_stride(planes, "out")
        return tuple(planes)

    def _check_in_planes(self, torch, comps, names):
        """Four device input planes: same device, dtype, shape, contiguous rows
        and one batch stride; returns 3-D views."""
        first = comps[0]
        self._check(first, names[0])
        if first.dim() not in (2, 3):
            raise ValueError(f"{names[0]} must be [rows, cols] or [B, rows, cols]")
        for c, n in zip(comps[1:], names[1:]):
            self._check(c, n)
            if c.shape != first.shape:
                raise ValueError("all four subbands must share dimensions")
        planes = []
        for c, n in zip(comps, names):
            _check_buffer(torch, c, n, first.shape, self.torch_dtype, first.device)
            planes.append(c if c.dim() == 3 else c.unsqueeze(0))
        _same_batch_stride(planes, "subbands")
        return planes

    def inverse(self, ll, hl, lh, hh, out=None, stream=None):
        torch = self._check(ll, "ll")
        comps = self._check_in_planes(torch, (ll, hl, lh, hh), ("ll", "hl", "lh", "hh"))
        b, rows, cols = comps[0].shape
        if out is None:
            out = torch.empty((b, 2 * rows, 2 * cols), dtype=ll.dtype, device=ll.device)
        else:
            _check_buffer(torch, out, "out", (b, 2 * rows, 2 * cols) if ll.dim() == 3 else (2 * rows, 2 * cols),
                          self.torch_dtype, ll.device)
        ob = out if out.dim() == 3 else out.unsqueeze(0)
        pl = _native.planes([_ptr(c) for c in comps], [c.stride(1) for c in comps], comps[0].stride(0))
        _native.check(
            _native.load().b2dwt_inverse(self.inv_plan.handle, pl, _ptr(ob), ob.stride(1), ob.stride(0), 2 * rows,
                                         2 * cols, b, _stream_handle(torch, stream)),
            "inverse",
        )
        return ob if ll.dim() == 3 else ob[0]

    def run_components(self, comps, program=None, out=None, stream=None):
        torch = self._check(comps[0], "comps")
        plan = self.fwd_plan if program is None else plan_for(program, self.dtype, self.flags)
        if len(comps) != 4:
            raise ValueError("run_components takes four component planes")
        cs = self._check_in_planes(torch, tuple(comps), tuple(f"comps[{i}]" for i in range(4)))
        b, rows, cols = cs[0].shape
        if out is None:
            out = [torch.empty_like(c) for c in cs]
        else:
            out = list(self._check_out_planes(torch, out, (b, rows, cols), comps[0].device, comps[0].dim() == 3))
        pin = _native.planes([_ptr(c) for c in cs], [c.stride(1) for c in cs], cs[0].stride(0))
        pout = _native.planes([_ptr(c) for c in out], [c.stride(1) for c in out], out[0].stride(0))
        _native.check(
            _native.load().b2dwt_run_components(plan.handle, pin, pout, rows, cols, b,
                                                _stream_handle(torch, stream)),
            "run_components",
        )
        return out if comps[0].dim() == 3 else [o[0] for o in out]

    def forward_rows(self, band, band_row0, global_height, out_row_begin, out_row_end, out=None, stream=None):
        """Forward transform of quad rows [out_row_begin, out_row_end) of a
        global_height x W image from a row band that starts at pixel row
        ``band_row0`` (must include the cone; see :attr:`cone`)."""
        torch = self._check(band, "band")
        if band.dim() != 2:
            raise ValueError("band must be [rows, W]")
        rows_b, w = band.shape
        n = out_row_end - out_row_begin
        if n < 1:
            raise ValueError("bad output row range")
        if out is None:
            out = tuple(torch.empty((n, w // 2), dtype=band.dtype, device=band.device) for _ in range(4))
        else:
            out = tuple(p[0] for p in self._check_out_planes(torch, out, (1, n, w // 2), band.device, False))
        pl = _native.planes([_ptr(o) for o in out], [o.stride(0) for o in out], 0)
        _native.check(
            _native.load().b2dwt_forward_rows(self.fwd_plan.handle, _ptr(band), band.stride(0), band_row0, rows_b,
                                              global_height, w, out_row_begin, out_row_end, pl,
                                              _stream_handle(torch, stream)),
            "forward_rows",
        )
        return out

    def forward2(self, x, det0=None, out1=None, stream=None):
        """Levels 0 and 1 of the pyramid of one ``[H, W]`` image in ONE kernel
        (b2dwt_forward2): level 0's LL band never reaches HBM.  Returns
        ``((hl0, lh0, hh0), (ll1, hl1, lh1, hh1))``, or ``None`` when the plan or
        geometry does not fit the fused kernel (run two :meth:`forward` calls)."""
        torch = self._check(x, "x")
        if x.dim() != 2:
            raise ValueError("forward2 takes one [H, W] image")
        h, w = x.shape
        if h % 4 or w % 4:
            raise ValueError(f"dimensions must be divisible by 4, got {w}x{h}")
        if det0 is None:
            det0 = tuple(torch.empty((h // 2, w // 2), dtype=x.dtype, device=x.device) for _ in range(3))
        if out1 is None:
            out1 = tuple(torch.empty((h // 4, w // 4), dtype=x.dtype, device=x.device) for _ in range(4))
        if len(det0) != 3 or len(out1) != 4:
            raise ValueError("det0 holds (hl, lh, hh) and out1 (ll, hl, lh, hh)")
        for b, n in zip(det0, ("hl", "lh", "hh")):
            _check_buffer(torch, b, f"det0.{n}", (h // 2, w // 2), self.torch_dtype, x.device)
        for b, n in zip(out1, ("ll", "hl", "lh", "hh")):
            _check_buffer(torch, b, f"out1.{n}", (h // 4, w // 4), self.torch_dtype, x.device)
        p0 = _native.planes([0] + [_ptr(b) for b in det0], [0] + [b.stride(0) for b in det0], 0)
        p1 = _native.planes([_ptr(b) for b in out1], [b.stride(0) for b in out1], 0)
        rc = _native.load().b2dwt_forward2(self.fwd_plan.handle, _ptr(x), x.stride(0), h, w, p0, p1,
                                           _stream_handle(torch, stream))
        if rc == _native.B2DWT_EUNSUPPORTED:
            return None
        _native.check(rc, "forward2")
        return det0, out1

    @property
    def cone(self):
        """(up, down, left, right) dependency cone of the fused forward kernel, quads."""
        return self.fwd_plan.cone

    # multi level -----------------------------------------------------------------------
    def dwt(self, x, levels: int, stream=None):
        """Return (ll, [(hl, lh, hh) per level, finest first]).  ``x`` is one
        ``[H, W]`` image or a ``[B, H, W]`` batch (every level then runs as one
        batched launch sequence; outputs gain the leading batch dimension)."""
        torch = self._check(x, "x")
        if x.dim() == 3:
            return self._dwt_batch(x, levels, stream)
        if x.dim() != 2:
            raise ValueError("dwt takes one [H, W] image or a [B, H, W] batch")
        h, w = x.shape
        if levels < 1:
            raise ValueError("levels must be >= 1")
        if h % (1 << levels) or w % (1 << levels):
            raise ValueError(f"dimensions must be divisible by 2^{levels}, got {w}x{h}")
        details = []
        for lvl in range(levels):
            hh_, ww_ = h >> (lvl + 1), w >> (lvl + 1)
            details.append(tuple(torch.empty((hh_, ww_), dtype=x.dtype, device=x.device) for _ in range(3)))
        ll = torch.empty((h >> levels, w >> levels), dtype=x.dtype, device=x.device)
        scratch = torch.empty(((h // 2) * (w // 2) + (h // 4) * (w // 4),), dtype=x.dtype, device=x.device) \
            if levels > 1 else None
        self.dwt_into(x, levels, details, ll, scratch, stream)
        return ll, details

    def _dwt_batch(self, x, levels, stream=None):
        torch = _torch()
        b, h, w = x.shape
        if levels < 1:
            raise ValueError("levels must be >= 1")
        if h % (1 << levels) or w % (1 << levels):
            raise ValueError(f"dimensions must be divisible by 2^{levels}, got {w}x{h}")
        details, src = [], x
        for lvl in range(levels):
            shp = (b, h >> (lvl + 1), w >> (lvl + 1))
            ll = torch.empty(shp, dtype=x.dtype, device=x.device)
            bands = tuple(torch.empty(shp, dtype=x.dtype, device=x.device) for _ in range(3))
            self.forward(src, out=(ll,) + bands, stream=stream)
            details.append(bands)
            src = ll
        return src, details

    def _idwt_batch(self, ll, details, out=None, stream=None):
        torch = _torch()
        cur = ll
        for lvl in range(len(details) - 1, -1, -1):
            hl, lh, hh = details[lvl]
            dst = out if lvl == 0 and out is not None else None
            cur = self.inverse(cur, hl, lh, hh, out=dst, stream=stream)
        return cur

    def _check_pyramid(self, torch, h, w, levels, details, ll, device=None, host=False):
        """Caller-supplied pyramid buffers: per level (hl, lh, hh) of
        (H >> (l+1)) x (W >> (l+1)) and the final LL."""
        if len(details) != levels:
            raise ValueError(f"details must hold {levels} levels, got {len(details)}")
        for lvl, d in enumerate(details):
            if len(d) != 3:
                raise ValueError("each level holds three detail planes (hl, lh, hh)")
            for b, n in zip(d, ("hl", "lh", "hh")):
                _check_buffer(torch, b, f"details[{lvl}].{n}", (h >> (lvl + 1), w >> (lvl + 1)), self.torch_dtype,
                              device, host)
        _check_buffer(torch, ll, "ll", (h >> levels, w >> levels), self.torch_dtype, device, host)

    def dwt_into(self, x, levels, details, ll, scratch, stream=None):
        torch = self._check(x, "x")
        if x.dim() != 2:
            raise ValueError("dwt_into takes one [H, W] image")
        h, w = x.shape
        if levels < 1:
            raise ValueError("levels must be >= 1")
        if h % (1 << levels) or w % (1 << levels):
            raise ValueError(f"dimensions must be divisible by 2^{levels}, got {w}x{h}")
        self._check_pyramid(torch, h, w, levels, details, ll, x.device)
        if levels > 1:
            need = (h // 2) * (w // 2) + (h // 4) * (w // 4)
            if scratch is None or not scratch.is_cuda or scratch.device != x.device or \
                    scratch.dtype != self.torch_dtype or not scratch.is_contiguous() or scratch.numel() < need:
                raise ValueError(f"scratch must be a contiguous {self.torch_dtype} device buffer of >= {need} elements")
        arr = (_native.Planes * levels)()
        for lvl, (hl, lh, hh) in enumerate(details):
            arr[lvl] = _native.planes([0, _ptr(hl), _ptr(lh), _ptr(hh)],
                                      [0, hl.stride(0), lh.stride(0), hh.stride(0)], 0)
        _native.check(
            _native.load().b2dwt_dwt(self.fwd_plan.handle, _ptr(x), x.stride(0), h, w, levels, arr, _ptr(ll),
                                     ll.stride(0), _ptr(scratch) if scratch is not None else None,
                                     _stream_handle(torch, stream)),
            "dwt",
        )

    def dwt_host(self, x, levels: int, details=None, ll=None, bands: int = 16, stream=None, sync: bool = True):
        """Pyramid of a HOST image into HOST subbands (b2dwt_dwt_host).

        ``x`` is a CPU tensor or NumPy array ``[H, W]``.  The upload, the
        band-by-band kernels and the downloads are pipelined (pinned host
        memory gives the copy overlap; pageable memory still works).  Outputs
        default to new pinned CPU tensors; pass ``details`` /  ``ll`` to reuse
        them.  Returns ``(ll, details)``; with ``sync=False`` they are valid
        once ``stream`` (default: current) has reached this point.
        """
        torch = _require_cuda()
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(np.ascontiguousarray(x))
        if x.device.type != "cpu":
            raise ValueError("dwt_host takes a host (CPU) image; use dwt() for device tensors")
        if x.dim() != 2 or x.stride(1) != 1:
            raise ValueError("dwt_host takes one [H, W] image with contiguous rows")
        if x.dtype != self.torch_dtype:
            raise TypeError(f"expected {self.torch_dtype}, got {x.dtype}")
        h, w = x.shape
        if levels < 1:
            raise ValueError("levels must be >= 1")
        if h % (1 << levels) or w % (1 << levels):
            raise ValueError(f"dimensions must be divisible by 2^{levels}, got {w}x{h}")
        pin = x.is_pinned()
        if details is None:
            details = [tuple(torch.empty((h >> (l + 1), w >> (l + 1)), dtype=x.dtype, pin_memory=pin)
                             for _ in range(3)) for l in range(levels)]
        if ll is None:
            ll = torch.empty((h >> levels, w >> levels), dtype=x.dtype, pin_memory=pin)
        self._check_pyramid(torch, h, w, levels, details, ll, host=True)
        lib = _native.load()
        need = int(lib.b2dwt_dwt_host_workspace(self.fwd_plan.handle, h, w, levels))
        if need < 0:
            raise ValueError("bad dwt_host geometry")
        ws = _call_workspace(torch, need, stream)
        arr = (_native.Planes * levels)()
        for lvl, (hl, lh, hh) in enumerate(details):
            arr[lvl] = _native.planes([0, _ptr(hl), _ptr(lh), _ptr(hh)],
                                      [0, hl.stride(0), lh.stride(0), hh.stride(0)], 0)
        s = _stream_handle(torch, stream)
        _native.check(
            lib.b2dwt_dwt_host(self.fwd_plan.handle, _ptr(x), x.stride(0), h, w, levels, arr, _ptr(ll),
                               ll.stride(0), _ptr(ws), ws.numel(), bands, s),
            "dwt_host",
        )
        if sync:
            (stream if stream is not None else torch.cuda.current_stream()).synchronize()
        return ll, details

    def capture_dwt(self, x, levels: int, level_events: bool = False):
        """Capture the whole ``levels``-deep pyramid of the device image ``x``
        into a CUDA graph (one host submission per pyramid).  Returns a
        :class:`PyramidGraph`; write new pixels into ``x`` and ``replay()``."""
        return PyramidGraph(self, x, levels, level_events)

    def idwt(self, ll, details, out=None, stream=None):
        torch = self._check(ll, "ll")
        if ll.dim() == 3:
            return self._idwt_batch(ll, details, out, stream)
        levels = len(details)
        if levels < 1:
            raise ValueError("levels must be >= 1")
        if ll.dim() != 2:
            raise ValueError("ll must be [rows, cols] or [B, rows, cols]")
        h, w = ll.shape[0] << levels, ll.shape[1] << levels
        self._check_pyramid(torch, h, w, levels, details, ll, ll.device)
        if out is None:
            out = torch.empty((h, w), dtype=ll.dtype, device=ll.device)
        else:
            _check_buffer(torch, out, "out", (h, w), self.torch_dtype, ll.device)
        scratch = torch.empty(((h // 2) * (w // 2) + (h // 4) * (w // 4),), dtype=ll.dtype, device=ll.device) \
            if levels > 1 else None
        arr = (_native.Planes * levels)()
        for lvl, (hl, lh, hh) in enumerate(details):
            arr[lvl] = _native.planes([0, _ptr(hl), _ptr(lh), _ptr(hh)],
                                      [0, hl.stride(0), lh.stride(0), hh.stride(0)], 0)
        _native.check(
            _native.load().b2dwt_idwt(self.inv_plan.handle, _ptr(ll), ll.stride(0), arr, levels, _ptr(out),
                                      out.stride(0), h, w, _ptr(scratch) if scratch is not None else None,
                                      _stream_handle(torch, stream)),
            "idwt",
        )
        return out


    def idwt_host(self, ll, details, out=None, bands: int = 16, stream=None, sync: bool = True):
        """Host subbands -> host image (b2dwt_idwt_host): the inverse of
        :meth:`dwt_host`, with level 0's upload, kernels and download
        overlapped in row bands.  ``ll`` / ``details`` are CPU tensors or NumPy
        arrays (pinned memory gives the overlap); returns a CPU tensor."""
        torch = _require_cuda()

        def host(a):
            t = torch.from_numpy(np.ascontiguousarray(a)) if isinstance(a, np.ndarray) else a
            if t.device.type != "cpu" or t.dim() != 2 or t.stride(1) != 1:
                raise ValueError("idwt_host takes host (CPU) [H, W] planes with contiguous rows")
            if t.dtype != self.torch_dtype:
                raise TypeError(f"expected {self.torch_dtype}, got {t.dtype}")
            return t

        ll = host(ll)
        details = [tuple(host(b) for b in d) for d in details]
        levels = len(details)
        if levels < 1:
            raise ValueError("levels must be >= 1")
        h, w = ll.shape[0] << levels, ll.shape[1] << levels
        for lvl, d in enumerate(details):
            for b in d:
                if tuple(b.shape) != (h >> (lvl + 1), w >> (lvl + 1)):
                    raise ValueError("all four subbands must share dimensions")
        if out is None:
            out = torch.empty((h, w), dtype=ll.dtype, pin_memory=ll.is_pinned())
        _check_buffer(torch, out, "out", (h, w), self.torch_dtype, host=True)
        lib = _native.load()
        need = int(lib.b2dwt_idwt_host_workspace(self.inv_plan.handle, h, w, levels))
        if need < 0:
            raise ValueError("bad idwt_host geometry")
        ws = _call_workspace(torch, need, stream)
        arr = (_native.Planes * levels)()
        for lvl, (hl, lh, hh) in enumerate(details):
            arr[lvl] = _native.planes([0, _ptr(hl), _ptr(lh), _ptr(hh)],
                                      [0, hl.stride(0), lh.stride(0), hh.stride(0)], 0)
        _native.check(
            lib.b2dwt_idwt_host(self.inv_plan.handle, _ptr(ll), ll.stride(0), arr, levels, _ptr(out), out.stride(0),
                                h, w, _ptr(ws), ws.numel(), bands, _stream_handle(torch, stream)),
            "idwt_host",
        )
        if sync:
            (stream if stream is not None else torch.cuda.current_stream()).synchronize()
        return out

    def forward_host_batch(self, x, out=None, chunk: int = 16, sync: bool = True):
        """Single-level forward of a HOST batch ``[B, H, W]`` into HOST subbands
        (LL, HL, LH, HH), each ``[B, H/2, W/2]``, streaming chunks of images: the
        upload of chunk k+1, the kernel of chunk k and the download of chunk
        k-1 run concurrently (two device slots, three streams).  Pinned host
        memory gives the overlap.  Bit-identical to :meth:`forward`."""
        torch = _require_cuda()
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(np.ascontiguousarray(x))
        if x.device.type != "cpu" or x.dim() != 3 or not x.is_contiguous():
            raise ValueError("forward_host_batch takes a contiguous host [B, H, W] tensor")
        if x.dtype != self.torch_dtype:
            raise TypeError(f"expected {self.torch_dtype}, got {x.dtype}")
        b, h, w = x.shape
        if h % 2 or w % 2:
            raise ValueError(f"dimensions must be even, got {w}x{h}")
        if out is None:
            out = tuple(torch.empty((b, h // 2, w // 2), dtype=x.dtype, pin_memory=x.is_pinned()) for _ in range(4))
        if not isinstance(out, (tuple, list)) or len(out) != 4:
            raise ValueError("out must be four planes (ll, hl, lh, hh)")
        for o, n in zip(out, ("ll", "hl", "lh", "hh")):
            _check_buffer(torch, o, f"out[{n}]", (b, h // 2, w // 2), self.torch_dtype, host=True)
        chunk = max(1, min(chunk, b))
        dev_in = [torch.empty((chunk, h, w), dtype=x.dtype, device="cuda") for _ in range(2)]
        dev_out = [torch.empty((4, chunk, h // 2, w // 2), dtype=x.dtype, device="cuda") for _ in range(2)]
        main = torch.cuda.current_stream()
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        s_in.wait_stream(main)
        s_out.wait_stream(main)
        freed = [None, None]  # event: slot's previous download finished
        for k, i0 in enumerate(range(0, b, chunk)):
            n = min(chunk, b - i0)
            slot = k % 2
            with torch.cuda.stream(s_in):
                if freed[slot] is not None:
                    s_in.wait_event(freed[slot])
                dev_in[slot][:n].copy_(x[i0:i0 + n], non_blocking=True)
                up = torch.cuda.Event()
                up.record(s_in)
            main.wait_event(up)
            self.forward(dev_in[slot][:n], out=tuple(dev_out[slot][c, :n] for c in range(4)))
            done = torch.cuda.Event()
            done.record(main)
            with torch.cuda.stream(s_out):
                s_out.wait_event(done)
                for c in range(4):  # contiguous slabs: one plain copy per plane
                    out[c][i0:i0 + n].copy_(dev_out[slot][c, :n], non_blocking=True)
                freed[slot] = torch.cuda.Event()
                freed[slot].record(s_out)
        main.wait_stream(s_out)  # later work on the caller's stream (and slot reuse) sees it all
        if sync:
            main.synchronize()
        return out

    def inverse_rows(self, band, band_row0, global_height, out_row_begin, out_row_end, out=None, stream=None):
        """Image rows [2*out_row_begin, 2*out_row_end) of the inverse from a row
        band of the four subband planes (quad rows [band_row0, band_row0 +
        rows)); mirror of :meth:`forward_rows` (b2dwt_inverse_rows)."""
        torch = _require_cuda()
        if len(band) != 4:
            raise ValueError("band must be the four subband planes")
        for b in band:
            if b.dim() != 2:
                raise ValueError("band planes must be [rows, cols]")
        band = [p[0] for p in self._check_in_planes(torch, tuple(band), ("ll", "hl", "lh", "hh"))]
        ll = band[0]
        w = 2 * ll.shape[1]
        if out_row_end <= out_row_begin:
            raise ValueError("bad output row range")
        if out is None:
            out = torch.empty((2 * (out_row_end - out_row_begin), w), dtype=ll.dtype, device=ll.device)
        else:
            _check_buffer(torch, out, "out", (2 * (out_row_end - out_row_begin), w), self.torch_dtype, ll.device)
        pin = _native.planes([_ptr(b) for b in band], [b.stride(0) for b in band], 0)
        _native.check(
            _native.load().b2dwt_inverse_rows(self.inv_plan.handle, pin, band_row0, ll.shape[0], _ptr(out),
                                              out.stride(0), global_height, w, out_row_begin, out_row_end,
                                              _stream_handle(torch, stream)),
            "inverse_rows",
        )
        return out


class PyramidGraph:
    """A multi-level forward transform captured as one CUDA graph.

    The graph bakes in the device addresses of ``x`` and of the outputs
    (``ll``, ``details``), which it owns; each :meth:`replay` recomputes the
    pyramid of whatever ``x`` holds.  With ``level_events=True`` an external
    CUDA event node is recorded before every level and after the last one, so
    per-level kernel times can be read after a replay (:meth:`level_ms`).
    """

    def __init__(self, tr: Transform, x, levels: int, level_events: bool = False):
        torch = tr._check(x, "x")
        h, w = x.shape
        self.x = x
        self.levels = levels
        self.ll, self.details = tr.dwt(x, levels)  # allocates + warms up every level
        self.scratch = torch.empty(((h // 2) * (w // 2) + (h // 4) * (w // 4),), dtype=x.dtype, device=x.device) \
            if levels > 1 else None
        # launch groups: the levels b2dwt_dwt runs in one kernel (fused pairs),
        # and where each group's LL lands: the scratch half it does not read
        # (b2dwt_host.cu b2dwt_dwt), the final one in ``ll``
        self.groups = self._groups(tr)
        half = (h // 2) * (w // 2)
        self._ll_views = [None] * levels
        in_sc = -1
        for a, b in self.groups:
            hh_, ww_ = h >> (b + 1), w >> (b + 1)
            if b == levels - 1:
                self._ll_views[b] = self.ll
                continue
            in_sc = 1 if in_sc == 0 else 0 if in_sc == 1 else (0 if b == 0 else 1)
            off = 0 if in_sc == 0 else half
            self._ll_views[b] = self.scratch[off:off + hh_ * ww_].view(hh_, ww_)
        self.events = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(len(self.groups) + 1)] \
            if level_events else None
        self._run(tr)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._run(tr)

    def _groups(self, tr):
        """[(first level, last level)] in launch order, as b2dwt_dwt groups them
        (b2dwt_host.cu: a pair starts where B2DWT_FUSE2_PAIRS allows, on levels of
        at least B2DWT_FUSE2_MIN_QUADS quads, when the fused kernel takes it)."""
        import os

        min_quads = int(os.environ.get("B2DWT_FUSE2_MIN_QUADS", 1 << 20))
        if not (tr.flags & _native.FAST) and os.environ.get("B2DWT_FUSE2_STRICT", "1") == "0":
            min_quads = 0  # strict plans held at one launch per level (b2dwt_host.cu fuse2_starts_at)
        starts = os.environ.get("B2DWT_FUSE2_PAIRS")
        starts = None if starts is None else {int(v) for v in starts.split(",") if v.strip()}
        h, w = self.x.shape
        torch = _torch()
        # does the plan have a fused kernel at all? (a tiny probe; geometry below)
        probe = torch.zeros((16, 256), dtype=self.x.dtype, device=self.x.device)
        fusable = not (tr.flags & _native.NO_FUSE) and tr.forward2(probe) is not None
        groups, lvl = [], 0
        while lvl < self.levels:
            hl, wl = h >> lvl, w >> lvl
            if fusable and lvl + 1 < self.levels and min_quads > 0 and (hl // 2) * (wl // 2) >= min_quads \
                    and (starts is None or lvl in starts) and hl % 4 == 0 and wl % 4 == 0 and wl >= 256 \
                    and (self.x.stride(0) * self.x.element_size()) % 16 == 0:
                groups.append((lvl, lvl + 1))
                lvl += 2
                continue
            groups.append((lvl, lvl))
            lvl += 1
        return groups

    def _run(self, tr):
        if self.events is None:
            # the product path: one b2dwt_dwt call (fused level pairs, PDL-chained)
            tr.dwt_into(self.x, self.levels, self.details, self.ll, self.scratch)
            return
        for i, (a, b) in enumerate(self.groups):
            self.events[i].record()
            src = self.x if a == 0 else self._ll_views[a - 1]
            if a == b:
                hl, lh, hh = self.details[a]
                tr.forward(src, out=(self._ll_views[a], hl, lh, hh))
            else:
                tr.forward2(src, self.details[a], (self._ll_views[b],) + tuple(self.details[b]))
        self.events[len(self.groups)].record()

    def replay(self):
        self.graph.replay()
        return self.ll, self.details

    def level_ms(self):
        """Kernel time of each launch group (:attr:`groups`: a level, or a fused
        pair of levels) in the last replay (needs level_events=True)."""
        return [self.events[i].elapsed_time(self.events[i + 1]) for i in range(len(self.groups))]


def _call_workspace(torch, nbytes, stream):
    """Device workspace for one host-pipeline call, from torch's caching
    allocator on the call's stream: calls on different streams never share it,
    and the block is recycled only after the stream has passed the call (the
    library joins its internal copy streams back to that stream)."""
    if stream is None:
        return torch.empty((nbytes,), dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(stream):
        return torch.empty((nbytes,), dtype=torch.uint8, device="cuda")


_TRANSFORMS: "OrderedDict" = None
_TRANSFORMS_MAX = 16
_SCHEME_KEYS: dict = {}  # id(scheme) -> (weakref to it, compiled-program key)


def _transform(scheme, precision: str) -> Transform:
    """Transform for the reference-shaped API, cached by the compiled programs
    (not the scheme object's identity: callers that rebuild the scheme per call
    reuse one entry) in a small LRU; entries hold no device workspace."""
    global _TRANSFORMS
    import weakref
    from collections import OrderedDict

    if _TRANSFORMS is None:
        _TRANSFORMS = OrderedDict()
    # fast path: the same scheme object again (compiling + inverting a scheme
    # costs ~1 ms, as much as a whole 1024^2 host-array call) -- held weakly
    hit = _SCHEME_KEYS.get(id(scheme))
    key = hit[1] if hit is not None and hit[0]() is scheme else None
    if key is None:
        fwd, inv = _programs(scheme)
        key = (_signature(fwd), _signature(inv))
        try:
            _SCHEME_KEYS[id(scheme)] = (weakref.ref(scheme), key)
            while len(_SCHEME_KEYS) > 4 * _TRANSFORMS_MAX:
                _SCHEME_KEYS.pop(next(iter(_SCHEME_KEYS)))
        except TypeError:  # not weakly referenceable: no fast path
            pass
    key = key + (precision,)
    t = _TRANSFORMS.get(key)
    if t is None:
        t = Transform(scheme, precision)
        _TRANSFORMS[key] = t
        while len(_TRANSFORMS) > _TRANSFORMS_MAX:
            _TRANSFORMS.popitem(last=False)
    else:
        _TRANSFORMS.move_to_end(key)
    return t


def _to_device(torch, arr: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(arr)).to("cuda", non_blocking=False)


def _to_host(t) -> np.ndarray:
    return t.cpu().numpy()


# -- reference-shaped host API ------------------------------------------------------------


def forward(image: Image2D, scheme, cfg: TileConfig | None = None) -> SubbandQuad:
    """Single-level forward transform of an even-dimensioned image (engine.py:481-487)."""
    cfg = cfg or TileConfig()
    a = image.data
    if a.shape[0] % 2 or a.shape[1] % 2:
        raise ValueError(f"dimensions must be even, got {a.shape[1]}x{a.shape[0]}")
    if cfg.tile is not None:  # (compiling costs ~0.3 ms: only when there is a tile to check)
        _check_tile(cfg, compile_scheme(scheme))
    torch = _require_cuda()
    tr = _transform(scheme, image.precision)
    h, w = a.shape
    # the four subbands in one device block: one download instead of four
    block = torch.empty((4, h // 2, w // 2), dtype=tr.torch_dtype, device="cuda")
    tr.forward(_to_device(torch, a), out=tuple(block[c] for c in range(4)))
    host = block.cpu().numpy()
    return SubbandQuad.from_components([host[c] for c in range(4)])


def inverse(quad: SubbandQuad, scheme, cfg: TileConfig | None = None) -> Image2D:
    """Invert :func:`forward`; ``scheme`` is the forward scheme (engine.py:490-495)."""
    cfg = cfg or TileConfig()
    if cfg.tile is not None:
        _check_tile(cfg, compile_scheme(invert_scheme(_adopt_scheme(scheme))))
    torch = _require_cuda()
    tr = _transform(scheme, quad.ll.precision)
    comps = [_to_device(torch, c) for c in quad.components()]
    return Image2D(_to_host(tr.inverse(*comps)))


def run_tiled(program, comps, cfg: TileConfig) -> list:
    """Run a compiled program over 4 component arrays (engine.py:404-439)."""
    if cfg.tile is not None:
        _check_tile(cfg, program)
    torch = _require_cuda()
    dtype = np.dtype(comps[0].dtype)
    if dtype not in _NP2NATIVE:
        raise TypeError("components must be float32 or float64")
    plan = plan_for(program, _NP2NATIVE[dtype])
    dev = [_to_device(torch, c) for c in comps]
    out = [torch.empty_like(d) for d in dev]
    rows, cols = comps[0].shape
    pin = _native.planes([_ptr(c) for c in dev], [c.stride(0) for c in dev], 0)
    pout = _native.planes([_ptr(c) for c in out], [c.stride(0) for c in out], 0)
    _native.check(
        _native.load().b2dwt_run_components(plan.handle, pin, pout, rows, cols, 1, _stream_handle(torch, None)),
        "run_tiled",
    )
    return [_to_host(o) for o in out]


def run_without_barriers(program, comps, cfg: TileConfig) -> list:
    """Fault model: the inter-pass barriers dropped (engine.py:454-475).

    Tiles run one after another, each taking the whole program to completion
    in place on the shared state, so later tiles read a mix of fresh and stale
    neighbours -- the race a barrier prevents, made deterministic as a
    regression witness.  On the GPU: per (tile, sub-step), the sub-step is
    evaluated over the current state (reflection at the image edges, as the
    reference) and only the tile's window is written back.  Bit-identical to
    the reference's fault model (tests/golden/nobarrier.npz).
    """
    from .program import PassProgram, StencilProgram

    torch = _require_cuda()
    dtype = np.dtype(comps[0].dtype)
    if dtype not in _NP2NATIVE:
        raise TypeError("components must be float32 or float64")
    rows, cols = comps[0].shape
    state = [_to_device(torch, np.ascontiguousarray(c)).clone() for c in comps]
    scratch = [torch.empty_like(c) for c in state]
    subs = [sub for p in program.passes for sub in p.substeps]
    plans = [plan_for(StencilProgram(program.scheme_name if hasattr(program, "scheme_name") else "custom",
                                     getattr(program, "wavelet", "custom"),
                                     (PassProgram(f"sub{i}", "lift", True, (sub,)),)),
                      _NP2NATIVE[dtype], _native.NO_TILE)
             for i, sub in enumerate(subs)]
    if cfg.tile is None:
        tiles = [(0, rows, 0, cols)]
    else:
        tw, th = cfg.tile
        tiles = [(r, min(r + th, rows), c, min(c + tw, cols)) for r in range(0, rows, th) for c in range(0, cols, tw)]
    lib = _native.load()
    pin = _native.planes([_ptr(c) for c in state], [c.stride(0) for c in state], 0)
    pout = _native.planes([_ptr(c) for c in scratch], [c.stride(0) for c in scratch], 0)
    stream = _stream_handle(torch, None)
    for r0, r1, c0, c1 in tiles:
        for plan in plans:
            _native.check(lib.b2dwt_run_components(plan.handle, pin, pout, rows, cols, 1, stream),
                          "run_without_barriers")
            for t in range(4):
                state[t][r0:r1, c0:c1] = scratch[t][r0:r1, c0:c1]
    return [_to_host(c) for c in state]


def run_reference(program, comps) -> list:
    """Untiled executor (engine.py:442-451): the same device path."""
    return run_tiled(program, comps, TileConfig())


def dwt(image: Image2D, scheme, levels: int = 1, cfg: TileConfig | None = None) -> Pyramid:
    """Multi-level forward transform: level l is :func:`forward` of level l-1's LL."""
    cfg = cfg or TileConfig()
    if cfg.tile is not None:
        _check_tile(cfg, compile_scheme(scheme))
    torch = _require_cuda()
    tr = _transform(scheme, image.precision)
    a = image.data
    if tr.fwd_plan.fused and a.size >= _HOST_PIPELINE_MIN_PX and a.shape[0] % (1 << levels) == 0 \
            and a.shape[1] % (1 << levels) == 0:
        # large host image: uploads, kernels and downloads overlapped in row bands
        ll, details = tr.dwt_host(a, levels)
        return Pyramid(Image2D(ll.numpy()), tuple(tuple(Image2D(b.numpy()) for b in d) for d in details))
    ll, details = tr.dwt(_to_device(torch, a), levels)
    return Pyramid(Image2D(_to_host(ll)), tuple(tuple(Image2D(_to_host(b)) for b in d) for d in details))


_HOST_PIPELINE_MIN_PX = 1 << 22  # below ~4 Mpx the copies are too short to pipeline


def idwt(pyramid: Pyramid, scheme, cfg: TileConfig | None = None) -> Image2D:
    """Invert :func:`dwt` level by level, coarsest first."""
    torch = _require_cuda()
    tr = _transform(scheme, pyramid.ll.precision)
    levels = len(pyramid.details)
    if tr.inv_plan.fused and pyramid.ll.data.size << (2 * levels) >= _HOST_PIPELINE_MIN_PX:
        # large host pyramid: level 0's upload, kernels and download overlapped
        out = tr.idwt_host(pyramid.ll.data, [tuple(b.data for b in d) for d in pyramid.details])
        return Image2D(out.numpy())
    details = [tuple(_to_device(torch, b.data) for b in d) for d in pyramid.details]
    return Image2D(_to_host(tr.idwt(_to_device(torch, pyramid.ll.data), details)))
