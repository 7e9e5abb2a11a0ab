"""ctypes binding of libb2dwt.so (the C ABI declared in include/b2dwt.h).

This is the only way the package computes pixels.  If the library is missing
or no CUDA device is visible, every compute call raises -- there is no CPU
fallback (the CPU oracle under oracle/ is test infrastructure only).
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# B2DWT_LIB: another in-tree build of the same library (development
# experiments, e.g. tools/ variants built with extra -D flags)
LIB_PATH = os.environ.get("B2DWT_LIB") or os.path.join(HERE, "libb2dwt.so")

B2DWT_OK = 0
B2DWT_EINVAL = -22
B2DWT_EUNSUPPORTED = -95
B2DWT_ECUDA = -5
F32, F64 = 0, 1
STRICT, FAST, FORCE_GENERIC, NO_TMA, NO_TILE, FORCE_TILE, NO_FUSE = 1, 2, 4, 8, 16, 32, 64

# Every symbol include/b2dwt.h declares (tests check the .so exports all of them).
EXPORTS = (
    "b2dwt_abi_version",
    "b2dwt_last_error",
    "b2dwt_device_count",
    "b2dwt_plan_create",
    "b2dwt_plan_destroy",
    "b2dwt_plan_get_info",
    "b2dwt_run_components",
    "b2dwt_forward",
    "b2dwt_inverse",
    "b2dwt_forward_rows",
    "b2dwt_dwt",
    "b2dwt_forward2",
    "b2dwt_idwt",
    "b2dwt_dwt_host_workspace",
    "b2dwt_dwt_host",
    "b2dwt_inverse_rows",
    "b2dwt_idwt_host_workspace",
    "b2dwt_idwt_host",
    "b2dwt_lift1d",
    "b2dwt_unlift1d",
)


class Term(ctypes.Structure):
    _fields_ = [
        ("src", ctypes.c_int32),
        ("dm", ctypes.c_int32),
        ("dn", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("coeff", ctypes.c_double),
    ]


class Program(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("n_substeps", ctypes.c_int32),
        ("term_counts", ctypes.POINTER(ctypes.c_int32)),
        ("terms", ctypes.POINTER(Term)),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("kernel", ctypes.c_int32),
        ("program_id", ctypes.c_int32),
        ("halo_left", ctypes.c_int32),
        ("halo_right", ctypes.c_int32),
        ("halo_up", ctypes.c_int32),
        ("halo_down", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("key", ctypes.c_char * 64),
    ]


class Planes(ctypes.Structure):
    _fields_ = [
        ("ptr", ctypes.c_void_p * 4),
        ("ld", ctypes.c_int64 * 4),
        ("bstride", ctypes.c_int64),
    ]


class NativeError(RuntimeError):
    pass


_lib = None
_lock = threading.Lock()


def library_path() -> str:
    return LIB_PATH


def load():
    """Load libb2dwt.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1705_08266_b200.build` "
                "(or __graft_entry__.build()); there is no CPU fallback"
            )
        lib = ctypes.CDLL(LIB_PATH)
        i32, i64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
        P = ctypes.POINTER
        sig = {
            "b2dwt_abi_version": (i32, []),
            "b2dwt_last_error": (ctypes.c_char_p, []),
            "b2dwt_device_count": (i32, []),
            "b2dwt_plan_create": (ctypes.c_int, [P(Program), i32, i32, P(vp)]),
            "b2dwt_plan_destroy": (ctypes.c_int, [vp]),
            "b2dwt_plan_get_info": (ctypes.c_int, [vp, P(PlanInfo)]),
            "b2dwt_run_components": (ctypes.c_int, [vp, P(Planes), P(Planes), i64, i64, i32, vp]),
            "b2dwt_forward": (ctypes.c_int, [vp, vp, i64, i64, i64, i64, P(Planes), i32, vp]),
            "b2dwt_inverse": (ctypes.c_int, [vp, P(Planes), vp, i64, i64, i64, i64, i32, vp]),
            "b2dwt_forward_rows": (ctypes.c_int, [vp, vp, i64, i64, i64, i64, i64, i64, i64, P(Planes), vp]),
            "b2dwt_dwt": (ctypes.c_int, [vp, vp, i64, i64, i64, i32, P(Planes), vp, i64, vp, vp]),
            "b2dwt_forward2": (ctypes.c_int, [vp, vp, i64, i64, i64, P(Planes), P(Planes), vp]),
            "b2dwt_idwt": (ctypes.c_int, [vp, vp, i64, P(Planes), i32, vp, i64, i64, i64, vp, vp]),
            "b2dwt_dwt_host_workspace": (i64, [vp, i64, i64, i32]),
            "b2dwt_dwt_host": (ctypes.c_int, [vp, vp, i64, i64, i64, i32, P(Planes), vp, i64, vp, i64, i32, vp]),
            "b2dwt_inverse_rows": (ctypes.c_int, [vp, P(Planes), i64, i64, vp, i64, i64, i64, i64, i64, vp]),
            "b2dwt_idwt_host_workspace": (i64, [vp, i64, i64, i32]),
            "b2dwt_lift1d": (ctypes.c_int, [i32, i32, vp, vp, vp, vp, vp, vp, i64, vp, vp, i64, i64, i32, vp]),
            "b2dwt_unlift1d": (ctypes.c_int, [i32, i32, vp, vp, vp, vp, vp, vp, vp, i64, vp, i64, i64, i32, vp]),
            "b2dwt_idwt_host": (ctypes.c_int, [vp, vp, i64, P(Planes), i32, vp, i64, i64, i64, vp, i64, i32, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.b2dwt_abi_version() != 1:
            raise NativeError("libb2dwt.so ABI version mismatch")
        _lib = lib
    return _lib


def check(rc: int, what: str = "b2dwt") -> None:
    if rc == B2DWT_OK:
        return
    msg = load().b2dwt_last_error().decode(errors="replace")
    if rc == B2DWT_EINVAL:
        raise ValueError(msg)
    if rc == B2DWT_EUNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    raise NativeError(f"{what} failed ({rc}): {msg}")


def device_count() -> int:
    return int(load().b2dwt_device_count())


def planes(ptrs, lds, bstride=0) -> Planes:
    p = Planes()
    for c in range(4):
        p.ptr[c] = ptrs[c]
        p.ld[c] = int(lds[c])
    p.bstride = int(bstride)
    return p


class Plan:
    """Owned b2dwt_plan handle for one compiled program at one precision."""

    def __init__(self, program, dtype: int, flags: int = 0):
        lib = load()
        subs = [s for p in program.passes for s in p.substeps]
        counts = (ctypes.c_int32 * (4 * len(subs)))()
        flat = []
        for si, sub in enumerate(subs):
            for t in range(4):
                counts[4 * si + t] = len(sub.terms[t])
                for (src, dm, dn, c) in sub.terms[t]:
                    flat.append(Term(int(src), int(dm), int(dn), 0, float(c)))
        terms = (Term * max(1, len(flat)))(*flat)
        prog = Program(1, len(subs), counts, terms)
        handle = ctypes.c_void_p()
        check(lib.b2dwt_plan_create(ctypes.byref(prog), dtype, flags, ctypes.byref(handle)), "plan_create")
        self._h = handle
        self.dtype = dtype
        self.flags = flags
        info = PlanInfo()
        check(lib.b2dwt_plan_get_info(self._h, ctypes.byref(info)), "plan_get_info")
        self.info = info
        self.key = info.key.decode()
        self.fused = bool(info.kernel)
        self.cone = (info.halo_up, info.halo_down, info.halo_left, info.halo_right)

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.b2dwt_plan_destroy(h)
            self._h = None
