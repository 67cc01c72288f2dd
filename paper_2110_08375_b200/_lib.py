"""ctypes binding of libmdls.so (include/mdls.h).  Argument marshalling only.

The library is loaded from this package directory; there is no fallback: if
``libmdls.so`` is missing the import of the compute API raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmdls.so")

PRECS = ("dd", "qd", "od", "d")
NSTAGES = 9
STAGES = ("house", "panel", "wy", "trailing", "form_q", "qtb", "invert", "mulinv", "bsupdate")
FAMILIES = ("gemm", "panel", "invert", "backsub", "other")
OP_QR, OP_BACKSUB, OP_LSTSQ, OP_APPLY_QT, OP_LSTSQ_NOQ, OP_ZLSTSQ = 0, 1, 2, 3, 4, 5
ERR_CUDA, ERR_UNSUPPORTED = -100, -101

_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_int64
_Z = ctypes.c_size_t


class Counts(ctypes.Structure):
    _fields_ = [
        ("add", ctypes.c_int64 * NSTAGES),
        ("mul", ctypes.c_int64 * NSTAGES),
        ("div", ctypes.c_int64 * NSTAGES),
        ("sqrt", ctypes.c_int64 * NSTAGES),
        ("flops", ctypes.c_double * NSTAGES),
        ("total_flops", ctypes.c_double),
    ]


# (name, restype, argtypes) for each per-precision entry point
_SIGS = {
    "mdls_workspace_": (_Z, [_I, _L, _L, _L]),
    "mdls_count_": (_I, [_I, _L, _L, _L, ctypes.POINTER(Counts)]),
    "mdls_md_op_": (_I, [_I, _L, _P, _P, _P, _L, _P]),
    "mdls_qr_": (_I, [_L, _L, _L, _P, _L, _L, _P, _L, _L, _P, _L, _L, _P, _Z, _P, _P]),
    "mdls_apply_qt_": (_I, [_L, _L, _L, _P, _L, _L, _P, _L, _L, _P, _L, _P, _L, _P, _Z, _P]),
    "mdls_qt_b_": (_I, [_L, _L, _P, _L, _L, _P, _L, _P, _L, _P, _Z, _P]),
    "mdls_gemm_": (_I, [_L, _L, _L, _I, _I, _P, _L, _L, _P, _L, _L, _P, _L, _L, _I, _P, _Z, _P]),
    "mdls_invert_tiles_": (_I, [_L, _L, _P, _L, _L, _P, _L, _L, _P, _P]),
    "mdls_backsub_": (_I, [_L, _L, _P, _L, _L, _P, _L, _P, _L, _P, _Z, _P, _P]),
    "mdls_lstsq_": (_I, [_L, _L, _L, _P, _L, _L, _P, _L, _P, _L, _I, _P, _L, _L, _P, _L, _L, _P, _L, _P, _Z, _P,
                         _P]),
    "mdls_norm2_": (_I, [_L, _P, _L, _P, _L, _P]),
    "mdls_lstsq_batched_": (_I, [_L, _L, _L, _L, _P, _L, _L, _L, _P, _L, _L, _P, _L, _L, _I, _I, _P, _Z, _P, _P]),
    "mdls_workspace_batched_": (_Z, [_I, _L, _L, _L, _I]),
    "mdls_zlstsq_": (_I, [_L, _L, _L, _P, _P, _L, _L, _P, _P, _L, _P, _P, _L, _I, _P, _Z, _P, _P]),
    "mdls_lstsq_plan_": (_I, [_L, _L, _L, _P, _L, _L, _P, _L, _P, _L, _I, _P, _Z, _P, ctypes.POINTER(_P)]),
    "mdls_lstsq_host_": (_I, [_L, _L, _L, _P, _L, _L, _P, _L, _P, _L, _I, _P, _Z, _P, _P]),
    "mdls_lstsq_host_plan_": (_I, [_L, _L, _L, _P, _L, _L, _P, _L, _P, _L, _I, _P, _Z, _P, ctypes.POINTER(_P)]),
    "mdls_lstsq_batched_plan_": (_I, [_L, _L, _L, _L, _P, _L, _L, _L, _P, _L, _L, _P, _L, _L, _I, _I, _P, _Z, _P,
                                      ctypes.POINTER(_P)]),
    "mdls_qr_panel_": (_I, [_L, _L, _L, _P, _L, _L, _P, _L, _L, _P, _L, _L, _P, _Z, _P, _P]),
    "mdls_qr_update_": (_I, [_L, _L, _L, _P, _L, _L, _P, _L, _L, _P, _L, _L, _L, _L, _P, _Z, _P]),
}

# every symbol include/mdls.h declares
EXPORTED = ["mdls_strerror", "mdls_version", "mdls_limbs", "mdls_launch_count", "mdls_trace_enable",
            "mdls_trace_collect", "mdls_plan_launch", "mdls_plan_launches", "mdls_plan_destroy"] + [f"{n}{p}" for n in _SIGS for p in PRECS]

_lib: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libmdls.so not found at {LIB_PATH}: the CUDA extension is not built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    lib.mdls_strerror.restype = ctypes.c_char_p
    lib.mdls_strerror.argtypes = [_I]
    lib.mdls_version.restype = _I
    lib.mdls_limbs.restype = _I
    lib.mdls_limbs.argtypes = [_I]
    lib.mdls_launch_count.restype = _L
    lib.mdls_trace_enable.argtypes = [_I]
    lib.mdls_trace_enable.restype = None
    lib.mdls_trace_collect.argtypes = [_P, _P, _P]
    lib.mdls_trace_collect.restype = _I
    lib.mdls_plan_launch.argtypes = [_P, _P]
    lib.mdls_plan_launch.restype = _I
    lib.mdls_plan_launches.argtypes = [_P]
    lib.mdls_plan_launches.restype = _L
    lib.mdls_plan_destroy.argtypes = [_P]
    lib.mdls_plan_destroy.restype = None
    for name, (res, args) in _SIGS.items():
        for p in PRECS:
            f = getattr(lib, f"{name}{p}")
            f.restype = res
            f.argtypes = args
    _lib = lib
    return lib


def fn(name: str, prec: str):
    return getattr(load(), f"{name}{prec}")


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().mdls_strerror(rc).decode()
        raise RuntimeError(f"{what} failed: rc={rc} ({msg})")
