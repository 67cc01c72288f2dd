"""CPU oracle for the multiple-double least-squares path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product package ``paper_2110_08375_b200`` never imports it, and the C source
``mdls_oracle.c`` shares no code with the CUDA path.

Every function here is a thin ctypes marshaller over ``liboracle.so`` (plain C,
``-O2 -ffp-contract=off``).  Arrays use the paper's staggered storage
(PAPER.md P:371-385): an md matrix with ``ld`` rows and ``cols`` columns is a
numpy float64 array of shape ``(m, cols, ld)`` (plane-major, each plane
column-major); an md vector of length n is ``(m, n)``.

Pins (tests/test_oracle_*.py): exact rationals for the error-free
transformations, mpmath at 2000 bits for md add/mul/div/sqrt, the paper's
Table 1 operation counts through the counting build
``liboracle_count.so``, closed-form QR/BS special cases, the Cholesky
characterisation of R, exact rational normal equations for least squares, and
the invariants E1/E2/E3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mdls_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_LIB_COUNT = os.path.join(_HERE, "liboracle_count.so")

PRECISIONS = {"d": 1, "dd": 2, "qd": 4, "od": 8}  # "d": plain double
OPS = {"add": 0, "sub": 1, "mul": 2, "div": 3, "sqrt": 4}

_CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11", "-Wall",
           "-Wno-unknown-pragmas", "-Wno-maybe-uninitialized"]


def build(force: bool = False) -> None:
    """Compile liboracle.so (OpenMP over independent columns) and liboracle_count.so."""
    for out, extra in ((_LIB, ["-fopenmp"]), (_LIB_COUNT, ["-DMDLS_ORACLE_COUNT"])):
        if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
            subprocess.check_call(["gcc", *_CFLAGS, *extra, "-o", out, _SRC, "-lm"])


_libs: dict[str, ctypes.CDLL] = {}

_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.c_int64


def _load(counting: bool = False) -> ctypes.CDLL:
    key = "count" if counting else "plain"
    if key in _libs:
        return _libs[key]
    build()
    lib = ctypes.CDLL(_LIB_COUNT if counting else _LIB)
    lib.oracle_md_op.argtypes = [ctypes.c_int, ctypes.c_int, _I64, _D, _D, _D]
    lib.oracle_renorm.argtypes = [ctypes.c_int, _D, _D]
    for fn in ("oracle_two_sum", "oracle_quick_two_sum", "oracle_two_prod"):
        getattr(lib, fn).argtypes = [ctypes.c_double, ctypes.c_double, _D]
    lib.oracle_split.argtypes = [ctypes.c_double, _D]
    lib.oracle_house.argtypes = [ctypes.c_int, _I64, _D, _D, _D, _D]
    lib.oracle_qr.argtypes = [ctypes.c_int, _I64, _I64, _D, _I64, _D, ctypes.c_int]
    lib.oracle_form_q.argtypes = [ctypes.c_int, _I64, _I64, _D, _I64, _D, _D, _I64, ctypes.c_int]
    lib.oracle_apply_qt.argtypes = [ctypes.c_int, _I64, _I64, _D, _I64, _D, _D, _D]
    lib.oracle_qt_b_explicit.argtypes = [ctypes.c_int, _I64, _D, _I64, _D, _D, ctypes.c_int]
    lib.oracle_backsub.argtypes = [ctypes.c_int, _I64, _D, _I64, _I64, _D, _I64, _D]
    lib.oracle_lstsq.argtypes = [ctypes.c_int, _I64, _I64, _D, _I64, _D, _D, _D, _D, ctypes.c_int]
    lib.oracle_zlstsq.argtypes = [ctypes.c_int, _I64, _I64, _D, _D, _I64, _D, _D, _D, _D, _D, _D]
    lib.oracle_inv_orth.argtypes = [ctypes.c_int, _I64, _D, _I64, ctypes.POINTER(_I64), _I64, ctypes.c_int]
    lib.oracle_inv_orth.restype = ctypes.c_double
    lib.oracle_inv_recon.argtypes = [ctypes.c_int, _I64, _I64, _D, _I64, _D, _I64, _D, _I64,
                                     ctypes.POINTER(_I64), _I64, ctypes.c_int]
    lib.oracle_inv_recon.restype = ctypes.c_double
    lib.oracle_inv_normal.argtypes = [ctypes.c_int, _I64, _I64, _D, _I64, _D, _D, ctypes.c_int]
    lib.oracle_inv_normal.restype = ctypes.c_double
    lib.oracle_dot.argtypes = [ctypes.c_int, _I64, _D, _I64, _I64, _D, _I64, _I64, _D]
    lib.oracle_blocked.argtypes = [ctypes.c_int, ctypes.c_int, _I64, _I64, _I64, _D, _D, _D, _D, _D, _D,
                                   ctypes.POINTER(_I64), ctypes.POINTER(_I64)]
    lib.oracle_norm2.argtypes = [ctypes.c_int, _I64, _D, _I64, _D]
    lib.oracle_residual_direct.argtypes = [ctypes.c_int, _I64, _I64, _D, _I64, _D, _D, _D]
    lib.oracle_count_get.argtypes = [ctypes.POINTER(ctypes.c_uint64)]
    lib.oracle_selfcheck.restype = ctypes.c_int
    if lib.oracle_selfcheck() != 0:
        raise RuntimeError("oracle self-check two_sum(2^53, 1) failed: reassociation or wrong rounding")
    _libs[key] = lib
    return lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def _m_of(prec) -> int:
    return PRECISIONS[prec] if isinstance(prec, str) else int(prec)


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# --------------------------------------------------------------------------- EFTs
def two_sum(a: float, b: float) -> tuple[float, float]:
    out = np.zeros(2)
    _load().oracle_two_sum(a, b, _p(out))
    return float(out[0]), float(out[1])


def quick_two_sum(a: float, b: float) -> tuple[float, float]:
    out = np.zeros(2)
    _load().oracle_quick_two_sum(a, b, _p(out))
    return float(out[0]), float(out[1])


def two_prod(a: float, b: float) -> tuple[float, float]:
    out = np.zeros(2)
    _load().oracle_two_prod(a, b, _p(out))
    return float(out[0]), float(out[1])


def split(a: float) -> tuple[float, float]:
    out = np.zeros(2)
    _load().oracle_split(a, _p(out))
    return float(out[0]), float(out[1])


# --------------------------------------------------------------------------- md ops
def md_op(op: str, prec, a: np.ndarray, b: np.ndarray | None = None, counting: bool = False) -> np.ndarray:
    """Elementwise md op on (m, n) limb-planar vectors."""
    m = _m_of(prec)
    a = np.ascontiguousarray(a, dtype=np.float64)
    assert a.ndim == 2 and a.shape[0] == m
    n = a.shape[1]
    c = np.zeros_like(a)
    bb = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
    rc = _load(counting).oracle_md_op(OPS[op], m, n, _p(a), _p(bb) if bb is not None else None, _p(c))
    if rc:
        raise ValueError(f"oracle_md_op rc={rc}")
    return c


def renorm(prec, f: np.ndarray) -> np.ndarray:
    m = _m_of(prec)
    f = np.ascontiguousarray(f, dtype=np.float64)
    assert f.shape == (m + 1,)
    r = np.zeros(m)
    _load().oracle_renorm(m, _p(f), _p(r))
    return r


def op_counts(op: str, prec, a: np.ndarray, b: np.ndarray | None = None) -> tuple[int, int, int, int]:
    """Base-double (+, -, *, /) counts of ONE md operation (counting build)."""
    lib = _load(counting=True)
    lib.oracle_count_reset()
    md_op(op, prec, a[:, :1], None if b is None else b[:, :1], counting=True)
    out = (ctypes.c_uint64 * 4)()
    lib.oracle_count_get(out)
    return tuple(int(v) for v in out)


# --------------------------------------------------------------------------- linear algebra
def house(prec, x: np.ndarray):
    m = _m_of(prec)
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = x.shape[1]
    v = np.zeros_like(x)
    beta = np.zeros(m)
    mu = np.zeros(m)
    _load().oracle_house(m, n, _p(x), _p(v), _p(beta), _p(mu))
    return v, beta, mu


def qr(prec, A: np.ndarray, nthreads: int = 0):
    """Unblocked Householder QR.  A: (m, K, M).  Returns (F, beta): F holds R in
    its upper triangle and v_j(2:) below the diagonal; beta is (m, K)."""
    m = _m_of(prec)
    F = np.array(A, dtype=np.float64, order="C", copy=True)
    _, K, M = F.shape
    beta = np.zeros((m, K))
    rc = _load().oracle_qr(m, M, K, _p(F), M, _p(beta), nthreads or default_threads())
    if rc:
        raise ValueError(f"oracle_qr rc={rc}")
    return F, beta


def r_of(F: np.ndarray) -> np.ndarray:
    """Upper triangle of a factored array, strictly-lower part zero."""
    m, K, M = F.shape
    mask = np.arange(M)[None, :] <= np.arange(K)[:, None]  # (K, M): row i <= col j
    return np.where(mask[None, :, :], F, 0.0)


def form_q(prec, F: np.ndarray, beta: np.ndarray, nthreads: int = 0) -> np.ndarray:
    m = _m_of(prec)
    _, K, M = F.shape
    Q = np.zeros((m, M, M))
    rc = _load().oracle_form_q(m, M, K, _p(F), M, _p(np.ascontiguousarray(beta)), _p(Q), M,
                               nthreads or default_threads())
    if rc:
        raise ValueError(f"oracle_form_q rc={rc}")
    return Q


def apply_qt(prec, F: np.ndarray, beta: np.ndarray, b: np.ndarray) -> np.ndarray:
    m = _m_of(prec)
    _, K, M = F.shape
    b = np.ascontiguousarray(b, dtype=np.float64)
    y = np.zeros_like(b)
    _load().oracle_apply_qt(m, M, K, _p(F), M, _p(np.ascontiguousarray(beta)), _p(b), _p(y))
    return y


def qt_b_explicit(prec, Q: np.ndarray, b: np.ndarray, nthreads: int = 0) -> np.ndarray:
    m = _m_of(prec)
    M = Q.shape[1]
    b = np.ascontiguousarray(b, dtype=np.float64)
    y = np.zeros_like(b)
    _load().oracle_qt_b_explicit(m, M, _p(np.ascontiguousarray(Q)), M, _p(b), _p(y), nthreads or default_threads())
    return y


def backsub(prec, R: np.ndarray, y: np.ndarray, n: int | None = None) -> tuple[np.ndarray, int]:
    """Plain back substitution on the leading n x n block of R (m, cols, ld)."""
    m = _m_of(prec)
    R = np.ascontiguousarray(R, dtype=np.float64)
    _, cols, ld = R.shape
    n = cols if n is None else n
    y = np.ascontiguousarray(y, dtype=np.float64)
    x = np.zeros((m, n))
    info = _load().oracle_backsub(m, n, _p(R), ld, cols, _p(y), y.shape[1], _p(x))
    return x, int(info)


def zlstsq(prec, Are: np.ndarray, Aim: np.ndarray, bre: np.ndarray, bim: np.ndarray):
    """Complex least squares (unblocked complex Householder QR with Hermitian reflectors, Q^H b, complex back
    substitution; mdls_oracle.c oracle_zlstsq).  Re/im parts as separate (m, K, M) / (m, M) arrays.
    Returns (xre, xim, Rre, Rim, info); R_jj = -phase(x_1) ||x|| (complex)."""
    m = _m_of(prec)
    Are = np.ascontiguousarray(Are, dtype=np.float64)
    Aim = np.ascontiguousarray(Aim, dtype=np.float64)
    _, K, M = Are.shape
    bre = np.ascontiguousarray(bre, dtype=np.float64)
    bim = np.ascontiguousarray(bim, dtype=np.float64)
    xre, xim = np.zeros((m, K)), np.zeros((m, K))
    Rre, Rim = np.zeros_like(Are), np.zeros_like(Aim)
    info = _load().oracle_zlstsq(m, M, K, _p(Are), _p(Aim), M, _p(bre), _p(bim), _p(xre), _p(xim), _p(Rre), _p(Rim))
    if info < 0:
        raise ValueError(f"oracle_zlstsq rc={info}")
    return xre, xim, Rre, Rim, info


def lstsq(prec, A: np.ndarray, b: np.ndarray, nthreads: int = 0):
    """x minimising ||b - Ax|| (QR, Q^T b by reflectors, back substitution).
    Returns (x, R, y) with R the (m, K, M) upper-triangular factor and y = Q^T b."""
    m = _m_of(prec)
    A = np.ascontiguousarray(A, dtype=np.float64)
    _, K, M = A.shape
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros((m, K))
    R = np.zeros_like(A)
    y = np.zeros((m, M))
    info = _load().oracle_lstsq(m, M, K, _p(A), M, _p(b), _p(x), _p(R), _p(y), nthreads or default_threads())
    if info < 0:
        raise ValueError(f"oracle_lstsq rc={info}")
    return x, R, y


def norm2(prec, y: np.ndarray) -> np.ndarray:
    """||y||_2 of an (m, n) md vector, as an (m,) md number."""
    m = _m_of(prec)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.zeros(m)
    _load().oracle_norm2(m, y.shape[1], _p(y), y.shape[1], _p(out))
    return out


def residual_direct(prec, A: np.ndarray, x: np.ndarray, b: np.ndarray) -> np.ndarray:
    """||b - A x||_2 evaluated directly in md, as an (m,) md number."""
    m = _m_of(prec)
    A = np.ascontiguousarray(A, dtype=np.float64)
    _, K, M = A.shape
    out = np.zeros(m)
    _load().oracle_residual_direct(m, M, K, _p(A), M, _p(np.ascontiguousarray(x, dtype=np.float64)),
                                   _p(np.ascontiguousarray(b, dtype=np.float64)), _p(out))
    return out


def _cols_arg(cols):
    if cols is None:
        return None, 0
    arr = np.ascontiguousarray(np.asarray(cols, dtype=np.int64))
    return arr.ctypes.data_as(ctypes.POINTER(_I64)), len(arr), arr


def inv_orth(prec, Q: np.ndarray, cols=None, nthreads: int = 0) -> float:
    m = _m_of(prec)
    Q = np.ascontiguousarray(Q)
    M = Q.shape[1]
    c = _cols_arg(cols)
    return _load().oracle_inv_orth(m, M, _p(Q), M, c[0], c[1], nthreads or default_threads())


def inv_recon(prec, A: np.ndarray, Q: np.ndarray, R: np.ndarray, cols=None, nthreads: int = 0) -> float:
    m = _m_of(prec)
    A = np.ascontiguousarray(A)
    _, K, M = A.shape
    c = _cols_arg(cols)
    return _load().oracle_inv_recon(m, M, K, _p(A), M, _p(np.ascontiguousarray(Q)), M,
                                    _p(np.ascontiguousarray(R)), R.shape[2], c[0], c[1],
                                    nthreads or default_threads())


def inv_normal(prec, A: np.ndarray, x: np.ndarray, b: np.ndarray, nthreads: int = 0) -> float:
    m = _m_of(prec)
    A = np.ascontiguousarray(A)
    _, K, M = A.shape
    return _load().oracle_inv_normal(m, M, K, _p(A), M, _p(np.ascontiguousarray(x)), _p(np.ascontiguousarray(b)),
                                     nthreads or default_threads())


def dot(prec, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """md dot product of two (m, n) md vectors (ascending accumulation)."""
    m = _m_of(prec)
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = a.shape[1]
    out = np.zeros(m)
    _load().oracle_dot(m, n, _p(a), n, 1, _p(b), n, 1, _p(out))
    return out


# --------------------------------------------------------------------------- blocked, counted pipelines
STAGES = ("house", "panel", "wy", "trailing", "form_q", "qtb", "invert", "mulinv", "bsupdate")
BLOCKED_OPS = {"qr": 0, "backsub": 1, "lstsq": 2, "apply_qt": 3, "lstsq_noq": 4}


def blocked(op: str, prec, A: np.ndarray, b: np.ndarray, nb: int):
    """Algorithm 2 (blocked Householder QR) / Algorithm 1 (tiled back substitution) step by step
    with per-stage md-op counters (mdls_oracle.c ``oracle_blocked``).  A: (m, K, M), or the upper
    triangular (m, K, K) for ``backsub``; b: (m, M).  Returns a dict with x, R, Q, y (None where the
    op has none), ``counts`` {stage: {add, mul, div, sqrt}}, ``nonpos`` (columns that took GVL's
    x1 <= 0 branch) and ``info``."""
    m = _m_of(prec)
    A = np.ascontiguousarray(A, dtype=np.float64)
    _, K, M = A.shape
    b = np.ascontiguousarray(b, dtype=np.float64)
    code = BLOCKED_OPS[op]
    x = np.zeros((m, K))
    R = np.zeros((m, K, M)) if code in (0, 2, 4) else None
    Q = np.zeros((m, M, M)) if code in (0, 2) else None
    y = np.zeros((m, M)) if code in (2, 3, 4) else None
    cnt = np.zeros((9, 4), dtype=np.int64)
    nonpos = ctypes.c_int64(0)
    nul = ctypes.POINTER(ctypes.c_double)()
    info = _load().oracle_blocked(code, m, M, K, nb, _p(A), _p(b), _p(x), _p(R) if R is not None else nul,
                                  _p(Q) if Q is not None else nul, _p(y) if y is not None else nul,
                                  cnt.ctypes.data_as(ctypes.POINTER(_I64)), ctypes.byref(nonpos))
    if info < 0:
        raise ValueError(f"oracle_blocked rc={info}")
    counts = {s: {"add": int(cnt[i, 0]), "mul": int(cnt[i, 1]), "div": int(cnt[i, 2]), "sqrt": int(cnt[i, 3])}
              for i, s in enumerate(STAGES)}
    return {"x": x if code != 3 and code != 0 else None, "R": R, "Q": Q, "y": y, "counts": counts,
            "nonpos": int(nonpos.value), "info": int(info)}
