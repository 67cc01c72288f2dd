"""Multiple-double least squares on B200 (arXiv 2110.08375), Python binding.

Thin marshalling over the C-ABI of ``include/mdls.h`` (``libmdls.so``): every
step of the path runs in the library's sm_100a kernels; torch only supplies
device memory and the current CUDA stream.  There is no CPU fallback.

Layout (the paper's staggered storage): an md matrix with ``ld``
rows and ``cols`` columns is a CUDA float64 tensor of shape ``(m, cols, ld)``
(limb planes, most significant first, each column-major); an md vector of
length n is ``(m, n)``.  m = 2 (dd), 4 (qd), 8 (od).
"""
from __future__ import annotations

import ctypes

from . import _lib

PRECISIONS = {"dd": 2, "qd": 4, "od": 8, "d": 1}  # "d": plain double
OPS = {"add": 0, "sub": 1, "mul": 2, "div": 3, "sqrt": 4, "sqrt_fast": 5, "recip_fast": 6, "wmul": 7, "wsqrt_fast": 8,
       "wrecip_fast": 9}
T1_SUMS = {"dd": (20, 23, 70), "qd": (89, 336, 893), "od": (269, 1742, 5126), "d": (1, 1, 1)}  # P:102-136 (add, mul, div)

__all__ = ["md_op", "qr", "apply_qt", "qt_b", "invert_tiles", "backsub", "lstsq", "lstsq_host", "norm2", "counts",
           "workspace_bytes", "PRECISIONS"]


def _torch():
    import torch

    return torch


def _stream():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _check_md(t, prec, ndim, name):
    torch = _torch()
    m = PRECISIONS[prec]
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name}: expected a CUDA tensor")
    if t.dtype != torch.float64 or t.dim() != ndim or t.shape[0] != m or not t.is_contiguous():
        raise ValueError(f"{name}: expected contiguous float64 of {ndim} dims with {m} limb planes, got "
                         f"{tuple(t.shape)} {t.dtype}")


def _mat(t):
    """(ptr, ld, ps) of an (m, cols, ld) tensor"""
    return ctypes.c_void_p(t.data_ptr()), t.shape[2], t.shape[1] * t.shape[2]


def _vec(t):
    return ctypes.c_void_p(t.data_ptr()), t.shape[1]


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


def workspace_bytes(prec: str, op: int, M: int, K: int, nb: int) -> int:
    return int(_lib.fn("mdls_workspace_", prec)(op, M, K, nb))


def _work(prec, op, M, K, nb, device):
    torch = _torch()
    n = workspace_bytes(prec, op, M, K, nb)
    if n == 0:
        raise ValueError(f"invalid sizes M={M} K={K} nb={nb}")
    return torch.empty(n, dtype=torch.uint8, device=device), n


def _info(device):
    torch = _torch()
    return torch.zeros(1, dtype=torch.int32, device=device)


def md_op(op: str, prec: str, a, b=None):
    """Elementwise md arithmetic on (m, n) CUDA vectors (A0)."""
    torch = _torch()
    _check_md(a, prec, 2, "a")
    unary = OPS[op] >= 4 and OPS[op] != 7
    if not unary:
        _check_md(b, prec, 2, "b")
    c = torch.empty_like(a)
    n = a.shape[1]
    rc = _lib.fn("mdls_md_op_", prec)(OPS[op], n, _ptr(a), _ptr(None if unary else b), _ptr(c), n, _stream())
    _lib.check(rc, "md_op")
    return c


def qr(prec: str, A, nb: int, form_q: bool = True, want_w: bool = False):
    """Blocked Householder QR (Algorithm 2).  Returns (F, Q, W, info): F = factored
    copy of A (R upper, v below), Q (m, M, M) or None, W (m, K, M) or None,
    info a device int32 tensor (0 ok, k>0 first zero/non-finite R_kk)."""
    torch = _torch()
    _check_md(A, prec, 3, "A")
    m, K, M = A.shape
    F = A.clone()
    Q = torch.empty((m, M, M), dtype=torch.float64, device=A.device) if form_q else None
    W = torch.empty((m, K, M), dtype=torch.float64, device=A.device) if want_w else None
    work, nbytes = _work(prec, _lib.OP_QR, M, K, nb, A.device)
    info = _info(A.device)
    qp, qld, qps = _mat(Q) if Q is not None else (ctypes.c_void_p(0), 0, 0)
    wp, wld, wps = _mat(W) if W is not None else (ctypes.c_void_p(0), 0, 0)
    rc = _lib.fn("mdls_qr_", prec)(M, K, nb, *_mat(F), qp, qld, qps, wp, wld, wps, _ptr(work), nbytes,
                                   _ptr(info), _stream())
    _lib.check(rc, "qr")
    return F, Q, W, info


def apply_qt(prec: str, F, W, b, nb: int):
    """y = Q^T b from a factored F and its W (panels applied)."""
    torch = _torch()
    _check_md(F, prec, 3, "F")
    _check_md(b, prec, 2, "b")
    m, K, M = F.shape
    y = torch.empty_like(b)
    work, nbytes = _work(prec, _lib.OP_APPLY_QT, M, K, nb, F.device)
    rc = _lib.fn("mdls_apply_qt_", prec)(M, K, nb, *_mat(F), *_mat(W), *_vec(b), *_vec(y), _ptr(work), nbytes,
                                         _stream())
    _lib.check(rc, "apply_qt")
    return y


def gemm(prec: str, A, B, C=None, trans_a: bool = False, trans_b: bool = False, mode: int = 0, work=None):
    """md tile product C (mode)= op(A) op(B) (mdls_gemm_<p>): operands are (m, cols, rows) limb-planar tensors,
    op(X) = X or X^T; mode 0 C = P, 1 C += P, 2 C -= P, 3 C = -P.  Returns C."""
    torch = _torch()
    _check_md(A, prec, 3, "A")
    _check_md(B, prec, 3, "B")
    m_l, ca, ra = A.shape
    _, cb, rb = B.shape
    m, k = (ca, ra) if trans_a else (ra, ca)
    kb, n = (cb, rb) if trans_b else (rb, cb)
    if kb != k:
        raise ValueError(f"gemm: inner dimensions {k} and {kb} differ")
    if C is None:
        C = torch.zeros((m_l, n, m), dtype=torch.float64, device=A.device)
    _check_md(C, prec, 3, "C")
    if work is None:
        work = torch.empty(8 * m_l * 8 * max(m * n, 1), dtype=torch.uint8, device=A.device)
    rc = _lib.fn("mdls_gemm_", prec)(m, n, k, int(trans_a), int(trans_b), *_mat(A), *_mat(B), *_mat(C), mode,
                                     _ptr(work), work.numel(), _stream())
    _lib.check(rc, "gemm")
    return C


def qt_b(prec: str, Q, b):
    """y = Q^T b with an explicit Q of shape (m, N, M) (N columns of M rows); y has N entries."""
    torch = _torch()
    _check_md(Q, prec, 3, "Q")
    _check_md(b, prec, 2, "b")
    m, N, M = Q.shape
    y = torch.empty((m, N), dtype=torch.float64, device=Q.device)
    work = torch.empty(8 * m * 8 * max(N, 1), dtype=torch.uint8, device=Q.device)
    rc = _lib.fn("mdls_qt_b_", prec)(M, N, *_mat(Q), *_vec(b), *_vec(y), _ptr(work), work.numel(), _stream())
    _lib.check(rc, "qt_b")
    return y


def invert_tiles(prec: str, U, nb: int, n: int | None = None):
    """Transposed inverses of the n/nb diagonal tiles of U (A7): Vt (m, n, nb)."""
    torch = _torch()
    _check_md(U, prec, 3, "U")
    n = U.shape[1] if n is None else n
    Vt = torch.empty((PRECISIONS[prec], n, nb), dtype=torch.float64, device=U.device)
    info = _info(U.device)
    rc = _lib.fn("mdls_invert_tiles_", prec)(n, nb, *_mat(U), *_mat(Vt), _ptr(info), _stream())
    _lib.check(rc, "invert_tiles")
    return Vt, info


def backsub(prec: str, U, y, nb: int, n: int | None = None):
    """Tiled back substitution (Algorithm 1) on the leading n x n of U.  Returns (x, info)."""
    torch = _torch()
    _check_md(U, prec, 3, "U")
    _check_md(y, prec, 2, "y")
    n = U.shape[1] if n is None else n
    x = torch.empty((PRECISIONS[prec], n), dtype=torch.float64, device=U.device)
    work, nbytes = _work(prec, _lib.OP_BACKSUB, n, n, nb, U.device)
    info = _info(U.device)
    rc = _lib.fn("mdls_backsub_", prec)(n, nb, *_mat(U), *_vec(y), *_vec(x), _ptr(work), nbytes, _ptr(info),
                                        _stream())
    _lib.check(rc, "backsub")
    return x, info


def norm2(prec: str, y):
    """||y||_2 of an (m, n) md vector, as an (m, 1) md tensor (mdls_norm2_<p>)."""
    torch = _torch()
    _check_md(y, prec, 2, "y")
    out = torch.empty((PRECISIONS[prec], 1), dtype=torch.float64, device=y.device)
    rc = _lib.fn("mdls_norm2_", prec)(y.shape[1], _ptr(y), y.shape[1], _ptr(out), 1, _stream())
    _lib.check(rc, "norm2")
    return out


class LstsqResult:
    __slots__ = ("x", "R", "Q", "y", "info", "residual")

    def __init__(self, x, R, Q, y, info, residual=None):
        self.x, self.R, self.Q, self.y, self.info, self.residual = x, R, Q, y, info, residual


def lstsq(prec: str, A, b, nb: int, form_q: bool = True, want_R: bool = False, want_Q: bool = False,
          want_y: bool = False, want_residual: bool = False, work=None):
    """Least squares x = argmin ||b - A x|| (QR, Q^T b, tiled back substitution).  With want_residual the
    result carries ``residual`` = ||(Q^T b)(K+1:M)||_2 = ||b - A x||_2 as an (m, 1) md tensor."""
    torch = _torch()
    _check_md(A, prec, 3, "A")
    _check_md(b, prec, 2, "b")
    m, K, M = A.shape
    dev = A.device
    x = torch.empty((m, K), dtype=torch.float64, device=dev)
    R = torch.empty((m, K, M), dtype=torch.float64, device=dev) if want_R else None
    Q = torch.empty((m, M, M), dtype=torch.float64, device=dev) if (want_Q and form_q) else None
    y = torch.empty((m, M), dtype=torch.float64, device=dev) if (want_y or want_residual) else None
    op = _lib.OP_LSTSQ if form_q else _lib.OP_LSTSQ_NOQ
    if work is None:
        work, nbytes = _work(prec, op, M, K, nb, dev)
    else:
        nbytes = work.numel()
    info = _info(dev)
    rp = _mat(R) if R is not None else (ctypes.c_void_p(0), 0, 0)
    qp = _mat(Q) if Q is not None else (ctypes.c_void_p(0), 0, 0)
    yp = _vec(y) if y is not None else (ctypes.c_void_p(0), 0)
    rc = _lib.fn("mdls_lstsq_", prec)(M, K, nb, *_mat(A), *_vec(b), *_vec(x), int(form_q), *rp, *qp, *yp,
                                      _ptr(work), nbytes, _ptr(info), _stream())
    _lib.check(rc, "lstsq")
    res = norm2(prec, y[:, K:].contiguous()) if want_residual else None
    return LstsqResult(x, R, Q, y if want_y else None, info, res)


def zlstsq(prec: str, Are, Aim, bre, bim, nb: int, form_q: bool = True, work=None):
    """Complex least squares (mdls_zlstsq_<p>, row f2): A = Are + i Aim (m, K, M each), b = bre + i bim (m, M).
    Returns (xre, xim, info)."""
    torch = _torch()
    for t, nm in ((Are, "Are"), (Aim, "Aim")):
        _check_md(t, prec, 3, nm)
    for t, nm in ((bre, "bre"), (bim, "bim")):
        _check_md(t, prec, 2, nm)
    m, K, M = Are.shape
    if Aim.shape != Are.shape or bre.shape != (m, M) or bim.shape != (m, M):
        raise ValueError("re/im shapes differ")
    dev = Are.device
    xre = torch.empty((m, K), dtype=torch.float64, device=dev)
    xim = torch.empty((m, K), dtype=torch.float64, device=dev)
    nbytes = int(_lib.fn("mdls_workspace_", prec)(_lib.OP_ZLSTSQ, M, K, nb))
    if nbytes == 0:
        raise ValueError("invalid complex least-squares shape (need M >= K, nb | 2K, nb <= 256)")
    if work is None or work.numel() < nbytes:
        work = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    info = _info(dev)
    rc = _lib.fn("mdls_zlstsq_", prec)(M, K, nb, _ptr(Are), _ptr(Aim), M, K * M, _ptr(bre), _ptr(bim), M, _ptr(xre),
                                       _ptr(xim), K, int(form_q), _ptr(work), work.numel(), _ptr(info), _stream())
    _lib.check(rc, "zlstsq")
    return xre, xim, info


def batch_workspace_bytes(prec: str, op: int, M: int, K: int, nb: int, groups: int) -> int:
    return int(_lib.fn("mdls_workspace_batched_", prec)(op, M, K, nb, groups))


def lstsq_batched(prec: str, A, b, nb: int, form_q: bool = True, groups: int = 4, work=None):
    """Independent least-squares problems (mdls_lstsq_batched_<p>): A (B, m, K, M), b (B, m, M) -> x (B, m, K),
    info (B,).  Problem p runs on stream group p mod ``groups``; up to ``groups`` solves overlap."""
    torch = _torch()
    if A.dim() != 4 or b.dim() != 3:
        raise ValueError("A must be (B, m, K, M) and b (B, m, M)")
    Bn, m, K, M = A.shape
    _check_md(A[0], prec, 3, "A")
    _check_md(b[0], prec, 2, "b")
    if not (A.is_contiguous() and b.is_contiguous()):
        raise ValueError("A and b must be contiguous")
    dev = A.device
    x = torch.empty((Bn, m, K), dtype=torch.float64, device=dev)
    info = torch.zeros(max(Bn, 1), dtype=torch.int32, device=dev)
    op = _lib.OP_LSTSQ if form_q else _lib.OP_LSTSQ_NOQ
    groups = max(1, min(int(groups), 16))
    nbytes = batch_workspace_bytes(prec, op, M, K, nb, groups)
    if nbytes == 0:
        raise ValueError("invalid batched least-squares shape")
    if work is None or work.numel() < nbytes:
        work = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    rc = _lib.fn("mdls_lstsq_batched_", prec)(Bn, M, K, nb, _ptr(A), M, K * M, m * K * M, _ptr(b), M, m * M,
                                              _ptr(x), K, m * K, int(form_q), groups, _ptr(work), work.numel(),
                                              _ptr(info), _stream())
    _lib.check(rc, "lstsq_batched")
    return x, info[:Bn]


class _Plan:
    """Owner of a libmdls plan (a library-owned CUDA graph of one call) and of the device buffers it was
    captured with.  run() replays it on the current stream."""

    def _capture(self, fn, args):
        h = ctypes.c_void_p(0)
        rc = fn(*args, ctypes.byref(h))
        _lib.check(rc, "plan")
        self._h = h

    def run(self):
        rc = _lib.load().mdls_plan_launch(self._h, _stream())
        _lib.check(rc, "plan_launch")

    @property
    def launches(self) -> int:
        return int(_lib.load().mdls_plan_launches(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().mdls_plan_destroy(h)
            except Exception:  # pragma: no cover (interpreter shutdown)
                pass


class LstsqPlan(_Plan):
    """Least squares of one M x K shape as a replayable plan (mdls_lstsq_plan_<p>): the plan owns A (m, K, M),
    b (m, M), x (m, K), info and the workspace.  solve(A, b) copies the inputs in (device tensors or pinned host
    tensors, asynchronously), replays the captured solve and returns x (the plan's buffer; copy it before the
    next solve)."""

    def __init__(self, prec: str, M: int, K: int, nb: int, form_q: bool = True, device=None):
        torch = _torch()
        dev = torch.device("cuda") if device is None else torch.device(device)
        m = PRECISIONS[prec]
        self.prec, self.M, self.K, self.nb = prec, M, K, nb
        self.A = torch.zeros((m, K, M), dtype=torch.float64, device=dev)
        self.b = torch.zeros((m, M), dtype=torch.float64, device=dev)
        self.x = torch.empty((m, K), dtype=torch.float64, device=dev)
        self.info = torch.zeros(1, dtype=torch.int32, device=dev)
        op = _lib.OP_LSTSQ if form_q else _lib.OP_LSTSQ_NOQ
        self.work, nbytes = _work(prec, op, M, K, nb, dev)
        self._capture(_lib.fn("mdls_lstsq_plan_", prec),
                      (M, K, nb, *_mat(self.A), *_vec(self.b), *_vec(self.x), int(form_q), _ptr(self.work), nbytes,
                       _ptr(self.info)))

    def solve(self, A=None, b=None):
        if A is not None:
            self.A.copy_(A, non_blocking=True)
        if b is not None:
            self.b.copy_(b, non_blocking=True)
        self.run()
        return self.x


class HostLstsqPlan(_Plan):
    """Least squares from and to page-locked HOST memory as a replayable plan (mdls_lstsq_host_plan_<p>): pinned
    host buffers A (m, K, M), b (m, M), x (m, K) -- the caller's (captured by address) or the plan's own -- plus the
    device workspace and info.  run() replays the captured call: b and then A's column panels cross PCIe while the
    factorisation of the first panels runs, x comes back at the end.  solve(A, b) first writes new inputs into the
    pinned buffers (host copies), replays and returns the pinned x after synchronising the current stream."""

    def __init__(self, prec: str, M: int, K: int, nb: int, form_q: bool = True, device=None, A=None, b=None, x=None):
        torch = _torch()
        dev = torch.device("cuda") if device is None else torch.device(device)
        m = PRECISIONS[prec]
        self.prec, self.M, self.K, self.nb = prec, M, K, nb

        def pinned(t, shape, name):  # the caller's pinned buffer (captured by address) or a new one
            if t is None:
                return torch.zeros(shape, dtype=torch.float64).pin_memory()
            if t.is_cuda or not t.is_pinned() or t.dtype != torch.float64 or tuple(t.shape) != shape \
                    or not t.is_contiguous():
                raise ValueError(f"HostLstsqPlan: {name} must be a pinned contiguous float64 host tensor {shape}")
            return t
        self.A = pinned(A, (m, K, M), "A")
        self.b = pinned(b, (m, M), "b")
        self.x = pinned(x, (m, K), "x")
        self.info = torch.zeros(1, dtype=torch.int32, device=dev)
        op = _lib.OP_LSTSQ if form_q else _lib.OP_LSTSQ_NOQ
        self.work, nbytes = _work(prec, op, M, K, nb, dev)
        self._capture(_lib.fn("mdls_lstsq_host_plan_", prec),
                      (M, K, nb, _ptr(self.A), M, K * M, _ptr(self.b), M, _ptr(self.x), K, int(form_q),
                       _ptr(self.work), nbytes, _ptr(self.info)))

    def solve(self, A=None, b=None):
        torch = _torch()
        if A is not None:
            self.A.copy_(torch.as_tensor(A))
        if b is not None:
            self.b.copy_(torch.as_tensor(b))
        self.run()
        torch.cuda.current_stream().synchronize()
        return self.x


def lstsq_host(prec: str, A, b, nb: int, form_q: bool = True):
    """Least squares from pinned host tensors A (m, K, M) and b (m, M) (mdls_lstsq_host_<p>): returns (x, info),
    x a pinned host (m, K) tensor, valid after the current stream synchronises (done here)."""
    torch = _torch()
    m = PRECISIONS[prec]
    if A.is_cuda or b.is_cuda or not A.is_pinned() or not b.is_pinned():
        raise ValueError("lstsq_host: A and b must be page-locked host tensors (tensor.pin_memory())")
    if A.dtype != torch.float64 or A.dim() != 3 or A.shape[0] != m or not A.is_contiguous():
        raise ValueError(f"lstsq_host: A must be contiguous float64 (m={m}, K, M)")
    _, K, M = A.shape
    x = torch.empty((m, K), dtype=torch.float64).pin_memory()
    dev = torch.device("cuda")
    work, nbytes = _work(prec, _lib.OP_LSTSQ if form_q else _lib.OP_LSTSQ_NOQ, M, K, nb, dev)
    info = _info(dev)
    rc = _lib.fn("mdls_lstsq_host_", prec)(M, K, nb, _ptr(A), M, K * M, _ptr(b), b.shape[1], _ptr(x), K, int(form_q),
                                           _ptr(work), nbytes, _ptr(info), _stream())
    _lib.check(rc, "lstsq_host")
    torch.cuda.current_stream().synchronize()
    return x, info


class BatchedLstsqPlan(_Plan):
    """mdls_lstsq_batched_plan_<p>: `batch` problems of one shape on `groups` stream groups, as one plan; owns
    A (B, m, K, M), b (B, m, M), x (B, m, K), info (B,) and the workspace."""

    def __init__(self, prec: str, batch: int, M: int, K: int, nb: int, form_q: bool = True, groups: int = 8,
                 device=None):
        torch = _torch()
        dev = torch.device("cuda") if device is None else torch.device(device)
        m = PRECISIONS[prec]
        self.prec, self.batch, self.M, self.K, self.nb = prec, batch, M, K, nb
        self.A = torch.zeros((batch, m, K, M), dtype=torch.float64, device=dev)
        self.b = torch.zeros((batch, m, M), dtype=torch.float64, device=dev)
        self.x = torch.empty((batch, m, K), dtype=torch.float64, device=dev)
        self.info = torch.zeros(max(batch, 1), dtype=torch.int32, device=dev)
        op = _lib.OP_LSTSQ if form_q else _lib.OP_LSTSQ_NOQ
        groups = max(1, min(int(groups), 16))
        nbytes = batch_workspace_bytes(prec, op, M, K, nb, groups)
        if nbytes == 0:
            raise ValueError("invalid batched least-squares shape")
        self.work = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self._capture(_lib.fn("mdls_lstsq_batched_plan_", prec),
                      (batch, M, K, nb, _ptr(self.A), M, K * M, m * K * M, _ptr(self.b), M, m * M, _ptr(self.x), K,
                       m * K, int(form_q), groups, _ptr(self.work), nbytes, _ptr(self.info)))

    def solve(self, A=None, b=None):
        if A is not None:
            self.A.copy_(A, non_blocking=True)
        if b is not None:
            self.b.copy_(b, non_blocking=True)
        self.run()
        return self.x


def launch_count() -> int:
    """Kernels launched by libmdls since load (host counter)."""
    return int(_lib.load().mdls_launch_count())


def trace_enable(on: bool = True) -> None:
    """Bracket every library launch with CUDA events (per-stage kernel times)."""
    _lib.load().mdls_trace_enable(int(on))


def trace_collect() -> dict:
    """Per-stage and per-kernel-family event times (ms) of the traced launches."""
    import numpy as np

    st = np.zeros(_lib.NSTAGES + 1)
    fm = np.zeros(len(_lib.FAMILIES))
    fl = np.zeros(len(_lib.FAMILIES), dtype=np.int64)
    rc = _lib.load().mdls_trace_collect(ctypes.c_void_p(st.ctypes.data), ctypes.c_void_p(fm.ctypes.data),
                                        ctypes.c_void_p(fl.ctypes.data))
    if rc < 0:
        raise RuntimeError(f"trace_collect failed rc={rc}")
    return {
        "stages_ms": {s: float(v) for s, v in zip(_lib.STAGES + ("setup",), st)},
        "family_ms": {f: float(v) for f, v in zip(_lib.FAMILIES, fm)},
        "family_launches": {f: int(v) for f, v in zip(_lib.FAMILIES, fl)},
        "launches": int(rc),
    }


def counts(prec: str, op: int, M: int, K: int, nb: int) -> dict:
    """Canonical md-op counts and Table-1 flops per stage (host, A10 ledger)."""
    c = _lib.Counts()
    rc = _lib.fn("mdls_count_", prec)(op, M, K, nb, ctypes.byref(c))
    _lib.check(rc, "count")
    return {
        "stages": {s: {"add": c.add[i], "mul": c.mul[i], "div": c.div[i], "sqrt": c.sqrt[i], "flops": c.flops[i]}
                   for i, s in enumerate(_lib.STAGES)},
        "total_flops": c.total_flops,
    }


# ---------------------------------------------------------------------------- multi-GPU building blocks
def _view(t, col0: int, ncols: int):
    """(ptr, ld, ps) of columns [col0, col0+ncols) of an (m, cols, ld) contiguous tensor."""
    ld = t.shape[2]
    return ctypes.c_void_p(t.data_ptr() + 8 * col0 * ld), ld, t.shape[1] * ld


def _trimmed(t, row0: int):
    """(ptr, ld, ps) of an (m, cols, ld) tensor holding only rows row0.. of an operand indexed by global row:
    the pointer is moved back by row0 rows (rows < row0 are never accessed, include/mdls.h)."""
    return ctypes.c_void_p(t.data_ptr() - 8 * row0), t.shape[2], t.shape[1] * t.shape[2]


def qr_panel(prec: str, A, col0: int, k: int, nb: int, W, Y, work=None):
    """Factor panel k stored in columns [col0, col0+nb) of A (rows global); W and Y receive the panel's
    P_WY = I + W Y^T, either as full (m, nb, M) tensors or row-trimmed (m, nb, M - k nb) ones (rows k nb..M-1).
    Returns the device info tensor."""
    M = A.shape[2]
    if work is None:
        work, nbytes = _work(prec, _lib.OP_QR, M, nb, nb, A.device)
    else:
        nbytes = work.numel()
    info = _info(A.device)
    r0 = M - W.shape[2]
    rc = _lib.fn("mdls_qr_panel_", prec)(M, nb, k, *_view(A, col0, nb), *_trimmed(W, r0), *_trimmed(Y, r0),
                                         _ptr(work), nbytes, _ptr(info), _stream())
    _lib.check(rc, "qr_panel")
    return info


def qr_update(prec: str, Wk, Yk, A, k: int, nb: int, c0: int, c1: int, work=None):
    """C += Yk (Wk^T C) on columns [c0, c1) of A (rows k*nb..M-1); Wk, Yk full or row-trimmed as in qr_panel."""
    M = A.shape[2]
    if c1 <= c0:
        return
    if work is None:
        work, nbytes = _work(prec, _lib.OP_QR, M, nb, nb, A.device)
    else:
        nbytes = work.numel()
    r0 = M - Wk.shape[2]
    rc = _lib.fn("mdls_qr_update_", prec)(M, nb, k, *_trimmed(Wk, r0), *_trimmed(Yk, r0), *_mat(A), c0, c1,
                                          _ptr(work), nbytes, _stream())
    _lib.check(rc, "qr_update")
