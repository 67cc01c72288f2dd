"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic: it only draws random doubles
and places them in the paper's staggered (limb-planar) storage.

Recipe (reading of P:654-663 "Random numbers were
generated for the input matrices ... upper triangular matrices ... as the
output of an LU factorization ... well conditioned problems"):

* generator: numpy ``Philox`` counter-based bit generator keyed by ``seed``
  (platform independent);
* an md value: limb 0 uniform in [-1, 1); limb k (k >= 1) = u_k * ulp(limb k-1) / 2
  with u_k uniform in (-1, 1).  Every limb is populated and the expansion is
  non-overlapping by construction (|x_k| < ulp(x_{k-1})/2), so no
  renormalisation (md arithmetic) is needed here;
* general matrices (least squares, QR): independent md values as above;
* upper-triangular matrices for the stand-alone back substitution: the U factor
  of a partially pivoted LU of a uniform [-1, 1) matrix (fp64, leading limb),
  lower limbs populated as above, strictly-lower part exactly zero.

Layout: an md matrix with ``rows`` rows and ``cols`` columns is a float64
array of shape ``(m, cols, rows)`` -- plane ``l`` (0 = most significant) is
column-major; an md vector of length n is ``(m, n)``.
"""
from __future__ import annotations

import numpy as np

PRECISIONS = {"d": 1, "dd": 2, "qd": 4, "od": 8}


def limbs(prec) -> int:
    return PRECISIONS[prec] if isinstance(prec, str) else int(prec)


def rng(seed: int, stream: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[int(seed) & 0xFFFFFFFFFFFFFFFF, int(stream)]))


def _lower_limbs(lead: np.ndarray, m: int, g: np.random.Generator) -> np.ndarray:
    out = np.empty((m,) + lead.shape, dtype=np.float64)
    out[0] = lead
    for k in range(1, m):
        u = g.uniform(-1.0, 1.0, size=lead.shape)
        # spacing(x) = ulp(x), a power of two: the product is exact
        out[k] = np.where(out[k - 1] != 0.0, u * np.spacing(np.abs(out[k - 1])) * 0.5, 0.0)
    return out


def random_md(shape, prec, seed: int, stream: int = 0) -> np.ndarray:
    """md array of the given element shape, returned as (m, *shape)."""
    m = limbs(prec)
    g = rng(seed, stream)
    lead = g.uniform(-1.0, 1.0, size=shape)
    return _lower_limbs(lead, m, g)


def random_matrix(rows: int, cols: int, prec, seed: int, stream: int = 1) -> np.ndarray:
    """(m, cols, rows) limb-planar column-major md matrix, entries as random_md."""
    x = random_md((cols, rows), prec, seed, stream)
    return np.ascontiguousarray(x)


def random_vector(n: int, prec, seed: int, stream: int = 2) -> np.ndarray:
    return np.ascontiguousarray(random_md((n,), prec, seed, stream))


def lu_upper(n: int, prec, seed: int, stream: int = 3) -> np.ndarray:
    """(m, n, n) upper-triangular md matrix: U of a partially pivoted LU."""
    import scipy.linalg

    m = limbs(prec)
    g = rng(seed, stream)
    a = g.uniform(-1.0, 1.0, size=(n, n))
    lu, _ = scipy.linalg.lu_factor(a, overwrite_a=True, check_finite=False)
    u = np.triu(lu)
    out = _lower_limbs(u.T.copy(), m, g)  # (m, cols, rows): transpose to column-major planes
    mask = np.tril(np.ones((n, n), dtype=bool), 0)  # mask[col, row] True where row <= col
    out[:, ~mask] = 0.0
    return np.ascontiguousarray(out)


def lstsq_problem(M: int, K: int, prec, seed: int):
    """(A, b): A (m, K, M), b (m, M)."""
    return random_matrix(M, K, prec, seed), random_vector(M, prec, seed)


def to_mp(x: np.ndarray):
    """Exact value of each md element as a python Fraction (for tests)."""
    from fractions import Fraction

    m = x.shape[0]
    flat = x.reshape(m, -1)
    return [sum((Fraction(float(flat[k, i])) for k in range(m)), Fraction(0)) for i in range(flat.shape[1])]


def lu_upper_torch(n: int, prec, seed: int, device="cuda"):
    """Large-n variant of lu_upper generated on the device with torch (seeded
    Philox/cuRAND stream + cuSOLVER LU, fp64): returns a CUDA tensor (m, n, n),
    column-major planes, strict lower part exactly zero.  Lower limbs are
    u * ulp(limb above) / 2 as in random_md (ulp via nextafter: exact)."""
    import torch

    m = limbs(prec)
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    a = torch.rand((n, n), generator=g, dtype=torch.float64, device=device) * 2.0 - 1.0
    lu, _ = torch.linalg.lu_factor(a)
    del a
    u = torch.triu(lu)
    del lu
    out = torch.empty((m, n, n), dtype=torch.float64, device=device)
    out[0] = u.T  # column-major plane: out[0, col, row] = U[row, col]
    del u
    mask = torch.triu(torch.ones((n, n), dtype=torch.bool, device=device)).T  # [col, row]: row <= col
    for k in range(1, m):
        prev = out[k - 1].abs()
        ulp = torch.nextafter(prev, torch.full_like(prev, float("inf"))) - prev
        r = torch.rand((n, n), generator=g, dtype=torch.float64, device=device) * 2.0 - 1.0
        out[k] = torch.where(mask & (out[k - 1] != 0), r * ulp * 0.5, torch.zeros_like(r))
        del prev, ulp, r
    return out


def random_vector_torch(n: int, prec, seed: int, device="cuda"):
    import torch

    m = limbs(prec)
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) + 7919)
    out = torch.empty((m, n), dtype=torch.float64, device=device)
    out[0] = torch.rand(n, generator=g, dtype=torch.float64, device=device) * 2.0 - 1.0
    for k in range(1, m):
        prev = out[k - 1].abs()
        ulp = torch.nextafter(prev, torch.full_like(prev, float("inf"))) - prev
        out[k] = (torch.rand(n, generator=g, dtype=torch.float64, device=device) * 2.0 - 1.0) * ulp * 0.5
    return out


def random_matrix_torch(rows: int, cols: int, prec, seed: int, device="cuda"):
    """Large-size variant of random_matrix generated on the device (seeded torch Philox): (m, cols, rows),
    limb 0 uniform in [-1, 1), limb k = u * ulp(limb k-1) / 2 with u uniform in (-1, 1)."""
    import torch

    m = limbs(prec)
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) + 104729)
    out = torch.empty((m, cols, rows), dtype=torch.float64, device=device)
    out[0] = torch.rand((cols, rows), generator=g, dtype=torch.float64, device=device) * 2.0 - 1.0
    for k in range(1, m):
        prev = out[k - 1].abs()
        ulp = torch.nextafter(prev, torch.full_like(prev, float("inf"))) - prev
        r = torch.rand((cols, rows), generator=g, dtype=torch.float64, device=device) * 2.0 - 1.0
        out[k] = torch.where(out[k - 1] != 0, r * ulp * 0.5, torch.zeros_like(r))
        del prev, ulp, r
    return out
