"""Parity helpers: compare GPU md results with the oracle's (tests only).

Tolerance (north_star): componentwise, scaled by the
column (or vector) max norm of the oracle result:
    |R_gpu - R_orc|_ij <= 1e3 * n * u * max_i |R_orc(i, j)|
    |x_gpu - x_orc|_i  <= 1e3 * n * u * max_i |x_orc(i)|
with u = 2^-53 (d, plain double), 2^-104 (dd), 2^-208 (qd), 2^-416 (od) and n the number of columns.
Differences are taken in md arithmetic (oracle md sub), leading limb.
"""
from __future__ import annotations

import numpy as np

U_OF = {"d": 2.0 ** -53, "dd": 2.0 ** -104, "qd": 2.0 ** -208, "od": 2.0 ** -416}


def md_diff(orc, prec, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """|a - b| (leading limb of the md difference), element shape of a."""
    m = a.shape[0]
    shape = a.shape[1:]
    d = orc.md_op("sub", prec, a.reshape(m, -1), b.reshape(m, -1))
    return np.abs(d[0]).reshape(shape)


def vec_ok(orc, prec, got, ref, n, factor=1e3):
    err = md_diff(orc, prec, got, ref)
    scale = float(np.max(np.abs(ref[0])))
    tol = factor * n * U_OF[prec] * scale
    return float(np.max(err)), tol


def mat_cols_ok(orc, prec, got, ref, n, factor=1e3):
    """got/ref: (m, cols, rows).  Returns (worst ratio err/tol over columns)."""
    err = md_diff(orc, prec, got, ref)  # (cols, rows)
    colmax = np.max(np.abs(ref[0]), axis=1)  # (cols,)
    tol = factor * n * U_OF[prec] * np.maximum(colmax, np.finfo(float).tiny)
    ratio = np.max(err, axis=1) / tol
    return float(np.max(ratio))
