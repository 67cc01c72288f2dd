"""Pins of the oracle's complex least squares (oracle_zlstsq: complex Householder QR with Hermitian
reflectors; row f2).  The complex path is checked against what the
mathematics fixes, not against itself: exact rational solutions of the complex normal equations
A^H A x = A^H b on Gaussian-integer problems, the reduction to the (separately pinned) real oracle on real
data, and phase equivariance (A -> iA gives x -> -i x; scaling column j by i gives x_j -> -i x_j), which a
missing conjugate or a transposed operand breaks."""
from fractions import Fraction

import numpy as np
import pytest

from paper_2110_08375_b200 import inputs

U = {"dd": 2.0 ** -104, "qd": 2.0 ** -208, "od": 2.0 ** -416}
M_OF = {"dd": 2, "qd": 4, "od": 8}


def _val(x, idx):  # exact value of md element idx of an (m, n) array
    return sum((Fraction(float(x[k, idx])) for k in range(x.shape[0])), Fraction(0))


def _solve_exact(A, b):
    """A: list of rows of (re, im) Fraction pairs (M x K); solve A^H A x = A^H b exactly."""
    M, K = len(A), len(A[0])

    def mul(p, q):
        return (p[0] * q[0] - p[1] * q[1], p[0] * q[1] + p[1] * q[0])

    def conj(p):
        return (p[0], -p[1])

    G = [[(Fraction(0), Fraction(0)) for _ in range(K)] for _ in range(K)]
    h = [(Fraction(0), Fraction(0)) for _ in range(K)]
    for r in range(K):
        for c in range(K):
            s = (Fraction(0), Fraction(0))
            for i in range(M):
                t = mul(conj(A[i][r]), A[i][c])
                s = (s[0] + t[0], s[1] + t[1])
            G[r][c] = s
        s = (Fraction(0), Fraction(0))
        for i in range(M):
            t = mul(conj(A[i][r]), b[i])
            s = (s[0] + t[0], s[1] + t[1])
        h[r] = s
    # Gaussian elimination (Hermitian positive definite: no pivoting needed)
    for p in range(K):
        d = G[p][p]
        dd = d[0] * d[0] + d[1] * d[1]
        inv = (d[0] / dd, -d[1] / dd)
        for r in range(p + 1, K):
            f = mul(G[r][p], inv)
            for c in range(p, K):
                t = mul(f, G[p][c])
                G[r][c] = (G[r][c][0] - t[0], G[r][c][1] - t[1])
            t = mul(f, h[p])
            h[r] = (h[r][0] - t[0], h[r][1] - t[1])
    x = [None] * K
    for r in range(K - 1, -1, -1):
        s = h[r]
        for c in range(r + 1, K):
            t = mul(G[r][c], x[c])
            s = (s[0] - t[0], s[1] - t[1])
        d = G[r][r]
        dd = d[0] * d[0] + d[1] * d[1]
        x[r] = mul(s, (d[0] / dd, -d[1] / dd))
    return x


@pytest.mark.parametrize("prec", ["dd", "qd", "od"])
@pytest.mark.parametrize("M,K,seed", [(5, 3, 1), (7, 4, 2), (6, 6, 3)])
def test_exact_normal_equations(orc, prec, M, K, seed):
    g = np.random.default_rng(seed)
    m = M_OF[prec]
    ar = g.integers(-4, 5, size=(K, M)).astype(float)
    ai = g.integers(-4, 5, size=(K, M)).astype(float)
    br = g.integers(-4, 5, size=M).astype(float)
    bi = g.integers(-4, 5, size=M).astype(float)
    Are, Aim = np.zeros((m, K, M)), np.zeros((m, K, M))
    Are[0], Aim[0] = ar, ai
    bre, bim = np.zeros((m, M)), np.zeros((m, M))
    bre[0], bim[0] = br, bi
    xr, xi, Rr, Ri, info = orc.zlstsq(prec, Are, Aim, bre, bim)
    assert info == 0
    A = [[(Fraction(ar[j, i]), Fraction(ai[j, i])) for j in range(K)] for i in range(M)]
    b = [(Fraction(br[i]), Fraction(bi[i])) for i in range(M)]
    x = _solve_exact(A, b)
    scale = max(max(abs(float(v[0])), abs(float(v[1]))) for v in x)
    for j in range(K):
        for got, ex in ((_val(xr, j), x[j][0]), (_val(xi, j), x[j][1])):
            assert abs(float(got - ex)) <= 1e3 * K * U[prec] * scale, (j, float(got - ex))


@pytest.mark.parametrize("prec", ["dd", "qd"])
def test_real_data_reduces_to_real_oracle(orc, prec):
    A, b = inputs.lstsq_problem(30, 20, prec, seed=9)
    xr, xi, Rr, Ri, info = orc.zlstsq(prec, A, np.zeros_like(A), b, np.zeros_like(b))
    x, _, _ = orc.lstsq(prec, A, b)
    assert info == 0 and np.all(xi == 0.0) and np.all(Ri == 0.0)
    d = orc.md_op("sub", prec, xr, x)
    assert np.max(np.abs(d[0])) <= 1e3 * 20 * U[prec] * np.max(np.abs(x[0]))


@pytest.mark.parametrize("prec", ["dd", "od"])
def test_phase_equivariance_and_triangular_R(orc, prec):
    M, K = 14, 9
    Are, bre = inputs.lstsq_problem(M, K, prec, seed=4)
    Aim, bim = inputs.lstsq_problem(M, K, prec, seed=5)
    xr, xi, Rr, Ri, info = orc.zlstsq(prec, Are, Aim, bre, bim)
    assert info == 0
    tol = 1e3 * K * U[prec] * max(np.max(np.abs(xr[0])), np.max(np.abs(xi[0])))
    # i A x' = b  =>  x' = -i x  (re x' = im x, im x' = -re x): multiplying by i is exact (limb swap / negation)
    yr, yi, _, _, _ = orc.zlstsq(prec, -Aim, Are, bre, bim)
    assert np.max(np.abs(orc.md_op("sub", prec, yr, xi)[0])) <= tol
    assert np.max(np.abs(orc.md_op("add", prec, yi, xr)[0])) <= tol
    # column j scaled by i: x'_j = -i x_j, the others unchanged
    j = 3
    Cr, Ci = Are.copy(), Aim.copy()
    Cr[:, j], Ci[:, j] = -Aim[:, j], Are[:, j]
    zr, zi, _, _, _ = orc.zlstsq(prec, Cr, Ci, bre, bim)
    er, ei = xr.copy(), xi.copy()
    er[:, j], ei[:, j] = xi[:, j], -xr[:, j]
    assert np.max(np.abs(orc.md_op("sub", prec, zr, er)[0])) <= tol
    assert np.max(np.abs(orc.md_op("sub", prec, zi, ei)[0])) <= tol
    # R upper triangular, |R_00| = ||A(:, 0)||
    for c in range(K):
        assert np.all(Rr[:, c, c + 1:] == 0.0) and np.all(Ri[:, c, c + 1:] == 0.0)
    n0 = np.sqrt(np.sum(Are[0, 0] ** 2 + Aim[0, 0] ** 2))
    assert abs(np.hypot(Rr[0, 0, 0], Ri[0, 0, 0]) - n0) <= 1e-14 * n0
