"""Pin the oracle's Householder QR, Q, Q^T b, back substitution and least squares.

Pins (none re-types the oracle's own formulas):
* house (GVL Alg. 5.1.1): exact dyadic cases x=(0,1), x=(1,1,1,1),
  rounded case x=(3,4) -> v=(1,-2), beta=0.4, Px=(5,0) (reading Z1).
* QR special cases with all-dyadic intermediates: A=I, A=positive diagonal,
  A = Sylvester Hadamard H4 -> R = 2I, Q = H4/2 exactly.
* R is the unique upper-triangular factor with positive diagonal, so R^T R =
  A^T A: R is compared with the Cholesky factor of the EXACT A^T A (fractions),
  taken in mpmath at 2000 bits; for square A, Q = A R^-1 likewise.
* x is compared with the exact rational solution of the normal equations
  A^T A x = A^T b (fraction-free); SPEC's K=1 examples.
* back substitution: U = I gives x = b limb for limb; unit upper-triangular
  integer U with integer b gives the integer x exactly; [[2,1],[0,4]]^-1 column
  solves; exact rational solves for random md U.
* invariants E1/E2/E3 <= 1e3 * M * u (north_star).
"""
from fractions import Fraction

import mpmath
import numpy as np
import pytest

from paper_2110_08375_b200 import inputs

mpmath.mp.prec = 2000
U_OF = {"d": 2.0 ** -53, "dd": 2.0 ** -104, "qd": 2.0 ** -208, "od": 2.0 ** -416}
PRECS = ["d", "dd", "qd", "od"]


def md_from(mat2d, m):
    """plain double matrix (rows, cols) -> (m, cols, rows) md with zero lower limbs."""
    a = np.zeros((m,) + mat2d.T.shape)
    a[0] = mat2d.T
    return np.ascontiguousarray(a)


def exact(x):
    """(m, ...) md -> nested object array of Fractions over the element shape."""
    m = x.shape[0]
    out = np.empty(x.shape[1:], dtype=object)
    for idx in np.ndindex(*x.shape[1:]):
        out[idx] = sum((Fraction(float(x[(k,) + idx])) for k in range(m)), Fraction(0))
    return out


def mpf_of(frac):
    return mpmath.mpf(frac.numerator) / frac.denominator


@pytest.mark.parametrize("prec", PRECS)
def test_house_exact_cases(orc, prec):
    m = inputs.limbs(prec)
    def vec(vals):
        x = np.zeros((m, len(vals)))
        x[0] = vals
        return x
    v, beta, mu = orc.house(prec, vec([0.0, 1.0]))
    assert list(v[0]) == [1.0, -1.0] and beta[0] == 1.0 and mu[0] == 1.0
    v, beta, mu = orc.house(prec, vec([1.0, 1.0, 1.0, 1.0]))
    assert list(v[0]) == [1.0, -1.0, -1.0, -1.0] and beta[0] == 0.5 and mu[0] == 2.0
    assert np.all(v[1:] == 0) and np.all(beta[1:] == 0) and np.all(mu[1:] == 0)
    v, beta, mu = orc.house(prec, vec([3.0, 4.0]))
    u = U_OF[prec]
    assert v[0, 0] == 1.0 and abs(sum(v[:, 1]) + 2.0) <= 4 * u
    assert abs(sum(beta) - 0.4) <= 4 * u and abs(sum(mu) - 5.0) <= 8 * u
    # degenerate column (sigma = 0): beta = 0, P = I, R_jj = x1 (reading Z2)
    v, beta, mu = orc.house(prec, vec([-2.0, 0.0, 0.0]))
    assert np.all(beta == 0) and mu[0] == -2.0 and list(v[0]) == [1.0, 0.0, 0.0]


@pytest.mark.parametrize("prec", PRECS)
def test_qr_identity_diagonal_hadamard(orc, prec):
    m = inputs.limbs(prec)
    for A2 in (np.eye(6), np.diag([3.0, 0.5, 2.0, 7.0])):
        F, beta = orc.qr(prec, md_from(A2, m))
        R = orc.r_of(F)
        Q = orc.form_q(prec, F, beta)
        assert np.array_equal(R[0], A2.T) and np.all(R[1:] == 0)
        assert np.array_equal(Q[0], np.eye(A2.shape[0])) and np.all(Q[1:] == 0)
        assert np.all(beta == 0)
    H = np.array([[1, 1, 1, 1], [1, -1, 1, -1], [1, 1, -1, -1], [1, -1, -1, 1]], dtype=float)
    F, beta = orc.qr(prec, md_from(H, m))
    R = orc.r_of(F)
    Q = orc.form_q(prec, F, beta)
    assert np.array_equal(R[0], 2 * np.eye(4)) and np.all(R[1:] == 0)
    assert np.array_equal(Q[0], (H / 2).T) and np.all(Q[1:] == 0)


def _chol_exact(A):
    """Upper Cholesky factor of the exact A^T A, in mpmath (2000 bits)."""
    Ae = exact(A)  # (K, M) object array: Ae[j, i] = A(i, j)
    K, M = Ae.shape
    G = mpmath.matrix(K, K)
    for p in range(K):
        for q in range(K):
            G[p, q] = mpf_of(sum((Ae[p, i] * Ae[q, i] for i in range(M)), Fraction(0)))
    L = mpmath.cholesky(G)
    return L.T, Ae


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("M,K", [(8, 8), (12, 7)])
def test_qr_matches_cholesky_of_normal_matrix(orc, prec, M, K):
    A = inputs.random_matrix(M, K, prec, seed=M * 100 + K)
    F, beta = orc.qr(prec, A)
    R = orc.r_of(F)
    Rx, Ae = _chol_exact(A)
    Re = exact(R)
    tol = mpmath.mpf(1e3 * M) * mpmath.mpf(U_OF[prec])
    scale = max(abs(mpf_of(Re[j, i])) for j in range(K) for i in range(M))
    for j in range(K):
        for i in range(M):
            if i <= j:
                assert abs(mpf_of(Re[j, i]) - Rx[i, j]) <= tol * scale, (i, j)
            else:
                assert Re[j, i] == 0
    if M == K:  # Q = A R^-1 is unique as well
        Q = orc.form_q(prec, F, beta)
        Qe = exact(Q)
        Amp = mpmath.matrix([[mpf_of(Ae[j, i]) for j in range(K)] for i in range(M)])
        Qx = Amp * mpmath.inverse(Rx)
        for j in range(K):
            for i in range(M):
                assert abs(mpf_of(Qe[j, i]) - Qx[i, j]) <= tol, (i, j)


@pytest.mark.parametrize("prec", PRECS)
def test_qr_invariants(orc, prec):
    M, K = 48, 32
    A = inputs.random_matrix(M, K, prec, seed=3)
    F, beta = orc.qr(prec, A)
    R = orc.r_of(F)
    Q = orc.form_q(prec, F, beta)
    bound = 1e3 * M * U_OF[prec]
    assert orc.inv_orth(prec, Q) <= bound
    assert orc.inv_recon(prec, A, Q, R) <= bound
    assert np.all(np.diag(R[0].T)[:K] > 0)
    # Q^T b by reflectors agrees with the explicit product
    b = inputs.random_vector(M, prec, 3)
    y1 = orc.apply_qt(prec, F, beta, b)
    y2 = orc.qt_b_explicit(prec, Q, b)
    assert np.max(np.abs(y1[0] - y2[0])) <= bound


def _exact_solve_upper(Ue, ye):
    n = len(ye)
    x = [Fraction(0)] * n
    for i in range(n - 1, -1, -1):
        s = ye[i] - sum((Ue[l, i] * x[l] for l in range(i + 1, n)), Fraction(0))
        x[i] = s / Ue[i, i]
    return x


@pytest.mark.parametrize("prec", PRECS)
def test_backsub_exact_cases(orc, prec):
    m = inputs.limbs(prec)
    b = inputs.random_vector(10, prec, 4)
    x, info = orc.backsub(prec, md_from(np.eye(10), m), b)
    assert info == 0 and np.array_equal(x, b)
    rng = np.random.default_rng(5)
    U = np.triu(rng.integers(-3, 4, size=(12, 12)).astype(float), 1) + np.eye(12)
    xi = rng.integers(-5, 6, size=12).astype(float)
    bi = U @ xi
    bb = np.zeros((m, 12))
    bb[0] = bi
    x, info = orc.backsub(prec, md_from(U, m), bb)
    assert np.array_equal(x[0], xi) and np.all(x[1:] == 0)
    # columns of [[2,1],[0,4]]^-1 = [[1/2,-1/8],[0,1/4]]
    T = md_from(np.array([[2.0, 1.0], [0.0, 4.0]]), m)
    for k, col in enumerate(([0.5, 0.0], [-0.125, 0.25])):
        e = np.zeros((m, 2))
        e[0, k] = 1.0
        x, _ = orc.backsub(prec, T, e)
        assert list(x[0]) == col and np.all(x[1:] == 0)
    # zero diagonal reported 1-based
    Z = md_from(np.array([[1.0, 1.0], [0.0, 0.0]]), m)
    _, info = orc.backsub(prec, Z, np.ones((m, 2)))
    assert info == 2


@pytest.mark.parametrize("prec", PRECS)
def test_backsub_vs_exact_rationals(orc, prec):
    n = 12
    U = inputs.lu_upper(n, prec, seed=8)
    y = inputs.random_vector(n, prec, 8)
    x, info = orc.backsub(prec, U, y)
    xe = _exact_solve_upper(exact(U), list(exact(y)))
    xnorm = max(abs(v) for v in xe)
    tol = Fraction(1000 * n) * Fraction(U_OF[prec])
    for i in range(n):
        got = sum((Fraction(float(x[k, i])) for k in range(x.shape[0])), Fraction(0))
        assert abs(got - xe[i]) <= tol * xnorm, i


def _exact_lstsq(A, b):
    Ae = exact(A)  # (K, M)
    be = exact(b)
    K, M = Ae.shape
    G = [[sum((Ae[p, i] * Ae[q, i] for i in range(M)), Fraction(0)) for q in range(K)] for p in range(K)]
    r = [sum((Ae[p, i] * be[i] for i in range(M)), Fraction(0)) for p in range(K)]
    # Gaussian elimination over the rationals (exact)
    for c in range(K):
        piv = next(i for i in range(c, K) if G[i][c] != 0)
        G[c], G[piv], r[c], r[piv] = G[piv], G[c], r[piv], r[c]
        for i in range(c + 1, K):
            f = G[i][c] / G[c][c]
            for j in range(c, K):
                G[i][j] -= f * G[c][j]
            r[i] -= f * r[c]
    x = [Fraction(0)] * K
    for i in range(K - 1, -1, -1):
        x[i] = (r[i] - sum((G[i][j] * x[j] for j in range(i + 1, K)), Fraction(0))) / G[i][i]
    return x


@pytest.mark.parametrize("prec", PRECS)
def test_lstsq_spec_examples(orc, prec):
    m = inputs.limbs(prec)
    A = md_from(np.array([[1.0], [1.0]]), m)
    b = np.zeros((m, 2))
    b[0] = [0.0, 2.0]
    x, R, y = orc.lstsq(prec, A, b)
    assert abs(sum(x[:, 0]) - 1.0) <= 4 * U_OF[prec]
    A = md_from(np.array([[1.0], [0.0]]), m)
    b = np.zeros((m, 2))
    b[0] = [0.0, 1.0]
    x, R, y = orc.lstsq(prec, A, b)
    assert np.all(x == 0.0)
    assert abs(abs(y[0, 1]) - 1.0) == 0.0  # the residual norm |(Q^T b)_2| = 1


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("M,K,integer", [(8, 4, True), (12, 6, False), (10, 10, False)])
def test_lstsq_vs_exact_normal_equations(orc, prec, M, K, integer):
    m = inputs.limbs(prec)
    if integer:
        rng = np.random.default_rng(M + K)
        A = md_from(rng.integers(-9, 10, size=(M, K)).astype(float), m)
        b = np.zeros((m, M))
        b[0] = rng.integers(-9, 10, size=M)
    else:
        A, b = inputs.lstsq_problem(M, K, prec, seed=M * K)
    x, R, y = orc.lstsq(prec, A, b)
    xe = _exact_lstsq(A, b)
    xnorm = max(abs(v) for v in xe)
    tol = Fraction(1000 * K) * Fraction(U_OF[prec])
    for i in range(K):
        got = sum((Fraction(float(x[k, i])) for k in range(m)), Fraction(0))
        assert abs(got - xe[i]) <= tol * xnorm, i
    assert orc.inv_normal(prec, A, x, b) <= 1e3 * M * U_OF[prec]


@pytest.mark.parametrize("prec", PRECS)
def test_dot_exact_rationals(orc, prec):
    a = inputs.random_md((40,), prec, 21)
    b = inputs.random_md((40,), prec, 22)
    got = sum(Fraction(float(v)) for v in orc.dot(prec, a, b))
    ea, eb = exact(a), exact(b)
    ref = sum((ea[i] * eb[i] for i in range(40)), Fraction(0))
    scale = sum((abs(ea[i] * eb[i]) for i in range(40)), Fraction(0))
    assert abs(got - ref) <= Fraction(1000 * 40) * Fraction(U_OF[prec]) * scale
