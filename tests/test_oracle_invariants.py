"""Known-answer pins of the oracle's invariants (north_star: ||Q^T Q - I||, ||A - QR|| / ||A||
and the normal-equation residual ||A^T (b - A x)||).  The GPU tests evaluate
E1/E2/E3 on GPU outputs with these very functions, so each is pinned here against an exact
rational evaluation (Python Fractions) on inputs whose true value is known: small-integer and
dyadic matrices (every md sum exact), non-symmetric cases that tell Q^T Q from Q Q^T, M != K cases
that tell A^T r from A r, column subsets, and a perturbation below double precision that only an
md (multi-limb) evaluation can see."""
from fractions import Fraction

import numpy as np
import pytest

PRECS = ["d", "dd", "qd", "od"]
PRECS_MD = ["dd", "qd", "od"]
M_OF = {"d": 1, "dd": 2, "qd": 4, "od": 8}


def _md(prec, mat):
    """(cols, rows) float array -> (m, cols, rows) with zero lower limbs"""
    out = np.zeros((M_OF[prec],) + mat.shape)
    out[0] = mat
    return out


def _fr(v):
    return Fraction(float(v))


def e1_exact(Q, cols=None):  # Q: rows x cols numpy (math layout), entries exact doubles
    n = Q.shape[1]
    cols = range(n) if cols is None else cols
    worst = Fraction(0)
    for c in cols:
        for r in range(n):
            s = sum(_fr(Q[i, r]) * _fr(Q[i, c]) for i in range(Q.shape[0])) - (1 if r == c else 0)
            worst = max(worst, abs(s))
    return worst


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("seed", range(3))
def test_inv_orth_integer_exact(orc, prec, seed):
    rng = np.random.default_rng(seed)
    n = 5
    Q = rng.integers(-3, 4, size=(n, n)).astype(float)
    got = orc.inv_orth(prec, _md(prec, Q.T))
    assert got == float(e1_exact(Q))
    cols = [1, 3]
    assert orc.inv_orth(prec, _md(prec, Q.T), cols=cols) == float(e1_exact(Q, cols))


def test_inv_orth_tells_qtq_from_qqt(orc):
    # Q = [[1, 0], [a, b]]: column 0 of Q^T Q - I is (a^2, a b), of Q Q^T - I is (0, a)
    a, b = 2.0 ** -10, 2.0 ** -5
    Q = np.array([[1.0, 0.0], [a, b]])
    got = orc.inv_orth("dd", _md("dd", Q.T), cols=[0])
    assert got == max(a * a, a * b) == 2.0 ** -15  # Q Q^T would give 2^-10


@pytest.mark.parametrize("prec", PRECS_MD)  # needs > 53 bits: multi-limb only
def test_inv_orth_hadamard_dyadic_perturbation(orc, prec):
    H = np.array([[1, 1, 1, 1], [1, -1, 1, -1], [1, 1, -1, -1], [1, -1, -1, 1]], dtype=float) / 2
    assert orc.inv_orth(prec, _md(prec, H.T)) == 0.0
    d = 2.0 ** -30
    Hp = H.copy()
    Hp[0, 0] += d  # (Q^T Q - I)_00 = 2 (1/2) d + d^2 = d + d^2 (exact double: 30 bits apart)
    assert orc.inv_orth(prec, _md(prec, Hp.T)) == d + d * d


@pytest.mark.parametrize("prec", PRECS_MD)  # needs > 53 bits: multi-limb only
def test_inv_orth_sub_double_perturbation(orc, prec):
    """Q = I + eps E with eps = 2^-70 held in the second limb: Q^T Q - I = eps (E + E^T) + eps^2 E^T E
    is invisible to plain doubles (1 + 2^-70 rounds to 1) and is recovered only in md arithmetic."""
    n = 3
    E = np.array([[5, 1, 0], [-1, 4, 1], [0, 1, 6]], dtype=float)  # diagonal in the 2nd limb
    eps = 2.0 ** -70
    Q = np.zeros((M_OF[prec], n, n))
    for r in range(n):
        Q[0, r, r] = 1.0
        for c in range(n):
            if E[r, c] != 0.0:
                Q[0 if r != c else 1, c, r] += E[r, c] * eps
    exact = Fraction(0)
    eF = Fraction(1, 2 ** 70)
    for c in range(n):
        for r in range(n):
            s = eF * (int(E[c, r]) + int(E[r, c])) + eF * eF * sum(int(E[i, r]) * int(E[i, c]) for i in range(n))
            exact = max(exact, abs(s))
    got = orc.inv_orth(prec, Q)
    assert got > 10 * eps  # the diagonal 2 eps E_rr dominates; a leading-limb evaluation sees only 2 eps
    rel = {"dd": 2.0 ** -30, "qd": 2.0 ** -52, "od": 2.0 ** -52}[prec]
    assert abs(got - float(exact)) <= rel * float(exact), (got, float(exact))


def e2_exact(A, Q, R, cols=None):
    M, K = A.shape
    cols = range(K) if cols is None else cols
    worst = Fraction(0)
    for c in cols:
        for i in range(M):
            s = _fr(A[i, c]) - sum(_fr(Q[i, l]) * _fr(R[l, c]) for l in range(c + 1))
            worst = max(worst, abs(s))
    amax = max(abs(_fr(v)) for v in A.ravel())
    return worst / amax


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("M,K", [(6, 4), (5, 5)])
def test_inv_recon_integer_exact(orc, prec, M, K):
    rng = np.random.default_rng(M * 10 + K)
    A = rng.integers(-4, 5, size=(M, K)).astype(float)
    Q = rng.integers(-2, 3, size=(M, M)).astype(float)
    R = np.triu(rng.integers(-3, 4, size=(M, K))).astype(float)
    got = orc.inv_recon(prec, _md(prec, A.T), _md(prec, Q.T), _md(prec, R.T))
    assert got == float(e2_exact(A, Q, R))
    assert orc.inv_recon(prec, _md(prec, A.T), _md(prec, Q.T), _md(prec, R.T), cols=[K - 1]) == \
        float(e2_exact(A, Q, R, [K - 1]))


def test_inv_recon_factorisation_is_zero_and_perturbation_exact(orc):
    # A = Q R exactly (Hadamard/2 times an integer upper triangle) -> 0; perturb R(1,2) by 2^-40
    H = np.array([[1, 1, 1, 1], [1, -1, 1, -1], [1, 1, -1, -1], [1, -1, -1, 1]], dtype=float) / 2
    R = np.triu(np.arange(1, 17, dtype=float).reshape(4, 4))
    A = H @ R
    assert orc.inv_recon("qd", _md("qd", A.T), _md("qd", H.T), _md("qd", R.T)) == 0.0
    Rp = R.copy()
    Rp[1, 2] += 2.0 ** -40
    expect = (2.0 ** -40) * 0.5 / np.max(np.abs(A))  # |Q(i,1)| = 1/2 for every i
    assert orc.inv_recon("qd", _md("qd", A.T), _md("qd", H.T), _md("qd", Rp.T)) == expect


def e3_exact(A, x, b):
    M, K = A.shape
    r = [_fr(b[i]) - sum(_fr(A[i, j]) * _fr(x[j]) for j in range(K)) for i in range(M)]
    atr = [sum(_fr(A[i, j]) * r[i] for i in range(M)) for j in range(K)]
    anorm = max(sum(abs(_fr(A[i, j])) for j in range(K)) for i in range(M))
    den = anorm * (anorm * max(abs(_fr(v)) for v in x) + max(abs(_fr(v)) for v in b))
    return max(abs(v) for v in atr) / den


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("M,K", [(7, 3), (4, 4), (9, 5)])
def test_inv_normal_integer_exact(orc, prec, M, K):
    rng = np.random.default_rng(M + 100 * K)
    A = rng.integers(-3, 4, size=(M, K)).astype(float)
    x = rng.integers(-5, 6, size=K).astype(float)
    b = rng.integers(-9, 10, size=M).astype(float)
    xm = np.zeros((M_OF[prec], K))
    xm[0] = x
    bm = np.zeros((M_OF[prec], M))
    bm[0] = b
    got = orc.inv_normal(prec, _md(prec, A.T), xm, bm)
    assert got == float(e3_exact(A, x, b))


def test_inv_normal_exact_solution_is_zero(orc):
    # x solves the normal equations exactly when b = A x: residual 0
    A = np.array([[1.0, 2.0], [3.0, -1.0], [0.5, 4.0]])
    x = np.array([0.25, -1.5])
    b = A @ x
    xm = np.zeros((2, 2))
    xm[0] = x
    bm = np.zeros((2, 3))
    bm[0] = b
    assert orc.inv_normal("dd", _md("dd", A.T), xm, bm) == 0.0
