"""Pins of the oracle's plain double ("1d") rows (the paper's double precision
version).

With m = 1 the oracle's md operations are single IEEE 754 operations, so:
* add/sub/mul/div/sqrt equal numpy's (IEEE, round to nearest) bit for bit;
* its Householder QR, Q^T b and back substitution are the textbook algorithms in double, so x agrees
  with LAPACK's least-squares solution (numpy.linalg.lstsq, a different algorithm: SVD-based gelsd)
  and R with LAPACK's QR (dgeqrf, made unique by a positive diagonal) within the backward-stable
  bound c * kappa * n * u, u = 2^-53;
* back substitution agrees with scipy's triangular solve (dtrtrs) to the forward-error bound.
The md-generic pins (exact dyadic QR cases, exact rational normal equations, Cholesky of the exact
A^T A, invariants E1/E2/E3) also run on m = 1 in tests/test_oracle_linalg.py and
tests/test_oracle_invariants.py.
"""
import numpy as np
import pytest
import scipy.linalg

from paper_2110_08375_b200 import inputs

U = 2.0 ** -53


def test_ops_are_ieee(orc):
    g = np.random.default_rng(5)
    a = g.standard_normal((1, 4000)) * np.exp2(g.integers(-40, 40, (1, 4000)))
    b = g.standard_normal((1, 4000)) * np.exp2(g.integers(-40, 40, (1, 4000)))
    for op, f in (("add", np.add), ("sub", np.subtract), ("mul", np.multiply), ("div", np.divide)):
        assert np.array_equal(orc.md_op(op, "d", a, b)[0], f(a[0], b[0])), op
    assert np.array_equal(orc.md_op("sqrt", "d", np.abs(a))[0], np.sqrt(np.abs(a[0])))


@pytest.mark.parametrize("M,K", [(64, 64), (200, 128), (300, 17)])
def test_lstsq_vs_lapack(orc, M, K):
    A, b = inputs.lstsq_problem(M, K, "d", seed=M + K)
    x, R, y = orc.lstsq("d", A, b)
    An, bn = A[0].T, b[0]
    kappa = np.linalg.cond(An)
    xl = np.linalg.lstsq(An, bn, rcond=None)[0]
    assert np.max(np.abs(x[0] - xl)) <= 10 * kappa * K * U * np.max(np.abs(xl))
    # R: LAPACK's R with its rows signed so that diag(R) > 0 is the same unique factor
    Rl = np.linalg.qr(An, mode="r")
    Rl = np.sign(np.diag(Rl))[:, None] * Rl
    Ro = np.triu(R[0].T[:K, :K])
    assert np.max(np.abs(Ro - Rl)) <= 10 * K * U * kappa * np.max(np.abs(Rl))
    # the residual tail: ||(Q^T b)_{K+1:M}|| = ||b - A x||
    if M > K:
        r = np.linalg.norm(bn - An @ xl)
        assert abs(np.linalg.norm(y[0, K:]) - r) <= 10 * kappa * M * U * np.linalg.norm(bn)


@pytest.mark.parametrize("n", [8, 96, 250])
def test_backsub_vs_lapack(orc, n):
    U_ = inputs.lu_upper(n, "d", seed=n)
    y = inputs.random_vector(n, "d", seed=n + 1)
    x, info = orc.backsub("d", U_, y)
    assert info == 0
    Un = U_[0].T
    xl = scipy.linalg.solve_triangular(Un, y[0], lower=False)
    kappa = np.linalg.cond(Un)
    assert np.max(np.abs(x[0] - xl)) <= 10 * n * U * kappa * np.max(np.abs(xl))
