"""f1: the least-squares residual ||b - A x||_2 from the trailing entries of
Q^T b (Q orthogonal).  Oracle pins: the md 2-norm on exact cases, and the
tail norm ||(Q^T b)(K+1:M)|| against a direct md evaluation of ||b - A x|| -- equal in exact
arithmetic, and to second order in the solution error because A^T r = 0 at the minimiser."""
import mpmath
import numpy as np
import pytest

from paper_2110_08375_b200 import inputs

from ._parity import U_OF

M_OF = {"d": 1, "dd": 2, "qd": 4, "od": 8}


@pytest.mark.parametrize("prec", ["d", "dd", "qd", "od"])
def test_norm2_exact_cases(orc, prec):
    m = M_OF[prec]
    y = np.zeros((m, 2))
    y[0] = [3.0, 4.0]
    out = orc.norm2(prec, y)
    mpmath.mp.prec = 2000
    assert out[0] == 5.0 and abs(sum(mpmath.mpf(float(v)) for v in out) - 5) <= mpmath.mpf(2) ** (-53 * m + 4) * 5
    y[0] = [1.0, 1.0]
    out = orc.norm2(prec, y)
    exact = mpmath.sqrt(2)
    got = sum(mpmath.mpf(float(v)) for v in out)
    assert abs(got - exact) <= mpmath.mpf(2) ** (-53 * m + 4) * exact
    assert orc.norm2(prec, np.zeros((m, 0)))[0] == 0.0


@pytest.mark.parametrize("prec", ["d", "dd", "qd", "od"])
def test_residual_spec_examples(orc, prec):
    m = M_OF[prec]
    A = np.zeros((m, 1, 2))
    A[0, 0] = [1.0, 0.0]
    b = np.zeros((m, 2))
    b[0] = [0.0, 1.0]  # x = 0, residual 1
    x, R, y = orc.lstsq(prec, A, b)
    assert x[0, 0] == 0.0
    assert orc.norm2(prec, y[:, 1:])[0] == 1.0
    assert orc.residual_direct(prec, A, x, b)[0] == 1.0


@pytest.mark.parametrize("prec", ["d", "dd", "qd", "od"])
@pytest.mark.parametrize("M,K", [(40, 12), (33, 32), (64, 8)])
def test_tail_norm_equals_direct_residual(orc, prec, M, K):
    A, b = inputs.lstsq_problem(M, K, prec, seed=M + K)
    x, R, y = orc.lstsq(prec, A, b)
    tail = orc.norm2(prec, y[:, K:])
    direct = orc.residual_direct(prec, A, x, b)
    d = orc.md_op("sub", prec, tail[:, None], direct[:, None])[0, 0]
    scale = np.max(np.sum(np.abs(A[0]), axis=0)) * np.max(np.abs(x[0])) + np.max(np.abs(b[0]))
    assert tail[0] > 0.1  # random overdetermined systems have an O(1) residual
    assert abs(d) <= 1e3 * M * U_OF[prec] * scale, (d, tail[0])
