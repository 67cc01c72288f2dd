"""Pin the oracle's error-free transformations and md arithmetic.

* two_sum / quick_two_sum / two_prod / split: exact rational arithmetic
  (fractions.Fraction of the doubles) -- s + e = a + b and p + e = a*b exactly;
  SPEC S:46-57 worked examples.
* md add/sub/mul/div/sqrt: mpmath at 2000 bits, relative error
  <= 2^(-53 m + 4) over random operands spanning exponents (SPEC S:89 target).
* special cases: x - x = 0, x * 1 = x, (2,0,0,0)*(3,0,0,0) = 6;
  renormalisation examples.
"""
from fractions import Fraction

import mpmath
import numpy as np
import pytest

from paper_2110_08375_b200 import inputs

mpmath.mp.prec = 2000


def F(x):
    return Fraction(float(x))


def test_two_sum_examples(orc):
    assert orc.two_sum(1.0, 2.0 ** -60) == (1.0, 2.0 ** -60)
    assert orc.two_sum(1.0, 2.0) == (3.0, 0.0)
    assert orc.two_sum(2.0 ** 53, 1.0) == (2.0 ** 53, 1.0)  # round-to-nearest-even


def test_two_prod_examples(orc):
    assert orc.two_prod(2.0, 3.0) == (6.0, 0.0)
    u = 1.0 + 2.0 ** -52
    assert orc.two_prod(u, u) == (1.0 + 2.0 ** -51, 2.0 ** -104)


def test_efts_exact_random(orc):
    rng = np.random.default_rng(7)
    a = rng.uniform(-1, 1, 3000) * 2.0 ** rng.integers(-40, 40, 3000)
    b = rng.uniform(-1, 1, 3000) * 2.0 ** rng.integers(-40, 40, 3000)
    for x, y in zip(a, b):
        s, e = orc.two_sum(x, y)
        assert F(s) + F(e) == F(x) + F(y) and s == x + y
        p, e = orc.two_prod(x, y)
        assert F(p) + F(e) == F(x) * F(y) and p == x * y
        assert e == float(F(x) * F(y) - F(p))  # == fma(x, y, -p): the GPU's FMA two_prod agrees bitwise
        hi, lo = orc.split(x)
        assert F(hi) + F(lo) == F(x)
        assert abs(hi) == 0.0 or np.frexp(hi)[0] * 2 ** 27 == int(np.frexp(hi)[0] * 2 ** 27)  # hi has <= 27 bits
        big, small = (x, y) if abs(x) >= abs(y) else (y, x)
        s, e = orc.quick_two_sum(big, small)
        assert F(s) + F(e) == F(x) + F(y)


def _val(col):
    return sum(mpmath.mpf(float(v)) for v in col)


@pytest.mark.parametrize("prec", ["dd", "qd", "od"])
@pytest.mark.parametrize("op", ["add", "sub", "mul", "div", "sqrt"])
def test_md_ops_vs_mpmath(orc, prec, op):
    m = inputs.limbs(prec)
    n = 300
    a = inputs.random_md((n,), prec, 101)
    b = inputs.random_md((n,), prec, 202)
    a = a * 2.0 ** np.random.default_rng(1).integers(-30, 30, size=n)  # exact rescaling of all limbs
    if op == "sqrt":
        a = np.where(a[0] < 0, -a, a)  # negate whole expansions: positive, still valid
    c = orc.md_op(op, prec, a, None if op == "sqrt" else b)
    bound = mpmath.mpf(2) ** (-53 * m + 4)
    for i in range(n):
        x, y, z = _val(a[:, i]), _val(b[:, i]), _val(c[:, i])
        exact = {"add": x + y, "sub": x - y, "mul": x * y, "div": x / y, "sqrt": mpmath.sqrt(x)}[op]
        scale = abs(x) + abs(y) if op in ("add", "sub") else abs(exact)
        assert abs(z - exact) <= bound * scale, (prec, op, i)


@pytest.mark.parametrize("prec", ["dd", "qd", "od"])
def test_md_special_cases(orc, prec):
    m = inputs.limbs(prec)
    x = inputs.random_md((50,), prec, 5)
    assert np.all(orc.md_op("sub", prec, x, x) == 0.0)
    one = np.zeros_like(x)
    one[0] = 1.0
    assert np.array_equal(orc.md_op("mul", prec, x, one), x)
    assert np.array_equal(orc.md_op("div", prec, x, one), x)
    two, three = np.zeros((m, 1)), np.zeros((m, 1))
    two[0], three[0] = 2.0, 3.0
    six = orc.md_op("mul", prec, two, three)
    assert six[0, 0] == 6.0 and np.all(six[1:] == 0.0)
    four = np.zeros((m, 1))
    four[0] = 4.0
    r = orc.md_op("sqrt", prec, four)
    assert r[0, 0] == 2.0 and np.all(r[1:] == 0.0)
    zero = np.zeros((m, 1))
    assert np.all(orc.md_op("sqrt", prec, zero) == 0.0)


@pytest.mark.parametrize("prec", ["dd", "qd", "od"])
def test_md_results_nonoverlapping(orc, prec):
    """Outputs are valid expansions: |limb k+1| <= ulp(limb k)/2."""
    m = inputs.limbs(prec)
    a = inputs.random_md((400,), prec, 9)
    b = inputs.random_md((400,), prec, 10)
    for op in ("add", "mul", "div"):
        c = orc.md_op(op, prec, a, b)
        for k in range(m - 1):
            nz = c[k] != 0
            assert np.all(np.abs(c[k + 1][nz]) <= np.spacing(np.abs(c[k][nz])) / 2 * (1 + 1e-15))


def test_renorm_examples(orc):
    assert list(orc.renorm("dd", np.array([1.0, 1.0, 0.0]))) == [2.0, 0.0]
    assert list(orc.renorm("qd", np.array([1.0, 2.0 ** -60, 0.0, 0.0, 0.0]))) == [1.0, 2.0 ** -60, 0.0, 0.0]
    # exact value preserved when the terms fit in m limbs
    f = np.array([1.0, 2.0 ** -30, 2.0 ** -60, 2.0 ** -200, 0.0])
    r = orc.renorm("qd", f)
    assert sum(F(v) for v in r) == sum(F(v) for v in f)
