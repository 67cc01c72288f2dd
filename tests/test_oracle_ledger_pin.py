"""A10 ledger pin: the canonical md-operation counts of ``mdls_count_<p>`` (the numbers the
headline metric is computed from) equal, integer for integer and stage by stage, the md
operations the oracle's blocked pipelines actually execute (``oracle.blocked``: Algorithm 2,
P:525-565, and Algorithm 1, step by step, every md add/mul/div/sqrt counted) --
the paper's per-kernel accumulation of operation counts.

Also pins the blocked oracle to the unblocked one: blocked Householder QR and tiled back
substitution reach the same R, Q and x in exact arithmetic, so the two
oracle paths must agree to the parity tolerance."""
import numpy as np
import pytest

import paper_2110_08375_b200 as mdls
from paper_2110_08375_b200 import inputs

from ._parity import U_OF, mat_cols_ok, vec_ok

OP = {"qr": 0, "backsub": 1, "lstsq": 2, "apply_qt": 3, "lstsq_noq": 4}
SHAPES = [(12, 8, 4), (10, 6, 2), (9, 9, 3), (16, 8, 8), (7, 4, 1), (20, 12, 4)]


def _upper(K, prec, seed):
    U = inputs.random_matrix(K, K, prec, seed=seed)
    for j in range(K):
        U[:, j, j + 1:] = 0.0
        U[0, j, j] += 3.0
    return U


def _assert_counts_equal(orc_counts, led, nonpos=0):
    for stage, c in orc_counts.items():
        s = led["stages"][stage]
        for k in ("add", "mul", "sqrt"):
            assert c[k] == s[k], (stage, k, c[k], s[k])
        # the ledger prices GVL's x1 > 0 branch: one division per column more than x1 <= 0
        assert c["div"] + (nonpos if stage == "house" else 0) == s["div"], (stage, c["div"], s["div"], nonpos)


@pytest.mark.parametrize("prec", ["d", "dd", "qd"])
@pytest.mark.parametrize("M,K,nb", SHAPES)
@pytest.mark.parametrize("op", ["qr", "lstsq", "lstsq_noq", "apply_qt"])
def test_ledger_equals_executed_counts(orc, prec, M, K, nb, op):
    A = inputs.random_matrix(M, K, prec, seed=M * K + nb)
    b = inputs.random_vector(M, prec, seed=nb)
    r = orc.blocked(op, prec, A, b, nb)
    _assert_counts_equal(r["counts"], mdls.counts(prec, OP[op], M, K, nb), nonpos=0 if op == "apply_qt" else r["nonpos"])


@pytest.mark.parametrize("M,K,nb", [(7, 4, 1), (12, 6, 3), (9, 5, 5)])
def test_ledger_exact_when_every_pivot_positive(orc, M, K, nb):
    """the ledger prices GVL's x1 > 0 branch for every column; on inputs where every column takes it,
    the executed counts equal the ledger with no correction at all"""
    for seed in range(2000):
        A = inputs.random_matrix(M, K, "dd", seed=seed)
        b = inputs.random_vector(M, "dd", seed=seed)
        r = orc.blocked("lstsq", "dd", A, b, nb)
        if r["nonpos"] == 0:
            break
    assert r["nonpos"] == 0, "no all-positive-pivot seed found"
    _assert_counts_equal(r["counts"], mdls.counts("dd", OP["lstsq"], M, K, nb))


@pytest.mark.parametrize("prec", ["dd", "od"])
@pytest.mark.parametrize("K,nb", [(8, 4), (12, 3), (16, 16), (5, 1), (24, 8)])
def test_ledger_backsub_counts(orc, prec, K, nb):
    U = _upper(K, prec, seed=K + nb)
    y = inputs.random_vector(K, prec, seed=3)
    r = orc.blocked("backsub", prec, U, y, nb)
    assert r["info"] == 0
    _assert_counts_equal(r["counts"], mdls.counts(prec, OP["backsub"], K, K, nb))


@pytest.mark.parametrize("M,K,nb", [(14, 10, 5), (9, 9, 3)])
def test_ledger_generic_inputs_branch_accounting(orc, M, K, nb):
    """uniform inputs take both branches of GVL's v1; the counts still agree once the x1 <= 0
    columns (one division fewer each) are accounted for"""
    A = inputs.random_matrix(M, K, "dd", seed=7)
    b = inputs.random_vector(M, "dd", seed=8)
    r = orc.blocked("lstsq", "dd", A, b, nb)
    assert r["nonpos"] > 0
    _assert_counts_equal(r["counts"], mdls.counts("dd", OP["lstsq"], M, K, nb), nonpos=r["nonpos"])


@pytest.mark.parametrize("prec", ["dd", "qd", "od"])
@pytest.mark.parametrize("M,K,nb", [(24, 16, 4), (17, 12, 6), (32, 32, 8)])
def test_blocked_oracle_matches_unblocked(orc, prec, M, K, nb):
    A, b = inputs.lstsq_problem(M, K, prec, seed=M + nb)
    rb = orc.blocked("lstsq", prec, A, b, nb)
    x, R, y = orc.lstsq(prec, A, b)
    err, tol = vec_ok(orc, prec, rb["x"], x, K)
    assert err <= tol, (err, tol)
    assert mat_cols_ok(orc, prec, rb["R"], R, K) <= 1.0
    Fo, beta = orc.qr(prec, A)
    Qo = orc.form_q(prec, Fo, beta)
    assert mat_cols_ok(orc, prec, np.ascontiguousarray(rb["Q"][:, :K]), np.ascontiguousarray(Qo[:, :K]), K) <= 1.0
    # Q^T b: explicit product (LSTSQ) and panel application (LSTSQ_NOQ) vs the reflectors
    rn = orc.blocked("lstsq_noq", prec, A, b, nb)
    for yy in (rb["y"], rn["y"]):
        e, t = vec_ok(orc, prec, np.ascontiguousarray(yy[:, :K]), np.ascontiguousarray(y[:, :K]), K)
        assert e <= t
    e, t = vec_ok(orc, prec, rn["x"], x, K)
    assert e <= t


def test_blocked_backsub_exact_integer_case(orc):
    """unit upper-triangular integer U with integer b: every tile inverse and x are integers, so the
    tiled solve is exact (SURVEY 8(c) BS pin) -- x equals the exact rational solution"""
    from fractions import Fraction

    K, nb = 12, 4
    rng = np.random.default_rng(5)
    Ui = np.triu(rng.integers(-2, 3, size=(K, K)), 1) + np.eye(K, dtype=np.int64)
    bi = rng.integers(-5, 6, size=K)
    U = np.zeros((2, K, K))
    U[0] = Ui.T.astype(float)  # (cols, rows) layout
    y = np.zeros((2, K))
    y[0] = bi
    r = orc.blocked("backsub", "dd", U, y, nb)
    xs = [Fraction(0)] * K
    for i in range(K - 1, -1, -1):
        xs[i] = Fraction(int(bi[i])) - sum(Fraction(int(Ui[i, l])) * xs[l] for l in range(i + 1, K))
    assert np.array_equal(r["x"][0], np.array([float(v) for v in xs]))
    assert np.all(r["x"][1] == 0.0)
