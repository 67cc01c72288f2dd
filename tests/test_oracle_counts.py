"""Pin the oracle's md arithmetic to the paper's Table 1.

The paper prints the base-double (+, -, *, /) counts of one dd/qd/od add, mul
and div.  The counting build of the oracle tallies every base operation its
algorithms execute.  A dropped term, an extra renormalisation step or a
different division algorithm changes these integers, so the match is a pin on
the *structure* of the md algorithms.

Exact cells: every octo double cell; the qd -, *, / columns; dd add; dd mul
* and -; dd div * and /.  The remaining cells differ from the printed table by
amounts no QDlib/CAMPARY variant reproduces (reading Z11);
they are asserted at their documented deltas so any change is noticed.
"""
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1.json")))

# (prec, op) -> per-column delta (ours - paper) for the cells T1 does not reproduce
KNOWN_DELTAS = {
    ("dd", "mul"): (1, 0, 0, 0),     # QDlib dd mul adds both cross products: 6 additions, T1 prints 5
    ("dd", "div"): (-2, 36, 0, 0),   # QDlib accurate_div +/- tally not reproducible from T1's 33/18
    ("qd", "add"): (-4, 0, 0, 0),
    ("qd", "mul"): (-4, 0, 0, 0),
    ("qd", "div"): (5, 0, 0, 0),
}


def _operands(m):
    a = np.zeros((m, 1))
    b = np.zeros((m, 1))
    a[0, 0], b[0, 0] = 1.1, 3.3
    for k in range(1, m):  # populated lower limbs: every branch-free path is exercised
        a[k, 0] = a[k - 1, 0] * 2.0 ** -54
        b[k, 0] = -b[k - 1, 0] * 2.0 ** -55
    return a, b


@pytest.mark.parametrize("prec,m", [("dd", 2), ("qd", 4), ("od", 8)])
@pytest.mark.parametrize("op", ["add", "mul", "div"])
def test_table1_counts(orc, prec, m, op):
    a, b = _operands(m)
    ours = orc.op_counts(op, prec, a, b)
    paper = tuple(GOLD[prec][op][:4])
    delta = KNOWN_DELTAS.get((prec, op), (0, 0, 0, 0))
    assert tuple(o - p for o, p in zip(ours, paper)) == delta, (prec, op, ours, paper)


def test_octo_double_row_exact(orc):
    a, b = _operands(8)
    for op in ("add", "mul", "div"):
        assert orc.op_counts(op, "od", a, b) == tuple(GOLD["od"][op][:4])


def test_table1_sums_and_averages():
    for prec in ("dd", "qd", "od"):
        rows = GOLD[prec]
        for op in ("add", "mul", "div"):
            assert sum(rows[op][:4]) == rows[op][4]
        avg = sum(rows[op][4] for op in ("add", "mul", "div")) / 3.0
        assert round(avg, 1) == rows["average"]
    # predicted overhead factors follow from the averages
    assert round(GOLD["qd"]["average"] / GOLD["dd"]["average"], 1) == 11.7
    assert round(GOLD["od"]["average"] / GOLD["qd"]["average"], 1) == 5.4


def test_counts_independent_of_values(orc):
    """The md algorithms are branch-free except renormalisation's zero tests:
    counts must not depend on the operand values."""
    rng = np.random.default_rng(3)
    for prec, m in (("qd", 4), ("od", 8)):
        base = orc.op_counts("mul", prec, *_operands(m))
        for _ in range(5):
            a = rng.uniform(-1, 1, size=(m, 1)) * 2.0 ** (-53 * np.arange(m))[:, None]
            b = rng.uniform(-1, 1, size=(m, 1)) * 2.0 ** (-53 * np.arange(m))[:, None]
            assert orc.op_counts("mul", prec, a, b) == base
