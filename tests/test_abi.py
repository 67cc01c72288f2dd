"""CPU checks of the C-ABI boundary (no GPU needed): libmdls.so loads, exports
every symbol include/mdls.h declares, rejects invalid arguments on the host
before launching anything, and its ledger (A10) matches closed forms that
follow from the algorithm definitions."""
import ctypes
import os
import re

import pytest

import paper_2110_08375_b200 as mdls
from paper_2110_08375_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "mdls.h")


def declared_symbols():
    src = open(HEADER).read()
    names = set(re.findall(r"\b(mdls_[a-z0-9_]+)\s*\(", src.split("#define MDLS_DECLARE")[0]))
    block = src.split("#define MDLS_DECLARE(P)")[1].split("MDLS_DECLARE(dd)")[0]
    stems = set(re.findall(r"\b(mdls_[a-z0-9_]+_)##P\s*\(", block))
    for p in re.findall(r"^MDLS_DECLARE\((\w+)\)", src, re.M):
        names |= {s + p for s in stems}
    return names


def test_header_and_exports_agree():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 36
    for n in names:
        assert hasattr(lib, n), n
    assert set(_lib.EXPORTED) == names


def test_version_limbs_strerror():
    lib = _lib.load()
    assert lib.mdls_version() >= 1
    assert [lib.mdls_limbs(i) for i in range(3)] == [2, 4, 8]
    assert b"invalid" in lib.mdls_strerror(-3)


@pytest.mark.parametrize("prec", ["d", "dd", "qd", "od"])
def test_host_argument_checks(prec):
    """Invalid sizes are rejected with -i before any CUDA call (works without a GPU)."""
    qr = _lib.fn("mdls_qr_", prec)
    nul = ctypes.c_void_p(0)
    assert qr(10, 20, 4, nul, 10, 200, nul, 0, 0, nul, 0, 0, nul, 0, nul, nul) == -1       # M < K
    assert qr(20, 10, 4, nul, 20, 200, nul, 0, 0, nul, 0, 0, nul, 0, nul, nul) == -3       # nb does not divide K
    assert qr(20, 8, 4, nul, 20, 160, nul, 0, 0, nul, 0, 0, nul, 0, nul, nul) == -4        # NULL A
    fake = ctypes.c_void_p(0x1000)
    assert qr(20, 8, 4, fake, 10, 160, nul, 0, 0, nul, 0, 0, nul, 0, nul, nul) == -4       # lda < M
    assert qr(20, 8, 4, fake, 20, 160, nul, 0, 0, nul, 0, 0, nul, 0, nul, nul) == -14      # no workspace
    bs = _lib.fn("mdls_backsub_", prec)
    assert bs(0, 4, fake, 4, 16, fake, 4, fake, 4, fake, 1 << 20, nul, nul) == -1
    assert bs(10, 4, fake, 10, 100, fake, 10, fake, 10, fake, 1 << 20, nul, nul) == -2
    assert bs(8, 4, fake, 8, 64, fake, 4, fake, 8, fake, 1 << 20, nul, nul) == -6          # psy < n
    op = _lib.fn("mdls_md_op_", prec)
    assert op(10, 10, fake, fake, fake, 10, nul) == -1
    assert op(0, 10, fake, nul, fake, 10, nul) == -4
    assert op(7, 10, fake, nul, fake, 10, nul) == -4                                       # warp mul needs b
    bat = _lib.fn("mdls_lstsq_batched_", prec)
    m = {"d": 1, "dd": 2, "qd": 4, "od": 8}[prec]
    args = [4, 64, 64, 8, fake, 64, 4096, m * 4096, fake, 64, m * 64, fake, 64, m * 64, 1, 2, fake, 1 << 40, nul, nul]
    for i, v, rc in ((0, -1, -1), (3, 7, -4), (7, 100, -8), (10, 10, -11), (13, 1, -14), (15, 0, -16), (15, 17, -16),
                     (17, 10, -18)):
        bad = list(args)
        bad[i] = v
        assert bat(*bad) == rc, (i, v)
    bws = _lib.fn("mdls_workspace_batched_", prec)
    assert bws(2, 64, 64, 8, 3) == 3 * (bws(2, 64, 64, 8, 1))
    assert bws(0, 64, 64, 8, 3) == 0 and bws(2, 64, 64, 8, 0) == 0
    plan = ctypes.c_void_p(0)
    lp = _lib.fn("mdls_lstsq_plan_", prec)
    assert lp(10, 20, 4, fake, 10, 200, fake, 10, fake, 20, 1, fake, 1 << 30, nul, ctypes.byref(plan)) == -1
    assert plan.value is None
    bad = list(args[:-1]) + [ctypes.byref(plan)]
    bad[15] = 0
    assert _lib.fn("mdls_lstsq_batched_plan_", prec)(*bad) == -16
    assert _lib.load().mdls_plan_launch(nul, nul) == -1
    _lib.load().mdls_plan_destroy(nul)
    host = _lib.fn("mdls_lstsq_host_", prec)
    assert host(10, 20, 4, fake, 10, 200, fake, 10, fake, 20, 1, fake, 1 << 30, nul, nul) == -1   # M < K
    assert host(20, 8, 4, nul, 20, 160, fake, 20, fake, 8, 1, fake, 1 << 30, nul, nul) == -4     # NULL A
    assert host(20, 8, 4, fake, 20, 160, fake, 10, fake, 8, 1, fake, 1 << 30, nul, nul) == -7    # psb < M
    assert host(20, 8, 4, fake, 20, 160, fake, 20, fake, 4, 1, fake, 1 << 30, nul, nul) == -9    # psx < K
    assert host(20, 8, 4, fake, 20, 160, fake, 20, fake, 8, 1, nul, 0, nul, nul) == -13         # no workspace
    assert _lib.fn("mdls_lstsq_host_plan_", prec)(20, 8, 4, fake, 20, 160, fake, 20, fake, 8, 1, fake, 1 << 30, nul,
                                                  None) == -15                                      # NULL plan
    hp = ctypes.c_void_p(0)
    assert _lib.fn("mdls_lstsq_host_plan_", prec)(10, 20, 4, fake, 10, 200, fake, 10, fake, 20, 1, fake, 1 << 30, nul,
                                                  ctypes.byref(hp)) == -1 and hp.value is None
    assert _lib.fn("mdls_workspace_", prec)(0, 10, 20, 4) == 0
    assert _lib.fn("mdls_workspace_", prec)(2, 1024, 1024, 128) > 0


def _pairs(c, stage):
    return c["stages"][stage]["mul"]


@pytest.mark.parametrize("prec", ["d", "dd", "qd", "od"])
def test_ledger_closed_forms(prec):
    M, K = 96, 64
    # nb = 1: every reflector is its own panel, the in-panel work vanishes and the
    # trailing update is the textbook unblocked update: sum_j 2 (M-j)(K-j-1) pairs
    c1 = mdls.counts(prec, 0, M, K, 1)
    assert _pairs(c1, "panel") == 0
    assert c1["stages"]["trailing"]["add"] == sum(2 * (M - j) * (K - j - 1) for j in range(K))
    # nb = K: one panel, the whole update is in-panel: per column 2 (M-j)(K-j-1) pairs plus K-j-1 scalings
    cK = mdls.counts(prec, 0, M, K, K)
    assert _pairs(cK, "trailing") == 0
    assert cK["stages"]["panel"]["add"] == sum(2 * (M - j) * (K - j - 1) for j in range(K))
    # house: one sqrt per column
    assert cK["stages"]["house"]["sqrt"] == K
    # backward Q: panel k of width nb touches an (M - k nb)^2 block twice per column
    c = mdls.counts(prec, 0, 1024, 1024, 128)
    assert _pairs(c, "form_q") == sum(2 * 128 * (1024 - 128 * k) ** 2 for k in range(8))
    assert _pairs(c, "trailing") == 704643072  # 7.05e8 pairs at 1024, nb 128
    # back substitution, N tiles of nb: D^2/2-type update count and zero-exploiting inverses
    b = mdls.counts(prec, 1, 17920, 17920, 128)
    N, nb = 140, 128
    assert _pairs(b, "bsupdate") == nb * nb * N * (N - 1) // 2
    assert b["stages"]["invert"]["add"] == N * nb * (nb * nb - 1) // 6
    assert b["stages"]["invert"]["div"] == N * nb


@pytest.mark.parametrize("prec", ["d", "dd", "qd", "od"])
def test_ledger_table1_weighting(prec):
    add, mul, div = mdls.T1_SUMS[prec]
    c = mdls.counts(prec, 2, 256, 256, 64)
    tot = 0.0
    for s, v in c["stages"].items():
        sq = 1 if prec == "d" else div + 2 * mul  # md sqrt priced as 1 div + 2 mul (Z12); a double sqrt is 1 flop
        f = v["add"] * add + v["mul"] * mul + v["div"] * div + v["sqrt"] * sq
        assert f == pytest.approx(v["flops"], rel=1e-15)
        tot += f
    assert tot == pytest.approx(c["total_flops"], rel=1e-15)


def test_overhead_factors_from_ledger():
    """The predicted dd->qd->od cost factors follow from Table 1 when the
    op mix is fixed: the ledger's ratios sit between the mul-only and add-only ratios."""
    f = {p: mdls.counts(p, 2, 1024, 1024, 128)["total_flops"] for p in ("dd", "qd", "od")}
    r1, r2 = f["qd"] / f["dd"], f["od"] / f["qd"]
    assert 89 / 20 < r1 < 336 / 23 and 269 / 89 < r2 < 1742 / 336
