"""A1-A6 parity: blocked Householder QR (Algorithm 2), Q, Q^T b and least
squares vs the oracle's unblocked Householder QR on the same inputs
(north_star tolerance 1e3 * n * u, column-norm scaled), plus the invariants
E1 = |Q^T Q - I|, E2 = |A - QR|/|A|, E3 = normal-equation residual evaluated
by the oracle on the GPU's outputs."""
import numpy as np
import pytest
import torch

from paper_2110_08375_b200 import inputs

from ._parity import U_OF, mat_cols_ok, vec_ok

pytestmark = pytest.mark.gpu

PRECS = ["d", "dd", "qd", "od"]


def _gpu(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("M,K,nb", [(64, 64, 8), (100, 64, 16), (130, 96, 32), (200, 128, 128), (300, 256, 64)])
def test_qr_vs_oracle(orc, mdls, dev, prec, M, K, nb):
    A = inputs.random_matrix(M, K, prec, seed=M + K + nb)
    F, Q, W, info = mdls.qr(prec, _gpu(A, dev), nb, form_q=True, want_w=True)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    Fo, beta = orc.qr(prec, A)
    Ro = orc.r_of(Fo)
    Rg = orc.r_of(F.cpu().numpy())
    assert mat_cols_ok(orc, prec, Rg, Ro, K) <= 1.0
    # strictly-lower part of R: the factored array holds v there; R itself is upper
    Qg = Q.cpu().numpy()
    bound = 1e3 * M * U_OF[prec]
    assert orc.inv_orth(prec, Qg) <= bound
    assert orc.inv_recon(prec, A, Qg, Rg) <= bound
    # Q vs oracle Q on the first K columns (unique for full-rank A with R_jj > 0)
    Qo = orc.form_q(prec, Fo, beta)
    assert mat_cols_ok(orc, prec, np.ascontiguousarray(Qg[:, :K]), np.ascontiguousarray(Qo[:, :K]), K) <= 1.0
    # apply_qt from the panels == explicit Q^T b
    b = inputs.random_vector(M, prec, seed=M)
    y1 = mdls.apply_qt(prec, F, W, _gpu(b, dev), nb).cpu().numpy()
    y2 = mdls.qt_b(prec, Q, _gpu(b, dev)).cpu().numpy()
    yo = orc.apply_qt(prec, Fo, beta, b)
    for y in (y1, y2):
        err, tol = vec_ok(orc, prec, y[:, :K].copy(), yo[:, :K].copy(), K)
        assert err <= tol


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("seed", range(5))
def test_lstsq_config1(orc, mdls, dev, prec, seed):
    """BASELINE config 1: 64 x 64, tile 8, 5 seeds."""
    M = K = 64
    A, b = inputs.lstsq_problem(M, K, prec, seed)
    for form_q in (True, False):
        r = mdls.lstsq(prec, _gpu(A, dev), _gpu(b, dev), 8, form_q=form_q, want_R=True, want_y=True)
        torch.cuda.synchronize()
        assert int(r.info.item()) == 0
        xo, Ro, yo = orc.lstsq(prec, A, b)
        err, tol = vec_ok(orc, prec, r.x.cpu().numpy(), xo, K)
        assert err <= tol, (form_q, err, tol)
        Rg = r.R.cpu().numpy()
        assert mat_cols_ok(orc, prec, Rg, Ro, K) <= 1.0
        assert np.all(Rg[:, np.tril_indices(M, -1)[1], np.tril_indices(M, -1)[0]] == 0.0)
        assert orc.inv_normal(prec, A, r.x.cpu().numpy(), b) <= 1e3 * M * U_OF[prec]


@pytest.mark.parametrize("prec", PRECS)
def test_lstsq_overdetermined_ragged(orc, mdls, dev, prec):
    M, K, nb = 203, 96, 32
    A, b = inputs.lstsq_problem(M, K, prec, 11)
    for form_q in (True, False):
        r = mdls.lstsq(prec, _gpu(A, dev), _gpu(b, dev), nb, form_q=form_q, want_y=True, want_residual=True)
        xo, Ro, yo = orc.lstsq(prec, A, b)
        err, tol = vec_ok(orc, prec, r.x.cpu().numpy(), xo, K)
        assert err <= tol
        _residual_ok(orc, prec, r, yo, A, b, K)
        assert orc.inv_normal(prec, A, r.x.cpu().numpy(), b) <= 1e3 * M * U_OF[prec]


def _residual_ok(orc, prec, r, yo, A, b, K):
    """f1: the residual ||b - A x|| = ||(Q^T b)(K+1:M)|| at md precision: the GPU's md norm
    (mdls_norm2 on its Q^T b tail) vs the oracle's, and the Q^T b tail entries themselves element by
    element (unique up to the sign convention of Q's trailing columns only through their norm, so the
    norm is compared, plus the direct ||b - A x_gpu||)."""
    M = A.shape[2]
    res_g = r.residual.cpu().numpy()[:, 0]
    res_o = orc.norm2(prec, yo[:, K:])
    d = orc.md_op("sub", prec, res_g[:, None], res_o[:, None])[0, 0]
    tol = 1e3 * M * U_OF[prec] * max(1.0, float(res_o[0]))
    assert abs(d) <= tol, (d, tol)
    direct = orc.residual_direct(prec, A, r.x.cpu().numpy(), b)
    d2 = orc.md_op("sub", prec, res_g[:, None], direct[:, None])[0, 0]
    scale = np.max(np.sum(np.abs(A[0]), axis=0)) * np.max(np.abs(r.x.cpu().numpy()[0])) + np.max(np.abs(b[0]))
    assert abs(d2) <= 1e3 * M * U_OF[prec] * scale, (d2, scale)


def test_lstsq_spec_examples(mdls, dev):
    for prec in PRECS:
        m = inputs.limbs(prec)
        A = np.zeros((m, 1, 2))
        A[0, 0] = [1.0, 1.0]
        b = np.zeros((m, 2))
        b[0] = [0.0, 2.0]
        r = mdls.lstsq(prec, _gpu(A, dev), _gpu(b, dev), 1)
        x = r.x.cpu().numpy()
        assert abs(x[0, 0] - 1.0) <= 4 * U_OF[prec] and abs(x[:2, 0].sum() - 1.0) <= 4 * U_OF[prec]


def test_qr_zero_column_reports_info(mdls, dev):
    m, M, K = 2, 32, 16
    A = inputs.random_matrix(M, K, "dd", seed=5)
    A[:, 5, :] = 0.0
    F, Q, W, info = mdls.qr("dd", _gpu(A, dev), 8, form_q=False)
    torch.cuda.synchronize()
    assert int(info.item()) > 0


def test_lstsq_nonfinite_input(mdls, dev):
    A, b = inputs.lstsq_problem(32, 16, "dd", 1)
    A[0, 3, 4] = np.nan
    r = mdls.lstsq("dd", _gpu(A, dev), _gpu(b, dev), 8)
    torch.cuda.synchronize()
    assert int(r.info.item()) == -1


@pytest.mark.parametrize("prec", ["d", "dd", "qd", "od"])
def test_lstsq_config2_full(orc, mdls, dev, prec):
    """BASELINE configs 2 and 3 at full size (dd/qd/od, 1024 x 1024, tile 128): full x and R parity."""
    M = K = 1024
    A, b = inputs.lstsq_problem(M, K, prec, 0)
    r = mdls.lstsq(prec, _gpu(A, dev), _gpu(b, dev), 128, form_q=True, want_R=True)
    torch.cuda.synchronize()
    assert int(r.info.item()) == 0
    xo, Ro, yo = orc.lstsq(prec, A, b)
    err, tol = vec_ok(orc, prec, r.x.cpu().numpy(), xo, K)
    rr = mat_cols_ok(orc, prec, r.R.cpu().numpy(), Ro, K)
    print(f"config 2/3 {prec}: x err/tol = {err / tol:.3e}, R worst column err/tol = {rr:.3e}")
    assert err <= tol, (err, tol)
    assert rr <= 1.0


@pytest.mark.parametrize("prec,M,K,nb", [("dd", 1536, 1024, 128), ("qd", 1280, 256, 64), ("dd", 2048, 128, 16),
                                        ("od", 1100, 64, 8)])
def test_lstsq_tall_512_thread_leaf(orc, mdls, dev, prec, M, K, nb):
    """Overdetermined systems taller than 1024 rows: the register leaf's 512-thread variant (rows per CTA in
    (64, 128]) in the chained factorisation, plus the residual entries of Q^T b."""
    A, b = inputs.lstsq_problem(M, K, prec, 3)
    r = mdls.lstsq(prec, _gpu(A, dev), _gpu(b, dev), nb, form_q=True, want_R=True, want_y=True,
                   want_residual=True)
    torch.cuda.synchronize()
    assert int(r.info.item()) == 0
    xo, Ro, yo = orc.lstsq(prec, A, b)
    err, tol = vec_ok(orc, prec, r.x.cpu().numpy(), xo, K)
    assert err <= tol, (err, tol)
    assert mat_cols_ok(orc, prec, r.R.cpu().numpy(), Ro, K) <= 1.0
    _residual_ok(orc, prec, r, yo, A, b, K)
