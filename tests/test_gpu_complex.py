"""Row f2: complex least squares on the GPU (mdls_zlstsq_<p>, re/im limb planes, solved through the real
embedding by the real pipeline) vs the oracle's complex Householder QR (oracle_zlstsq) on the same inputs,
componentwise in Re x and Im x to the north_star tolerance 1e3 n u -- the least-squares solution is unique,
the two factorisations are not (reading C1)."""
import numpy as np
import pytest
import torch

from paper_2110_08375_b200 import inputs

from ._parity import vec_ok

pytestmark = pytest.mark.gpu


def _problem(M, K, prec, seed):
    Are, bre = inputs.lstsq_problem(M, K, prec, seed)
    Aim, bim = inputs.lstsq_problem(M, K, prec, seed + 1000)
    return Are, Aim, bre, bim


@pytest.mark.parametrize("prec", ["dd", "qd", "od"])
@pytest.mark.parametrize("M,K,nb", [(32, 32, 8), (80, 48, 16), (130, 64, 32)])
def test_zlstsq_vs_oracle(orc, mdls, dev, prec, M, K, nb):
    Are, Aim, bre, bim = _problem(M, K, prec, seed=M + K)
    g = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    for form_q in (True, False):
        xr, xi, info = mdls.zlstsq(prec, g(Are), g(Aim), g(bre), g(bim), nb, form_q=form_q)
        torch.cuda.synchronize()
        assert int(info.item()) == 0
        oxr, oxi, _, _, oinfo = orc.zlstsq(prec, Are, Aim, bre, bim)
        assert oinfo == 0
        scale = max(np.max(np.abs(oxr[0])), np.max(np.abs(oxi[0])))
        for got, ref in ((xr, oxr), (xi, oxi)):
            err, _ = vec_ok(orc, prec, got.cpu().numpy(), ref, K)
            assert err <= 1e3 * K * {"dd": 2.0 ** -104, "qd": 2.0 ** -208, "od": 2.0 ** -416}[prec] * scale


def test_zlstsq_t5_dd512(orc, mdls, dev):
    """T5's complex double double shape (512 x 512), tile 64."""
    Are, Aim, bre, bim = _problem(512, 512, "dd", seed=5)
    g = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    xr, xi, info = mdls.zlstsq("dd", g(Are), g(Aim), g(bre), g(bim), 64)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    oxr, oxi, _, _, _ = orc.zlstsq("dd", Are, Aim, bre, bim)
    scale = max(np.max(np.abs(oxr[0])), np.max(np.abs(oxi[0])))
    for got, ref in ((xr, oxr), (xi, oxi)):
        err, _ = vec_ok(orc, "dd", got.cpu().numpy(), ref, 512)
        assert err <= 1e3 * 512 * 2.0 ** -104 * scale
