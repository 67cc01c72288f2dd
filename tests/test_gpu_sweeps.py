"""f3 parity: the sweep shapes of tools/sweeps.py (the paper's T5-T9 tilings) meet the same
oracle bar as the headline shapes -- T5's dd tilings of n = 512 from 32 x 16 to 2 x 256, and back substitution
with the non-power-of-two tiles of T7/T9 (nb = 96, 160, 224) in every precision."""
import numpy as np
import pytest
import torch

from paper_2110_08375_b200 import inputs

from ._parity import mat_cols_ok, vec_ok

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nb", [16, 256])
def test_t5_tilings_dd512(orc, mdls, dev, nb):
    M = K = 512
    A, b = inputs.lstsq_problem(M, K, "dd", seed=M + nb)
    r = mdls.lstsq("dd", torch.from_numpy(A).to(dev), torch.from_numpy(b).to(dev), nb, want_R=True)
    torch.cuda.synchronize()
    assert int(r.info.item()) == 0
    xo, Ro, _ = orc.lstsq("dd", A, b)
    err, tol = vec_ok(orc, "dd", r.x.cpu().numpy(), xo, K)
    assert err <= tol
    assert mat_cols_ok(orc, "dd", r.R.cpu().numpy(), Ro, K) <= 1.0


@pytest.mark.parametrize("prec,nb,tiles", [("dd", 96, 5), ("qd", 224, 3), ("od", 160, 3), ("qd", 160, 4)])
def test_t7_t9_backsub_tiles(orc, mdls, dev, prec, nb, tiles):
    n = nb * tiles
    U = inputs.lu_upper(n, prec, seed=n + 1)
    y = inputs.random_vector(n, prec, seed=n + 2)
    x, info = mdls.backsub(prec, torch.from_numpy(U).to(dev), torch.from_numpy(y).to(dev), nb)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    xr, _ = orc.backsub(prec, U, y)
    err, tol = vec_ok(orc, prec, x.cpu().numpy(), xr, n)
    assert err <= tol, (err, tol)
