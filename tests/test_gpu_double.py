"""Row f4: the plain double ("1d") path -- the same kernels instantiated for one limb (the paper's
double precision version) -- against the oracle's m = 1 rows (IEEE double Householder QR,
pinned to LAPACK in tests/test_oracle_double.py) at the benchmark shape, with the north_star rule
1e3 * n * u, u = 2^-53.  The small shapes run through the md-generic parity files (test_gpu_qr.py,
test_gpu_backsub.py, test_gpu_gemm.py, test_gpu_invariants.py, test_gpu_arith.py)."""
import numpy as np
import pytest
import torch

from paper_2110_08375_b200 import inputs

from ._parity import U_OF, mat_cols_ok, vec_ok

pytestmark = pytest.mark.gpu


def _gpu(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


@pytest.mark.parametrize("form_q", [True, False])
def test_lstsq_1024(orc, mdls, dev, form_q):
    M = K = 1024
    A, b = inputs.lstsq_problem(M, K, "d", seed=3)
    r = mdls.lstsq("d", _gpu(A, dev), _gpu(b, dev), 128, form_q=form_q, want_R=True)
    torch.cuda.synchronize()
    assert int(r.info.item()) == 0
    xo, Ro, _ = orc.lstsq("d", A, b)
    err, tol = vec_ok(orc, "d", r.x.cpu().numpy(), xo, K)
    assert err <= tol, (err, tol)
    Rg = r.R.cpu().numpy()
    assert mat_cols_ok(orc, "d", Rg, Ro, K) <= 1.0
    assert orc.inv_normal("d", A, r.x.cpu().numpy(), b) <= 1e3 * M * U_OF["d"]


def test_lstsq_tall_residual(orc, mdls, dev):
    M, K, nb = 2048, 512, 128
    A, b = inputs.lstsq_problem(M, K, "d", seed=9)
    r = mdls.lstsq("d", _gpu(A, dev), _gpu(b, dev), nb, form_q=False, want_y=True, want_residual=True)
    torch.cuda.synchronize()
    xo, _, yo = orc.lstsq("d", A, b)
    err, tol = vec_ok(orc, "d", r.x.cpu().numpy(), xo, K)
    assert err <= tol
    ro = orc.norm2("d", yo[:, K:].copy())
    assert abs(float(r.residual.cpu().numpy()[0, 0]) - ro[0]) <= 1e3 * M * U_OF["d"] * ro[0]


def test_deterministic(mdls, dev):
    A, b = inputs.lstsq_problem(512, 512, "d", seed=1)
    xs = [mdls.lstsq("d", _gpu(A, dev), _gpu(b, dev), 64, form_q=True).x.cpu().numpy() for _ in range(3)]
    assert all(np.array_equal(xs[0], x) for x in xs[1:])
