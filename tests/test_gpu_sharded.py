"""Block-column sharded least squares through the real kernels on one GPU: P virtual ranks in one process
(broadcasts are shared references), the same host orchestration -- look-ahead on a critical stream, the bulk
trailing update on a second stream, row-trimmed panel factors -- that runs one rank per GPU over NCCL.
Every update is issued one panel at a time, so the result is bitwise independent of P; and it
meets the oracle parity rule (north_star tolerance)."""
import numpy as np
import pytest
import torch

from paper_2110_08375_b200 import inputs, sharded

from ._parity import vec_ok

pytestmark = pytest.mark.gpu


def _solve(prec, A, b, nb, P, dev):
    M, K = A.shape[2], A.shape[1]
    st = sharded.plan(prec, M, K, nb, P)
    A_loc = {r: torch.from_numpy(np.ascontiguousarray(A[:, sharded.local_columns(st, r), :])).to(dev)
             for r in range(P)}
    bd = torch.from_numpy(b).to(dev)
    new = lambda shape: torch.zeros(shape, dtype=torch.float64, device=dev)  # noqa: E731
    x, F, y, info = sharded.sharded_lstsq(prec, A_loc, bd, M, K, nb, P, sharded.GpuOps(), None, new,
                                          sharded.Streams(dev))
    torch.cuda.synchronize()
    return x, F, y, info


@pytest.mark.parametrize("prec,M,K,nb", [("dd", 200, 192, 32), ("qd", 200, 192, 32), ("od", 136, 128, 16),
                                         ("dd", 520, 512, 64)])
def test_sharded_lstsq_virtual_ranks(orc, mdls, dev, prec, M, K, nb):
    A, b = inputs.lstsq_problem(M, K, prec, seed=M + nb)
    ref = _solve(prec, A, b, nb, 1, dev)
    assert int(ref[3].item()) == 0
    for P in (2, 3):
        got = _solve(prec, A, b, nb, P, dev)
        assert int(got[3].item()) == 0
        for g, r in zip(got[:3], ref[:3]):
            assert torch.equal(g, r), f"P={P} differs from the single-rank result"
    xo, Ro, yo = orc.lstsq(prec, A, b)
    err, tol = vec_ok(orc, prec, ref[0].cpu().numpy(), xo, K)
    assert err <= tol, (err, tol)


def test_sharded_singular_reports_info(orc, mdls, dev):
    """A zero column reaches the caller through the panel infos (first zero R_jj, 1-based)."""
    A, b = inputs.lstsq_problem(96, 64, "dd", seed=3)
    A[:, 40, :] = 0.0
    x, F, y, info = _solve("dd", A, b, 16, 2, dev)
    assert int(info.item()) == 41
