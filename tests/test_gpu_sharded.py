"""Block-column sharded least squares through the real kernels on one GPU:
P virtual ranks in one process (broadcasts are shared references), the same
host orchestration that runs one rank per GPU over NCCL.  Parity with the
oracle (north_star tolerance) and with the single-GPU lstsq."""
import numpy as np
import pytest
import torch

from paper_2110_08375_b200 import inputs, sharded

from ._parity import U_OF, vec_ok

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec", ["dd", "qd"])
@pytest.mark.parametrize("P", [2, 3])
def test_sharded_lstsq_virtual_ranks(orc, mdls, dev, prec, P):
    M, K, nb = 200, 192, 32
    A, b = inputs.lstsq_problem(M, K, prec, seed=P)
    st = sharded.plan(prec, M, K, nb, P)
    A_loc = {r: torch.from_numpy(np.ascontiguousarray(A[:, sharded.local_columns(st, r), :])).to(dev)
             for r in range(P)}
    bd = torch.from_numpy(b).to(dev)
    new = lambda shape: torch.zeros(shape, dtype=torch.float64, device=dev)
    x, F, y, info = sharded.sharded_lstsq(prec, A_loc, bd, M, K, nb, P, sharded.GpuOps(), None, new)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    xo, Ro, yo = orc.lstsq(prec, A, b)
    err, tol = vec_ok(orc, prec, x.cpu().numpy(), xo, K)
    assert err <= tol, (err, tol)
    r1 = mdls.lstsq(prec, torch.from_numpy(A).to(dev), bd, nb)
    err, tol = vec_ok(orc, prec, x.cpu().numpy(), r1.x.cpu().numpy(), K)
    assert err <= tol
