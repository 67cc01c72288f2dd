"""Plans (library-owned CUDA graphs, mdls_lstsq_plan_<p> / mdls_lstsq_batched_plan_<p>): a replay computes
exactly what the direct call computes (bitwise), for new inputs copied into the plan's buffers between
replays, and counts its kernels."""
import numpy as np
import pytest
import torch

from paper_2110_08375_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec,M,K,nb", [("dd", 96, 64, 16), ("qd", 64, 64, 8), ("od", 80, 48, 16),
                                         ("dd", 1024, 1024, 128)])
def test_lstsq_plan_bitwise(mdls, dev, prec, M, K, nb):
    plan = mdls.LstsqPlan(prec, M, K, nb, form_q=True, device=dev)
    assert plan.launches > 0
    for seed in (3, 4):
        A, b = inputs.lstsq_problem(M, K, prec, seed)
        At, bt = torch.from_numpy(A).to(dev), torch.from_numpy(b).to(dev)
        x = plan.solve(torch.from_numpy(A).pin_memory(), torch.from_numpy(b).pin_memory()).clone()
        r = mdls.lstsq(prec, At, bt, nb, form_q=True)
        torch.cuda.synchronize()
        assert int(plan.info.item()) == 0
        assert torch.equal(x, r.x)


def test_batched_plan_bitwise(mdls, dev):
    B, M, K, nb = 5, 96, 64, 16
    probs = [inputs.lstsq_problem(M, K, "qd", s) for s in range(B)]
    A = torch.from_numpy(np.stack([a for a, _ in probs])).to(dev)
    b = torch.from_numpy(np.stack([bb for _, bb in probs])).to(dev)
    plan = mdls.BatchedLstsqPlan("qd", B, M, K, nb, groups=3, device=dev)
    x = plan.solve(A, b).clone()
    xd, info = mdls.lstsq_batched("qd", A, b, nb, groups=3)
    torch.cuda.synchronize()
    assert plan.info.cpu().tolist() == [0] * B
    assert torch.equal(x, xd)
    n0 = mdls.launch_count()
    plan.run()
    torch.cuda.synchronize()
    assert mdls.launch_count() - n0 == plan.launches
