"""The end-to-end call with HOST buffers (mdls_lstsq_host_<p>, the HostLstsqPlan graph): A's column panels are
copied on a library stream while the factorisation of the first panels runs, every lane waiting only for the
panels it touches.  The arithmetic is the device path's, in the same order, so x is bitwise equal to
mdls_lstsq on the same inputs (register-leaf chain and the GEMM-chained overlap path), and matches the oracle."""
import numpy as np
import pytest
import torch

from paper_2110_08375_b200 import inputs

from ._parity import vec_ok

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec,M,K,nb", [("dd", 1024, 1024, 128), ("qd", 300, 256, 64), ("d", 512, 384, 128),
                                         ("od", 1040, 64, 32)])
@pytest.mark.parametrize("form_q", [True, False])
def test_host_io_bitwise_equals_device_path(orc, mdls, dev, prec, M, K, nb, form_q):
    A, b = inputs.lstsq_problem(M, K, prec, seed=M + K)
    r = mdls.lstsq(prec, torch.from_numpy(A).to(dev), torch.from_numpy(b).to(dev), nb, form_q=form_q)
    x_dev = r.x.cpu()
    x_h, info = mdls.lstsq_host(prec, torch.from_numpy(A).pin_memory(), torch.from_numpy(b).pin_memory(), nb,
                                form_q=form_q)
    assert int(info.item()) == 0
    assert torch.equal(x_h, x_dev)
    if M <= 512:
        xo, _, _ = orc.lstsq(prec, A, b)
        err, tol = vec_ok(orc, prec, x_h.numpy(), xo, K)
        assert err <= tol


def test_host_plan_replays_new_inputs(mdls, dev):
    prec, M, K, nb = "dd", 512, 512, 64
    plan = mdls.HostLstsqPlan(prec, M, K, nb, form_q=True, device=dev)
    for seed in (1, 2):
        A, b = inputs.lstsq_problem(M, K, prec, seed=seed)
        x = plan.solve(A, b).clone()
        ref = mdls.lstsq(prec, torch.from_numpy(A).to(dev), torch.from_numpy(b).to(dev), nb, form_q=True).x.cpu()
        assert int(plan.info.item()) == 0
        assert torch.equal(x, ref)


def test_host_io_copy_modes_bitwise(tmp_path):
    """the copy-engine and zero-copy panel transfers (MDLS_HOST_ZC=0 / 1, read once per process) give the same x"""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2110_08375_b200 as mdls
from paper_2110_08375_b200 import inputs
A, b = inputs.lstsq_problem(512, 384, "qd", 5)
x, info = mdls.lstsq_host("qd", torch.from_numpy(A).pin_memory(), torch.from_numpy(b).pin_memory(), 64)
assert int(info.item()) == 0
np.save(sys.argv[1], x.numpy())
"""
    outs = []
    for zc in ("0", "1"):
        out = str(tmp_path / f"x{zc}.npy")
        p = subprocess.run([sys.executable, "-c", code, out], env={**os.environ, "MDLS_HOST_ZC": zc},
                           capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])
