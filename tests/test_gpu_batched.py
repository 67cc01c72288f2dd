"""Batched least squares (mdls_lstsq_batched_<p>, SURVEY 8(e) batch sharding,
BASELINE config 5b): every problem of a batch solved on the library's stream
groups must equal the single-problem mdls_lstsq result bit for bit (same
kernels, fixed-order reductions; concurrency must not change a bit), and
sampled problems must meet the oracle parity rule (1e3 n u)."""
import numpy as np
import pytest
import torch

from paper_2110_08375_b200 import batch, inputs

from ._parity import vec_ok

pytestmark = pytest.mark.gpu


def _stack(M, K, prec, seeds, dev):
    probs = [inputs.lstsq_problem(M, K, prec, s) for s in seeds]
    A = torch.from_numpy(np.stack([a for a, _ in probs])).to(dev)
    b = torch.from_numpy(np.stack([bb for _, bb in probs])).to(dev)
    return probs, A, b


@pytest.mark.parametrize("prec", ["d", "dd", "qd", "od"])
@pytest.mark.parametrize("M,K,nb,B,groups", [(96, 64, 16, 6, 3), (130, 128, 32, 5, 2), (64, 64, 8, 3, 4)])
def test_batched_equals_single(orc, mdls, dev, prec, M, K, nb, B, groups):
    probs, A, b = _stack(M, K, prec, range(100, 100 + B), dev)
    for form_q in (True, False):
        x, info = mdls.lstsq_batched(prec, A, b, nb, form_q=form_q, groups=groups)
        torch.cuda.synchronize()
        assert info.cpu().tolist() == [0] * B
        for p in range(B):
            r = mdls.lstsq(prec, A[p], b[p], nb, form_q=form_q)
            torch.cuda.synchronize()
            assert torch.equal(r.x, x[p]), f"problem {p} differs from the single solve"
    # the oracle on two sampled problems
    for p in (0, B - 1):
        xo, _, _ = orc.lstsq(prec, *probs[p])
        err, tol = vec_ok(orc, prec, x[p].cpu().numpy(), xo, K)
        assert err <= tol


def test_batched_cfg5b_sampled(orc, mdls, dev):
    """Config 5b shape (dd 1024 x 1024, tile 128) on one GPU: a batch of 8 with 4 stream groups; problems 0 and
    7 vs the oracle, all vs the single-solve bits."""
    M = K = 1024
    B = 8
    probs, A, b = _stack(M, K, "dd", range(B), dev)
    x, info = mdls.lstsq_batched("dd", A, b, 128, form_q=True, groups=4)
    torch.cuda.synchronize()
    assert info.cpu().tolist() == [0] * B
    for p in range(B):
        r = mdls.lstsq("dd", A[p], b[p], 128, form_q=True)
        torch.cuda.synchronize()
        assert torch.equal(r.x, x[p])
    for p in (0, B - 1):
        xo, _, _ = orc.lstsq("dd", *probs[p])
        err, tol = vec_ok(orc, "dd", x[p].cpu().numpy(), xo, K)
        assert err <= tol


def test_batched_edge_cases(mdls, dev):
    from paper_2110_08375_b200 import _lib
    import ctypes

    fn = _lib.fn("mdls_lstsq_batched_", "dd")
    nbytes = mdls.batch_workspace_bytes("dd", _lib.OP_LSTSQ, 64, 64, 8, 2)
    assert nbytes > 0
    assert mdls.batch_workspace_bytes("dd", _lib.OP_LSTSQ, 64, 64, 8, 0) == 0
    assert mdls.batch_workspace_bytes("dd", _lib.OP_QR, 64, 64, 8, 2) == 0
    work = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    A = torch.zeros((1, 2, 64, 64), dtype=torch.float64, device=dev)
    b = torch.zeros((1, 2, 64), dtype=torch.float64, device=dev)
    x = torch.zeros((1, 2, 64), dtype=torch.float64, device=dev)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    # batch 0: nothing enqueued, success
    assert fn(0, 64, 64, 8, P(A), 64, 4096, 8192, P(b), 64, 128, P(x), 64, 128, 1, 2, P(work), nbytes,
              ctypes.c_void_p(0), st) == 0
    # groups out of range, overlapping problems, short workspace
    assert fn(1, 64, 64, 8, P(A), 64, 4096, 8192, P(b), 64, 128, P(x), 64, 128, 1, 0, P(work), nbytes,
              ctypes.c_void_p(0), st) == -16
    assert fn(1, 64, 64, 8, P(A), 64, 4096, 100, P(b), 64, 128, P(x), 64, 128, 1, 2, P(work), nbytes,
              ctypes.c_void_p(0), st) == -8
    assert fn(1, 64, 64, 8, P(A), 64, 4096, 8192, P(b), 64, 128, P(x), 64, 128, 1, 2, P(work), nbytes - 1,
              ctypes.c_void_p(0), st) == -18
    # a singular problem reports through its own dev_info slot only
    A2 = torch.stack([torch.from_numpy(inputs.lstsq_problem(64, 64, "dd", 1)[0])] * 2).to(dev)
    A2[1, :, 5, :] = 0.0  # column 5 of problem 1 is zero -> R_55 = 0
    b2 = torch.stack([torch.from_numpy(inputs.lstsq_problem(64, 64, "dd", 1)[1])] * 2).to(dev)
    xs, info = mdls.lstsq_batched("dd", A2, b2, 8, groups=2)
    torch.cuda.synchronize()
    assert int(info[0]) == 0 and int(info[1]) > 0
    assert batch.shard_range(256, 3, 8) == (96, 128)
