"""A3-A6 building block: the md tile product mdls_gemm_<p> (C (mode)= op(A) op(B)) vs
the oracle's md dot products (the plain definition C_ij = sum_k a_ik b_kj, each
product one md mul, each sum one md add, ascending k; oracle/mdls_oracle.c
oracle_dot).  Tolerance: the north_star 1e3 * k * u, scaled by the entry's
sum_k |a_ik b_kj| (the accumulation error bound of any summation order), so the
test pins the dd pair accumulator and the qd/od level-bin accumulators (md.cuh
Acc) on long reductions, split-K included (k up to 2000 > 8 k-tiles)."""
import numpy as np
import pytest
import torch

from paper_2110_08375_b200 import inputs

from ._parity import U_OF

pytestmark = pytest.mark.gpu


def _gpu(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def _op(X, trans):
    # X: (m, cols, rows) limb-planar column-major; returns op(X) as (m, rows_op, cols_op) row-major view
    Xr = np.transpose(X, (0, 2, 1))  # (m, rows, cols)
    return np.transpose(Xr, (0, 2, 1)) if trans else Xr


@pytest.mark.parametrize("prec", ["d", "dd", "qd", "od"])
@pytest.mark.parametrize("m,n,k,ta,tb,mode", [(37, 29, 61, 0, 0, 0), (16, 70, 2000, 1, 0, 1), (130, 3, 513, 0, 1, 2),
                                              (9, 11, 7, 1, 1, 3), (64, 64, 128, 0, 0, 1)])
def test_gemm_vs_oracle_dots(orc, mdls, dev, prec, m, n, k, ta, tb, mode):
    ml = inputs.limbs(prec)
    A = inputs.random_matrix(k if ta else m, m if ta else k, prec, seed=m + 3 * k)
    B = inputs.random_matrix(n if tb else k, k if tb else n, prec, seed=n + 5 * k)
    C0 = inputs.random_matrix(m, n, prec, seed=m * n)
    Cg = mdls.gemm(prec, _gpu(A, dev), _gpu(B, dev), C=_gpu(C0, dev).clone(), trans_a=bool(ta), trans_b=bool(tb),
                   mode=mode)
    torch.cuda.synchronize()
    Cg = Cg.cpu().numpy()  # (m, n cols, m rows)
    Aop = _op(A, ta)  # (ml, m, k)
    Bop = _op(B, tb)  # (ml, k, n)
    for i in range(m):
        for j in range(n):
            p = orc.dot(prec, np.ascontiguousarray(Aop[:, i, :]), np.ascontiguousarray(Bop[:, :, j]))
            c0 = C0[:, j, i]
            if mode == 0:
                ref = p
            elif mode == 1:
                ref = orc.md_op("add", prec, c0[:, None], p[:, None])[:, 0]
            elif mode == 2:
                ref = orc.md_op("sub", prec, c0[:, None], p[:, None])[:, 0]
            else:
                ref = -p
            d = orc.md_op("sub", prec, Cg[:, j, i][:, None], ref[:, None])[0, 0]
            scale = float(np.sum(np.abs(Aop[0, i, :] * Bop[0, :, j]))) + abs(float(c0[0])) * (mode in (1, 2))
            tol = 1e3 * k * U_OF[prec] * max(scale, 1e-300)
            assert abs(d) <= tol, (prec, i, j, d, tol)
    assert Cg.shape == (ml, n, m)


def test_gemm_argument_errors(mdls, dev):
    from paper_2110_08375_b200 import _lib

    A = torch.zeros((2, 4, 4), dtype=torch.float64, device=dev)
    f = _lib.fn("mdls_gemm_", "dd")
    import ctypes

    p = ctypes.c_void_p(A.data_ptr())
    assert f(-1, 4, 4, 0, 0, p, 4, 16, p, 4, 16, p, 4, 16, 0, None, 0, None) == -1
    assert f(4, 4, 4, 2, 0, p, 4, 16, p, 4, 16, p, 4, 16, 0, None, 0, None) == -4
    assert f(4, 4, 4, 0, 0, p, 4, 16, p, 4, 16, p, 4, 16, 0, None, 0, None) == -12  # C aliases A


@pytest.mark.parametrize("prec,m,n,k,tb", [("dd", 1024, 1024, 128, 1), ("dd", 600, 700, 300, 0), ("qd", 512, 640, 128, 1),
                                           ("od", 256, 480, 96, 0)])
def test_gemm_stream_k(orc, mdls, dev, prec, m, n, k, tb):
    """One- and two-wave shapes take the stream-K path (tiles x k-tiles split evenly over the CTA slots, a tile's
    last CTA merging the others' partials in k order): sampled entries vs the oracle dots, and the result is
    bitwise identical run to run (fixed segmentation, fixed merge order)."""
    A = inputs.random_matrix(m, k, prec, seed=m + k)
    B = inputs.random_matrix(n if tb else k, k if tb else n, prec, seed=n + k)
    C0 = inputs.random_matrix(m, n, prec, seed=7)
    outs = []
    for _ in range(2):
        outs.append(mdls.gemm(prec, _gpu(A, dev), _gpu(B, dev), C=_gpu(C0, dev).clone(), trans_b=bool(tb), mode=1))
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    Cg = outs[0].cpu().numpy()
    Bop = _op(B, tb)
    rng = np.random.default_rng(3)
    for i, j in zip(rng.integers(0, m, 40), rng.integers(0, n, 40)):
        p = orc.dot(prec, np.ascontiguousarray(A.transpose(0, 2, 1)[:, i, :]), np.ascontiguousarray(Bop[:, :, j]))
        ref = orc.md_op("add", prec, C0[:, j, i][:, None], p[:, None])[:, 0]
        d = orc.md_op("sub", prec, Cg[:, j, i][:, None], ref[:, None])[0, 0]
        scale = float(np.sum(np.abs(A[0, :, i] * Bop[0, :, j]))) + abs(float(C0[0, j, i]))
        assert abs(d) <= 1e3 * k * U_OF[prec] * scale, (i, j, d)
