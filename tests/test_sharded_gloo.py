"""Block-column sharded QR orchestration (paper_2110_08375_b200/sharded.py) on
CPU: world_size 2 over gloo, and P virtual ranks in one process.

The compute steps are replaced by plain fp64 test implementations (numpy
Householder on the leading limb) so the HOST logic is what is checked: panel
ownership, broadcast of W/Y from the owner, which columns each rank updates,
backward column-sharded Q formation and the all-gather of Q^T b.  The result
must reproduce the unsharded computation: A = Q R, Q^T Q = I, R upper
triangular with R_jj >= 0, and the same R as a single-rank run.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_08375_b200 import sharded


class PlainOps(sharded.Ops):
    """fp64 stand-ins for the libmdls steps (test-only; limb 0 carries the value)."""

    def panel(self, prec, A, col0, k, nb, W, Y):
        a = A[0].numpy().T  # (M, cols) view -> work on a copy of the panel
        M = a.shape[0]
        j0 = k * nb
        P = a[:, col0:col0 + nb].copy()
        Ym = np.zeros((M, nb))
        betas = np.zeros(nb)
        for l in range(nb):
            j = j0 + l
            x = P[j:, l].copy()
            sigma = float(x[1:] @ x[1:])
            v = np.concatenate([[1.0], x[1:]])
            if sigma == 0.0:
                beta, mu = 0.0, x[0]
            else:
                mu = np.sqrt(x[0] ** 2 + sigma)
                v1 = x[0] - mu if x[0] <= 0 else -sigma / (x[0] + mu)
                beta = 2 * v1 ** 2 / (sigma + v1 ** 2)
                v = np.concatenate([[v1], x[1:]]) / v1
            P[j:, l:] -= beta * np.outer(v, v @ P[j:, l:])
            P[j, l] = mu
            P[j + 1:, l] = v[1:]
            Ym[j:, l] = v
            betas[l] = beta
        # W by the paper's recurrence z = -beta (v + W Y^T v)
        Wm = np.zeros((M, nb))
        for l in range(nb):
            v = Ym[:, l]
            Wm[:, l] = -betas[l] * (v + Wm[:, :l] @ (Ym[:, :l].T @ v))
        A[0, col0:col0 + nb, :] = torch.from_numpy(P.T.copy())
        r0 = M - W.shape[2]  # row-trimmed panel buffers hold rows r0..M-1
        W.zero_()
        Y.zero_()
        W[0] = torch.from_numpy(Wm.T[:, r0:].copy())
        Y[0] = torch.from_numpy(Ym.T[:, r0:].copy())

    def update(self, prec, Wk, Yk, A, k, nb, c0, c1):
        if c1 <= c0:
            return
        j0 = k * nb
        r0 = A.shape[2] - Wk.shape[2]
        C = A[0, c0:c1, j0:].numpy().T  # (rows, cols)
        Wm = Wk[0, :, j0 - r0:].numpy().T
        Ym = Yk[0, :, j0 - r0:].numpy().T
        C2 = C + Ym @ (Wm.T @ C)
        A[0, c0:c1, j0:] = torch.from_numpy(C2.T.copy())

    def identity_cols(self, prec, Q, cols):
        Q.zero_()
        for j, c in enumerate(cols):
            Q[0, j, c] = 1.0

    def qt_b_cols(self, prec, Q, b):
        y = torch.zeros((Q.shape[0], Q.shape[1]), dtype=torch.float64)
        y[0] = torch.from_numpy(Q[0].numpy() @ b[0].numpy())
        return y

    def backsub(self, prec, R, y, nb):
        K = R.shape[1]
        U = np.triu(R[0].numpy().T[:K, :K])
        x = torch.zeros((R.shape[0], K), dtype=torch.float64)
        x[0] = torch.from_numpy(np.linalg.solve(U, y[0].numpy()[:K]))
        return x, 0


def run_sharded(A, nb, P, local_ranks, comm):
    m, K, M = A.shape
    st = sharded.plan("dd", M, K, nb, P)
    A_loc = {r: A[:, sharded.local_columns(st, r), :].clone() for r in local_ranks}
    new = lambda shape: torch.zeros(shape, dtype=torch.float64)
    W, Y, _ = sharded.sharded_qr(st, A_loc, PlainOps(), comm, new)
    Q = sharded.sharded_form_q(st, W, Y, PlainOps(), new, local_ranks)
    return st, A_loc, Q


def _check(A, st, A_loc, Q, local_ranks):
    m, K, M = A.shape
    R = np.zeros((K, M))
    for r in local_ranks:
        R[sharded.local_columns(st, r)] = A_loc[r][0].numpy()
    R = np.triu(R.T[:K, :K])  # (K, K) upper part
    Qf = np.zeros((M, M))
    for r in local_ranks:
        Qf[:, sharded.local_q_columns(st, r)] = Q[r][0].numpy().T
    return R, Qf


def _problem(M, K, seed=0):
    g = np.random.default_rng(seed)
    A = np.zeros((2, K, M))
    A[0] = g.uniform(-1, 1, size=(K, M))
    return torch.from_numpy(A)


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_virtual_ranks_reproduce_qr(P):
    M, K, nb = 48, 32, 8
    A = _problem(M, K)
    st, A_loc, Q = run_sharded(A, nb, P, list(range(P)), None)
    R, Qf = _check(A, st, A_loc, Q, list(range(P)))
    A0 = A[0].numpy().T
    assert np.allclose(Qf[:, :K] @ R, A0, atol=1e-12)
    assert np.allclose(Qf.T @ Qf, np.eye(M), atol=1e-12)
    assert np.all(np.diag(R) > 0)
    # identical to the single-rank result (ownership does not change the arithmetic)
    st1, A1, Q1 = run_sharded(A, nb, 1, [0], None)
    R1, Qf1 = _check(A, st1, A1, Q1, [0])
    assert np.array_equal(R, R1) and np.array_equal(Qf, Qf1)


def test_plan_ownership():
    st = sharded.plan("dd", 1024, 1024, 128, 3)
    assert st.panels == {0: [0, 3, 6], 1: [1, 4, 7], 2: [2, 5]}
    cols = sorted(c for r in range(3) for c in sharded.local_columns(st, r))
    assert cols == list(range(1024))
    qcols = sorted(c for r in range(3) for c in sharded.local_q_columns(st, r))
    assert qcols == list(range(1024))


def _worker(rank, world, port, M, K, nb, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = _problem(M, K)
        comm = sharded.Comm()
        st, A_loc, Q = run_sharded(A, nb, world, [rank], comm)
        # gather every rank's R columns and Q columns to rank 0 (byte movement)
        Rl = A_loc[rank].contiguous()
        Ql = Q[rank].contiguous()
        sizes = [len(sharded.local_columns(st, r)) for r in range(world)]
        qsizes = [len(sharded.local_q_columns(st, r)) for r in range(world)]
        padR = torch.zeros((2, max(sizes), M), dtype=torch.float64)
        padR[:, :Rl.shape[1]] = Rl
        padQ = torch.zeros((2, max(qsizes), M), dtype=torch.float64)
        padQ[:, :Ql.shape[1]] = Ql
        gR = [torch.zeros_like(padR) for _ in range(world)]
        gQ = [torch.zeros_like(padQ) for _ in range(world)]
        dist.all_gather(gR, padR)
        dist.all_gather(gQ, padQ)
        if rank == 0:
            A_all = {r: gR[r][:, :sizes[r]] for r in range(world)}
            Q_all = {r: gQ[r][:, :qsizes[r]] for r in range(world)}
            R, Qf = _check(A, st, A_all, Q_all, list(range(world)))
            np.save(out + "_R.npy", R)
            np.save(out + "_Q.npy", Qf)
    finally:
        dist.destroy_process_group()


def test_gloo_world2(tmp_path):
    M, K, nb = 40, 32, 8
    port = 29500 + os.getpid() % 1000
    out = str(tmp_path / "res")
    mp.start_processes(_worker, args=(2, port, M, K, nb, out), nprocs=2, join=True, start_method="spawn")
    R = np.load(out + "_R.npy")
    Qf = np.load(out + "_Q.npy")
    A = _problem(M, K)
    st1, A1, Q1 = run_sharded(A, nb, 1, [0], None)
    R1, Qf1 = _check(A, st1, A1, Q1, [0])
    assert np.array_equal(R, R1)
    assert np.array_equal(Qf, Qf1)
    assert np.allclose(Qf[:, :K] @ R, A[0].numpy().T, atol=1e-12)


@pytest.mark.parametrize("P", [1, 3])
def test_sharded_lstsq_virtual(P):
    M, K, nb = 40, 24, 8
    A = _problem(M, K, seed=4)
    g = np.random.default_rng(5)
    b = torch.zeros((2, M), dtype=torch.float64)
    b[0] = torch.from_numpy(g.uniform(-1, 1, M))
    st = sharded.plan("dd", M, K, nb, P)
    A_loc = {r: A[:, sharded.local_columns(st, r), :].clone() for r in range(P)}
    new = lambda shape: torch.zeros(shape, dtype=torch.float64)
    x, F, y, info = sharded.sharded_lstsq("dd", A_loc, b, M, K, nb, P, PlainOps(), None, new)
    x_ref = np.linalg.lstsq(A[0].numpy().T, b[0].numpy(), rcond=None)[0]
    assert np.allclose(x[0].numpy(), x_ref, atol=1e-12)
