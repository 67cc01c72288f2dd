"""Batch sharding host logic (paper_2110_08375_b200/batch.py) on CPU: the shard
blocks partition the batch exactly, and a world_size-2 gloo run that solves its
shard (plain fp64 stand-in solver on limb 0, test-only) and all-gathers the
solutions reproduces the single-rank result bit for bit."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_08375_b200 import batch


@pytest.mark.parametrize("B", [0, 1, 5, 7, 256])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_partition(B, world):
    seen = []
    sizes = []
    for r in range(world):
        lo, hi = batch.shard_range(B, r, world)
        assert 0 <= lo <= hi <= B
        seen.extend(range(lo, hi))
        sizes.append(hi - lo)
    assert seen == list(range(B))  # contiguous, in rank order, each problem exactly once
    assert max(sizes) - min(sizes) <= 1


def test_shard_bad_args():
    with pytest.raises(ValueError):
        batch.shard_range(4, 2, 2)
    with pytest.raises(ValueError):
        batch.shard_range(4, 0, 0)


M, K = 12, 8


def _problem(p):
    rng = np.random.default_rng(1000 + p)
    A = np.zeros((2, K, M))
    b = np.zeros((2, M))
    A[0] = rng.uniform(-1, 1, (K, M))
    b[0] = rng.uniform(-1, 1, M)
    return A, b


def _plain_solver(prec, A, b, nb, form_q=True, groups=1):
    xs = []
    for p in range(A.shape[0]):
        a = A[p, 0].numpy().T
        x, *_ = np.linalg.lstsq(a, b[p, 0].numpy(), rcond=None)
        xx = np.zeros((2, K))
        xx[0] = x
        xs.append(xx)
    return torch.from_numpy(np.stack(xs)), torch.zeros(A.shape[0], dtype=torch.int32)


def _worker(rank, world, B, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi, x, info = batch.solve_shard("dd", _problem, B, rank, world, nb=4, solver=_plain_solver)
    if x is None:
        x = torch.zeros((0, 2, K), dtype=torch.float64)
    xall = batch.gather_solutions(x, B, rank, world)
    if rank == 0:
        torch.save(xall, out)
    dist.destroy_process_group()


@pytest.mark.parametrize("B", [5, 8])
def test_gloo_world2_matches_single(tmp_path, B):
    out = str(tmp_path / "x.pt")
    port = 29631 + B
    mp.spawn(_worker, args=(2, B, port, out), nprocs=2, join=True)
    xall = torch.load(out)
    _, _, xs, _ = batch.solve_shard("dd", _problem, B, 0, 1, nb=4, solver=_plain_solver)
    assert xall.shape == (B, 2, K)
    assert torch.equal(xall, xs)
