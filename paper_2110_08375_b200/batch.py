"""Batch sharding of independent least-squares problems across GPUs (SURVEY 8(e),
BASELINE config 5b: a batch of 256 dd 1024 x 1024 solves).

Each rank owns a contiguous, balanced block of problem indices (`shard_range`);
it solves them with one `mdls_lstsq_batched_<p>` call (several problems in
flight on the GPU's stream groups); no collective touches the data path.  The
solutions are gathered only on request (`gather_solutions`, a byte movement over
the process group), e.g. to hand the whole batch to one consumer.  Problem p is
generated from seed p, so any rank layout produces the same batch.
"""
from __future__ import annotations


def shard_range(batch: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of the problems owned by `rank`: contiguous blocks whose sizes differ by at most one."""
    if world < 1 or not (0 <= rank < world) or batch < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_solutions(x_local, batch: int, rank: int, world: int, group=None):
    """All-gather the per-rank solution blocks (B_r, m, K) into the whole batch (batch, m, K) on every rank.
    Blocks are padded to the largest shard for the collective and trimmed afterwards."""
    import torch
    import torch.distributed as dist

    sizes = [shard_range(batch, r, world) for r in range(world)]
    cap = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((cap,) + tuple(x_local.shape[1:]), dtype=x_local.dtype, device=x_local.device)
    pad[: x_local.shape[0]] = x_local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([parts[r][: hi - lo] for r, (lo, hi) in enumerate(sizes)], dim=0)


def solve_shard(prec: str, make_problem, batch: int, rank: int, world: int, nb: int, groups: int = 4,
                form_q: bool = True, device=None, solver=None):
    """Solve this rank's block of the batch.  make_problem(p) -> (A_p, b_p) host arrays of problem p;
    solver(prec, A (B_r, m, K, M), b (B_r, m, M), nb, form_q, groups) -> (x, info), by default the library's
    lstsq_batched.  Returns (lo, hi, x, info)."""
    import numpy as np
    import torch

    lo, hi = shard_range(batch, rank, world)
    if solver is None:
        from . import lstsq_batched as solver
    if hi == lo:
        return lo, hi, None, None
    probs = [make_problem(p) for p in range(lo, hi)]
    A = torch.from_numpy(np.stack([a for a, _ in probs]))
    b = torch.from_numpy(np.stack([bb for _, bb in probs]))
    if device is not None:
        A, b = A.to(device), b.to(device)
    x, info = solver(prec, A, b, nb, form_q=form_q, groups=groups)
    return lo, hi, x, info
