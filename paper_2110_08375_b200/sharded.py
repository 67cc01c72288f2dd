"""Block-column sharded least squares over P ranks (north_star multi-GPU).

Host orchestration only: every arithmetic step is a libmdls call (``qr_panel``,
``qr_update``, ``qt_b``, ``backsub``) and every exchange is byte movement
through ``torch.distributed`` (NCCL over NVLink on GPUs; gloo in the CPU tests),
never an md sum inside a collective.

Algorithm 2 distributed by panels: panel k (columns [k nb,
(k+1) nb)) lives on rank k mod P.  For k = 0..N-1:
  1. the owner factors panel k (A1-A3)                 -> W_k, Y_k (M x nb each)
  2. broadcast W_k, Y_k from the owner                  (NCCL broadcast)
  3. every rank applies panel k to its panels > k      (A4, C += Y (W^T C))
Q formation (A5) is column-sharded without further communication: every rank
keeps all (W_k, Y_k) and accumulates Q(:, own column blocks) backward,
Q_tr += W_k (Y_k^T Q_tr).  Q^T b (A6): y(own blocks) = Q(:, own)^T b, then an
all-gather of the slices.  Back substitution (A7-A9, about 1/100 of the QR work
at 1024) runs on every rank after an all-gather of R's panels.

The same driver serves P "virtual" ranks in one process (``local_ranks`` with
several entries, ``comm=None``): broadcasts become shared references.  That is
how the sharded path is exercised on a single GPU.
"""
from __future__ import annotations

from dataclasses import dataclass, field


class Ops:
    """The per-rank compute steps.  GpuOps maps them onto libmdls; tests may
    substitute plain implementations to check the orchestration on CPU."""

    def panel(self, prec, A, col0, k, nb, W, Y):  # pragma: no cover - interface
        raise NotImplementedError

    def update(self, prec, Wk, Yk, A, k, nb, c0, c1):  # pragma: no cover
        raise NotImplementedError

    def identity_cols(self, prec, Q, cols):  # pragma: no cover
        raise NotImplementedError

    def qt_b_cols(self, prec, Q, b):  # pragma: no cover
        raise NotImplementedError

    def backsub(self, prec, R, y, nb):  # pragma: no cover
        raise NotImplementedError


class GpuOps(Ops):
    def __init__(self):
        import paper_2110_08375_b200 as mdls

        self.mdls = mdls

    def panel(self, prec, A, col0, k, nb, W, Y):
        return self.mdls.qr_panel(prec, A, col0, k, nb, W, Y)

    def update(self, prec, Wk, Yk, A, k, nb, c0, c1):
        self.mdls.qr_update(prec, Wk, Yk, A, k, nb, c0, c1)

    def identity_cols(self, prec, Q, cols):
        import torch

        Q.zero_()
        if len(cols):
            idx = torch.arange(len(cols), device=Q.device)
            Q[0, idx, torch.tensor(cols, device=Q.device)] = 1.0

    def qt_b_cols(self, prec, Q, b):
        return self.mdls.qt_b(prec, Q, b)

    def backsub(self, prec, R, y, nb):
        return self.mdls.backsub(prec, R, y, nb)


@dataclass
class ShardState:
    prec: str
    M: int
    K: int
    nb: int
    P: int
    panels: dict = field(default_factory=dict)   # rank -> global panel indices owned (ascending)
    qblocks: dict = field(default_factory=dict)  # rank -> global Q column blocks owned


def owner(k: int, P: int) -> int:
    return k % P


def plan(prec: str, M: int, K: int, nb: int, P: int) -> ShardState:
    if K % nb or M < K:
        raise ValueError("need nb | K and M >= K")
    N = K // nb
    st = ShardState(prec, M, K, nb, P)
    nqb = -(-M // nb)
    for r in range(P):
        st.panels[r] = [k for k in range(N) if owner(k, P) == r]
        st.qblocks[r] = [q for q in range(nqb) if owner(q, P) == r]
    return st


def local_columns(st: ShardState, r: int):
    """global column indices held by rank r, in local order"""
    return [k * st.nb + c for k in st.panels[r] for c in range(st.nb)]


def local_q_columns(st: ShardState, r: int):
    return [q * st.nb + c for q in st.qblocks[r] for c in range(st.nb) if q * st.nb + c < st.M]


class Comm:
    """torch.distributed wrapper (rank-local tensors); None = virtual ranks."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def broadcast(self, tensors, src):
        for t in tensors:
            self.dist.broadcast(t, src=src, group=self.group)

    def all_gather(self, t):
        out = [t.new_empty(t.shape) for _ in range(self.size)]
        self.dist.all_gather(out, t.contiguous(), group=self.group)
        return out


def sharded_qr(st: ShardState, A_loc: dict, ops: Ops, comm: Comm | None, new_empty):
    """Factor in place.  A_loc[r]: (m, n_loc_cols, M) tensor of rank r's panels.
    Returns (W, Y): lists over k of (m, nb, M) panel factors (every local rank
    sees every panel).  new_empty(shape) allocates a float64 tensor."""
    m = {"dd": 2, "qd": 4, "od": 8}[st.prec]
    N = st.K // st.nb
    local = sorted(A_loc)
    W, Y = [], []
    for k in range(N):
        o = owner(k, st.P)
        Wk = new_empty((m, st.nb, st.M))
        Yk = new_empty((m, st.nb, st.M))
        if o in local:
            lk = st.panels[o].index(k)
            ops.panel(st.prec, A_loc[o], lk * st.nb, k, st.nb, Wk, Yk)
        if comm is not None:
            comm.broadcast([Wk, Yk], src=o)
        for r in local:  # trailing update of the panels > k this rank holds
            later = [i for i, kk in enumerate(st.panels[r]) if kk > k]
            if later:
                ops.update(st.prec, Wk, Yk, A_loc[r], k, st.nb, later[0] * st.nb, len(st.panels[r]) * st.nb)
        W.append(Wk)
        Y.append(Yk)
    return W, Y


def sharded_form_q(st: ShardState, W, Y, ops: Ops, new_empty, local_ranks):
    """Q(:, own column blocks) by backward accumulation Q_tr += W_k (Y_k^T Q_tr)."""
    m = {"dd": 2, "qd": 4, "od": 8}[st.prec]
    Q = {}
    for r in local_ranks:
        cols = local_q_columns(st, r)
        Q[r] = new_empty((m, len(cols), st.M))
        ops.identity_cols(st.prec, Q[r], cols)
    N = st.K // st.nb
    for k in range(N - 1, -1, -1):
        for r in local_ranks:
            cols = local_q_columns(st, r)
            first = next((i for i, c in enumerate(cols) if c >= k * st.nb), len(cols))
            # exchanged roles: C += W_k (Y_k^T C)
            ops.update(st.prec, Y[k], W[k], Q[r], k, st.nb, first, len(cols))
    return Q


def gather_columns(st: ShardState, pieces: dict, cols_of, comm: Comm | None, total: int, new_empty):
    """Assemble a (m, total, L) array from per-rank column pieces (all ranks get it)."""
    import torch

    ranks = range(st.P)
    some = next(iter(pieces.values()))
    m, L = some.shape[0], some.shape[2]
    if comm is not None:
        sizes = [len(cols_of(st, r)) for r in ranks]
        pad = new_empty((m, max(sizes), L))
        mine = pieces[comm.rank]
        pad[:, :mine.shape[1]] = mine
        parts = comm.all_gather(pad)
        pieces = {r: parts[r][:, :sizes[r]] for r in ranks}
    out = new_empty((m, total, L))
    for r, t in pieces.items():
        idx = torch.tensor(cols_of(st, r), dtype=torch.long, device=t.device)
        out[:, idx] = t
    return out


def sharded_lstsq(prec: str, A_loc: dict, b, M: int, K: int, nb: int, P: int, ops: Ops, comm: Comm | None,
                  new_empty):
    """x = argmin ||b - A x|| with A column-sharded over P ranks (A_loc[r] holds the
    columns local_columns(st, r)).  Every rank returns the same x (and R, y)."""
    st = plan(prec, M, K, nb, P)
    W, Y = sharded_qr(st, A_loc, ops, comm, new_empty)
    local = sorted(A_loc)
    Q = sharded_form_q(st, W, Y, ops, new_empty, local)
    # Q^T b: own column blocks, then all-gather the slices (byte movement)
    ysl = {r: ops.qt_b_cols(prec, Q[r], b)[:, :, None] for r in local}
    y = gather_columns(st, ysl, local_q_columns, comm, M, new_empty)[:, :, 0].contiguous()
    # R: all-gather the factored panels, back substitution on the leading K x K
    F = gather_columns(st, {r: A_loc[r] for r in local}, local_columns, comm, K, new_empty).contiguous()
    x, info = ops.backsub(prec, F, y, nb)
    return x, F, y, info
