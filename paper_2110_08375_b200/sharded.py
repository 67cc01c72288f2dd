"""Block-column sharded least squares over P ranks (north_star multi-GPU).

Host orchestration only: every arithmetic step is a libmdls call (``qr_panel``,
``qr_update``, ``qt_b``, ``backsub``) and every exchange is byte movement
through ``torch.distributed`` (NCCL over NVLink on GPUs; gloo in the CPU tests),
never an md sum inside a collective.

Algorithm 2 distributed by panels: panel k (columns [k nb,
(k+1) nb)) lives on rank k mod P.  With look-ahead, step k is
  1. (critical stream) the owner of panel k+1 applies panel k to panel k+1 only,
     factors panel k+1 (A1-A3) and the owner broadcasts W_{k+1}, Y_{k+1};
  2. (bulk stream) every rank applies panel k to its panels beyond k+1
     (A4, C += Y (W^T C)), one panel per call,
so the factorisation of panel k+1 and its broadcast overlap the bulk of step k.
W_k and Y_k are zero above row k nb: only rows k nb..M-1 are stored and
broadcast (row-trimmed buffers, include/mdls.h).  Every update is issued one
panel (nb columns) at a time, so each column block sees exactly the same
launches whatever P is: the sharded result is bitwise independent of the rank
count (tests/test_gpu_sharded.py).
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

from contextlib import nullcontext
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
        self._work = {}  # (stream, prec, M, nb) -> scratch of one panel (one per stream: they run concurrently)

    def _scratch(self, prec, M, nb, device):
        import torch

        key = (torch.cuda.current_stream(device).cuda_stream, prec, M, nb)
        if key not in self._work:
            self._work[key] = torch.empty(self.mdls.workspace_bytes(prec, 0, M, nb, nb), dtype=torch.uint8,
                                          device=device)
        return self._work[key]

    def panel(self, prec, A, col0, k, nb, W, Y):
        return self.mdls.qr_panel(prec, A, col0, k, nb, W, Y, work=self._scratch(prec, A.shape[2], nb, A.device))

    def update(self, prec, Wk, Yk, A, k, nb, c0, c1):
        self.mdls.qr_update(prec, Wk, Yk, A, k, nb, c0, c1, work=self._scratch(prec, A.shape[2], nb, A.device))

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


class Streams:
    """The critical (look-ahead panel) and bulk (trailing update) streams of this process on a GPU; no-ops on
    CPU tensors.  The critical stream has the higher priority."""

    def __init__(self, device=None):
        import torch

        self.gpu = device is not None and torch.device(device).type == "cuda"
        if self.gpu:
            self.crit = torch.cuda.Stream(device=device, priority=-1)
            self.bulk = torch.cuda.Stream(device=device, priority=0)
            self.crit.wait_stream(torch.cuda.current_stream(device))
            self.bulk.wait_stream(torch.cuda.current_stream(device))

    def on(self, which):
        import torch

        return torch.cuda.stream(getattr(self, which)) if self.gpu else nullcontext()

    def record(self, which):
        return getattr(self, which).record_event() if self.gpu else None

    def wait(self, which, ev):
        if self.gpu and ev is not None:
            getattr(self, which).wait_event(ev)

    def join(self):
        import torch

        if self.gpu:
            cur = torch.cuda.current_stream(self.crit.device)
            cur.wait_stream(self.crit)
            cur.wait_stream(self.bulk)


def sharded_qr(st: ShardState, A_loc: dict, ops: Ops, comm: Comm | None, new_empty, streams: Streams | None = None):
    """Factor in place.  A_loc[r]: (m, n_loc_cols, M) tensor of rank r's panels.  Returns (W, Y, info): lists
    over k of the row-trimmed (m, nb, M - k nb) panel factors (every local rank sees every panel) and the
    owners' panel info tensors.  new_empty(shape) allocates a float64 tensor (zeroed)."""
    m = {"dd": 2, "qd": 4, "od": 8}[st.prec]
    N = st.K // st.nb
    nb = st.nb
    local = sorted(A_loc)
    S = streams if streams is not None else Streams(None)
    W, Y, infos = [None] * N, [None] * N, []
    bulk_done = {}  # (rank, k): bulk updates of step k issued on this rank

    def factor_and_broadcast(k):  # on the critical stream
        o = owner(k, st.P)
        Wk = new_empty((m, nb, st.M - k * nb))
        Yk = new_empty((m, nb, st.M - k * nb))
        if o in local:
            infos.append(ops.panel(st.prec, A_loc[o], st.panels[o].index(k) * nb, k, nb, Wk, Yk))
        if comm is not None:
            comm.broadcast([Wk, Yk], src=o)
        W[k], Y[k] = Wk, Yk
        return S.record("crit")

    with S.on("crit"):
        ev_panel = factor_and_broadcast(0)
    for k in range(N):
        ev_next = None
        if k + 1 < N:
            o1 = owner(k + 1, st.P)
            with S.on("crit"):
                if o1 in local:
                    # panel k+1 received the panels < k through the bulk of step k-1
                    S.wait("crit", bulk_done.get((o1, k - 1)))
                    j = st.panels[o1].index(k + 1)
                    ops.update(st.prec, W[k], Y[k], A_loc[o1], k, nb, j * nb, (j + 1) * nb)
                ev_next = factor_and_broadcast(k + 1)
        with S.on("bulk"):
            S.wait("bulk", ev_panel)  # W_k, Y_k factored and broadcast
            for r in local:
                for j, kk in enumerate(st.panels[r]):
                    if kk > k + 1:
                        ops.update(st.prec, W[k], Y[k], A_loc[r], k, nb, j * nb, (j + 1) * nb)
                bulk_done[(r, k)] = S.record("bulk")
        ev_panel = ev_next
    S.join()
    return W, Y, infos


def sharded_form_q(st: ShardState, W, Y, ops: Ops, new_empty, local_ranks):
    """Q(:, own column blocks) by backward accumulation Q_tr += W_k (Y_k^T Q_tr), one column block per call."""
    m = {"dd": 2, "qd": 4, "od": 8}[st.prec]
    nb = st.nb
    Q = {}
    for r in local_ranks:
        cols = local_q_columns(st, r)
        Q[r] = new_empty((m, len(cols), st.M))
        ops.identity_cols(st.prec, Q[r], cols)
    N = st.K // nb
    for k in range(N - 1, -1, -1):
        for r in local_ranks:
            for j, q in enumerate(st.qblocks[r]):
                if q >= k:  # exchanged roles: C += W_k (Y_k^T C)
                    c1 = min((j + 1) * nb, Q[r].shape[1])
                    ops.update(st.prec, Y[k], W[k], Q[r], k, nb, j * nb, c1)
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
                  new_empty, streams: Streams | None = None):
    """x = argmin ||b - A x|| with A column-sharded over P ranks (A_loc[r] holds the
    columns local_columns(st, r)).  Every rank returns the same x (and R, y, info: the
    minimum-positive-or-zero combination of the owners' panel infos and the back substitution's)."""
    st = plan(prec, M, K, nb, P)
    W, Y, pinfo = sharded_qr(st, A_loc, ops, comm, new_empty, streams)
    local = sorted(A_loc)
    Q = sharded_form_q(st, W, Y, ops, new_empty, local)
    # Q^T b: own column blocks (one block per call), then all-gather the slices (byte movement)
    ysl = {}
    for r in local:
        parts = [ops.qt_b_cols(prec, Q[r][:, j * nb:(j + 1) * nb].contiguous(), b)
                 for j in range(-(-Q[r].shape[1] // nb))]
        ysl[r] = (parts[0] if len(parts) == 1 else _cat1(parts))[:, :, None]
    y = gather_columns(st, ysl, local_q_columns, comm, M, new_empty)[:, :, 0].contiguous()
    # R: all-gather the factored panels, back substitution on the leading K x K
    F = gather_columns(st, {r: A_loc[r] for r in local}, local_columns, comm, K, new_empty).contiguous()
    x, info = ops.backsub(prec, F, y, nb)
    info = _combine_info(info, pinfo, comm)
    return x, F, y, info


def _cat1(parts):
    import torch

    return torch.cat(parts, dim=1)


def _combine_info(info, pinfo, comm):
    """Fold the panel infos (first zero/non-finite R_jj, 1-based global row; 0 = fine) into the back
    substitution's: the smallest positive code wins (every rank gets the same value)."""
    import torch

    if not isinstance(info, torch.Tensor):
        return info
    big = 1 << 30
    v = info.reshape(-1)[:1].clone().to(torch.int64)
    v = torch.where(v > 0, v, torch.full_like(v, big))
    for pi in pinfo:
        p = pi.reshape(-1)[:1].to(torch.int64)
        v = torch.minimum(v, torch.where(p > 0, p, torch.full_like(p, big)))
    if comm is not None:
        comm.dist.all_reduce(v, op=comm.dist.ReduceOp.MIN, group=comm.group)
    return torch.where(v == big, torch.zeros_like(v), v).to(info.dtype)
