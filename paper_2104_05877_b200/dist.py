"""Column-sharded randomized LUPP over a torch.distributed process group.

One process per GPU.  A (m x n) is split into contiguous column blocks, rank r owning columns
[col0_r, col0_r + ncols_r) (``shard``).  The path:

  sketch      X_r = Gamma A_r on every rank, no communication: Gamma(r, i) depends only on the
              seed and the row index i of A (R1), which is not sharded, so every rank
              regenerates the same Gamma and X = [X_0, X_1, ...] column-wise (Alg. 2 line 2).
  select_cols three exchange patterns, all equal to single-GPU LUPP on the unsharded sketch
              (ties to the lowest GLOBAL index, R6):
              "step" (the per-step design): the panel stays sharded; at each of the
              k pivot steps every rank proposes its best active row as one record (value,
              global index, the row) and ONE all-gather of P records lets every rank apply the
              same decision to its own rows (sk_lupp_dist_*; ``select_cols_stepwise``;
              ``CapturedStepwise`` replays the k steps as one CUDA graph).
              "replicate" (variant ii): the k sketch rows that column LUPP can read (R5) are
              all-gathered once (k x n doubles) and every rank runs the single-GPU cluster
              LUPP kernel on identical bytes.
              "p2p" (variant i, ``P2PStepwise``): the per-step design with the exchange inside
              the step kernel -- records stored into the peers' mailboxes over NVLink.
  gather C    each rank packs the skeleton columns it owns; ONE all-gather of the packed blocks
              (padded to the largest owner count) gives C = A(:, J_s) on every rank.
  select_rows row LUPP on the replicated C, identical on every rank (Alg. 2 line 4).
  residual    Q = ortho(C) by Cholesky QR distributed over row blocks of the basis (a local Gram
              matrix and ONE k x k all-reduce per pass, one all-gather of the row blocks); each
              rank returns ||A_r - Q Q^T A_r||_F^2 and ||A_r||_F^2 and one sum all-reduce gives the
              global Frobenius residual of the column ID.

On CUDA tensors (backend=None) the library does all of this itself: ``api.DistSession`` creates
a column-sharded context (sk_create_dist) that owns its NCCL communicator and issues every
collective above on its own stream (dist.cu).  With an explicit ``backend`` the same protocol
runs here over torch.distributed -- the multi-process CPU tests substitute a host backend to
exercise it with the gloo backend (tests/test_dist_gloo.py).
"""
import math

import torch
import torch.distributed as dist


def shard(n, world, rank):
    """(col0, ncols) of rank's contiguous column block; block sizes differ by at most one."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, rem = divmod(n, world)
    col0 = rank * base + min(rank, rem)
    return col0, base + (1 if rank < rem else 0)


class CudaBackend:
    """The product backend: every step in libskel.so kernels."""

    def __init__(self):
        from . import api
        self.api = api

    def sketch(self, A_local, l, embedding, seed, zeta):
        return self.api.sketch(A_local, l, embedding, seed, zeta)

    def select_cols(self, Xk, k):
        Js, Lf, U, _ = self.api.select_cols(Xk, k)
        return Js, Lf

    def lupp_dist(self, nloc, k, col0, world, device=None):
        return self.api.LuppDist(nloc, k, col0, world, device)

    def select_rows(self, C, k):
        Is, _, _, _ = self.api.select_rows(C, k)
        return Is

    def gather_cols_shard(self, A_local, Js, col0):
        return self.api.gather_cols_shard(A_local, Js, col0)

    def residual_cols(self, A_local, C):
        return self.api.residual_cols(A_local, C)


def _all_gather_cols(local, n_global, group, world):
    """Concatenate the ranks' column blocks (rows x ncols_r) into rows x n_global, in rank order."""
    rows = local.shape[0]
    nmax = -(-n_global // world)
    buf = torch.zeros((rows, nmax), dtype=local.dtype, device=local.device)
    buf[:, :local.shape[1]] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    cols = []
    for r in range(world):
        _, nc = shard(n_global, world, r)
        cols.append(parts[r][:, :nc])
    return torch.cat(cols, dim=1).contiguous()


def _stepwise_loop(sel, k, group):
    for t in range(1, k + 1):
        dist.all_gather_into_tensor(sel.gathered, sel.cand, group=group)
        sel.step(t)


def select_cols_stepwise(X_local, n_global, k, group=None, backend=None):
    """Column LUPP with one all-gather of P records per pivot step.
    X_local: this rank's l x ncols sketch block (row-major).  Returns (Js replicated, Lf rows of
    this rank's block, U replicated); raises on a rank failure (R7)."""
    backend = backend or CudaBackend()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    col0, nloc = shard(n_global, world, rank)
    if X_local.shape[1] != nloc:
        raise ValueError(f"rank {rank}: X_local has {X_local.shape[1]} columns, shard() expects {nloc}")
    if not (1 <= k <= X_local.shape[0]) or k > n_global:
        raise ValueError("need 1 <= k <= l and k <= n")
    sel = backend.lupp_dist(nloc, k, col0, world, X_local.device.index if X_local.is_cuda else None)
    sel.begin(X_local)
    _stepwise_loop(sel, k, group)
    sel.info()
    return sel.Js, sel.Lf, sel.U


class CapturedStepwise:
    """select_cols_stepwise with begin + the k (all-gather, step) pairs captured once in a CUDA
    graph over fixed buffers (NCCL collectives are graph-capturable): ``run()`` replays it with
    no per-step host work.  ``X_local`` is read at every replay (update it in place)."""

    def __init__(self, X_local, n_global, k, group=None):
        from . import api
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        col0, nloc = shard(n_global, world, rank)
        self.k, self.group, self.X = k, group, X_local
        self.sel = api.LuppDist(nloc, k, col0, world, X_local.device.index)
        self._eager()                                   # warm-up: NCCL communicator, library context
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.sel.begin(self.X)
            _stepwise_loop(self.sel, k, group)

    def _eager(self):
        self.sel.begin(self.X)
        _stepwise_loop(self.sel, self.k, self.group)
        self.sel.info()

    def run(self):
        self.graph.replay()
        return self.sel.Js, self.sel.Lf, self.sel.U


class P2PStepwise:
    """select_cols_stepwise with the exchange INSIDE the step kernel (SURVEY 8(e) variant i): each
    rank owns a mailbox in device memory, maps every peer's mailbox through CUDA IPC (NVLink peer
    memory on one node), and the step kernel stores its record straight into the peers' mailboxes
    and releases a flag -- no collective and no host call between pivot steps.  The group is used
    only once, to exchange the IPC handles.  ``run(X_local)`` -> (Js, Lf, U); ``close()`` unmaps."""

    def __init__(self, n_global, k, group=None, device=None):
        from . import api
        self.api = api
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        col0, nloc = shard(n_global, world, rank)
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.k, self.group, self.world, self.rank = k, group, world, rank
        self.mailbox = api.ipc_alloc(api.mailbox_bytes(k, world), dev.index)
        self.imported = []
        if world == 1:
            ptrs = [self.mailbox]
        else:
            handles = [None] * world
            dist.all_gather_object(handles, api.ipc_export(self.mailbox, dev.index), group=group)
            ptrs = []
            for r in range(world):
                if r == rank:
                    ptrs.append(self.mailbox)
                else:
                    p = api.ipc_import(handles[r], dev.index)
                    self.imported.append(p)
                    ptrs.append(p)
        self.peers = torch.tensor(ptrs, dtype=torch.int64, device=dev)
        self.sel = api.LuppDistP2P(nloc, k, col0, world, rank, self.peers, self.mailbox, dev.index)

    def run(self, X_local):
        self.sel.begin(X_local)
        for t in range(1, self.k + 1):
            self.sel.step(t)
        self.sel.info()
        return self.sel.Js, self.sel.Lf, self.sel.U

    def close(self):
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier(group=self.group)          # no peer still writes into our mailbox
        for p in self.imported:
            self.api.ipc_close(p)
        self.imported = []
        if self.mailbox:
            self.api.ipc_free(self.mailbox)
            self.mailbox = 0


def _owners(Js, n_global, world):
    """Owner rank of every skeleton column and each rank's columns in pivot order (host lists)."""
    blocks = [shard(n_global, world, r) for r in range(world)]
    owner = []
    for j in Js:
        owner.append(next((r for r, (c0, nc) in enumerate(blocks) if c0 <= j < c0 + nc), -1))
    return owner, blocks


def gather_cols_allgather(A_local, Js, n_global, group=None, backend=None):
    """C = A_global(:, J_s) on every rank (S3 on a column-sharded A): every rank packs the
    skeleton columns it owns (in pivot order) into a block padded to the largest owner count, ONE
    all-gather moves the blocks, and C's columns are taken from them in pivot order -- m k doubles
    received per rank, half of what a sum all-reduce of zero-padded copies moves."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    J = [int(j) for j in Js.tolist()]
    owner, blocks = _owners(J, n_global, world)
    col0 = blocks[rank][0]
    cnt = [owner.count(r) for r in range(world)]
    cmax = max(1, max(cnt))
    mine = [j - col0 for j, o in zip(J, owner) if o == rank]
    send = backend.pack_cols(A_local, mine, cmax)                   # (cmax, m): row i = packed column i
    parts = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(parts, send, group=group)
    seen = [0] * world
    cols = []
    for o in owner:
        cols.append(parts[o][seen[o]])
        seen[o] += 1
    return torch.stack(cols, 0).t()                                  # m x k, column-major


def cholqr_rows_dist(B, passes, shift, group=None, backend=None):
    """Q = ortho(B) for a replicated basis B (m x k) by Cholesky QR distributed over row blocks
    (rank r: rows [r mb, (r+1) mb), mb = ceil(m / P)): per pass a local Gram matrix, ONE k x k sum
    all-reduce, the replicated Cholesky factor L and the local solve B_r <- B_r L^{-T} (the first
    pass shifted for shifted CholeskyQR3); one all-gather of the row blocks replicates Q."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    m, k = B.shape
    mb = -(-m // world)
    r0 = min(m, rank * mb)
    Bl = backend.row_block(B, r0, min(mb, m - r0), mb)                # mb x k, zero rows past m
    for p in range(passes):
        G = backend.gram(Bl)
        dist.all_reduce(G, op=dist.ReduceOp.SUM, group=group)
        Bl = backend.chol_right_solve(Bl, G, m if (shift and p == 0) else 0)
    parts = [torch.empty_like(Bl) for _ in range(world)]
    dist.all_gather(parts, Bl.contiguous(), group=group)
    return torch.cat(parts, 0)[:m]


def _dist_rand_lupp_lib(A_local, n_global, k, l, embedding, seed, zeta, rows, residual, group, exchange):
    """The product path: a library-owned column-sharded context (api.DistSession); every exchange
    (sketch rows or per-step records, C's columns, Gram matrices, squared sums) is a collective the
    library issues on its own NCCL communicator."""
    from . import api
    out = {}
    sess = api.DistSession(n_global, group, A_local.device.index, "step" if exchange == "step" else "replicate")
    try:
        with sess:
            out["col0"], out["ncols"] = sess.col0, sess.ncols
            X_local = api.sketch(A_local, l, embedding, seed, zeta)
            if exchange == "p2p":
                p2p = P2PStepwise(n_global, k, group, A_local.device.index)
                try:
                    Js, Lf, _ = p2p.run(X_local)
                finally:
                    p2p.close()
            else:
                Js, Lf, _, _ = api.select_cols(X_local, k)
            out["Js"], out["Lf"] = Js, Lf
            if rows or residual:
                out["C"] = api.gather_cols(A_local, Js)
                if rows:
                    out["Is"] = api.select_rows(out["C"], k)[0]
                if residual:
                    out["residual"], out["normA"] = api.residual(A_local, Js, None, "col_id")
    finally:
        sess.close()
    return out


def dist_rand_lupp(A_local, n_global, k, l, embedding="gaussian", seed=0, zeta=8, rows=False,
                   residual=False, group=None, backend=None, exchange="replicate"):
    """Algorithm 2 on a column-sharded A.  A_local: this rank's block (m x ncols, column-major).

    Returns a dict with J_s (global column indices, replicated), I_s (if rows), the skeleton
    matrix C (replicated, if rows or residual) and the column-ID residual / ||A||_F (if residual).
    backend=None (CUDA tensors): the library's distributed context does everything.  An explicit
    backend runs the same protocol here over torch.distributed (the CPU tests' host backend).
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    col0, ncols = shard(n_global, world, rank)
    m = A_local.shape[0]
    if A_local.shape[1] != ncols:
        raise ValueError(f"rank {rank}: A_local has {A_local.shape[1]} columns, shard() expects {ncols}")
    if not (1 <= k <= l <= m) or k > n_global:
        raise ValueError("need 1 <= k <= l <= m and k <= n")
    if exchange not in ("step", "p2p", "replicate"):
        raise ValueError("exchange must be 'step', 'p2p' or 'replicate'")
    if backend is None:
        return _dist_rand_lupp_lib(A_local, n_global, k, l, embedding, seed, zeta, rows, residual, group, exchange)
    out = {"col0": col0, "ncols": ncols}
    X_local = backend.sketch(A_local, l, embedding, seed, zeta)               # l x ncols
    if exchange == "step":
        Js, Lf, _ = select_cols_stepwise(X_local, n_global, k, group, backend)  # Lf: this rank's rows
    elif exchange == "p2p":
        raise ValueError("exchange='p2p' needs the CUDA library (backend=None)")
    else:
        Xk = _all_gather_cols(X_local[:k], n_global, group, world)            # k x n (rows 0..k-1)
        Js, Lf = backend.select_cols(Xk, k)
    out["Js"] = Js
    out["Lf"] = Lf
    if rows or residual:
        C = gather_cols_allgather(A_local, Js, n_global, group, backend)
        out["C"] = C
        if rows:
            out["Is"] = backend.select_rows(C, k)
        if residual:
            B, passes, shift = backend.basis(C)                              # LUPP basis or C itself
            Q = cholqr_rows_dist(B, passes, shift, group, backend)
            r2, a2 = backend.residual_q(A_local, Q)
            sums = torch.tensor([r2, a2], dtype=torch.float64, device=A_local.device)
            dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
            out["residual"] = math.sqrt(max(float(sums[0]), 0.0))
            out["normA"] = math.sqrt(float(sums[1]))
    return out
