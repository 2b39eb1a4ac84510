"""Column-sharded randomized LUPP over a torch.distributed process group.

One process per GPU.  A (m x n) is split into contiguous column blocks, rank r owning columns
[col0_r, col0_r + ncols_r) (``shard``).  The path:

  sketch      X_r = Gamma A_r on every rank, no communication: Gamma(r, i) depends only on the
              seed and the row index i of A (R1), which is not sharded, so every rank
              regenerates the same Gamma and X = [X_0, X_1, ...] column-wise (Alg. 2 line 2).
  select_cols the k sketch rows that column LUPP can read (R5) are all-gathered
              (k x n doubles, one collective) and every rank runs the same deterministic
              cluster LUPP kernel on identical bytes -> identical J_s on every rank
              ("gather-then-replicate", SURVEY 8(e) variant ii).  Ties go to the lowest GLOBAL
              index (R6), so the result equals single-GPU LUPP on the unsharded sketch.
  gather C    each rank writes the skeleton columns it owns (zeros elsewhere,
              sk_gather_cols_shard) and a sum all-reduce assembles C = A(:, J_s) exactly.
  select_rows row LUPP on the replicated C, identical on every rank (Alg. 2 line 4).
  residual    Q = ortho(C) is computed identically on every rank; each rank returns
              ||A_r - Q Q^T A_r||_F^2 and ||A_r||_F^2 (sk_residual_cols) and one sum all-reduce
              gives the global Frobenius residual of the column ID.

All arithmetic runs in the library kernels (``backend``); this module only moves tensors
between ranks.  The backend is an object with the library's call signatures; the default is
the CUDA library (paper_2104_05877_b200.api).  The multi-process CPU tests substitute a
host backend to exercise this protocol with the gloo backend (tests/test_dist_gloo.py).
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


def dist_rand_lupp(A_local, n_global, k, l, embedding="gaussian", seed=0, zeta=8, rows=False,
                   residual=False, group=None, backend=None):
    """Algorithm 2 on a column-sharded A.  A_local: this rank's block (m x ncols, column-major).

    Returns a dict with J_s (global column indices, replicated), I_s (if rows), the skeleton
    matrix C (replicated, if rows or residual) and the column-ID residual / ||A||_F (if residual).
    """
    backend = backend or CudaBackend()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    col0, ncols = shard(n_global, world, rank)
    m = A_local.shape[0]
    if A_local.shape[1] != ncols:
        raise ValueError(f"rank {rank}: A_local has {A_local.shape[1]} columns, shard() expects {ncols}")
    if not (1 <= k <= l <= m) or k > n_global:
        raise ValueError("need 1 <= k <= l <= m and k <= n")
    out = {"col0": col0, "ncols": ncols}
    X_local = backend.sketch(A_local, l, embedding, seed, zeta)               # l x ncols
    Xk = _all_gather_cols(X_local[:k], n_global, group, world)                # k x n (rows 0..k-1)
    Js, Lf = backend.select_cols(Xk, k)
    out["Js"] = Js
    out["Lf"] = Lf
    if rows or residual:
        C = backend.gather_cols_shard(A_local, Js, col0)                      # m x k, zeros off-shard
        Ct = C.t().contiguous()                                                # k x m: row t = column t of C
        dist.all_reduce(Ct, op=dist.ReduceOp.SUM, group=group)                 # exact: one owner per column
        C = Ct.t()                                                             # column-major m x k
        out["C"] = C
        if rows:
            out["Is"] = backend.select_rows(C, k)
        if residual:
            r2, a2 = backend.residual_cols(A_local, C)
            sums = torch.tensor([r2, a2], dtype=torch.float64, device=Xk.device)
            dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
            out["residual"] = math.sqrt(max(float(sums[0]), 0.0))
            out["normA"] = math.sqrt(float(sums[1]))
    return out
