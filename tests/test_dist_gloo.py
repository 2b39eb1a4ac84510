"""The column-sharded path on CPU: the merge rule and the rank protocol.

* oracle.dist (per-step exchange with the lowest-global-index merge rule) == single-process LUPP,
  pivots and factors bit for bit, including exact ties that straddle a shard boundary.
* paper_2104_05877_b200.dist.dist_rand_lupp over world-size-2 and -3 gloo groups, with a host
  backend built from the oracle standing in for the CUDA kernels, reproduces the unsharded oracle
  path: J_s, C = A(:, J_s) (one all-gather of the owners' packed columns), I_s and the column-ID
  residual (Q by Cholesky QR distributed over row blocks: k x k all-reduces + one all-gather),
  with the gather-then-replicate and the per-step exchanges.
"""
import math
import os
import socket

import numpy as np
import pytest
import scipy.linalg as sla
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from inputs import kahan_witness, make_c1
from oracle import dist as o_dist
from oracle import lupp as o_lupp
from oracle import residual as o_res
from oracle import sketch as o_sketch
from paper_2104_05877_b200.dist import dist_rand_lupp, shard


@pytest.mark.parametrize("n,world", [(10, 3), (4096, 8), (7, 7), (5, 1), (1000, 6)])
def test_shard_partitions_columns(n, world):
    blocks = [shard(n, world, r) for r in range(world)]
    assert blocks[0][0] == 0
    for (c0, nc), (c1, _) in zip(blocks, blocks[1:]):
        assert c0 + nc == c1
    assert sum(nc for _, nc in blocks) == n
    assert max(nc for _, nc in blocks) - min(nc for _, nc in blocks) <= 1


@pytest.mark.parametrize("splits", [[40], [13, 27], [10, 10, 10, 10], [1, 38, 1]])
def test_sharded_merge_rule_equals_single_lupp(splits):
    rng = np.random.default_rng(len(splits))
    X = rng.standard_normal((12, sum(splits)))
    blocks = np.split(X, np.cumsum(splits)[:-1], axis=1)
    piv_d, Lf_d, U_d = o_dist.select_cols_sharded(blocks, 10)
    piv, Lf, U, _ = o_lupp.select_cols(X, 10)
    assert piv.tolist() == piv_d.tolist()
    np.testing.assert_array_equal(Lf, Lf_d)
    np.testing.assert_array_equal(U, U_d)


def test_sharded_ties_go_to_lowest_global_index():
    # Kahan witness: every step is an exact tie; shards split the tied columns, so a
    # rank-local "first maximum" rule would pick a later global index at a shard boundary.
    l = 8
    X = kahan_witness(l, 20)
    perm = np.r_[np.arange(l, 20), np.arange(l)]           # tied columns moved to the last shard
    Xp = X[:, perm]
    for splits in ([12, 8], [5, 7, 8], [19, 1]):
        blocks = np.split(Xp, np.cumsum(splits)[:-1], axis=1)
        piv_d, _, _ = o_dist.select_cols_sharded(blocks, l)
        piv, _, _, _ = o_lupp.select_cols(Xp, l)
        assert piv_d.tolist() == piv.tolist()


class HostBackend:
    """Test stand-in for the CUDA kernels (the oracle, on CPU tensors)."""

    def sketch(self, A_local, l, embedding, seed, zeta):
        return torch.from_numpy(o_sketch.sketch(A_local.numpy(), l, embedding, seed, zeta))

    def select_cols(self, Xk, k):
        piv, Lf, _, _ = o_lupp.select_cols(Xk.numpy(), k)
        return torch.from_numpy(piv), torch.from_numpy(Lf)

    def select_rows(self, C, k):
        piv, _, _, _ = o_lupp.select_rows(C.numpy(), k)
        return torch.from_numpy(piv)

    def gather_cols_shard(self, A_local, Js, col0):
        m, nc = A_local.shape
        C = torch.zeros((Js.numel(), m), dtype=torch.float64).t()
        for t, j in enumerate(Js.tolist()):
            if col0 <= j < col0 + nc:
                C[:, t] = A_local[:, j - col0]
        return C

    def residual_cols(self, A_local, C):
        A = A_local.numpy()
        Q = o_res.ortho(C.numpy())
        E = A - Q @ (Q.T @ A)
        return float(np.sum(E * E)), float(np.sum(A * A))

    # the pieces of the distributed residual protocol (dist.gather_cols_allgather, cholqr_rows_dist)
    def pack_cols(self, A_local, idx, cmax):
        out = torch.zeros((cmax, A_local.shape[0]), dtype=torch.float64)
        for i, j in enumerate(idx):
            out[i] = A_local[:, j]
        return out

    def basis(self, C):
        # as the library: the LUPP factor of C (range(C) = range(Lf_C)) with CholeskyQR2
        _, Lf, _, _ = o_lupp.select_rows(C.numpy(), C.shape[1])
        return torch.from_numpy(Lf), 2, False

    def row_block(self, B, r0, rows, mb):
        out = torch.zeros((mb, B.shape[1]), dtype=torch.float64)
        out[:rows] = B[r0:r0 + rows]
        return out

    def gram(self, Bl):
        return Bl.t() @ Bl

    def chol_right_solve(self, Bl, G, shift_rows):
        G = G.numpy().copy()
        k = G.shape[0]
        if shift_rows:
            G += 11.0 * (shift_rows * k + k * (k + 1)) * 2.0 ** -53 * np.trace(G) * np.eye(k)
        L = np.linalg.cholesky(G)
        return torch.from_numpy(sla.solve_triangular(L, Bl.numpy().T, lower=True).T.copy())

    def residual_q(self, A_local, Q):
        A = A_local.numpy()
        Qn = Q.numpy()
        E = A - Qn @ (Qn.T @ A)
        return float(np.sum(E * E)), float(np.sum(A * A))


def _worker(rank, world, port, A, k, l, seed, q, exchange="replicate"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = A.shape[1]
        c0, nc = shard(n, world, rank)
        A_local = torch.from_numpy(np.asfortranarray(A[:, c0:c0 + nc]))
        out = dist_rand_lupp(A_local, n, k, l, "gaussian", seed, rows=True, residual=True, backend=HostStepBackend(),
                             exchange=exchange)
        q.put((rank, out["Js"].tolist(), out["Is"].tolist(), out["C"].numpy().copy(), out["residual"], out["normA"]))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,exchange", [(2, "replicate"), (3, "replicate"), (2, "step"), (3, "step")])
def test_dist_rand_lupp_gloo_matches_unsharded_oracle(world, exchange):
    A, _ = make_c1(seed=1001)
    A = A[:, :251]                                           # ragged shards
    k, l, seed = 20, 40, 2001
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, A, k, l, seed, q, exchange)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    X = o_sketch.sketch(A, l, "gaussian", seed)
    piv, _, _, _ = o_lupp.select_cols(X, k)
    ipiv, _, _, _ = o_lupp.select_rows(A[:, piv], k)
    r_or, n_or = o_res.residual(A, piv, kind="col_id")
    for rank, Js, Is, C, r, nA in res:
        assert Js == piv.tolist(), rank
        np.testing.assert_array_equal(C, A[:, piv])          # assembled exactly by the all-gather
        assert Is == ipiv.tolist()
        assert abs(r - r_or) <= 1e-12 * r_or + 4 * 2.0 ** -53 * n_or
        assert abs(nA - n_or) <= 1e-14 * n_or
    assert math.isfinite(res[0][4])


# ---------------------------------------------------------------- per-step exchange
class HostLuppDist:
    """Test stand-in for api.LuppDist (the sk_lupp_dist_* kernels): the same record protocol --
    [|value| or -1, global index or -1, local max|panel|, 0, row] -- in numpy, so the per-step
    all-gather of dist.select_cols_stepwise runs over gloo on CPU."""

    def __init__(self, nloc, k, col0, world, device=None):
        self.nloc, self.k, self.col0, self.world = nloc, k, col0, world
        self.rec = k + 4
        self.cand = torch.zeros(self.rec, dtype=torch.float64)
        self.gathered = torch.zeros(world * self.rec, dtype=torch.float64)
        self.Js = torch.full((k,), -1, dtype=torch.int64)
        self.Lf = torch.zeros((nloc, k), dtype=torch.float64)
        self.U = torch.zeros((k, k), dtype=torch.float64)
        self.status = 0

    def begin(self, X_local):
        self.M = X_local[:self.k].numpy().T.copy()
        self.act = np.ones(self.nloc, dtype=bool)
        self.lmax = float(np.max(np.abs(self.M))) if self.M.size else 0.0
        self.status = 0
        self._propose(0)

    def _propose(self, t):
        c = np.zeros(self.rec)
        c[:3] = (-1.0, -1.0, self.lmax)
        if self.act.any():
            a = np.where(self.act, np.abs(self.M[:, t]), -1.0)
            i = int(np.argmax(a))
            c[0], c[1], c[4:] = a[i], self.col0 + i, self.M[i]
        self.cand.copy_(torch.from_numpy(c))

    def step(self, t):
        if self.status:
            return
        G = self.gathered.view(self.world, self.rec).numpy()
        gmax = float(G[:, 2].max())
        best = None
        for w in range(self.world):
            if G[w, 1] >= 0 and (best is None or G[w, 0] > G[best, 0] or
                                 (G[w, 0] == G[best, 0] and G[w, 1] < G[best, 1])):
                best = w
        if best is None or not (G[best, 0] > 1e-14 * gmax):
            self.status = t
            self.Js[t - 1:] = -1
            return
        g, row = int(G[best, 1]), G[best, 4:].copy()
        self.Js[t - 1] = g
        self.U[t - 1, t - 1:] = torch.from_numpy(row[t - 1:])
        Lf = self.Lf.numpy()
        if self.col0 <= g < self.col0 + self.nloc:
            self.act[g - self.col0] = False
            Lf[g - self.col0, t - 1] = 1.0
        rows = np.nonzero(self.act)[0]
        mult = self.M[rows, t - 1] / row[t - 1]
        Lf[rows, t - 1] = mult
        self.M[rows, t:] -= np.outer(mult, row[t:])
        if t < self.k:
            self._propose(t)

    def info(self):
        if self.status:
            raise o_lupp.RankError(self.status)
        return 0


class HostStepBackend(HostBackend):
    def lupp_dist(self, nloc, k, col0, world, device=None):
        return HostLuppDist(nloc, k, col0, world)


def _step_worker(rank, world, port, X, k, q):
    from paper_2104_05877_b200.dist import select_cols_stepwise
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = X.shape[1]
        c0, nc = shard(n, world, rank)
        Xl = torch.from_numpy(np.ascontiguousarray(X[:, c0:c0 + nc]))
        try:
            Js, Lf, U = select_cols_stepwise(Xl, n, k, backend=HostStepBackend())
            q.put((rank, "ok", Js.tolist(), Lf.numpy().copy(), U.numpy().copy()))
        except o_lupp.RankError as e:
            q.put((rank, "rank", e.step, None, None))
    finally:
        dist.destroy_process_group()


def _run_step(X, k, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_step_worker, args=(r, world, port, X, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("n,k,world", [(251, 20, 2), (100, 12, 3), (2, 2, 3)])
def test_stepwise_gloo_equals_single_lupp(n, k, world):
    # ragged shards; (2, 2, 3) leaves rank 2 with no columns (it proposes "none" every step)
    X = np.random.default_rng(n + world).standard_normal((k + 3, n))
    res = _run_step(X, k, world)
    piv, Lf, U, _ = o_lupp.select_cols(X, k)
    for rank, kind, Js, _, Ur in res:
        assert kind == "ok" and Js == piv.tolist(), rank
        np.testing.assert_array_equal(Ur, U)
    np.testing.assert_array_equal(np.vstack([r[3] for r in res]), Lf)    # rank blocks stack to Lf


def test_stepwise_gloo_ties_and_rank_failure():
    l = 6
    X = kahan_witness(l, 14)[:, np.r_[np.arange(l, 14), np.arange(l)]]   # tied columns in the last shard
    res = _run_step(X, l, 3)
    piv, _, _, _ = o_lupp.select_cols(X, l)
    assert all(r[2] == piv.tolist() for r in res)
    Z = np.zeros((4, 9))
    Z[0, 3] = 1.0                                                       # rank 1 after step 1
    res = _run_step(Z, 3, 2)
    assert all(r[1] == "rank" and r[2] == 2 for r in res)
