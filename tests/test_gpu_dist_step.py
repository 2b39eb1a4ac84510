"""GPU parity of the per-step-exchange column LUPP (sk_lupp_dist_*).

The P ranks of the column-sharded path are emulated in ONE process on one GPU: P LuppDist
states over the P column blocks of the sketch, and the all-gather of their records done as a
device copy between steps.  No kernel waits on another rank, so this is the exact per-step
protocol without a multi-GPU launch.  The update rounds like the oracle (no FMA contraction), so
pivots, U and the stacked Lf are compared BIT FOR BIT with oracle.lupp.select_cols on the
unsharded sketch.  The NCCL tests run the real collective at world size 1 (eager and captured
in a CUDA graph).
"""
import os

import numpy as np
import pytest
import torch

import paper_2104_05877_b200 as sk
from inputs import kahan_witness, make_c2
from oracle import lupp as o_lupp
from oracle import sketch as o_sketch
from paper_2104_05877_b200.dist import shard

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def emulate(X, k, world):
    """Run the P-rank protocol in one process. Returns (Js, Lf stacked, U, info)."""
    n = X.shape[1]
    sels, blocks = [], []
    for r in range(world):
        c0, nc = shard(n, world, r)
        sels.append(sk.LuppDist(nc, k, c0, world, 0))
        blocks.append(torch.from_numpy(np.ascontiguousarray(X[:, c0:c0 + nc])).to(DEV))
    for s, b in zip(sels, blocks):
        s.begin(b)
    for t in range(1, k + 1):
        g = torch.cat([s.cand for s in sels])
        for s in sels:
            s.gathered.copy_(g)
            s.step(t)
    infos = []
    for s in sels:
        try:
            infos.append(s.info())
        except sk.SkelError as e:
            infos.append(e.info)
    Js = [s.Js.cpu().numpy() for s in sels]
    for j in Js[1:]:
        np.testing.assert_array_equal(j, Js[0])                       # replicated
    Us = [s.U.cpu().numpy() for s in sels]
    for u in Us[1:]:
        np.testing.assert_array_equal(u, Us[0])
    Lf = np.vstack([s.Lf.cpu().numpy()[:s.nloc] for s in sels])
    return Js[0], Lf, Us[0], infos


@pytest.mark.parametrize("n,k,world", [(251, 20, 1), (251, 20, 3), (1000, 64, 8), (300, 40, 7), (5, 5, 8)])
def test_stepwise_bitwise_equals_oracle(n, k, world):
    # (5, 5, 8): three ranks own no column; (300, 40, 7): ragged blocks spanning several CTAs
    X = np.random.default_rng(7 * n + k).standard_normal((k + 5, n))
    Js, Lf, U, infos = emulate(X, k, world)
    piv, Lfo, Uo, _ = o_lupp.select_cols(X, k)
    assert infos == [0] * world
    np.testing.assert_array_equal(Js, piv)
    np.testing.assert_array_equal(U, Uo)
    np.testing.assert_array_equal(Lf, Lfo)


def test_stepwise_c2_k512_full_size():
    """C2 at the bench configuration: the oracle sketch (l = 522) of the 4096^2 input, 4 shards."""
    A, _ = make_c2(seed=1002)
    X = o_sketch.sketch(A, 522, "gaussian", 2002 + 512)
    Js, Lf, U, infos = emulate(X, 512, 4)
    piv, Lfo, Uo, _ = o_lupp.select_cols(X, 512)
    assert infos == [0] * 4
    np.testing.assert_array_equal(Js, piv)
    np.testing.assert_array_equal(U, Uo)
    np.testing.assert_array_equal(Lf, Lfo)


def test_stepwise_ties_straddle_shards():
    l = 10
    X = kahan_witness(l, 40)[:, np.r_[np.arange(l, 40), np.arange(l)]]
    for world in (2, 3, 5):
        Js, _, U, infos = emulate(X, l, world)
        piv, _, Uo, _ = o_lupp.select_cols(X, l)
        np.testing.assert_array_equal(Js, piv)
        np.testing.assert_array_equal(U, Uo)
        assert infos == [0] * world


def test_stepwise_rank_failure():
    Z = np.zeros((6, 50))
    Z[0, 31] = 3.0
    Z[1, 7] = 1e-20                                                    # below 1e-14 max|panel|
    Js, _, _, infos = emulate(Z, 4, 3)
    assert infos == [2, 2, 2]
    assert Js[0] == 31 and (Js[1:] == -1).all()


def _nccl_world1(port):
    import torch.distributed as tdist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device(DEV))
    return tdist


def test_stepwise_nccl_world1_eager_and_graph():
    from paper_2104_05877_b200.dist import CapturedStepwise, select_cols_stepwise
    tdist = _nccl_world1(29541)
    try:
        X = np.random.default_rng(5).standard_normal((70, 700))
        piv, Lfo, Uo, _ = o_lupp.select_cols(X, 64)
        Xd = torch.from_numpy(X).to(DEV)
        Js, Lf, U = select_cols_stepwise(Xd, 700, 64)
        np.testing.assert_array_equal(Js.cpu().numpy(), piv)
        np.testing.assert_array_equal(Lf.cpu().numpy(), Lfo)
        cap = CapturedStepwise(Xd, 700, 64)
        for _ in range(2):
            cap.sel.Js.fill_(-7)
            Js, Lf, U = cap.run()
            torch.cuda.synchronize()
            np.testing.assert_array_equal(Js.cpu().numpy(), piv)
            np.testing.assert_array_equal(U.cpu().numpy(), Uo)
        X2 = np.random.default_rng(6).standard_normal((70, 700))        # new data, same graph
        Xd.copy_(torch.from_numpy(X2))
        Js, _, _ = cap.run()
        piv2, _, _, _ = o_lupp.select_cols(X2, 64)
        np.testing.assert_array_equal(Js.cpu().numpy(), piv2)
    finally:
        tdist.destroy_process_group()


def test_dist_rand_lupp_step_exchange_nccl_world1():
    from inputs import make_c1
    from paper_2104_05877_b200.dist import dist_rand_lupp
    tdist = _nccl_world1(29543)
    try:
        A, _ = make_c1(seed=1001)
        Ad = sk.fortran(torch.from_numpy(A).to(DEV))
        out = dist_rand_lupp(Ad, 256, 20, 40, "gaussian", 2001, rows=True, exchange="step")
        X = o_sketch.sketch(A, 40, "gaussian", 2001)
        piv, _, _, _ = o_lupp.select_cols(X, 20)
        assert out["Js"].cpu().tolist() == piv.tolist()
        ipiv, _, _, _ = o_lupp.select_rows(A[:, piv], 20)
        assert out["Is"].cpu().tolist() == ipiv.tolist()
    finally:
        tdist.destroy_process_group()


# ---------------------------------------------------------------- exchange fused into the kernel
def emulate_p2p(X, k, world, reps=1):
    """P ranks on one GPU with P2P mailboxes: rank r's step-t kernel waits for the flags of all
    ranks' step t-1 kernels, which were launched before it in program order on the same stream
    (so no kernel ever waits for one that has not run).  Returns (Js, Lf, U, infos) of the last rep."""
    n = X.shape[1]
    boxes = [sk.ipc_alloc(sk.mailbox_bytes(k, world), 0) for _ in range(world)]
    peers = torch.tensor(boxes, dtype=torch.int64, device=DEV)
    try:
        sels, blocks = [], []
        for r in range(world):
            c0, nc = shard(n, world, r)
            sels.append(sk.LuppDistP2P(nc, k, c0, world, r, peers, boxes[r], 0))
            blocks.append(torch.from_numpy(np.ascontiguousarray(X[:, c0:c0 + nc])).to(DEV))
        for _ in range(reps):
            for s, b in zip(sels, blocks):
                s.begin(b)
            for t in range(1, k + 1):
                for s in sels:
                    s.step(t)
            infos = []
            for s in sels:
                try:
                    infos.append(s.info())
                except sk.SkelError as e:
                    infos.append(e.info)
        Js = [s.Js.cpu().numpy() for s in sels]
        for j in Js[1:]:
            np.testing.assert_array_equal(j, Js[0])
        Lf = np.vstack([s.Lf.cpu().numpy()[:s.nloc] for s in sels])
        return Js[0], Lf, sels[0].U.cpu().numpy(), infos
    finally:
        torch.cuda.synchronize()
        for b in boxes:
            sk.ipc_free(b, 0)


@pytest.mark.parametrize("n,k,world", [(251, 20, 1), (251, 20, 3), (1000, 64, 8), (5, 5, 8)])
def test_p2p_stepwise_bitwise_equals_oracle(n, k, world):
    X = np.random.default_rng(11 * n + k).standard_normal((k + 5, n))
    Js, Lf, U, infos = emulate_p2p(X, k, world, reps=2)                 # rep 2 reuses the mailboxes
    piv, Lfo, Uo, _ = o_lupp.select_cols(X, k)
    assert infos == [0] * world
    np.testing.assert_array_equal(Js, piv)
    np.testing.assert_array_equal(U, Uo)
    np.testing.assert_array_equal(Lf, Lfo)


def test_p2p_stepwise_ties_and_rank_failure():
    l = 10
    X = kahan_witness(l, 40)[:, np.r_[np.arange(l, 40), np.arange(l)]]
    Js, _, _, infos = emulate_p2p(X, l, 3)
    piv, _, _, _ = o_lupp.select_cols(X, l)
    np.testing.assert_array_equal(Js, piv)
    Z = np.zeros((6, 50))
    Z[0, 31] = 3.0
    Z[1, 7] = 1e-20
    Js, _, _, infos = emulate_p2p(Z, 4, 3)
    assert infos == [2, 2, 2] and Js[0] == 31 and (Js[1:] == -1).all()


def test_p2p_dist_rand_lupp_world1():
    from inputs import make_c1
    from paper_2104_05877_b200.dist import dist_rand_lupp
    tdist = _nccl_world1(29547)
    try:
        A, _ = make_c1(seed=1001)
        Ad = sk.fortran(torch.from_numpy(A).to(DEV))
        out = dist_rand_lupp(Ad, 256, 20, 40, "gaussian", 2001, rows=True, exchange="p2p")
        X = o_sketch.sketch(A, 40, "gaussian", 2001)
        piv, _, _, _ = o_lupp.select_cols(X, 20)
        assert out["Js"].cpu().tolist() == piv.tolist()
    finally:
        tdist.destroy_process_group()


def _ipc_child(handle, q):
    from cuda.bindings import runtime as cudart
    import paper_2104_05877_b200 as skc
    torch.cuda.set_device(0)
    ptr = skc.ipc_import(handle, 0)
    host = np.zeros(4, dtype=np.float64)
    err, = cudart.cudaMemcpy(host.ctypes.data, ptr, 32, cudart.cudaMemcpyKind.cudaMemcpyDeviceToHost)
    q.put((int(err), host.tolist()))
    skc.ipc_close(ptr, 0)


def test_ipc_handle_maps_the_buffer_in_another_process():
    """The mailbox plumbing of P2PStepwise: a second process maps the buffer by its handle and reads
    what the first wrote (no kernel waits on the other process)."""
    import torch.multiprocessing as mp
    from cuda.bindings import runtime as cudart
    ptr = sk.ipc_alloc(64, 0)
    try:
        vals = np.array([1.5, -2.25, 3.0, 7.0])
        err, = cudart.cudaMemcpy(ptr, vals.ctypes.data, 32, cudart.cudaMemcpyKind.cudaMemcpyHostToDevice)
        assert int(err) == 0
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        p = ctx.Process(target=_ipc_child, args=(sk.ipc_export(ptr, 0), q))
        p.start()
        err, got = q.get(timeout=120)
        p.join(timeout=60)
        assert p.exitcode == 0 and err == 0 and got == vals.tolist()
    finally:
        sk.ipc_free(ptr, 0)


_TIMEOUT_CHILD = r"""
import numpy as np, torch
import paper_2104_05877_b200 as sk
from paper_2104_05877_b200._lib import SK_E_STATE
k, world = 6, 2
X = torch.from_numpy(np.random.default_rng(1).standard_normal((k + 2, 40))).to("cuda:0")
boxes = [sk.ipc_alloc(sk.mailbox_bytes(k, world), 0) for _ in range(world)]
peers = torch.tensor(boxes, dtype=torch.int64, device="cuda:0")
s = sk.LuppDistP2P(20, k, 0, world, 0, peers, boxes[0], 0)   # rank 1 never runs
s.begin(X[:, :20].contiguous())
for t in range(1, k + 1):
    s.step(t)
try:
    s.info()
    raise SystemExit("no error")
except sk.SkelError as e:
    assert e.status == SK_E_STATE and e.info == -1, (e.status, e.info)
torch.cuda.synchronize()
print("TIMEOUT-OK")
"""


def test_p2p_missing_peer_times_out_instead_of_hanging():
    """Rank 1 of 2 never publishes: rank 0's step-1 kernel gives up after SKEL_PEER_TIMEOUT_MS,
    latches -1, and the remaining steps return at once (child process, bounded by timeout)."""
    import subprocess
    import sys
    env = dict(os.environ, SKEL_PEER_TIMEOUT_MS="300")
    r = subprocess.run([sys.executable, "-c", _TIMEOUT_CHILD], env=env, capture_output=True, text=True,
                       timeout=180, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "TIMEOUT-OK" in r.stdout, r.stdout + r.stderr
