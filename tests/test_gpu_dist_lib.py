"""GPU parity through the C-ABI column-sharded context (sk_nccl_unique_id / sk_create_dist,
SURVEY 8(b), 8(e)): the library owns the NCCL communicator and issues every exchange itself.

Run at world size 1 on the one GPU of this pool (NCCL with one rank: every collective is a local
copy, so the whole protocol -- packing, all-gathers, k x k all-reduces of the distributed Cholesky
QR, the captured per-step graph -- runs with real NCCL calls); the multi-rank protocol is checked
over gloo on CPU (tests/test_dist_gloo.py).  Everything is compared with the oracle on the same
seeded inputs: J_s / I_s identical, Z and eta within the S5 tolerance, residuals within
1e-9 r + 4u||A||_F.
"""
import os
import socket

import numpy as np
import pytest
import torch

import paper_2104_05877_b200 as sk
from inputs import make_c1, make_c2, make_lowrank
from oracle import idcoef as o_id
from oracle import lupp as o_lupp
from oracle import residual as o_res
from oracle import sketch as o_sketch
from tests.parity import lupp_parity, rel_fro

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
U = 2.0 ** -53


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl1():
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device(DEV))
    yield tdist
    tdist.destroy_process_group()


def dev_f(a):
    return sk.fortran(torch.from_numpy(np.ascontiguousarray(a)).to(DEV))


def res_ok(r, ro, nA):
    return abs(r - ro) <= 1e-9 * ro + 4 * U * nA


@pytest.mark.parametrize("exchange", ["replicate", "step"])
def test_dist_context_c1_whole_path(nccl1, exchange):
    A, _ = make_c1(seed=1001)
    k, l, seed = 20, 40, 2001
    Ad = dev_f(A)
    sess = sk.DistSession(256, None, 0, exchange)
    try:
        with sess:
            assert (sess.col0, sess.ncols) == (0, 256)
            X = sk.sketch(Ad, l, "gaussian", seed)
            Js, Lf, Ug, _ = sk.select_cols(X, k)
            Js2, _, _, _ = sk.select_cols(X, k)            # the per-step graph is replayed
            assert torch.equal(Js, Js2)
            C = sk.gather_cols(Ad, Js)
            Is, _, _, _ = sk.select_rows(C, k)
            Z, eta = sk.id_coeffs(Lf, Js, want_eta=True)
            res = {kind: sk.residual(Ad, Js, Is, kind) for kind in ("col_id", "row_id", "cur")}
            r_cz, _ = sk.residual(Ad, Js, None, "id_coeffs", Z)
            Jh, Ih = sk.rand_lupp(torch.from_numpy(np.asfortranarray(A)).t().contiguous().t(), k, l, seed=seed,
                                  rows=True)
            Jd, _ = sk.rand_lupp(Ad, k, l, seed=seed)
    finally:
        sess.close()
    Xo = o_sketch.sketch(A, l, "gaussian", seed)
    assert rel_fro(X.cpu().numpy(), Xo) <= 1e-12
    piv, Lo, Uo, _ = o_lupp.select_cols(Xo, k)
    assert Js.cpu().tolist() == piv.tolist()
    assert Jh.tolist() == piv.tolist() and Jd.tolist() == piv.tolist()
    assert rel_fro(Lf.cpu().numpy(), Lo) <= 1e-10 and rel_fro(Ug.cpu().numpy(), Uo) <= 1e-10
    np.testing.assert_array_equal(C.cpu().numpy(), A[:, piv])          # assembled exactly
    ipiv, _, _, _ = o_lupp.select_rows(A[:, piv], k)
    assert Is.cpu().tolist() == ipiv.tolist() and Ih.tolist() == ipiv.tolist()
    Zo, _, eta_o = o_id.id_coeffs(Lo, piv)
    np.testing.assert_array_equal(Z.cpu().numpy()[:, piv], np.eye(k))
    assert rel_fro(Z.cpu().numpy(), Zo) <= 1e-10 and abs(eta - eta_o) <= 1e-8 * eta_o
    for kind, (r, nA) in res.items():
        ro, nAo = o_res.residual(A, piv, ipiv, kind=kind)
        assert res_ok(r, ro, nAo), (kind, r, ro)
    rz, nAo = o_res.residual(A, piv, kind="id_coeffs", Z=Zo)
    assert res_ok(r_cz, rz, nAo), (r_cz, rz)


@pytest.mark.parametrize("exchange", ["replicate", "step"])
def test_dist_context_c2_k512(nccl1, exchange):
    """C2 at the bench's k = 512 through the distributed context: the ill-conditioned C
    (cond 1.6e11) goes through the LUPP basis + distributed CholeskyQR2."""
    A, sigma = make_c2(seed=1002)
    k, l, seed = 512, 522, 2002 + 512
    Ad = dev_f(A)
    sess = sk.DistSession(4096, None, 0, exchange)
    try:
        with sess:
            X = sk.sketch(Ad, l, "gaussian", seed)
            Js, _, _, _ = sk.select_cols(X, k)
            r, nA = sk.residual(Ad, Js, None, "col_id")
    finally:
        sess.close()
    Xo = o_sketch.sketch(A, l, "gaussian", seed)
    (piv, _, _, _), _ = lupp_parity(Js.cpu().numpy(), lambda f: o_lupp.select_cols(Xo, k, f))
    ro, nAo = o_res.residual(A, piv, kind="col_id")
    assert res_ok(r, ro, nAo), (r, ro)


def test_dist_context_tall_c_shifted_cholqr3(nccl1):
    """C taller than the LUPP basis handles (m > 65536): distributed shifted CholeskyQR3."""
    rng = np.random.default_rng(31)
    m, n, k, l = 70000, 300, 24, 40
    A = make_lowrank(m, n, 0.8 ** np.arange(n), rng)
    Ad = dev_f(A)
    sess = sk.DistSession(n, None, 0, "replicate")
    try:
        with sess:
            X = sk.sketch(Ad, l, "gaussian", 5)
            Js, _, _, _ = sk.select_cols(X, k)
            r, nA = sk.residual(Ad, Js, None, "col_id")
    finally:
        sess.close()
    piv, _, _, _ = o_lupp.select_cols(o_sketch.sketch(A, l, "gaussian", 5), k)
    assert Js.cpu().tolist() == piv.tolist()
    ro, nAo = o_res.residual(A, piv, kind="col_id")
    assert res_ok(r, ro, nAo), (r, ro)


@pytest.mark.parametrize("exchange", ["replicate", "step"])
def test_dist_rand_lupp_library_path_with_residual(nccl1, exchange):
    """dist.dist_rand_lupp on CUDA tensors (the library-owned communicator) with residual=True --
    the combination that used to fail in round 1 (ADVICE: Xk unbound)."""
    from paper_2104_05877_b200.dist import dist_rand_lupp
    A, _ = make_c1(seed=1001)
    out = dist_rand_lupp(dev_f(A), 256, 20, 40, "gaussian", 2001, rows=True, residual=True, exchange=exchange)
    piv, _, _, _ = o_lupp.select_cols(o_sketch.sketch(A, 40, "gaussian", 2001), 20)
    assert out["Js"].cpu().tolist() == piv.tolist()
    ro, nAo = o_res.residual(A, piv, kind="col_id")
    assert res_ok(out["residual"], ro, nAo)


def test_dist_context_bad_partition_and_info():
    """sk_create_dist rejects blocks that do not cover [0, n_global); sk_dist_info on a plain
    context reports world 1."""
    import ctypes
    L = sk.api.lib()
    h = sk.context(0)
    w = ctypes.c_int32(0)
    assert L.sk_dist_info(h, None, ctypes.byref(w), None, None, None) == 0 and w.value == 1
    uid = (ctypes.c_char * 128)()
    assert L.sk_nccl_unique_id(uid) == 0
    bad = ctypes.c_void_p()
    st = L.sk_create_dist(ctypes.byref(bad), 0, None, uid, 0, 1, 100, 0, 90)   # 90 of 100 columns
    assert st == 1 and not bad.value
