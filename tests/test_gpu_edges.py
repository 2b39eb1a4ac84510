"""GPU edge cases through the C ABI: empty and degenerate sizes, single rows/columns, k = 1,
l = m, ties, zero matrices, lda padding, argument errors -- each against the oracle or a closed form."""
import math

import numpy as np
import pytest
import torch

import paper_2104_05877_b200 as sk
from oracle import lupp as o_lupp
from oracle import residual as o_res
from oracle import sketch as o_sketch

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def dev_f(a):
    return sk.fortran(torch.from_numpy(np.ascontiguousarray(a)).to(DEV))


def test_sketch_empty_n():
    A = torch.empty((50, 0), dtype=torch.float64, device=DEV)
    X = sk.sketch(A, 10, "gaussian", 1)
    assert X.shape == (10, 0)


@pytest.mark.parametrize("emb", ["gaussian", "sparse_sign"])
def test_sketch_single_row_and_column(emb):
    rng = np.random.default_rng(0)
    A = rng.standard_normal((64, 1))
    l = 8
    X = sk.sketch(dev_f(A), l, emb, 5, 2 if emb == "sparse_sign" else 8).cpu().numpy()
    ref = o_sketch.sketch(A, l, emb, 5, 2 if emb == "sparse_sign" else 8)
    assert np.linalg.norm(X - ref) <= 1e-12 * np.linalg.norm(ref)
    A1 = rng.standard_normal((1, 7))                     # m = l = 1
    X1 = sk.sketch(dev_f(A1), 1, "gaussian", 5).cpu().numpy()
    np.testing.assert_allclose(X1, o_sketch.sketch(A1, 1, "gaussian", 5), rtol=1e-14)


def test_sketch_zero_matrix_is_zero():
    X = sk.sketch(dev_f(np.zeros((300, 40))), 20, "gaussian", 3).cpu().numpy()
    assert np.count_nonzero(X) == 0


def test_select_cols_k1_is_argmax_first_row():
    rng = np.random.default_rng(1)
    X = rng.standard_normal((3, 500))
    Js, Lf, U, _ = sk.select_cols(torch.from_numpy(X).to(DEV), 1)
    assert Js.item() == int(np.argmax(np.abs(X[0])))
    np.testing.assert_allclose(Lf.cpu().numpy()[:, 0], X[0] / X[0, Js.item()], rtol=1e-15)


def test_select_rows_single_column_and_k_equals_m():
    rng = np.random.default_rng(2)
    C = rng.standard_normal((40, 1))
    Is, _, _, _ = sk.select_rows(dev_f(C), 1)
    assert Is.item() == int(np.argmax(np.abs(C[:, 0])))
    Cs = rng.standard_normal((12, 12))
    Is, _, _, _ = sk.select_rows(dev_f(Cs), 12)
    piv, _, _, _ = o_lupp.select_rows(Cs, 12)
    assert Is.cpu().tolist() == piv.tolist()


def test_select_cols_all_zero_is_rank_failure_at_step_1():
    with pytest.raises(sk.SkelError) as e:
        sk.select_cols(torch.zeros((4, 100), dtype=torch.float64, device=DEV), 3)
    assert e.value.status == 2 and e.value.info == 1


@pytest.mark.parametrize("n", [70000, 131000])
def test_select_cols_tall_rank_failure_across_clusters(n):
    # two nonzero sketch columns in different clusters of a multi-cluster panel: steps 1-2 pick
    # them (the larger first), step 3 finds no pivot in any cluster -> SK_E_RANK, info 3, and the
    # asynchronous form leaves Js[2:] = -1
    X = np.zeros((4, n))
    X[:, 7] = [1.0, 2.0, 3.0, 4.0]
    X[:, n - 5] = [-2.0, 1.0, 0.5, 0.25]
    Xd = torch.from_numpy(X).to(DEV)
    with pytest.raises(sk.SkelError) as e:
        sk.select_cols(Xd, 4)
    assert e.value.status == 2 and e.value.info == 3
    Js, _, _, _ = sk.select_cols(Xd, 4, check=False)
    assert Js.cpu().tolist() == [n - 5, 7, -1, -1]


def test_select_cols_exact_ties_everywhere():
    # every entry of the first row equal: the lowest index wins each tie (R6)
    X = np.ones((2, 64))
    X[1] = np.arange(64)
    Js, _, _, _ = sk.select_cols(torch.from_numpy(X).to(DEV), 2)
    piv, _, _, _ = o_lupp.select_cols(X, 2)
    assert Js.cpu().tolist() == piv.tolist() == [0, 63]


def test_residual_full_rank_skeleton_is_zero_and_k_equals_n():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((80, 30))
    J = torch.arange(30, dtype=torch.int64, device=DEV)
    r, nA = sk.residual(dev_f(A), J, None, "col_id")       # C = A: the projector is exact
    assert r <= 1e-12 * nA


def test_padded_lda_everywhere():
    rng = np.random.default_rng(4)
    m, n, l, k = 200, 90, 24, 12
    A = rng.standard_normal((m, n))
    buf = torch.zeros((n, m + 5), dtype=torch.float64, device=DEV)
    buf[:, :m] = torch.from_numpy(A.T.copy()).to(DEV)
    Av = buf.t()[:m]                                       # lda = m + 5
    X = sk.sketch(Av, l, "gaussian", 9)
    Js, _, _, _ = sk.select_cols(X, k)
    r, nA = sk.residual(Av, Js, None, "col_id")
    ro, nAo = o_res.residual(A, Js.cpu().numpy(), kind="col_id")
    assert abs(r - ro) <= 1e-9 * ro + 4 * 2.0 ** -53 * nAo


@pytest.mark.parametrize("call", ["l_gt_m", "k_gt_l", "zeta_bad", "bad_kind"])
def test_argument_errors_are_reported(call):
    A = dev_f(np.ones((10, 10)))
    with pytest.raises((sk.SkelError, KeyError)) as e:
        if call == "l_gt_m":
            sk.sketch(A, 11, "gaussian", 1)
        elif call == "k_gt_l":
            sk.select_cols(torch.ones((3, 10), dtype=torch.float64, device=DEV), 4)
        elif call == "zeta_bad":
            sk.sketch(A, 5, "sparse_sign", 1, 9)
        else:
            sk.residual(A, torch.zeros(2, dtype=torch.int64, device=DEV), None, "nope")
    if isinstance(e.value, sk.SkelError):
        assert e.value.status == 1


def test_gather_cols_out_of_range_index_gives_zero_column():
    # Js is device data the host never reads: an index outside [0, n) must not read out of bounds
    A = np.random.default_rng(3).standard_normal((37, 9))
    Js = torch.tensor([4, 9, -1, 0, 1 << 40], dtype=torch.int64, device=DEV)
    C = sk.gather_cols(dev_f(A), Js).cpu().numpy()
    np.testing.assert_array_equal(C[:, 0], A[:, 4])
    np.testing.assert_array_equal(C[:, 3], A[:, 0])
    for t in (1, 2, 4):
        assert not C[:, t].any()


def test_rand_lupp_rank_failure_reports_the_step():
    # two nonzero columns, k = 4: the sketch has exactly two nonzero columns, so the column LUPP
    # finds no pivot at step 3; the error carries that step (device and host A)
    from paper_2104_05877_b200._lib import SK_E_RANK
    A = np.zeros((60, 40))
    A[:, 5] = np.random.default_rng(8).standard_normal(60)
    A[:, 17] = np.random.default_rng(9).standard_normal(60)
    for At in (torch.from_numpy(np.asfortranarray(A)), dev_f(A)):
        with pytest.raises(sk.SkelError) as e:
            sk.rand_lupp(At, 4, 12, "gaussian", 1)
        assert e.value.status == SK_E_RANK and e.value.info == 3


# ------------------------------------------------------------------ round-2 entry points at the edges
def rand_cm(m, n, seed):
    return np.random.default_rng(seed).standard_normal((m, n))


@pytest.mark.parametrize("m,n,l,chunk", [(1037, 5, 3, 256), (33, 300, 1, 16), (2049, 129, 17, 1024)])
def test_sketch_chunked_tiny_and_ragged(m, n, l, chunk):
    """K-chunked Omega with ragged chunks (m not a multiple of the chunk or of 16), l = 1 and n < one tile."""
    A = rand_cm(m, n, m + n)
    sk.set_sketch_tuning(chunk_rows=chunk)
    try:
        X = sk.sketch(dev_f(A), l, "gaussian", 3).cpu().numpy()
    finally:
        sk.set_sketch_tuning()
    ref = o_sketch.sketch(A, l, "gaussian", 3)
    assert np.linalg.norm(X - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("host", [False, True])
def test_sketch_dual_single_column_and_row(host):
    A = rand_cm(40, 1, 1)
    Ain = torch.from_numpy(np.asfortranarray(A)) if host else dev_f(A)
    X, Y = sk.sketch_dual(Ain, 1, 1, seed_x=4, seed_y=5)
    np.testing.assert_allclose(X.cpu().numpy(), o_sketch.sketch(A, 1, "gaussian", 4), rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(Y.cpu().numpy(), o_sketch.sketch_cols(A, 1, "gaussian", 5), rtol=1e-13, atol=1e-15)


def test_estimates_k1_and_square_pivot_block():
    """k = 1 and k = l (X_1 square: X_1^+ X = X_1^{-1} X, the sketch interpolation matrix itself)."""
    from oracle import estimates as o_est
    A = rand_cm(60, 50, 7)
    Ad = dev_f(A)
    for k, l in ((1, 4), (8, 8)):
        X = sk.sketch(Ad, l, "gaussian", 11)
        Js, _, _, _ = sk.select_cols(X, k)
        Z = sk.id_estimate_cols(X, Js).cpu().numpy()
        Zo = o_est.id_estimate_cols(o_sketch.sketch(A, l, "gaussian", 11), Js.cpu().numpy())
        assert np.linalg.norm(Z - Zo) <= 1e-9 * np.linalg.norm(Zo)
        Y = sk.sketch_cols(Ad, l, "gaussian", 12)
        Is, _, _, _ = sk.select_rows(Y, k)
        W = sk.id_estimate_rows(Y, Is).cpu().numpy()
        Wo = o_est.id_estimate_rows(o_sketch.sketch_cols(A, l, "gaussian", 12), Is.cpu().numpy())
        assert np.linalg.norm(W - Wo) <= 1e-9 * np.linalg.norm(Wo)
        r, _ = sk.residual(Ad, Js, Is, "cur_css")
        ro = float(np.linalg.norm(A - o_est.cur_css(A, Is.cpu().numpy(), Js.cpu().numpy())))
        assert abs(r - ro) <= 1e-8 * ro


def test_power_ortho_full_rank_l_equals_n():
    """l = n: ortho(Y) spans everything, X = Q^T A with Q m x n orthonormal: X^T X = A^T A."""
    A = rand_cm(70, 12, 9)
    X = sk.sketch_power(dev_f(A), 12, "gaussian", 3, 2, ortho=True).cpu().numpy()
    np.testing.assert_allclose(X.T @ X, A.T @ A, rtol=0, atol=1e-11 * np.abs(A.T @ A).max())


def test_dist_context_k1_and_gaps_fallback():
    """The distributed context at world size 1 with k = 1 (the per-step graph with one step) and with the
    gaps output requested under the per-step exchange (served by the gather-then-replicate path)."""
    import os
    import socket
    import torch.distributed as tdist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device(DEV))
    try:
        A = rand_cm(90, 40, 3)
        Ad = dev_f(A)
        sess = sk.DistSession(40, None, 0, "step")
        try:
            with sess:
                X = sk.sketch(Ad, 6, "gaussian", 8)
                J1, _, _, _ = sk.select_cols(X, 1)
                J5, _, _, g5 = sk.select_cols(X, 5, want_gaps=True)
        finally:
            sess.close()
        Xo = o_sketch.sketch(A, 6, "gaussian", 8)
        assert J1.cpu().tolist() == o_lupp.select_cols(Xo, 1)[0].tolist()
        piv, _, _, go = o_lupp.select_cols(Xo, 5)
        assert J5.cpu().tolist() == piv.tolist()
        np.testing.assert_allclose(g5.cpu().numpy(), go, atol=1e-9)
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("kind", ["col_id", "row_id", "cur"])
@pytest.mark.parametrize("scale", [1.0, 1e-2])
def test_residual_projection_identity_large_residual(kind, scale):
    """R25: when r^2 >= 1e-3 ||A||^2 the projection kinds take ||A||^2 - ||W||^2 (no second GEMM).
    A Gaussian matrix with a planted rank-20 part: scale 1 keeps r^2/||A||^2 ~ 0.9 (identity path),
    scale 1e-2 makes the noise small (r^2/||A||^2 ~ 1e-4: the explicit path) -- both vs the oracle."""
    rng = np.random.default_rng(77)
    m, n, k = 1500, 700, 20
    A = rng.standard_normal((m, 20)) @ rng.standard_normal((20, n)) + scale * rng.standard_normal((m, n))
    Ad = dev_f(A)
    X = sk.sketch(Ad, k + 10, "gaussian", 3)
    Js, _, _, _ = sk.select_cols(X, k)
    Is, _, _, _ = sk.select_rows(sk.gather_cols(Ad, Js), k)
    r, nA = sk.residual(Ad, Js, Is if kind != "col_id" else None, kind)
    ro, nAo = o_res.residual(A, Js.cpu().numpy(), Is.cpu().numpy(), kind=kind)
    assert abs(r - ro) <= 1e-9 * ro + 4 * 2.0 ** -53 * nAo, (kind, scale, r, ro, (ro / nAo) ** 2)
    assert abs(nA - nAo) <= 1e-12 * nAo
