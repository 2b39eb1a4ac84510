"""GPU parity at BASELINE.json's full sizes (configs C2, C3, C4), in the launch configuration
bench.py times (same entry points, same shapes, device-resident A).

Each case runs the whole hot path on the GPU and the oracle independently on the same
seeded input (the oracle computes its own sketch; nothing it consumes comes from the
CUDA path) and compares: sketch within 1e-12 relative Frobenius, skeleton sets identical
up to documented near-ties, residuals within 1e-9 r + 4u||A||_F.
"""
import numpy as np
import pytest
import scipy.sparse as sps
import torch

import paper_2104_05877_b200 as sk
from inputs import make_c2, make_c3, make_c4
from oracle import cpqr as o_cpqr
from oracle import idcoef as o_id
from oracle import lupp as o_lupp
from oracle import omega as o_omega
from oracle import residual as o_res
from oracle import sketch as o_sketch
from tests.parity import lupp_parity, rel_fro

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
U = 2.0 ** -53


def dev_f(a):
    return sk.fortran(torch.from_numpy(np.ascontiguousarray(a)).to(DEV))


def res_ok(r, ro, nA):
    return abs(r - ro) <= 1e-9 * ro + 4 * U * nA


@pytest.fixture(scope="module")
def c2():
    A, sigma = make_c2(seed=1002)
    return A, sigma, dev_f(A)


@pytest.mark.parametrize("k", [16, 64, 256, 512])
def test_c2_full_path(c2, k):
    """C2 at every k of BASELINE configs[1] (k = 512, l = 522 is the bench's C2 line)."""
    A, sigma, Ad = c2
    l, seed = k + 10, 2002 + k
    X = sk.sketch(Ad, l, "gaussian", seed)
    Js, Lf, _, _ = sk.select_cols(X, k)
    Z, eta = sk.id_coeffs(Lf, Js, want_eta=True)
    r, nA = sk.residual(Ad, Js, None, "col_id")
    torch.cuda.synchronize()

    Xo = o_sketch.sketch(A, l, "gaussian", seed)
    assert rel_fro(X.cpu().numpy(), Xo) <= 1e-12
    (piv, Lo, Uo, _), ties = lupp_parity(Js.cpu().numpy(), lambda f: o_lupp.select_cols(Xo, k, f))
    Zo, _, eta_o = o_id.id_coeffs(Lo, piv)
    kappa = abs(Uo[0, 0] / Uo[k - 1, k - 1])
    assert rel_fro(Z.cpu().numpy(), Zo) <= max(1e-9, 4 * k * U * kappa)
    assert abs(eta - eta_o) <= max(1e-8, 4 * k * U * kappa) * eta_o
    ro, nAo = o_res.residual(A, piv, kind="col_id")
    assert res_ok(r, ro, nAo), (r, ro)
    assert r >= o_res.optimal_error(sigma, k) * (1 - 1e-9)


@pytest.mark.parametrize("k", [64, 512])
def test_c2_cpqr_bench_shape(c2, k):
    """S2' at the shape bench.py times (X 522 x 4096, k = 512) and k = 64: CPQR on the GPU's
    sketch against the oracle's CPQR on the oracle's sketch (reading R9)."""
    A, _, Ad = c2
    l, seed = k + 10, 2002 + k
    X = sk.sketch(Ad, l, "gaussian", seed)
    Jc, R = sk.select_cols_cpqr(X, k, want_r=True)
    Xo = o_sketch.sketch(A, l, "gaussian", seed)
    piv, Ro = o_cpqr.select_cols_cpqr(Xo, k)
    assert Jc.cpu().tolist() == piv.tolist()
    # R's rows carry the Householder sign convention of both sides (alpha = -sign(x0) ||x||)
    assert rel_fro(R.cpu().numpy(), Ro) <= 1e-9


def test_c2_sketch_cluster_paths(c2):
    """The TMA sketch with a padded cluster grid (n-tiles not a multiple of the cluster size)."""
    A, _, Ad = c2
    for ncols, l in ((1300, 74), (2100, 266), (4095, 37)):
        X = sk.sketch(Ad[:, :ncols], l, "gaussian", 77)
        Xo = o_sketch.sketch(A[:, :ncols], l, "gaussian", 77)
        assert rel_fro(X.cpu().numpy(), Xo) <= 1e-12


@pytest.fixture(scope="module")
def c3():
    A, sigma = make_c3(seed=1003)
    return A, sigma, dev_f(A)


def oracle_sparse_sketch(A, l, seed, zeta):
    """X = Gamma A with the oracle's sparse-sign structure, as a sparse product (same definition
    as oracle.sketch, which would form the dense 510 x 16384 Gamma)."""
    rows, signs = o_omega.sparse_sign_structure(seed, l, A.shape[0], zeta)
    cols = np.repeat(np.arange(A.shape[0]), zeta)
    G = sps.csr_matrix((signs.ravel() / np.sqrt(zeta), (rows.ravel(), cols)), shape=(l, A.shape[0]))
    return np.asarray(G @ A)


def test_c3_full_cur(c3):
    """C3: 16384^2, sparse sign zeta=8, k=500, l=510, two-sided CUR."""
    A, sigma, Ad = c3
    k, l, seed = 500, 510, 2003
    X = sk.sketch(Ad, l, "sparse_sign", seed, 8)
    Js, _, _, _ = sk.select_cols(X, k)
    C = sk.gather_cols(Ad, Js)
    Is, _, _, _ = sk.select_rows(C, k)
    r_cur, nA = sk.residual(Ad, Js, Is, "cur")
    torch.cuda.synchronize()

    Xo = oracle_sparse_sketch(A, l, seed, 8)
    assert rel_fro(X.cpu().numpy(), Xo) <= 1e-12
    (piv, _, _, _), _ = lupp_parity(Js.cpu().numpy(), lambda f: o_lupp.select_cols(Xo, k, f, fast=True))
    Co = A[:, piv]
    np.testing.assert_array_equal(C.cpu().numpy(), Co)
    (ipiv, _, _, _), _ = lupp_parity(Is.cpu().numpy(), lambda f: o_lupp.select_rows(Co, k, f, fast=True))
    ro, nAo = o_res.residual(A, piv, ipiv, kind="cur")
    assert res_ok(r_cur, ro, nAo), (r_cur, ro)
    assert abs(nA - nAo) <= 1e-13 * nAo


@pytest.fixture(scope="module")
def c4():
    A, _ = make_c4(seed=1004)
    return A, dev_f(A)


@pytest.mark.parametrize("k", [50, 100, 200])
def test_c4_full_row_and_col_id(c4, k):
    """C4: 65536 x 784 nonnegative, Gaussian l=2k; column ID and row ID."""
    A, Ad = c4
    l, seed = 2 * k, 2004 + k
    X = sk.sketch(Ad, l, "gaussian", seed)
    Js, _, _, _ = sk.select_cols(X, k)
    Is, _, _, _ = sk.select_rows(sk.gather_cols(Ad, Js), k)
    r_col, nA = sk.residual(Ad, Js, None, "col_id")
    r_row, _ = sk.residual(Ad, None, Is, "row_id")
    torch.cuda.synchronize()

    Xo = o_sketch.sketch(A, l, "gaussian", seed)
    assert rel_fro(X.cpu().numpy(), Xo) <= 1e-12
    (piv, _, _, _), _ = lupp_parity(Js.cpu().numpy(), lambda f: o_lupp.select_cols(Xo, k, f))
    (ipiv, _, _, _), _ = lupp_parity(Is.cpu().numpy(), lambda f: o_lupp.select_rows(A[:, piv], k, f))
    rc, nAo = o_res.residual(A, piv, kind="col_id")
    rr, _ = o_res.residual(A, None, ipiv, kind="row_id")
    assert res_ok(r_col, rc, nAo), (r_col, rc)
    assert res_ok(r_row, rr, nAo), (r_row, rr)
