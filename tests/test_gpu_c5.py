"""C5 (BASELINE configs[4]) at full size on one B200: A 131072 x 65536 FP64 (68.7 GB), k=1000,
l=1100, Gaussian sketch, column LUPP, column-ID residual.

Two checks:
* test_c5_full: sampled columns of A against the reflector-by-reflector definition, sampled
  sketch columns X(:, j) = Gamma A(:, j) against the oracle's Gamma, and properties that hold at
  any size (first pivot = argmax |X(0, :)|, distinct pivots, |L| <= 1 with
  L(J_s[t], t) = 1, Eckart-Young);
* test_c5_oracle_streamed: the whole path against the oracle.  A does not fit in host memory at
  once, so the oracle takes it from the device in column blocks: its own X = Gamma A
  (column-separable), its own LUPP on X (the plain-C loop, bitwise equal to the numpy one) and
  its own column-ID residual with the residual blocks formed explicitly.  X within 1e-12, J_s
  identical up to documented near-ties, residual within 1e-9 r + 4u||A||_F.
"""
import numpy as np
import pytest
import torch

import paper_2104_05877_b200 as sk
from inputs import c5
from oracle import lupp as o_lupp
from oracle import omega as o_omega
from oracle import residual as o_res
from oracle import sketch as o_sketch
from tests.parity import lupp_parity, rel_fro

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def c5_data():
    fac = []
    A, sigma = c5.build_on_device(DEV, factors_out=fac)
    yield A, sigma, fac[0], fac[1]
    del A
    torch.cuda.empty_cache()


def test_c5_full(c5_data):
    A, sigma, Y, Yp = c5_data
    m, n = A.shape
    k, l, seed = 1000, 1100, 2005
    cols = [0, 1, 999, 31337, n - 1]
    for j in cols:
        ref = c5.column_by_reflectors(j, Y, Yp, sigma)
        np.testing.assert_allclose(A[:, j].cpu().numpy(), ref, atol=1e-14)
    X = sk.sketch(A, l, "gaussian", seed)
    # sampled sketch columns against the oracle's Gamma (generated in row chunks of A)
    acols = np.stack([c5.column_by_reflectors(j, Y, Yp, sigma) for j in cols], 1)
    Xo = np.zeros((l, len(cols)))
    for i0 in range(0, m, 16384):
        G = o_omega.gaussian_z(seed, l, np.arange(i0, min(m, i0 + 16384))) / np.sqrt(l)
        Xo += G @ acols[i0:i0 + G.shape[1]]
    Xg = X[:, cols].cpu().numpy()
    assert np.linalg.norm(Xg - Xo) <= 1e-12 * np.linalg.norm(Xo)
    Js, Lf, _, _ = sk.select_cols(X, k)
    J = Js.cpu().numpy()
    x0 = X[0].abs()
    assert J[0] == int(torch.argmax(x0).item())
    assert len(set(J.tolist())) == k and J.min() >= 0 and J.max() < n
    assert float(Lf.abs().max()) <= 1.0 + 1e-14
    assert torch.all(Lf[Js, torch.arange(k, device=DEV)] == 1.0)
    r, nA = sk.residual(A, Js, None, "col_id")
    opt = o_res.optimal_error(sigma, k)
    assert abs(nA - np.sqrt(np.sum(sigma ** 2))) <= 1e-12 * nA
    assert opt * (1 - 1e-9) <= r <= 100 * opt


def test_c5_oracle_streamed(c5_data):
    A, sigma, Y, Yp = c5_data
    m, n = A.shape
    k, l, seed = 1000, 1100, 2005
    At = A.t()                                               # n x m contiguous: row j = column j of A

    def get_cols(j0, j1):                                    # the input, column block by column block
        return At[j0:j1].cpu().numpy().T

    X = sk.sketch(A, l, "gaussian", seed)
    Js, Lf, _, _ = sk.select_cols(X, k)
    r, nA = sk.residual(A, Js, None, "col_id")
    Xg = X.cpu().numpy()
    jg = Js.cpu().numpy()
    del X, Lf
    torch.cuda.empty_cache()

    Xo = o_sketch.sketch_streamed(get_cols, m, n, l, "gaussian", seed)
    assert rel_fro(Xg, Xo) <= 1e-12
    (piv, _, _, _), ties = lupp_parity(jg, lambda f: o_lupp.select_cols(Xo, k, f, fast=True))
    del Xo
    ro, nAo = o_res.residual_col_id_streamed(get_cols, m, n, piv)
    assert abs(nA - nAo) <= 1e-12 * nAo
    assert abs(r - ro) <= 1e-9 * ro + 4 * 2.0 ** -53 * nAo, (r, ro)
    assert ro >= o_res.optimal_error(sigma, k) * (1 - 1e-9)


def test_c5_srtt(c5_data):
    """The SRTT embedding at C5's m = 131072 (the four-step cluster transform): sampled sketch
    columns against the oracle's FFT route, then the column LUPP properties and the residual's
    Eckart-Young bracket on the SRTT sketch."""
    A, sigma, Y, Yp = c5_data
    m, n = A.shape
    k, l, seed = 1000, 1100, 2006
    cols = [0, 1, 4097, 31337, n - 1]
    X = sk.sketch(A, l, "srtt", seed)
    acols = np.stack([c5.column_by_reflectors(j, Y, Yp, sigma) for j in cols], 1)
    Xo = o_sketch.sketch_srtt_fft(acols, l, seed)
    assert rel_fro(X[:, cols].cpu().numpy(), Xo) <= 1e-12
    Js, Lf, _, _ = sk.select_cols(X, k)
    J = Js.cpu().numpy()
    assert J[0] == int(torch.argmax(X[0].abs()).item())
    assert len(set(J.tolist())) == k
    assert float(Lf.abs().max()) <= 1.0 + 1e-14
    r, nA = sk.residual(A, Js, None, "col_id")
    opt = o_res.optimal_error(sigma, k)
    assert opt * (1 - 1e-9) <= r <= 100 * opt
