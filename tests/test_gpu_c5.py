"""C5 (BASELINE configs[4]) at full size on one B200: A 131072 x 65536 FP64 (68.7 GB), k=1000,
l=1100, Gaussian sketch, column LUPP, column-ID residual.

The oracle cannot run this size end to end, so parity is checked on outputs it can compute one
by one: sampled columns of A against the reflector-by-reflector definition,
sampled sketch columns X(:, j) = Gamma A(:, j) against the oracle's Gamma, and properties that
hold at any size: the first pivot is argmax |X(0, :)|, pivots are distinct, |L| <= 1
with L(J_s[t], t) = 1, and the residual respects Eckart-Young.
"""
import numpy as np
import pytest
import torch

import paper_2104_05877_b200 as sk
from inputs import c5
from oracle import omega as o_omega
from oracle import residual as o_res

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
